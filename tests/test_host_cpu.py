"""Host-side logic and the C ABI surface, without a GPU.

* the library loads and exports every function include/gridrogue_b200.h
  declares (no compute calls: there is no device here);
* the state field table of the ABI matches the reference SimState layout
  (state._SHAPES via the oracle's copy of it) for both tiers;
* the numpy RandomPolicy equals policies.RandomPolicy (via the oracle);
* shard bounds / exchange combination used by the multi-GPU path;
* the gymnax facade's variant table and error behaviour.
"""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    """Every function declared by the headers under include/ (the C ABI of
    the env step, gridrogue_b200.h, and the learner's objective,
    gridrogue_ppo.h)."""
    names = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if not h.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(grp?_[a-z_0-9]+)\s*\(", src))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    from paper_2402_16801_b200._build import LIB
    assert os.path.exists(LIB), "build() must have produced the CUDA library"
    lib = ctypes.CDLL(LIB)
    names = _declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_errors_without_device():
    from paper_2402_16801_b200 import _lib
    L = _lib.lib()
    assert L.gr_version() == 1
    cfg = _lib.GrConfig()
    cfg.tier = 7
    cfg.n_envs = 4
    h = ctypes.c_void_p()
    rc = L.gr_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc == _lib.GR_E_INVALID and b"unknown tier" in L.gr_last_error()
    cfg.tier = 1
    cfg.obs_mode = 2
    cfg.tile_px = 9
    assert L.gr_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.GR_E_INVALID
    assert b"tile_px" in L.gr_last_error()
    cfg.tile_px, cfg.obs_mode, cfg.n_envs = 10, 1, 0
    assert L.gr_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.GR_E_INVALID
    cfg.reset_ratio = 16
    cfg.n_envs, cfg.env_offset, cfg.n_envs_global = 8, 4, 10
    assert L.gr_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.GR_E_INVALID
    assert b"shard" in L.gr_last_error()


@pytest.mark.parametrize("tier", ["classic", "extended"])
def test_field_table_matches_reference_layout(oracle_lib, tier):
    from paper_2402_16801_b200 import _lib
    O = oracle_lib
    L = _lib.lib()
    assert _lib.FIELD_NAMES == O.FIELD_NAMES
    shapes = O.field_shapes(tier, 1)
    for fid, name in enumerate(_lib.FIELD_NAMES):
        n = ctypes.c_int64()
        esz = ctypes.c_int32()
        assert L.gr_field_info(_lib.TIER_IDS[tier], fid, ctypes.byref(n), ctypes.byref(esz)) == 0
        dt, shape = shapes[name]
        assert n.value == int(np.prod(shape[1:], dtype=np.int64)), name
        assert esz.value == np.dtype(dt).itemsize, name
    assert L.gr_field_info(0, 999, None, None) == _lib.GR_E_INVALID


@pytest.mark.parametrize("n_actions", [17, 43])
def test_numpy_random_policy_matches_reference_policy(oracle_lib, n_actions):
    from paper_2402_16801_b200.policies import RandomPolicy
    pol = RandomPolicy(12345, n_actions)
    for t in range(20):
        a = pol.actions(1000, env0=77)
        assert np.array_equal(a, oracle_lib.random_actions(12345, t, 1000, n_actions, env0=77))
        assert a.min() >= 0 and a.max() < n_actions


def test_shard_bounds_partition():
    from paper_2402_16801_b200.parallel import shard_bounds
    for n in (1, 7, 64, 65536, 1000003):
        for world in (1, 2, 3, 4, 8):
            if n < world:
                continue
            b = [shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_combine_exchange():
    from paper_2402_16801_b200.parallel import combine_exchange
    rec = np.array([[3, 1, 0, 0], [0, 4, 0, 0], [9, 2, 0, 0]], np.int32)
    assert combine_exchange(rec, 0, 5) == {"k_local": 3, "offset": 0, "n_pool": 3, "flags": 7}
    assert combine_exchange(rec, 2, 5) == {"k_local": 9, "offset": 3, "n_pool": 5, "flags": 7}


def test_gymnax_variant_table():
    from paper_2402_16801_b200 import make_craftax_env_from_name, VARIANTS
    assert VARIANTS["Craftax-Symbolic"] == ("extended", "symbolic")
    assert VARIANTS["Craftax-Classic-Pixels"] == ("classic", "pixels")
    env = make_craftax_env_from_name("Craftax-Classic-Symbolic-v1")
    assert env.num_actions() == 17
    assert env.observation_space().shape == (1345,)
    env = make_craftax_env_from_name("Craftax-Pixels")
    assert env.num_actions() == 43
    assert env.observation_space().shape == (110, 130, 3)
    with pytest.raises(ValueError):
        make_craftax_env_from_name("Craftax-Nope")
    with pytest.raises(ValueError):
        make_craftax_env_from_name("Craftax-Symbolic", auto_reset=False)


def test_product_does_not_import_oracle():
    """The checker is never part of the shipped path."""
    pkg = os.path.join(ROOT, "paper_2402_16801_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "libgr_oracle" not in txt, f


_GLIBC_CHECK = r"""
#include "gr_glibc_sincos.h"
#include <stdio.h>
int main(void) {
  float lo = 0.0f, hi = 6.2831853071795864769f;
  uint32_t a, b; memcpy(&a, &lo, 4); memcpy(&b, &hi, 4);
  long bad = 0, n = 0;
  for (uint32_t i = a; i <= b; ++i, ++n) {
    float f; memcpy(&f, &i, 4);
    double x = f, s1 = sin(x), s2 = gl_sin(x), c1 = cos(x), c2 = gl_cos(x);
    bad += memcmp(&s1, &s2, 8) != 0 || memcmp(&c1, &c2, 8) != 0;
  }
  uint64_t r = 88172645463325252ull;
  for (long k = 0; k < 20000000; ++k, ++n) {
    r ^= r << 13; r ^= r >> 7; r ^= r << 17;
    double x = ((double)(r >> 11) * 0x1p-53 - 0.5) * ((k & 1) ? 2e-2 : 2e4);
    double s1 = sin(x), s2 = gl_sin(x), c1 = cos(x), c2 = gl_cos(x);
    bad += memcmp(&s1, &s2, 8) != 0 || memcmp(&c1, &c2, 8) != 0;
  }
  printf("%ld %ld\n", n, bad);
  return 0;
}
"""


def test_glibc_sincos_port_equals_libm_exhaustively(tmp_path):
    """Hazard H3: the device's float64 sin / cos (csrc/gr_glibc_sincos.h, the
    code worldgen's cave noise runs) compiled for the host with the same
    operation sequence equals the system libm -- which numpy's float64
    sin / cos call -- bit for bit on every float32 angle in [0, 2*pi]
    (1,086,918,620 inputs: the cave gradients' whole domain) and on 2e7
    random doubles of both signs."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc") or pytest.skip("gcc not available")
    src = tmp_path / "glibc_check.c"
    src.write_text(_GLIBC_CHECK)
    exe = tmp_path / "glibc_check"
    inc = os.path.join(ROOT, "paper_2402_16801_b200", "csrc")
    subprocess.run([gcc, "-O2", "-ffp-contract=off", "-I", inc, str(src), "-o", str(exe), "-lm"], check=True)
    n, bad = map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split())
    assert n == 1_086_918_620 + 20_000_000
    assert bad == 0
