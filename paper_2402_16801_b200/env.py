"""Host-side mirror of the reference's batched-env interface.

``BatchEnv`` is a drop-in for ``gridrogue_gym.BatchEnv``
(/root/reference/pkg/bindings/src/gridrogue_gym/__init__.py:24-95): same
constructor, properties, ``reset() -> obs``, ``step(actions) -> (obs, reward,
done, info)``, error messages and single-owner rule, backed by the CUDA
library instead of numpy.  ``GridrogueBatch`` is the lower-level handle that
keeps everything on the device (torch tensors as carriers) for training
loops and the benchmark.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib
from ._lib import check, lib

TIERS = {
    "classic": dict(n_actions=17, n_achievements=22, obs=1345, view=(7, 9), side=0),
    "extended": dict(n_actions=43, n_achievements=67, obs=8268, view=(9, 11), side=2),
}
SUPPORTED_TILE_PX = (7, 10, 16)
DEFAULT_TILE_PX = {"classic": 7, "extended": 10}


def _tier_name(tier) -> str:
    name = getattr(tier, "name", tier)
    if name not in TIERS:
        raise ValueError(f"unknown tier {name!r}")   # constants.tier_by_name
    return name


def pixel_shape(tier: str, tile_px: int) -> tuple:
    t = TIERS[tier]
    vr, vc = t["view"]
    return ((vr + 2) * tile_px, (vc + t["side"]) * tile_px, 3)


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


class GridrogueBatch:
    """One shard of the batch on one GPU: device state + device I/O tensors.

    Output tensors are preallocated once and overwritten by every call
    (the reference allocates fresh arrays per step; clone if you keep them).
    """

    def __init__(self, n_envs: int, tier: str = "extended", seed: int = 0,
                 obs_mode: str = "symbolic", max_episode_length: int | None = None,
                 tile_px: int | None = None, device: int = 0, reset_ratio: int = 16,
                 env_offset: int = 0, n_envs_global: int | None = None,
                 newly: bool = True, info: bool = True):
        import torch
        self.torch = torch
        self.tier = _tier_name(tier)
        if obs_mode not in _lib.OBS_IDS:
            raise ValueError(f"unknown obs_mode {obs_mode!r}")
        self.obs_mode = obs_mode
        self.n = int(n_envs)
        self.tile_px = int(tile_px or DEFAULT_TILE_PX[self.tier])
        if obs_mode == "pixels" and self.tile_px not in SUPPORTED_TILE_PX:
            raise ValueError(f"tile_px must be one of {SUPPORTED_TILE_PX}")
        self.device = torch.device("cuda", device)
        cfg = _lib.GrConfig()
        cfg.tier = _lib.TIER_IDS[self.tier]
        cfg.obs_mode = _lib.OBS_IDS[obs_mode]
        cfg.tile_px = self.tile_px
        cfg.reset_ratio = int(reset_ratio)
        cfg.n_envs = self.n
        cfg.env_offset = int(env_offset)
        cfg.n_envs_global = int(n_envs_global or self.n)
        cfg.max_episode_length = int(max_episode_length or 0)
        cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        cfg.device = int(device)
        self.cfg = cfg
        self.h = ctypes.c_void_p()
        check(lib().gr_create(ctypes.byref(cfg), ctypes.byref(self.h)))
        t = TIERS[self.tier]
        self.n_actions = t["n_actions"]
        self.n_achievements = t["n_achievements"]
        dev = self.device
        n = self.n
        if obs_mode == "symbolic":
            self.obs = torch.empty((n, t["obs"]), dtype=torch.float32, device=dev)
        elif obs_mode == "pixels":
            self.obs = torch.empty((n,) + pixel_shape(self.tier, self.tile_px), dtype=torch.uint8, device=dev)
        else:
            self.obs = torch.empty((n, 0), dtype=torch.float32, device=dev)
        self.actions = torch.zeros(n, dtype=torch.int64, device=dev)
        self.reward = torch.empty(n, dtype=torch.float32, device=dev)
        self.done = torch.empty(n, dtype=torch.uint8, device=dev)
        self.newly = torch.empty((n, t["n_achievements"]), dtype=torch.uint8, device=dev) if newly else None
        self.time = torch.empty(n, dtype=torch.int32, device=dev) if info else None
        self.floor = torch.empty(n, dtype=torch.uint8, device=dev) if info else None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                lib().gr_destroy(h)
            except Exception:   # interpreter shutdown: module globals already gone
                pass
            self.h = None

    # --- hot path -----------------------------------------------------
    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def _obs_ptr(self):
        return _ptr(self.obs) if self.obs_mode != "none" else None

    def reset(self):
        check(lib().gr_reset(self.h, self._obs_ptr(), self._stream()))
        return self.obs

    def random_actions(self, seed: int, t: int, out=None):
        out = self.actions if out is None else out
        check(lib().gr_random_actions(self.h, seed & 0xFFFFFFFF, t, _ptr(out), self._stream()))
        return out

    def set_validate(self, on: bool) -> None:
        check(lib().gr_set_validate(self.h, 1 if on else 0))

    def step(self, actions=None):
        """Device step; returns (obs, reward, done, newly, time, floor) tensors."""
        a = self.actions if actions is None else actions
        if tuple(a.shape) != (self.n,):
            raise ValueError(f"actions must have shape ({self.n},), got {tuple(a.shape)}")
        if a is not self.actions:
            # one stable action buffer: the library replays a captured step
            # graph per set of buffer addresses
            self.actions.copy_(a)
            a = self.actions
        check(lib().gr_step(self.h, _ptr(a), self._obs_ptr(), _ptr(self.reward), _ptr(self.done),
                            _ptr(self.newly), _ptr(self.time), _ptr(self.floor), self._stream()))
        return self.obs, self.reward, self.done, self.newly, self.time, self.floor

    # sharded step (see parallel.py)
    def step_local(self, actions, exchange):
        check(lib().gr_step_local(self.h, _ptr(actions), _ptr(self.reward), _ptr(self.done),
                                  _ptr(self.newly), _ptr(self.time), _ptr(self.floor),
                                  _ptr(exchange), self._stream()))

    def step_finish(self, exchange_all, rank: int, world: int):
        check(lib().gr_step_finish(self.h, _ptr(exchange_all), rank, world, self._obs_ptr(),
                                   self._stream()))
        return self.obs, self.reward, self.done, self.newly, self.time, self.floor

    def obs_to_host(self, out: np.ndarray) -> np.ndarray:
        """Copy the current observation buffer into a host numpy array (every
        word written; symbolic observations travel packed, gr_obs_to_host)."""
        if self.obs_mode == "none":
            return out
        if out.nbytes != self.obs.numel() * self.obs.element_size() or not out.flags.c_contiguous:
            raise ValueError("obs_to_host needs a C-contiguous array of the observation buffer's size")
        check(lib().gr_obs_to_host(self.h, _ptr(self.obs), out.ctypes.data_as(ctypes.c_void_p), self._stream()))
        return out

    def observe(self):
        check(lib().gr_observe(self.h, self._obs_ptr(), self._stream()))
        return self.obs

    # --- state channel --------------------------------------------------
    def field_shape(self, name: str) -> tuple:
        n_el = ctypes.c_int64()
        esz = ctypes.c_int32()
        check(lib().gr_field_info(self.cfg.tier, _lib.FIELD_ID[name], ctypes.byref(n_el), ctypes.byref(esz)))
        return n_el.value, esz.value

    def export_field(self, name: str) -> np.ndarray:
        self.torch.cuda.synchronize(self.device)
        n_el, esz = self.field_shape(name)
        buf = np.empty(self.n * n_el * esz, np.uint8)
        check(lib().gr_export_field(self.h, _lib.FIELD_ID[name], buf.ctypes.data_as(ctypes.c_void_p)))
        return buf

    def import_field(self, name: str, arr: np.ndarray) -> None:
        self.torch.cuda.synchronize(self.device)
        a = np.ascontiguousarray(arr)
        n_el, esz = self.field_shape(name)
        if a.nbytes != self.n * n_el * esz:
            raise ValueError(f"field {name}: expected {self.n * n_el * esz} bytes, got {a.nbytes}")
        check(lib().gr_import_field(self.h, _lib.FIELD_ID[name], a.ctypes.data_as(ctypes.c_void_p)))

    def export_state(self, shapes: dict | None = None) -> dict:
        """Every SimState field as numpy in the reference layout (layout.field_shapes)."""
        if shapes is None:
            from .layout import field_shapes
            shapes = field_shapes(self.tier, self.n)
        out = {}
        for name in _lib.FIELD_NAMES:
            dt, shape = shapes[name]
            out[name] = self.export_field(name).view(dt).reshape(shape)
        return out

    def import_state(self, fields: dict) -> None:
        for name in _lib.FIELD_NAMES:
            self.import_field(name, fields[name])

    # --- metrics ------------------------------------------------------
    def stats(self) -> dict:
        s = _lib.GrStats()
        check(lib().gr_stats_get(self.h, ctypes.byref(s)))
        return {"episodes": s.episodes, "total_return": s.total_return, "total_steps": s.total_steps,
                "ach_episodes": np.array(s.ach_episodes[:self.n_achievements], np.int64)}

    def episode_progress(self) -> tuple:
        """BatchState.ep_return (f64[N]) and ep_length (i64[N]) of the running episodes."""
        self.torch.cuda.synchronize(self.device)
        ret = np.zeros(self.n, np.float64)
        length = np.zeros(self.n, np.int64)
        check(lib().gr_export_episode(self.h, ret.ctypes.data_as(ctypes.c_void_p),
                                      length.ctypes.data_as(ctypes.c_void_p)))
        return ret, length

    def set_episode_progress(self, ep_return: np.ndarray, ep_length: np.ndarray) -> None:
        ret = np.ascontiguousarray(ep_return, np.float64)
        length = np.ascontiguousarray(ep_length, np.int64)
        if ret.shape != (self.n,) or length.shape != (self.n,):
            raise ValueError(f"episode arrays must have shape ({self.n},)")
        self.torch.cuda.synchronize(self.device)
        check(lib().gr_import_episode(self.h, ret.ctypes.data_as(ctypes.c_void_p),
                                      length.ctypes.data_as(ctypes.c_void_p)))

    @property
    def step_index(self) -> int:
        v = ctypes.c_int64()
        check(lib().gr_get_step_index(self.h, ctypes.byref(v)))
        return v.value

    @step_index.setter
    def step_index(self, value: int) -> None:
        self.torch.cuda.synchronize(self.device)
        check(lib().gr_set_step_index(self.h, int(value)))

    def set_stats(self, stats: dict) -> None:
        """Restore EpisodeStats (checkpoint / resume)."""
        s = _lib.GrStats()
        s.episodes = int(stats["episodes"])
        s.total_steps = int(stats["total_steps"])
        s.total_return = float(stats["total_return"])
        ach = np.asarray(stats["ach_episodes"], np.int64)
        for k in range(min(len(ach), 67)):
            s.ach_episodes[k] = int(ach[k])
        check(lib().gr_stats_set(self.h, ctypes.byref(s)))

    def episodes_completed(self) -> int:
        v = ctypes.c_int64()
        check(lib().gr_episodes_completed(self.h, ctypes.byref(v)))
        return v.value

    def level_seeds(self) -> np.ndarray:
        self.torch.cuda.synchronize(self.device)
        out = np.empty(self.n, np.uint64)
        check(lib().gr_level_seeds(self.h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def kernel_launches(self) -> int:
        return int(lib().gr_kernel_launches(self.h))

    KERNEL_CLASSES = ("step", "scan", "info", "worldgen", "install", "obs", "policy", "other", "obs_reset",
                      "obs_prep")

    def set_profiling(self, on: bool) -> None:
        check(lib().gr_set_profiling(self.h, 1 if on else 0))

    def kernel_times(self) -> dict:
        """{class: (device ms, launches)} since the last call (CUDA events)."""
        k = len(self.KERNEL_CLASSES)
        ms = (ctypes.c_double * k)()
        cnt = (ctypes.c_int64 * k)()
        check(lib().gr_kernel_times(self.h, ms, cnt, k))
        return {c: (ms[i], cnt[i]) for i, c in enumerate(self.KERNEL_CLASSES)}

    def worldgen_counters(self) -> dict:
        c = (ctypes.c_int64 * 5)()
        check(lib().gr_worldgen_counters(self.h, c))
        return dict(zip(("worlds", "retried_floors", "template_floors", "potion_ties", "fragile_caves"), c))


class BatchEnv:
    """N parallel episodes behind a (obs, reward, done, info) step contract.

    Drop-in for gridrogue_gym.BatchEnv (__init__.py:24-95) with numpy
    inputs/outputs; the work runs on the GPU through the C ABI with
    host<->device copies inside ``step``.  obs_mode "pixels" adds the RGB
    frame of tiles.render_tiles per env (the reference renders one env).
    """

    metadata = {"obs_modes": ("symbolic", "none", "pixels")}

    def __init__(self, n_envs: int, tier: str = "extended", seed: int = 0,
                 obs_mode: str = "symbolic", max_episode_length: int | None = None,
                 tile_px: int | None = None, device: int = 0, obs_transfer: str = "dense",
                 _batch: GridrogueBatch | None = None):
        if obs_mode not in self.metadata["obs_modes"]:
            raise ValueError(f"unknown obs_mode {obs_mode!r}")
        if obs_transfer not in ("dense", "delta"):
            raise ValueError(f"unknown obs_transfer {obs_transfer!r}")
        if obs_transfer == "delta" and obs_mode != "symbolic":
            raise ValueError("obs_transfer='delta' needs obs_mode='symbolic'")
        self.obs_transfer = obs_transfer
        self.tier_name = _tier_name(tier)
        self.n_envs = int(n_envs)
        self.obs_mode = obs_mode
        self.seed = int(seed)
        self._batch = _batch if _batch is not None else GridrogueBatch(
            self.n_envs, self.tier_name, self.seed, obs_mode, max_episode_length, tile_px, device)
        self._stepping = threading.Lock()
        self._ready = _batch is not None
        import torch
        n = self.n_envs
        t = TIERS[self.tier_name]
        pin = dict(pin_memory=True)
        if obs_mode == "symbolic":
            self._obs_alloc = lambda: torch.empty((n, t["obs"]), dtype=torch.float32, **pin).numpy()
        elif obs_mode == "pixels":
            shape = (n,) + pixel_shape(self.tier_name, self._batch.tile_px)
            self._obs_alloc = lambda: torch.empty(shape, dtype=torch.uint8, **pin).numpy()
        else:
            self._obs_alloc = lambda: np.zeros((n, 0), np.float32)
        # observations: the reference returns a fresh array per call.  Copying
        # a 2 GB pinned buffer into a new array per step cost 5x the PCIe
        # transfer, so the obs land in one of two pinned buffers that is
        # handed out as is; a buffer is only reused once the caller holds no
        # reference to it (refcount), else the step falls back to a copy
        self._h_obs = self._obs_alloc()          # staging buffer of the fallback
        self._obs_pool = [self._obs_alloc(), self._obs_alloc()] if obs_mode != "none" else []
        # obs_transfer "delta": the handle owns the buffers' contents
        # (gr_host_obs_attach) and moves only the words that changed since the
        # buffer's last observation; arrays are handed out read-only so a
        # caller cannot make the buffer and the handle's copy of it disagree
        self._attached = []
        if obs_transfer == "delta":
            for b in [self._h_obs, *self._obs_pool]:
                check(lib().gr_host_obs_attach(self._batch.h, b.ctypes.data_as(ctypes.c_void_p)))
                self._attached.append(b.ctypes.data)   # the address only: refcounts pick free buffers
                b.flags.writeable = False   # views handed out cannot be made writable again
        self._h_act = torch.empty(n, dtype=torch.int64, **pin).numpy()
        self._h_rew = torch.empty(n, dtype=torch.float32, **pin).numpy()
        self._h_done = torch.empty(n, dtype=torch.bool, **pin).numpy()
        self._h_newly = torch.empty((n, t["n_achievements"]), dtype=torch.bool, **pin).numpy()
        self._h_time = torch.empty(n, dtype=torch.int32, **pin).numpy()
        self._h_floor = torch.empty(n, dtype=torch.uint8, **pin).numpy()

    @classmethod
    def from_batch(cls, batch: GridrogueBatch, obs_transfer: str = "dense") -> "BatchEnv":
        """The numpy contract over an existing device batch that has been
        reset (and possibly stepped) -- e.g. a benchmark's pre-rolled batch."""
        return cls(batch.n, batch.tier, int(batch.cfg.seed), batch.obs_mode, None, batch.tile_px,
                   batch.device.index or 0, obs_transfer, _batch=batch)

    def close(self) -> None:
        """Detach the delta-transfer buffers from the handle (idempotent): the
        handle may outlive this object (``env.batch``), and its attachments
        are keyed by host address."""
        att = getattr(self, "_attached", None)
        b = getattr(self, "_batch", None)
        while att:
            addr = att.pop()
            if b is not None and getattr(b, "h", None) is not None and b.h.value:
                try:
                    lib().gr_host_obs_detach(b.h, ctypes.c_void_p(addr))
                except Exception:   # interpreter shutdown
                    pass

    def __del__(self):
        self.close()

    @property
    def n_actions(self) -> int:
        return TIERS[self.tier_name]["n_actions"]

    @property
    def obs_width(self) -> int:
        if self.obs_mode == "symbolic":
            return TIERS[self.tier_name]["obs"]
        if self.obs_mode == "pixels":
            return int(np.prod(pixel_shape(self.tier_name, self._batch.tile_px)))
        return 0

    @property
    def batch(self) -> GridrogueBatch:
        return self._batch

    def _vp(self, a):
        return a.ctypes.data_as(ctypes.c_void_p)

    def _free_obs_buffer(self):
        """A pool buffer no caller holds (None: all held)."""
        import sys
        for k in range(len(self._obs_pool)):
            if sys.getrefcount(self._obs_pool[k]) <= 2:   # the pool list + getrefcount's argument
                return k
        return None

    def _obs_target(self):
        if self.obs_mode == "none":
            return None, self._h_obs
        k = self._free_obs_buffer()
        return k, (self._obs_pool[k] if k is not None else self._h_obs)

    def _obs_result(self, k, buf):
        if self.obs_mode == "none":
            return self._h_obs.copy()
        if k is None:
            return buf.copy()
        return buf.view() if self.obs_transfer == "delta" else buf

    def reset(self) -> np.ndarray:
        k, buf = self._obs_target()
        obs_p = self._vp(buf) if self.obs_mode != "none" else None
        check(lib().gr_reset_host(self._batch.h, obs_p))
        self._ready = True
        return self._obs_result(k, buf)

    def step(self, actions):
        if not self._ready:
            raise RuntimeError("call reset() before step()")
        if not self._stepping.acquire(blocking=False):
            raise RuntimeError("BatchEnv is single-owner: concurrent step() calls are not allowed")
        try:
            actions = np.ascontiguousarray(actions, dtype=np.int64)
            if actions.shape != (self.n_envs,):
                raise ValueError(f"actions must have shape ({self.n_envs},), got {actions.shape}")
            bad = (actions < 0) | (actions >= self.n_actions)
            if bad.any():
                i = int(np.argmax(bad))
                raise ValueError(f"invalid action {int(actions[i])} for env {i}")
            np.copyto(self._h_act, actions)
            k, buf = self._obs_target()
            obs_p = self._vp(buf) if self.obs_mode != "none" else None
            check(lib().gr_step_host(self._batch.h, self._vp(self._h_act), obs_p, self._vp(self._h_rew),
                                     self._vp(self._h_done), self._vp(self._h_newly),
                                     self._vp(self._h_time), self._vp(self._h_floor)))
            info = {"time": self._h_time.view(np.uint32).copy(), "floor": self._h_floor.copy(),
                    "newly_unlocked": self._h_newly.copy(),
                    "episodes_completed": self._batch.episodes_completed()}
            return self._obs_result(k, buf), self._h_rew.copy(), self._h_done.copy(), info
        finally:
            self._stepping.release()

    def level_seeds(self) -> np.ndarray:
        return self._batch.level_seeds()
