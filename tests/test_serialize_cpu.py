"""The game_state format of paper_2402_16801_b200.serialize vs the reference (no GPU).

Golden blobs were written by the reference's own serializer
(tests/golden/make_serialize_golden.py); the reader must accept them, and
blobs packed here must load in the reference's reader when it is present.
"""

import io
import json
import os
import sys

import numpy as np
import pytest

from paper_2402_16801_b200 import serialize as S
from paper_2402_16801_b200._lib import FIELD_NAMES

GOLD = os.path.join(os.path.dirname(__file__), "golden")
BLOBS = ["game_state_classic.bin", "game_state_extended.bin", "game_state_classic_batch.bin",
         "game_state_extended_batch.bin"]


def _blob(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name", BLOBS)
def test_reader_accepts_reference_blobs(name):
    meta, data = S._unpack(_blob(name), "game_state")
    assert meta["tier"] in ("classic", "extended") and meta["version"] == 1
    fields = S._fields_of(data, meta["tier"])
    assert list(fields) == list(FIELD_NAMES)
    assert int(data["max_episode_length"]) == 100_000


def test_reader_rejects_wrong_kind_and_version():
    blob = _blob(BLOBS[0])
    with pytest.raises(ValueError):
        S._unpack(blob, "world")
    meta, data = S._unpack(blob, "game_state")
    arrays = {k: data[k] for k in data.files if k != "__meta__"}
    bad = io.BytesIO()
    np.savez(bad, __meta__=np.frombuffer(json.dumps(dict(meta, version=2)).encode(), np.uint8), **arrays)
    with pytest.raises(ValueError):
        S._unpack(bad.getvalue(), "game_state")


@pytest.mark.parametrize("name", BLOBS)
def test_packed_blob_loads_in_reference_reader(name):
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.path.insert(0, ref)
    from gridrogue.serialize import state_from_bytes
    meta, data = S._unpack(_blob(name), "game_state")
    arrays = S._fields_of(data, meta["tier"])
    arrays["max_episode_length"] = np.int64(data["max_episode_length"])
    st = state_from_bytes(S._pack("game_state", meta["tier"], arrays))
    for f in FIELD_NAMES:
        assert np.array_equal(getattr(st.sim, f), arrays[f]), f
