"""blake2b-64 digests, identical to tests/golden/make_golden.py:digest."""

import hashlib

import numpy as np


def digest(*arrays) -> int:
    h = hashlib.blake2b(digest_size=8)
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return int.from_bytes(h.digest(), "little")


def state_digest(fields: dict, names) -> int:
    return digest(*[fields[n] for n in names])
