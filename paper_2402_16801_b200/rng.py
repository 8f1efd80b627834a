"""Host-side stream keys of the reference's counter-based RNG (rng.py:23-113).

Only what the host needs to hand streams to the device: ``make_stream``
(key = splitmix64 finalizer of the seed) and ``split``; the draws
themselves (hash2(key, counter)) happen in the kernels.
"""

from __future__ import annotations

_MASK = (1 << 64) - 1


def mix64(z: int) -> int:
    """rng._mix: the splitmix64 finalizer (rng.py:23-31)."""
    z = (z + 0x9E3779B97F4A7C15) & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def hash2(k: int, n: int) -> int:
    """rng.hash2 = mix(k ^ mix(n)) (rng.py:34-36)."""
    return mix64((k & _MASK) ^ mix64(n & _MASK))


class Stream:
    """rng.RngStream: immutable (key, counter)."""

    __slots__ = ("key", "counter")

    def __init__(self, key: int, counter: int = 0):
        self.key = key & _MASK
        self.counter = counter & _MASK

    def __repr__(self) -> str:
        return f"Stream(key={self.key:#x}, counter={self.counter})"


def make_stream(seed: int) -> Stream:
    return Stream(mix64(seed & _MASK))


def split(parent: Stream, stream_id: int) -> Stream:
    return Stream(hash2(parent.key, hash2(stream_id & _MASK, parent.counter)))
