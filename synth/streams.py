"""Counter-based SplitMix64 random streams (vectorised numpy, version-stable).

A stream is identified by (seed, label).  Element i of a stream is
``mix64(state0 + (i + 1) * GAMMA)`` -- exactly the i-th output of a SplitMix64
generator started at ``state0`` -- so any slice of a stream can be produced
without generating the prefix, and two programs that agree on (seed, label)
agree on every value.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _label_hash(label: str) -> int:
    # FNV-1a 64 over the UTF-8 bytes: a fixed, documented label -> integer map.
    h = 0xCBF29CE484222325
    for b in label.encode("utf-8"):
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def stream_state(seed: int, label: str) -> np.uint64:
    s = np.uint64((int(seed) * 0x9E3779B97F4A7C15 + _label_hash(label)) & 0xFFFFFFFFFFFFFFFF)
    return mix64(np.array([s], dtype=np.uint64))[0]


def u64(seed: int, label: str, start: int, count: int) -> np.ndarray:
    """Raw uint64 values [start, start+count) of stream (seed, label)."""
    st = stream_state(seed, label)
    idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(st + idx * GAMMA)


def uniform(seed: int, label: str, start: int, count: int) -> np.ndarray:
    """Uniform doubles in [0, 1) with 53 random bits."""
    return (u64(seed, label, start, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_open(seed: int, label: str, start: int, count: int) -> np.ndarray:
    """Uniform doubles in (0, 1): (k + 0.5) * 2^-53."""
    return ((u64(seed, label, start, count) >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def permutation(seed: int, label: str, n: int) -> np.ndarray:
    """Uniform random permutation of [0, n): argsort of n random keys (ties broken by index)."""
    keys = u64(seed, label, 0, n)
    return np.argsort(keys, kind="stable").astype(np.int64)


def normal_f32(seed: int, label: str, count: int, chunk: int = 1 << 24) -> np.ndarray:
    """Standard normal fp32 values by Box-Muller on pairs of stream uniforms."""
    out = np.empty(count, dtype=np.float32)
    npairs = (count + 1) // 2
    for p0 in range(0, npairs, chunk):
        p1 = min(npairs, p0 + chunk)
        u = uniform_open(seed, label, 2 * p0, 2 * (p1 - p0))
        u0, u1 = u[0::2], u[1::2]
        r = np.sqrt(-2.0 * np.log(u0))
        t = 2.0 * np.pi * u1
        z = np.empty(2 * (p1 - p0), dtype=np.float64)
        z[0::2] = r * np.cos(t)
        z[1::2] = r * np.sin(t)
        e0, e1 = 2 * p0, min(count, 2 * p1)
        out[e0:e1] = z[: e1 - e0].astype(np.float32)
    return out
