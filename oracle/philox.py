"""The oracle's own Omega generator (Alg. 1 line 4: Q ~ N(0,1)^{c x 2k}).

TEST INFRASTRUCTURE ONLY.  The paper only says "standard normal";
the counter-based stream both sides implement independently is fixed in
DESIGN.md ("Omega stream", reading O11):

* Philox4x32-10 (Salmon et al., SC'11), key = (seed mod 2^32, seed >> 32),
  counter of block b = (b mod 2^32, b >> 32, 0x4F4D4547, 0).
* Element (i, j) of the c x l matrix (global row i) is entry e = i*l + j;
  block b = e >> 2 and lane t = e & 3.  The four words x0..x3 of block b give
  u_t = (x_t + 0.5) * 2^-32 and two Box-Muller pairs:
  z0 = r01 cos(2 pi u1), z1 = r01 sin(2 pi u1), r01 = sqrt(-2 ln u0);
  z2 = r23 cos(2 pi u3), z3 = r23 sin(2 pi u3), r23 = sqrt(-2 ln u2);
  evaluated in fp64 (each operation rounded once) and rounded to fp32.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)
TWO_PI = 6.283185307179586  # the double nearest 2*pi
OMEGA_TAG = 0x4F4D4547


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds on arrays of counters.

    ctr: uint32-valued array (..., 4); key: (k0, k1).  Returns uint64 array (..., 4)
    holding the four 32-bit output words."""
    c = np.asarray(ctr, dtype=np.uint64)
    c0, c1, c2, c3 = (c[..., i].copy() for i in range(4))
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
    return np.stack([c0, c1, c2, c3], axis=-1)


def omega(seed: int, row0: int, rows: int, l: int) -> np.ndarray:
    """Rows [row0, row0+rows) of the c x l Omega, fp32 (as the CUDA path stores it)."""
    e0 = row0 * l
    e1 = (row0 + rows) * l
    b0, b1 = e0 >> 2, (e1 + 3) >> 2
    b = np.arange(b0, b1, dtype=np.uint64)
    ctr = np.stack(
        [b & _MASK, b >> np.uint64(32), np.full_like(b, OMEGA_TAG), np.zeros_like(b)], axis=-1
    )
    x = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)).astype(np.float64)
    u = (x + 0.5) * (2.0 ** -32)
    z = np.empty_like(u)
    r01 = np.sqrt(-2.0 * np.log(u[:, 0]))
    r23 = np.sqrt(-2.0 * np.log(u[:, 2]))
    t1 = TWO_PI * u[:, 1]
    t3 = TWO_PI * u[:, 3]
    z[:, 0] = r01 * np.cos(t1)
    z[:, 1] = r01 * np.sin(t1)
    z[:, 2] = r23 * np.cos(t3)
    z[:, 3] = r23 * np.sin(t3)
    flat = z.reshape(-1)[e0 - 4 * b0 : e1 - 4 * b0]
    return flat.astype(np.float32).reshape(rows, l)
