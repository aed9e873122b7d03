"""Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers: as easy as 1, 2, 3").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper draws its sketches from NumPy's global RNG (P:L1284 ``np.random.choice``), which is
not reproducible across implementations.  DESIGN.md §3 (the sketch-stream contract) replaces
it by this counter-based generator so that the CUDA path and this oracle can produce the same
sketch bit for bit.  Written from the algorithm's definition: 10 rounds of

    (x0, x1, x2, x3) <- (hi(M1*x2) ^ x1 ^ k0, lo(M1*x2), hi(M0*x0) ^ x3 ^ k1, lo(M0*x0))

with the key bumped by the Weyl constants (W0, W1) between rounds.

Pinned by tests/test_oracle_philox.py against (a) the published known-answer vectors
(tests/golden/philox4x32_10_kat.txt) and (b) the CUDA toolkit's host-compiled
``curand_Philox4x32_10`` on a grid of counters/keys.
"""

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)
SH32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10.  All arguments: integers or arrays of 32-bit values.

    Returns a tuple of four uint64 arrays (each value < 2**32): the output words x, y, z, w.
    """
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & MASK32 for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    for rnd in range(10):
        p0 = M0 * c0            # < 2**64: exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> SH32, p0 & MASK32
        hi1, lo1 = p1 >> SH32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if rnd < 9:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
    return c0, c1, c2, c3


def seed_key(seed):
    """Sketch-stream key: key = (seed mod 2**32, seed >> 32)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32
