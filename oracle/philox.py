"""Philox4x32-10 counter-based generator, host (NumPy) implementation for the oracle.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import anything under oracle/.

Definition (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as
1, 2, 3", SC'11, the Philox-4x32 round function with R = 10 rounds):

    (hi0, lo0) = mulhilo32(M0, X0)       M0 = 0xD2511F53
    (hi1, lo1) = mulhilo32(M1, X2)       M1 = 0xCD9E8D57
    X' = (hi1 ^ X1 ^ K0,  lo1,  hi0 ^ X3 ^ K1,  lo0)
    K  <- K + (W0, W1) (mod 2^32) between rounds, W0 = 0x9E3779B9, W1 = 0xBB67AE85

The sketch (reading R6) uses it as a hash; the CUDA path implements the
same published generator independently (no shared code).  Pinned by the
published known-answer vectors in tests/golden/philox4x32_10_kat.txt.
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
SH = np.uint64(32)


def philox4x32_10(ctr, key):
    """ctr: (..., 4) uint32-valued array, key: (..., 2) -> (..., 4) uint32 array."""
    c = np.asarray(ctr, dtype=np.uint64)
    k = np.asarray(key, dtype=np.uint64)
    x0, x1, x2, x3 = c[..., 0], c[..., 1], c[..., 2], c[..., 3]
    k0 = k[..., 0] + np.zeros_like(x0)
    k1 = k[..., 1] + np.zeros_like(x0)
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * x0          # < 2^64, exact in uint64
        p1 = M1 * x2
        hi0, lo0 = p0 >> SH, p0 & MASK
        hi1, lo1 = p1 >> SH, p1 & MASK
        x0, x1, x2, x3 = hi1 ^ x1 ^ k0, lo1, hi0 ^ x3 ^ k1, lo0
    return np.stack([x0, x1, x2, x3], axis=-1).astype(np.uint32)
