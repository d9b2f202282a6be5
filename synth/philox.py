"""Counter-based generator shared (as a SPECIFICATION, not as code) by the client-side oracle and the
library's GPU encryption / key generation (hy_keygen / hy_encrypt).

Each side implements the same generator: the library in CUDA (csrc/kernels.cu), this module in
vectorised NumPy for the oracle tests.  No method arithmetic lives here: only random integers and
their documented mapping to the distributions the client draws (PAPER.md:242-253 [ign]: uniform
mask a, error e, secret s; readings R2/R3: ternary secret, centered binomial eta = 20).

Generator: Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3", SC'11):
128-bit counter (c0, c1, c2, c3), 64-bit key (k0, k1) = (seed mod 2^32, seed >> 32), ten rounds,
multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85.

Counter assignment (one Philox block per coefficient k):
  secret s[k]                       ctr = (k, 0, 0, 1)
  encryption j: mask a_l[k]         ctr = (k, j, l, 2)        error e[k]   ctr = (k, j, 0, 3)
  key for Galois element g, gadget digit dd (dd = i for one digit per limb, i V + v with a
  sub-digit base):                   mask a_{dd,l}[k]  ctr = (k, g, 256 dd + l, 4)
                                     error e_dd[k]     ctr = (k, g, 256 dd, 5)
Mappings of the block (x0, x1, x2, x3) (32-bit words):
  uniform residue mod q:  floor(X q / 2^128), X = x3 2^96 + x2 2^64 + x1 2^32 + x0  (exact, bias < 2^-64)
  ternary:                floor(Y 3 / 2^64) - 1,  Y = x1 2^32 + x0
  centered binomial(20):  popcount(Y & (2^20 - 1)) - popcount((Y >> 20) & (2^20 - 1))
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
U32 = np.uint64(0xFFFFFFFF)

P_SECRET, P_ENC_A, P_ENC_E, P_KEY_A, P_KEY_E = 1, 2, 3, 4, 5


def philox4x32(c0, c1, c2, c3, seed: int, rounds: int = 10):
    """Vectorised Philox4x32-R: counters are uint64 arrays holding 32-bit values; returns 4 arrays."""
    c = [np.asarray(x, dtype=np.uint64) & U32 for x in (c0, c1, c2, c3)]
    c = np.broadcast_arrays(*c)
    c = [x.copy() for x in c]
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    for r in range(rounds):
        if r:
            k0, k1 = (k0 + W0) & 0xFFFFFFFF, (k1 + W1) & 0xFFFFFFFF
        p0 = np.uint64(M0) * c[0]
        p1 = np.uint64(M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & U32
        hi1, lo1 = p1 >> np.uint64(32), p1 & U32
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return c


def _mul64(a, b):
    """Exact 64 x 64 -> 128-bit product of uint64 arrays / scalars: (hi, lo)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    a0, a1 = a & U32, a >> np.uint64(32)
    b0, b1 = b & U32, b >> np.uint64(32)
    p00, p01, p10, p11 = a0 * b0, a0 * b1, a1 * b0, a1 * b1
    mid = (p00 >> np.uint64(32)) + (p01 & U32) + (p10 & U32)
    lo = (p00 & U32) | ((mid & U32) << np.uint64(32))
    hi = p11 + (p01 >> np.uint64(32)) + (p10 >> np.uint64(32)) + (mid >> np.uint64(32))
    return hi, lo


def uniform_mod(x, q: int) -> np.ndarray:
    """floor(X q / 2^128) for the 128-bit blocks X = (x0, x1, x2, x3)."""
    xlo = x[0] | (x[1] << np.uint64(32))
    xhi = x[2] | (x[3] << np.uint64(32))
    a1, a0 = _mul64(xhi, q)
    b1, _ = _mul64(xlo, q)
    s = a0 + b1                      # wraps mod 2^64
    carry = (s < a0).astype(np.uint64)
    return a1 + carry


def ternary(x) -> np.ndarray:
    y = x[0] | (x[1] << np.uint64(32))
    hi, _ = _mul64(y, 3)
    return hi.astype(np.int64) - 1


def cbd20(x) -> np.ndarray:
    y = x[0] | (x[1] << np.uint64(32))
    m = np.uint64((1 << 20) - 1)

    def popcount(v):
        v = v.copy()
        c = np.zeros(v.shape, dtype=np.int64)
        for _ in range(20):
            c += (v & np.uint64(1)).astype(np.int64)
            v >>= np.uint64(1)
        return c

    return popcount(y & m) - popcount((y >> np.uint64(20)) & m)


# ---- the client's draws (oracle side) ----
def secret(seed: int, N: int) -> np.ndarray:
    k = np.arange(N, dtype=np.uint64)
    return ternary(philox4x32(k, 0, 0, P_SECRET, seed))


def enc_mask(seed: int, j: int, primes: Sequence[int], N: int) -> np.ndarray:
    """uint64 [L][N] uniform residues (mask a of encryption j)."""
    k = np.arange(N, dtype=np.uint64)
    return np.stack([uniform_mod(philox4x32(k, j, l, P_ENC_A, seed), q) for l, q in enumerate(primes)])


def enc_error(seed: int, j: int, N: int) -> np.ndarray:
    k = np.arange(N, dtype=np.uint64)
    return cbd20(philox4x32(k, j, 0, P_ENC_E, seed))


def key_mask(seed: int, g: int, primes: Sequence[int], N: int, ND: int = 0) -> np.ndarray:
    """uint64 [ND digits][L limbs][N] (masks a_dd of the key for Galois element g; ND = L default)."""
    k = np.arange(N, dtype=np.uint64)
    ND = ND or len(primes)
    return np.stack([np.stack([uniform_mod(philox4x32(k, g, 256 * i + l, P_KEY_A, seed), q)
                               for l, q in enumerate(primes)]) for i in range(ND)])


def key_error(seed: int, g: int, ND: int, N: int) -> np.ndarray:
    k = np.arange(N, dtype=np.uint64)
    return np.stack([cbd20(philox4x32(k, g, 256 * i, P_KEY_E, seed)) for i in range(ND)])
