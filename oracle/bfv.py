"""ORACLE (test infrastructure only) — textbook BFV over an RNS modulus Q = prod q_l.

Follows PAPER.md §2.3 (lines 236-378):
  * symmetric encryption (c0, c1) = ([Delta m + a s + e]_Q, -a), Delta = floor(Q/t)
    (Eq. bfv_enc, PAPER.md:244-253 [\\ignore], footnote :242);
  * decryption [round(t [c0 + c1 s]_Q / Q)]_t, correct iff ||v||_inf < Delta/2
    (Eq. bfv_dec2, PAPER.md:256-267 [\\ignore]);
  * HRot = automorphism + key switching with a decomposition, hoisted
    (decompose once, then per-rotation automorphism + key inner product; PAPER.md:373-378,
    :1472-1473 "PermDecomp"/"PermAuto").
Readings: RNS digits, one per limb, no special prime (R5); hoisted digit
definition d_i = [c1]_{q_i} taken BEFORE the automorphism (R6); ternary secret and
CBD errors come from synth/ and are passed in (R2).

Ciphertexts are uint64 arrays [2][L][N] of canonical residues (coefficient form).
Galois keys are uint64 [L digits][2: b, a][L limbs][N].
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import ring
from .params import is_prime


@dataclass
class BFVParams:
    N: int
    primes: List[int]
    t: int
    w: int = 0   # decomposition base 2^w INSIDE each RNS limb (0: one digit per limb, reading R5)

    def __post_init__(self):
        assert self.N & (self.N - 1) == 0
        for q in self.primes:
            assert is_prime(q) and q % (2 * self.N) == 1, q
        assert is_prime(self.t) and self.t % (2 * self.N) == 1
        self.Q = 1
        for q in self.primes:
            self.Q *= q
        self.delta = self.Q // self.t

    @property
    def L(self) -> int:
        return len(self.primes)

    @property
    def V(self) -> int:
        """Sub-digits per limb: ceil(max bit length / w) (1 without a sub-digit base)."""
        return 1 if not self.w else -(-max(q.bit_length() for q in self.primes) // self.w)

    @property
    def ND(self) -> int:
        """Gadget digits: limb i, sub-digit v -> digit i V + v."""
        return self.L * self.V


def crt(residues: Sequence[np.ndarray], primes: Sequence[int]) -> list:
    """x in [0, Q) with x = r_l mod q_l (Chinese remainder theorem, textbook form)."""
    Q = 1
    for q in primes:
        Q *= q
    n = len(residues[0])
    out = [0] * n
    for r, q in zip(residues, primes):
        Qi = Q // q
        c = Qi * pow(Qi, -1, q)
        for j in range(n):
            out[j] += int(r[j]) * c
    return [x % Q for x in out]


def _mul_sparse_first(x, y, q: int) -> np.ndarray:
    """x * y mod (X^N + 1, q), passing the operand with fewer nonzero coefficients first (the
    schoolbook product skips zero coefficients of its first operand; the product commutes)."""
    if np.count_nonzero(np.asarray(y)) < np.count_nonzero(np.asarray(x)):
        x, y = y, x
    return ring.nc_mul(x, y, q)


def encrypt(P: BFVParams, m, s, a, e) -> np.ndarray:
    """Symmetric BFV encryption: c0 = [Delta m + a s + e], c1 = [-a], per limb.
    m: [N] ints in [0,t); s: [N] ternary; a: uint64 [L][N] uniform residues; e: [N] small ints."""
    L, N = P.L, P.N
    ct = np.empty((2, L, N), dtype=np.uint64)
    m = [int(x) % P.t for x in m]
    for l, q in enumerate(P.primes):
        a_s = _mul_sparse_first(s, a[l], q)
        dm = np.array([(P.delta * x) % q for x in m], dtype=object)
        ct[0, l] = ((dm + a_s.astype(object) + np.asarray(e, dtype=np.int64).astype(object)) % q).astype(np.uint64)
        ct[1, l] = ring.canon(-(a[l].astype(object)), q)
    return ct


def phase(P: BFVParams, ct, s) -> list:
    """[c0 + c1 s]_Q as integers in [0, Q)  (Eq. bfv_dec)."""
    res = []
    for l, q in enumerate(P.primes):
        c1s = ring.nc_mul(s, ct[1, l], q)
        res.append(((ct[0, l].astype(object) + c1s.astype(object)) % q))
    return crt(res, P.primes)


def decrypt(P: BFVParams, ct, s) -> np.ndarray:
    """m = [round(t x / Q)]_t with x = [c0 + c1 s]_Q in [0, Q)  (Eq. bfv_dec2).
    round(y) = floor(y + 1/2); ties cannot occur because gcd(Q, 2t) = 1."""
    x = phase(P, ct, s)
    return np.array([((P.t * v + P.Q // 2) // P.Q) % P.t for v in x], dtype=np.int64)


def noise_bits(P: BFVParams, ct, s, m) -> float:
    """log2 ||[c0 + c1 s - Delta m]_Q||_inf (centered) — the noise v of Eq. bfv_dec.
    Decryption is correct iff this is < log2(Delta/2)  (PAPER.md:266-267 [\\ignore], :318)."""
    import math
    x = phase(P, ct, s)
    worst = 0
    for v, mm in zip(x, m):
        r = (v - P.delta * (int(mm) % P.t)) % P.Q
        if r > P.Q // 2:
            r -= P.Q
        worst = max(worst, abs(r))
    return math.log2(worst) if worst else 0.0


def noise_budget_bits(P: BFVParams) -> float:
    import math
    return math.log2(P.delta / 2)


def galois_keygen(P: BFVParams, s, g: int, a, e) -> np.ndarray:
    """Switching key for X -> X^g under the RNS-digit gadget (reading R5), optionally refined by a
    base-2^w decomposition inside each limb (PAPER.md:1470 [app] decomposition base; SURVEY §8(f)
    NEXT-4): digit (i, v) has gadget g_{i,v} = (Q/q_i)[(Q/q_i)^{-1}]_{q_i} 2^{w v}, whose residue mod
    q_l is [i == l] 2^{w v}:
        b_{(i,v),l} = [-a_{(i,v),l} s + e_{(i,v)} + [i == l] 2^{w v} s(X^g)]_{q_l},  a uniform.
    a: uint64 [ND][L][N], e: [ND][N].  Returns uint64 [ND][2][L][N] (b first, then a)."""
    L, N, V = P.L, P.N, P.V
    s_g = ring.automorphism(np.asarray(s, dtype=np.int64), g)
    key = np.empty((P.ND, 2, L, N), dtype=np.uint64)
    for dd in range(P.ND):
        i, v = divmod(dd, V)
        for l, q in enumerate(P.primes):
            a_s = _mul_sparse_first(s, a[dd, l], q)
            b = -(a_s.astype(object)) + np.asarray(e[dd], dtype=np.int64).astype(object)
            if i == l:
                b = b + s_g.astype(object) * ((1 << (P.w * v)) % q)
            key[dd, 0, l] = ring.canon(b % q, q)
            key[dd, 1, l] = a[dd, l]
    return key


def decompose(P: BFVParams, ct) -> List[np.ndarray]:
    """Hoisting step 1 ('PermDecomp'): digits d_i = [c1]_{q_i}
    as integer polynomials with coefficients in [0, q_i); with a sub-digit base 2^w each is
    split further into its base-2^w digits d_{i,v} = floor(d_i / 2^{w v}) mod 2^w, v < V, so that
    sum_v d_{i,v} 2^{w v} = d_i (digit order i V + v)."""
    if not P.w:
        return [ct[1, i].astype(np.int64) for i in range(P.L)]
    mask = np.uint64((1 << P.w) - 1)
    return [((ct[1, i] >> np.uint64(P.w * v)) & mask).astype(np.int64) for i in range(P.L) for v in range(P.V)]


def rotate_hoisted(P: BFVParams, ct, digits, g: int, key) -> np.ndarray:
    """Hoisting step 2 ('PermAuto'): for every limb l
        c0' = [sigma_g(c0) + sum_i sigma_g(d_i) b_{i,l}]_{q_l},   c1' = [sum_i sigma_g(d_i) a_{i,l}]_{q_l}
    with sigma_g applied to the integer digit polynomials (reading R6)."""
    L, N = P.L, P.N
    dg = [ring.automorphism(d, g) for d in digits]
    out = np.empty((2, L, N), dtype=np.uint64)
    for l, q in enumerate(P.primes):
        c0 = ring.automorphism_mod(ct[0, l], g, q).astype(object)
        c1 = np.zeros(N, dtype=object)
        for i in range(len(digits)):   # L digits, or L V sub-digits (the key has as many rows)
            di = ring.canon(dg[i], q)
            c0 = c0 + ring.nc_mul(di, key[i, 0, l], q).astype(object)
            c1 = c1 + ring.nc_mul(di, key[i, 1, l], q).astype(object)
        out[0, l] = (c0 % q).astype(np.uint64)
        out[1, l] = (c1 % q).astype(np.uint64)
    return out


def rotate_direct(P: BFVParams, ct, g: int, key) -> np.ndarray:
    """HRot WITHOUT hoisting (the ablation of PAPER.md Fig. 4 (b), :373-378, :778-787): the
    automorphism acts on every limb first (mod q_l), then the ROTATED c1 is decomposed (digits of
    [sigma_g(c1)]_{q_i}), so every rotation repeats the decomposition.  Bitwise different from the
    hoisted definition (reading R6), same decryption."""
    L, N = P.L, P.N
    rot = np.stack([np.stack([ring.automorphism_mod(ct[c, l], g, q) for l, q in enumerate(P.primes)])
                    for c in range(2)])
    digits = decompose(P, rot)
    out = np.empty((2, L, N), dtype=np.uint64)
    for l, q in enumerate(P.primes):
        c0 = rot[0, l].astype(object)
        c1 = np.zeros(N, dtype=object)
        for i in range(len(digits)):
            d = ring.canon(digits[i], q)
            c0 = c0 + ring.nc_mul(d, key[i, 0, l], q).astype(object)
            c1 = c1 + ring.nc_mul(d, key[i, 1, l], q).astype(object)
        out[0, l] = (c0 % q).astype(np.uint64)
        out[1, l] = (c1 % q).astype(np.uint64)
    return out


def hrot(P: BFVParams, ct, g: int, key) -> np.ndarray:
    """HRot by one automorphism (hoisted definition applied to a single rotation)."""
    return rotate_hoisted(P, ct, decompose(P, ct), g, key)
