"""ORACLE (test infrastructure only) — parameter selection (§3.2.1).

  1) (n, p, q) with p = 1 mod 2n and q = 1 mod 2n
  2) h_{p,n}: the non-zero coefficient of the plaintext whose slots hold [1, -1]
                                                              
  3) k minimising k*h_{p,n} mod p

h is computed by literally SIMD-encoding the slot vector [1..1 | -1..-1] with
oracle.encoding (no closed form), then checking the result has exactly two
equal non-zero coefficients (the paper's claim).
"""
from __future__ import annotations

from typing import List, Optional


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (bases = first 12 primes)."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37]
    for p in small:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_primes(N: int, bits: int, count: int) -> List[int]:
    """The `count` largest primes q < 2^bits with q = 1 mod 2N, descending (PAPER.md:611 step 1)."""
    out = []
    q = ((2**bits - 1) // (2 * N)) * (2 * N) + 1
    while len(out) < count and q > 2 * N:
        if q < 2**bits and is_prime(q):
            out.append(q)
        q -= 2 * N
    return out


def min_primitive_2n_root(t: int, N: int) -> int:
    """zeta_t: the smallest g in [2, t) with g^N = -1 (mod t), i.e. a primitive 2N-th root of unity.
    (this choice reproduces h_{307201,2048} = 84248 of PAPER.md:600.)"""
    assert (t - 1) % (2 * N) == 0, "t must be 1 mod 2N (PAPER.md:611)"
    for g in range(2, t):
        if pow(g, N, t) == t - 1:
            return g
    raise ValueError("no primitive 2N-th root")


def slot_exponents(N: int) -> List[int]:
    """Evaluation exponents of the 2 x (N/2) slot layout: row 0 slot i <-> zeta^{3^i mod 2N},
    row 1 slot i <-> zeta^{-3^i mod 2N}  (PAPER.md:316 SIMD encoding; layout reading A1).
    Returned in slot order [row 0 slots 0..N/2-1, row 1 slots 0..N/2-1]."""
    M = 2 * N
    r0 = [pow(3, i, M) for i in range(N // 2)]
    r1 = [(M - e) % M for e in r0]
    return r0 + r1


def galois_elt_for_step(N: int, step: int) -> int:
    """Left-rotation of both slot rows by `step` = automorphism X -> X^{3^step mod 2N}
    (HRot).  step is taken mod N/2."""
    return pow(3, step % (N // 2), 2 * N)


def rowswap_elt(N: int) -> int:
    """Swap of the two slot rows = X -> X^{2N-1} (alignment HRot)."""
    return 2 * N - 1


def h_pn(p: int, n: int) -> int:
    """h_{p,n} by encoding the slot vector [1,...,1 | -1,...,-1].
    Raises if the encoded polynomial is not the 2-term sparse form the paper states."""
    from .encoding import encode
    slots = [1] * (n // 2) + [p - 1] * (n // 2)
    m = encode(slots, p, n)
    nz = [(j, int(c)) for j, c in enumerate(m) if int(c) != 0]
    if len(nz) != 2 or nz[0][1] != nz[1][1]:
        raise AssertionError(f"[1,-1] plaintext is not 2-term sparse: {nz[:4]}")
    return nz[0][1]


def h_positions(p: int, n: int) -> List[int]:
    from .encoding import encode
    m = encode([1] * (n // 2) + [p - 1] * (n // 2), p, n)
    return [j for j, c in enumerate(m) if int(c) != 0]


def centered(x: int, p: int) -> int:
    """[x]_p in (-p/2, p/2]  (PAPER.md:255 [\\ignore] mod operation)."""
    x %= p
    return x - p if x > p // 2 else x


def find_k(p: int, h: int, k_max: int = 32) -> int:
    """k in [1, k_max] minimising |[k h]_p| (centered), ties -> smaller k.
    k_max = 32 is DESIGN.md reading R13 (the paper's k=11 needs 11 <= k_max <= 50)."""
    best, best_k = None, None
    for k in range(1, k_max + 1):
        v = abs(centered(k * h, p))
        if best is None or v < best:
            best, best_k = v, k
    return best_k
