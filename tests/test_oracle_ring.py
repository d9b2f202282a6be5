"""Pins for oracle/ring.py (schoolbook negacyclic product, automorphisms) — CPU only.

Each pin is independent of the code it checks: a library path (numpy.polynomial on
Python ints), the ring identity X^N = -1, and the evaluation homomorphism at
primitive 2N-th roots of unity (a property of Z_q[X]/(X^N+1), not of the code).
"""
import numpy as np
import pytest

from oracle import ring
from oracle.params import is_prime, ntt_primes

pytestmark = pytest.mark.filterwarnings("ignore")


def _np_poly_negacyclic(a, b, q):
    """Library path: full polynomial product (numpy.polynomial, Python ints) then X^N = -1."""
    from numpy.polynomial import polynomial as P
    n = len(a)
    full = P.polymul(np.array([int(x) for x in a], dtype=object), np.array([int(x) for x in b], dtype=object))
    full = list(full) + [0] * (2 * n - len(full))
    return [(int(full[k]) - int(full[k + n])) % q for k in range(n)]


@pytest.mark.parametrize("n,bits", [(8, 20), (16, 50), (32, 60), (64, 62)])
def test_nc_mul_matches_library_product(n, bits):
    q = ntt_primes(n, bits, 1)[0]
    g = np.random.default_rng(n * bits)
    for _ in range(3):
        a = g.integers(0, q, n, dtype=np.uint64)
        b = g.integers(0, q, n, dtype=np.uint64)
        assert list(ring.nc_mul(a, b, q)) == _np_poly_negacyclic(a, b, q)
        assert ring.nc_mul_py(a, b, q) == _np_poly_negacyclic(a, b, q)


def test_x_pow_n_is_minus_one():
    """x^{N-1} * x = -1 in Z_q[X]/(X^N+1)."""
    for n in (16, 4096):
        q = ntt_primes(n, 60, 1)[0]
        a = np.zeros(n, dtype=np.uint64)
        a[n - 1] = 1
        b = np.zeros(n, dtype=np.uint64)
        b[1] = 1
        c = ring.nc_mul(a, b, q)
        assert c[0] == q - 1 and not c[1:].any()


def test_evaluation_homomorphism():
    """c = a*b  =>  c(psi^e) = a(psi^e) b(psi^e) mod q for every primitive 2N-th root psi^e."""
    n, q = 32, ntt_primes(32, 40, 1)[0]
    gen = pow(next(x for x in range(2, q) if pow(x, (q - 1) // 2, q) == q - 1), (q - 1) // (2 * n), q)
    assert pow(gen, n, q) == q - 1
    g = np.random.default_rng(7)
    a = g.integers(0, q, n, dtype=np.uint64)
    b = g.integers(0, q, n, dtype=np.uint64)
    c = ring.nc_mul(a, b, q)
    ev = lambda p, x: sum(int(p[j]) * pow(x, j, q) for j in range(n)) % q
    for e in range(1, 2 * n, 2):
        x = pow(gen, e, q)
        assert ev(c, x) == ev(a, x) * ev(b, x) % q


def test_sparse_operand_and_large_n():
    """Zero-skipping is exact: a 2-term sparse first operand equals the sum of two shifted copies."""
    n = 8192
    q = ntt_primes(n, 60, 1)[0]
    g = np.random.default_rng(3)
    b = g.integers(0, q, n, dtype=np.uint64)
    a = np.zeros(n, dtype=np.uint64)
    a[n // 4] = 5
    a[3 * n // 4] = q - 7
    c = ring.nc_mul(a, b, q)

    def shift(p, k):      # X^k * p, negacyclic
        out = np.empty(n, dtype=object)
        for j in range(n):
            e = j + k
            out[e % n] = int(p[j]) if e < n else -int(p[j])
        return out
    ref = (5 * shift(b, n // 4) - 7 * shift(b, 3 * n // 4)) % q
    assert list(c) == list(ref)


def test_automorphism_properties():
    n = 16
    M = 2 * n
    p = np.arange(1, n + 1, dtype=np.int64)
    # sigma_g o sigma_h = sigma_{gh}
    for g in (3, 5, 9, M - 1):
        for h in (3, 7, M - 1):
            lhs = ring.automorphism(ring.automorphism(p, h), g)
            rhs = ring.automorphism(p, (g * h) % M)
            assert list(lhs) == list(rhs)
    # sigma_{2N-1}(X^j) = X^{-j} = -X^{N-j}
    for j in range(1, n):
        e = np.zeros(n, dtype=np.int64)
        e[j] = 1
        r = ring.automorphism(e, M - 1)
        assert r[n - j] == -1 and np.count_nonzero(r) == 1
    # automorphism_mod agrees with the signed version reduced mod q
    q = ntt_primes(n, 30, 1)[0]
    pm = np.arange(n, dtype=np.uint64) * np.uint64(12345) % np.uint64(q)
    for g in (3, 27, M - 1):
        assert list(ring.automorphism_mod(pm, g, q)) == [int(x) % q for x in ring.automorphism(pm.astype(np.int64), g)]


def test_is_prime_small():
    sieve = [True] * 5000
    sieve[0] = sieve[1] = False
    for i in range(2, 5000):
        if sieve[i]:
            for j in range(i * i, 5000, i):
                sieve[j] = False
    assert all(is_prime(i) == sieve[i] for i in range(5000))
    assert is_prime(2**61 - 1) and not is_prime(2**61 + 1)
