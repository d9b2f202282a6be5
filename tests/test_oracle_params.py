"""Pins for oracle/params.py and oracle/encoding.py against the paper's printed values
(tests/golden/paper_values.json, each with its PAPER.md line) and closed forms — CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import ring
from oracle.encoding import decode, decode_batch, encode, encode_batch
from oracle.params import (centered, find_k, galois_elt_for_step, h_pn, h_positions, is_prime,
                           min_primitive_2n_root, ntt_primes, rowswap_elt)
from synth import PRIMES, T_PLAIN

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_h_gazelle_params_matches_paper():
    """h_{307201,2048} = 84248, by literally encoding [1,-1] slots."""
    assert is_prime(307201) and 307201 % 4096 == 1
    assert h_pn(307201, 2048) == GOLD["h_307201_2048"]["value"]
    assert h_positions(307201, 2048) == [512, 1536]   # X^{N/4}, X^{3N/4}


def test_k_gazelle_params_matches_paper():
    """k = 11: [11 * 84248]_p = 5125."""
    k = find_k(307201, 84248)
    assert k == GOLD["k_307201_2048"]["value"]
    assert centered(11 * 84248, 307201) == 5125


def test_noise_bit_claims():
    """'at most 25 bits' (k=1), '21 bits' (k=11), conventional '29 bits':
    factor f0 + 2 f1 h with 8-bit kernel values, and n p / 2 for dense PMult."""
    assert round(math.log2(2 * 84248 * 2**8)) == GOLD["pmult_bits_k1"]["value"]
    assert round(math.log2(2 * 5125 * 2**8)) == GOLD["pmult_bits_k11"]["value"]
    assert math.ceil(math.log2(2048 * 307201 / 2)) == GOLD["pmult_bits_conventional"]["value"]


@pytest.mark.parametrize("p,n", [(97, 16), (17, 8), (7681, 256), (65537, 64), (65537, 4096)])
def test_h_closed_form(p, n):
    """Closed form: [1,-1] slots <=> h (X^{N/4} + X^{3N/4}) with h^2 = -1/2 mod p."""
    h = h_pn(p, n)
    assert h * h % p == (-pow(2, -1, p)) % p
    assert h_positions(p, n) == [n // 4, 3 * n // 4]


def test_t65537_values():
    """For t = 65537: h = 63481 (= -2056) at N = 4096/8192/16384, k = 32 with [k h]_t = -255."""
    for N in (4096, 8192, 16384):
        z = min_primitive_2n_root(T_PLAIN, N)
        assert pow(z, N, T_PLAIN) == T_PLAIN - 1
    h = h_pn(T_PLAIN, 4096)
    assert h == 63481
    assert find_k(T_PLAIN, h) == 32 and centered(32 * h, T_PLAIN) == -255
    assert find_k(T_PLAIN, h, k_max=31) == 31


def test_primes_in_synth_are_the_largest_ntt_primes():
    """synth.PRIMES = the largest primes < 2^b with q = 1 mod 2^32 (= ntt_primes with 2N = 2^32), so
    NTT-friendly (q = 1 mod 2N) for every configured N."""
    for (N, bits), ps in PRIMES.items():
        assert ntt_primes(2**31, bits, len(ps)) == ps
        assert all(q % (2 * N) == 1 and q % 2**32 == 1 and q < 2**bits for q in ps)


@pytest.mark.parametrize("t,N", [(97, 16), (65537, 64)])
def test_encode_roundtrip_and_constant(t, N):
    g = np.random.default_rng(N)
    v = g.integers(0, t, N)
    assert list(decode(encode(v, t, N), t, N)) == list(v)
    # "the plaintext whose slots are filled with only 1 is simply a constant 1"
    c = encode([1] * N, t, N)
    assert c[0] == 1 and not c[1:].any()


def test_simd_multiplication_and_rotation():
    """Slot-wise product = ring product (PAPER.md:316 SIMD); X -> X^{3^s} rotates both rows left by s
    and X -> X^{2N-1} swaps the rows (reading R7)."""
    t, N = 65537, 64
    g = np.random.default_rng(5)
    a = g.integers(0, t, N)
    b = g.integers(0, t, N)
    pa, pb = encode(a, t, N), encode(b, t, N)
    prod = ring.nc_mul(pa, pb, t)
    assert list(decode(prod, t, N)) == list(a * b % t)
    half = N // 2
    for s in (1, 3, -1, half - 1):
        gg = galois_elt_for_step(N, s)
        r = decode(ring.canon(ring.automorphism(pa, gg), t), t, N)
        exp = np.concatenate([np.roll(a[:half], -s), np.roll(a[half:], -s)])
        assert list(r) == list(exp)
    sw = decode(ring.canon(ring.automorphism(pa, rowswap_elt(N)), t), t, N)
    assert list(sw) == list(np.concatenate([a[half:], a[:half]]))


def test_batch_encode_matches_single():
    t, N = 65537, 128
    g = np.random.default_rng(9)
    V = g.integers(0, t, (3, N))
    E = encode_batch(V, t, N)
    for i in range(3):
        assert list(E[i]) == list(encode(V[i], t, N))
    assert (decode_batch(E, t, N) == V).all()
