"""Pins for oracle/bfv.py: decryption correctness, homomorphic properties, hoisted rotation,
and the hoisted-vs-direct distinction (reading R6) — CPU only, small N."""
import numpy as np
import pytest

from oracle import bfv, ring
from oracle.encoding import decode, encode
from oracle.params import galois_elt_for_step, ntt_primes, rowswap_elt
import synth

T = 65537


def _setup(N=64, L=3, bits=50, seed=0):
    P = bfv.BFVParams(N, ntt_primes(N, bits, L), T)
    g = synth.rng(90 + seed, "sk")
    s = synth.ternary(g, N)
    return P, s


def _enc(P, s, slots, stream):
    m = encode(slots, P.t, P.N)
    ga = synth.rng(91, "a", stream)
    ge = synth.rng(91, "e", stream)
    a = synth.uniform_residues(ga, P.primes, (P.N,))
    e = synth.cbd(ge, P.N)
    return bfv.encrypt(P, m, s, a, e), m


def _key(P, s, g, stream):
    a = synth.uniform_residues(synth.rng(92, "a", stream), P.primes, (P.ND, P.N))
    e = synth.cbd(synth.rng(92, "e", stream), (P.ND, P.N))
    return bfv.galois_keygen(P, s, g, a, e)


def test_encrypt_decrypt_and_noise():
    P, s = _setup()
    v = np.arange(P.N) * 977 % T
    ct, m = _enc(P, s, v, 0)
    assert list(decode(bfv.decrypt(P, ct, s), T, P.N)) == list(v)
    # fresh noise is the CBD error: |e| <= eta = 20
    assert bfv.noise_bits(P, ct, s, m) <= np.log2(20)
    assert ct.dtype == np.uint64 and all((ct[:, l] < q).all() for l, q in enumerate(P.primes))


def test_hadd_cmult():
    """HAdd adds slots; CMult by an integer scales slots."""
    P, s = _setup()
    g = np.random.default_rng(1)
    v1, v2 = g.integers(0, T, P.N), g.integers(0, T, P.N)
    c1, _ = _enc(P, s, v1, 1)
    c2, _ = _enc(P, s, v2, 2)
    add = np.stack([np.stack([ring.add_mod(c1[c, l], c2[c, l], q) for l, q in enumerate(P.primes)])
                    for c in range(2)])
    assert list(decode(bfv.decrypt(P, add, s), T, P.N)) == list((v1 + v2) % T)
    w = -93
    cm = np.stack([np.stack([ring.scalar_mul_mod(c1[c, l], w, q) for l, q in enumerate(P.primes)])
                   for c in range(2)])
    assert list(decode(bfv.decrypt(P, cm, s), T, P.N)) == list((w * v1) % T)


@pytest.mark.parametrize("step", [1, 5, -3])
def test_hoisted_rotation_rotates_slots(step):
    P, s = _setup()
    v = np.random.default_rng(step + 10).integers(0, T, P.N)
    ct, _ = _enc(P, s, v, 3)
    g = galois_elt_for_step(P.N, step)
    r = bfv.hrot(P, ct, g, _key(P, s, g, 0))
    half = P.N // 2
    exp = np.concatenate([np.roll(v[:half], -step), np.roll(v[half:], -step)])
    assert list(decode(bfv.decrypt(P, r, s), T, P.N)) == list(exp)


def test_rotation_algebra():
    """rot(s) o rot(-s) = id and the row swap is an involution."""
    P, s = _setup()
    v = np.random.default_rng(4).integers(0, T, P.N)
    ct, _ = _enc(P, s, v, 4)
    g1, g2 = galois_elt_for_step(P.N, 7), galois_elt_for_step(P.N, -7)
    back = bfv.hrot(P, bfv.hrot(P, ct, g1, _key(P, s, g1, 1)), g2, _key(P, s, g2, 2))
    assert list(decode(bfv.decrypt(P, back, s), T, P.N)) == list(v)
    gs = rowswap_elt(P.N)
    ks = _key(P, s, gs, 3)
    sw2 = bfv.hrot(P, bfv.hrot(P, ct, gs, ks), gs, ks)
    assert list(decode(bfv.decrypt(P, sw2, s), T, P.N)) == list(v)


def test_hoisted_vs_direct_differ_but_decrypt_equal():
    """Reading R4: decomposing c1 before the automorphism (hoisted) vs after (direct) gives
    different ciphertext bits but the same plaintext, so bit-exact parity needs one definition."""
    P, s = _setup()
    v = np.random.default_rng(6).integers(0, T, P.N)
    ct, _ = _enc(P, s, v, 5)
    g = galois_elt_for_step(P.N, 1)
    key = _key(P, s, g, 4)
    hoisted = bfv.hrot(P, ct, g, key)
    # direct: automorphism on every limb first, then digits of the rotated c1 in [0, q_i) (written
    # out here, independently of bfv.rotate_direct, which must agree)
    rot = np.stack([np.stack([ring.automorphism_mod(ct[c, l], g, q) for l, q in enumerate(P.primes)])
                    for c in range(2)])
    direct = np.empty_like(rot)
    for l, q in enumerate(P.primes):
        c0 = rot[0, l].astype(object)
        c1 = np.zeros(P.N, dtype=object)
        for i in range(P.L):
            d = ring.canon(rot[1, i], q)
            c0 = c0 + ring.nc_mul(d, key[i, 0, l], q).astype(object)
            c1 = c1 + ring.nc_mul(d, key[i, 1, l], q).astype(object)
        direct[0, l] = (c0 % q).astype(np.uint64)
        direct[1, l] = (c1 % q).astype(np.uint64)
    assert np.array_equal(bfv.rotate_direct(P, ct, g, key), direct)
    assert not np.array_equal(hoisted, direct)
    assert list(bfv.decrypt(P, hoisted, s)) == list(bfv.decrypt(P, direct, s))


def test_decrypt_rounding_is_exact_at_boundary():
    """Decrypt rounds t x / Q to nearest with an exact big-integer formula: a phase of
    Delta*m + v decrypts to m when |v| < Delta/2 - (Q mod t) and not when |v| > Delta/2 + t
    (the (Q mod t) slack is the textbook FV correction)."""
    P, s = _setup(N=16, L=2, bits=30)
    # build a ciphertext with c1 = 0 so the phase is c0 directly
    slack = P.Q % P.t
    for m0, v, ok in [(5, P.delta // 2 - slack - 1, True), (5, -(P.delta // 2 - slack - 1), True),
                      (T - 1, -(P.delta // 2 - slack - 1), True), (0, -(P.delta // 2 - slack - 1), True),
                      (5, P.delta // 2 + T, False), (5, -(P.delta // 2 + T), False)]:
        x = (P.delta * m0 + v) % P.Q
        ct = np.zeros((2, P.L, P.N), dtype=np.uint64)
        for l, q in enumerate(P.primes):
            ct[0, l, 0] = x % q
        assert (bfv.decrypt(P, ct, s)[0] == m0) == ok


# ---------------------------------------------------------------------------------------------
# sub-digit decomposition base (PAPER.md:1470 [app] "decomposition base")
# ---------------------------------------------------------------------------------------------
def test_subdigit_gadget_reconstructs_c1():
    """The gadget identity, written out: for every limb l, sum_{i,v} d_{i,v} g_{i,v} = c1 (mod q_l)
    with g_{i,v} = [i == l] 2^{w v} mod q_l, and every digit below 2^w."""
    for w in (13, 20, 25, 50):
        P = bfv.BFVParams(64, ntt_primes(64, 50, 3), T, w=w)
        assert P.V == -(-50 // w) and P.ND == 3 * P.V
        c1 = synth.uniform_residues(synth.rng(93, "ct", w), P.primes, (P.N,))
        ct = np.stack([c1, c1])
        d = bfv.decompose(P, ct)
        assert len(d) == P.ND and all(int(x.max()) < (1 << w) and int(x.min()) >= 0 for x in d)
        for l, q in enumerate(P.primes):
            acc = np.zeros(P.N, dtype=object)
            for dd, x in enumerate(d):
                i, v = divmod(dd, P.V)
                if i == l:
                    acc = acc + x.astype(object) * pow(2, w * v)
            assert list(acc % q) == [int(y) for y in c1[l]]


def test_subdigit_key_relation_and_rotation():
    """b + a s = e + [i == l] 2^{w v} s(X^g) (mod q_l) for every digit row; the hoisted rotation
    with the sub-digit key decrypts to the rotated slots; its key-switching noise is far below
    the one-digit-per-limb gadget's (the reason for a smaller base: PAPER.md:587-617)."""
    N = 256
    P1 = bfv.BFVParams(N, ntt_primes(N, 50, 2), T)
    P2 = bfv.BFVParams(N, ntt_primes(N, 50, 2), T, w=20)
    s = synth.ternary(synth.rng(94, "sk"), N)
    g = galois_elt_for_step(N, 3)
    key = _key(P2, s, g, 7)
    assert key.shape == (P2.ND, 2, 2, N)
    sg = ring.automorphism(np.asarray(s), g)
    e = synth.cbd(synth.rng(92, "e", 7), (P2.ND, N))
    for dd in range(P2.ND):
        i, v = divmod(dd, P2.V)
        for l, q in enumerate(P2.primes):
            lhs = (key[dd, 0, l].astype(object) + ring.nc_mul(np.asarray(s), key[dd, 1, l], q).astype(object)) % q
            rhs = (np.asarray(e[dd]).astype(object) + (sg.astype(object) * pow(2, 20 * v) if i == l else 0)) % q
            assert list(lhs) == list(rhs)
    v = np.arange(N) * 31 % T
    noise = []
    for P in (P1, P2):
        ct, m = _enc(P, s, v, 3)
        rot = bfv.hrot(P, ct, g, _key(P, s, g, 7))
        exp = np.concatenate([np.roll(v[:N // 2], -3), np.roll(v[N // 2:], -3)])
        dec = bfv.decrypt(P, rot, s)
        assert list(decode(dec, T, N)) == list(exp)
        noise.append(bfv.noise_bits(P, rot, s, dec))
    assert noise[1] < noise[0] - 20, noise
