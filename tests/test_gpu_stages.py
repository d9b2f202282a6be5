"""GPU parity, per stage (T1): NTT products and hoisted rotations through the C-ABI vs the oracle,
bit-exact.  Marked gpu."""
import numpy as np
import pytest

import synth
from oracle import bfv, ring
from oracle.params import galois_elt_for_step, ntt_primes, rowswap_elt

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hy():
    import paper_2311_12519_b200 as pkg
    from paper_2311_12519_b200 import build
    build.build()
    pkg.load_library()
    assert torch.cuda.is_available()
    return pkg


PARAMS = [(1024, 50, 2), (4096, 50, 2), (8192, 60, 3), (16384, 60, 5)]


@pytest.mark.parametrize("N,bits,L", PARAMS)
def test_poly_mul_matches_schoolbook(hy, N, bits, L):
    primes = ntt_primes(N, bits, L)
    p = hy.hy_params_create(N, primes, 65537)
    try:
        g = synth.rng(200 + L, "misc")
        n = 2
        a = synth.uniform_residues(g, primes, (n, N))
        b = synth.uniform_residues(g, primes, (n, N))
        # edge values: all q-1 in one poly, zeros in another
        for l, q in enumerate(primes):
            a[1, l, :] = q - 1
            b[1, l, : N // 2] = 0
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        dc = torch.empty_like(da)
        hy.hy_poly_mul(p, da, db, dc)
        c = dc.cpu().numpy()
        for i in range(n):
            for l, q in enumerate(primes):
                assert np.array_equal(c[i, l], ring.nc_mul(a[i, l], b[i, l], q)), (i, l)
    finally:
        hy.hy_params_destroy(p)


@pytest.mark.parametrize("N,bits,L", [(4096, 50, 2), (8192, 60, 3), (8192, 59, 2)])
def test_throughput_ntt_kernels(hy, N, bits, L):
    """Launches of >= 592 transforms take the one-CTA-per-transform kernels (ntt2_*: inline-PTX
    butterflies, conditional subtraction on every other forward stage): products of edge-valued and
    random polynomials against the schoolbook oracle, and NTT -> INTT = identity on all of them."""
    primes = ntt_primes(N, bits, L)
    p = hy.hy_params_create(N, primes, 65537)
    try:
        g = synth.rng(210 + L, "misc")
        n = 600 // L + 8
        a = synth.uniform_residues(g, primes, (n, N))
        b = synth.uniform_residues(g, primes, (n, N))
        for l, q in enumerate(primes):
            a[0, l, :], b[0, l, :] = q - 1, q - 1          # largest residues everywhere
            a[1, l, :], b[1, l, : N // 2] = q - 1, 0
            a[2, l, :] = 0
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        dc = torch.empty_like(da)
        hy.hy_poly_mul(p, da, db, dc)
        c = dc.cpu().numpy()
        for i in (0, 1, 2, 3, n - 1):
            for l, q in enumerate(primes):
                assert np.array_equal(c[i, l], ring.nc_mul(a[i, l], b[i, l], q)), (i, l)
        hy.hy_ntt_roundtrip(p, da)
        assert np.array_equal(da.cpu().numpy(), a)
    finally:
        hy.hy_params_destroy(p)


@pytest.mark.parametrize("N,bits,L", PARAMS)
def test_ntt_roundtrip(hy, N, bits, L):
    primes = ntt_primes(N, bits, L)
    p = hy.hy_params_create(N, primes, 65537)
    try:
        x = synth.uniform_residues(synth.rng(300, "misc"), primes, (8, N))
        for l, q in enumerate(primes):
            x[0, l, :] = q - 1
            x[1, l, :] = 0
        dx = torch.from_numpy(x).cuda()
        for _ in range(10):
            hy.hy_ntt_roundtrip(p, dx)
        assert np.array_equal(dx.cpu().numpy(), x)
    finally:
        hy.hy_params_destroy(p)


@pytest.mark.parametrize("N,bits,L,steps", [(1024, 50, 2, [1, -1, 17]), (4096, 50, 2, [1, -16]),
                                             (8192, 60, 3, [-65, 1]), (16384, 60, 5, [3])])
def test_hoisted_rotation_bit_exact(hy, N, bits, L, steps):
    """S1+S2 (PermDecomp + PermAuto) and S5 vs oracle.bfv.hrot on real encryptions; also the row swap."""
    primes = ntt_primes(N, bits, L)
    P = bfv.BFVParams(N, primes, 65537)
    s = synth.ternary(synth.rng(400, "sk"), N)
    from tests.hyena_client import encrypt_slots, keygen
    v = synth.uniform_int(synth.rng(400, "x"), 0, 65537, (2, N))
    cts = encrypt_slots(P, s, v, 400)
    elts = [galois_elt_for_step(N, st) for st in steps] + [rowswap_elt(N)]
    keys = keygen(P, s, elts, 400)
    p = hy.hy_params_create(N, primes, 65537)
    try:
        hy.hy_keys_upload(p, elts, np.stack([keys[g] for g in elts]))
        din = torch.from_numpy(cts).cuda()
        dout = torch.empty_like(din)
        for g in elts[:2] + [elts[-1]]:
            hy.hy_rotate(p, din, g, dout)
            got = dout.cpu().numpy()
            for i in range(len(cts)):
                ref = bfv.hrot(P, cts[i], g, keys[g])
                assert np.array_equal(got[i], ref), (g, i)
        # decryption of the GPU rotation (library debug decrypt) = rotated slots
        g = elts[0]
        hy.hy_rotate(p, din, g, dout)
        slots = hy.hy_decrypt_debug(p, s.astype(np.int8), dout, 1)
        half = N // 2
        for i in range(len(cts)):
            exp = np.concatenate([np.roll(v[i, :half], -steps[0]), np.roll(v[i, half:], -steps[0])])
            assert np.array_equal(slots[i].astype(np.int64), exp)
    finally:
        hy.hy_params_destroy(p)


def test_missing_key_is_reported(hy):
    N = 1024
    primes = ntt_primes(N, 50, 2)
    p = hy.hy_params_create(N, primes, 65537)
    try:
        x = torch.zeros((1, 2, 2, N), dtype=torch.uint64, device="cuda")
        with pytest.raises(hy.HyenaError, match="no Galois key"):
            hy.hy_rotate(p, x, 3, x)
    finally:
        hy.hy_params_destroy(p)
