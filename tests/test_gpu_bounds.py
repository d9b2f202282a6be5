"""Lazy-accumulation headroom at the planner's bounds (the
MAC accumulates unreduced products and reduces once per output).

The planner admits MAC depth K <= 2^16 and, for c_n = 2, K * k <= 2^21 (hy_plan_layout).  The
kernels' exactness arguments (int8 byte planes: |W x R_b| <= 128 * 255 * K < 2^31 in TMEM; FP64:
30-bit halves x |w| <= 128 summed over K <= 2^16 terms stays below 2^53; the epilogue's
k (B0 + B1) below the 2^62 offset) are checked here at exactly those bounds, on every MAC path
that applies, with every weight of the first output rows = -128 and inputs at the top of their
range:
  * 1x1 layers (K = Jc): coefficient-domain inputs all q - 1 (the tc_coef path reads them as is)
    or the constant polynomial -1, whose NTT is q - 1 in every slot (the NTT-domain paths);
  * 3x3 layers (K = 9 Jc): every input ciphertext is the same random ciphertext, so the oracle
    rotates it once (conv.rotations) and reuses the rotations for every channel (hoisted
    rotations are a deterministic function of the ciphertext); the GPU rotates all of them.
Ciphertext limbs are compared bit for bit with the oracle on output ciphertexts 0 and 1 (weights
rows shared by every Co used).  Marked gpu."""
import numpy as np
import pytest

import synth
from oracle import bfv, conv
from oracle.params import ntt_primes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N = 1024
PRIMES = ntt_primes(N, 50, 2)
OUTS = [0, 1]
_CACHE = {}


@pytest.fixture(scope="module")
def hy():
    import paper_2311_12519_b200 as pkg
    from paper_2311_12519_b200 import build
    build.build()
    pkg.load_library()
    assert torch.cuda.is_available()
    return pkg


def weights(Co, Ci, kk, seed):
    """Rows 0..3 all -128 (row 3 of a c_n = 2 pair: also -128), the rest uniform int8."""
    g = synth.rng(seed, "W")
    W = g.integers(-128, 128, size=(Co, Ci, kk, kk), dtype=np.int64).astype(np.int8)
    W[: min(Co, 4)] = -128
    return W


def inputs(J, domain, seed):
    """[J][2][L][N]: 'coef' = every coefficient q - 1; 'ntt' = the constant polynomial -1; a few
    uniform ciphertexts are mixed in (positions seeded) so an indexing error cannot hide."""
    ct = np.zeros((J, 2, len(PRIMES), N), dtype=np.uint64)
    for l, q in enumerate(PRIMES):
        if domain == "coef":
            ct[:, :, l, :] = q - 1
        else:
            ct[:, :, l, 0] = q - 1
    g = synth.rng(seed, "ct", 1)
    idx = g.choice(J, size=min(J, 16), replace=False)
    ct[idx] = synth.uniform_residues(g, PRIMES, (len(idx), 2, N))
    return ct


def run(hy, W, shape, ct, keys, path):
    p = hy.hy_params_create(N, PRIMES, synth.T_PLAIN, 0)
    try:
        if keys:
            elts = sorted(keys)
            hy.hy_keys_upload(p, elts, np.stack([keys[g] for g in elts]))
        w = hy.hy_encode_weights(p, W, **shape)
        try:
            try:
                hy.hy_weights_set_mac_path(w, path)
            except hy.HyenaError as e:
                assert "not valid" in str(e)
                pytest.skip(f"{path} does not apply")
            lay = hy.hy_weights_layout(w)
            assert lay.J == len(ct)
            d_in = torch.from_numpy(ct).cuda()
            d_out = torch.full((lay.Jout, 2, len(PRIMES), N), 9, dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, d_in, d_out)
            torch.cuda.synchronize()
            return d_out[OUTS[0]:OUTS[-1] + 1].cpu().numpy(), lay
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)


def oracle_1x1(cn, domain, Ci, W, ct, keys):
    key = ("1x1", cn, domain)
    if key not in _CACHE:
        P = bfv.BFVParams(N, PRIMES, synth.T_PLAIN)
        pl = conv.plan(N, 1, Ci, W.shape[0], 1, 1, 1, 1, 0, False, cn)
        ls = conv.setup(pl, synth.T_PLAIN)
        R = {(c, 0): ct[c] for c in range(pl.J)}       # identity tap: R = the ciphertext itself
        _CACHE[key] = conv.he_conv(P, ls, W, ct, keys, out_cts=OUTS, R=R), ls
    return _CACHE[key]


def oracle_3x3(cn, Ci, W, ct, keys):
    key = ("3x3", cn)
    if key not in _CACHE:
        P = bfv.BFVParams(N, PRIMES, synth.T_PLAIN)
        pl = conv.plan(N, 1, Ci, W.shape[0], 2, 2, 3, 3, 1, False, cn)
        ls = conv.setup(pl, synth.T_PLAIN)
        R1 = conv.rotations(P, pl, ct, keys, cts=[0])
        R = {(c, tau): R1[(0, tau)] for c in range(pl.J) for tau in range(len(pl.taps))}
        _CACHE[key] = conv.he_conv(P, ls, W, ct, keys, out_cts=OUTS, R=R), ls
    return _CACHE[key]


def uniform_keys(elts, seed):
    kk = synth.gen_uniform_keys(PRIMES, len(elts), N, seed)
    return {g: kk[n] for n, g in enumerate(elts)}


PATHS_1x1 = ["tc_coef", "tc_fused", "tc_split", "fp64_fused", "fp64_split"]


@pytest.mark.parametrize("path", PATHS_1x1)
def test_bound_1x1_cn1_K65536(hy, path):
    """c_n = 1, K = Jc = 2^16 (the planner's maximum), every weight of rows 0..3 = -128."""
    Ci = 1 << 16
    Co = 32 if path == "fp64_fused" else 34          # fp64_fused needs M <= 32, fp64_split M > 32
    W = weights(34, Ci, 1, 901)[:Co]
    domain = "coef" if path == "tc_coef" else "ntt"
    ct = inputs(Ci, domain, 902)
    shape = dict(Ci=Ci, Co=Co, H=1, W=1, kh=1, kw=1, pad=0, batch=1, force_cn=1)
    got, lay = run(hy, W, shape, ct, {}, path)
    assert lay.cn == 1 and lay.Jc * lay.n_taps == 1 << 16
    ref, _ = oracle_1x1(1, domain, Ci, weights(34, Ci, 1, 901), ct, {})
    for n, oc in enumerate(OUTS):
        assert np.array_equal(got[n], ref[oc]), f"{path}: output ct {oc} differs at K = 2^16"


@pytest.mark.parametrize("path", PATHS_1x1)
def test_bound_1x1_cn2_Kk2pow21(hy, path):
    """c_n = 2, k = 32, K = Jc = 2^16: K * k = 2^21 (the planner's maximum)."""
    Ci = 1 << 17
    Co = 16 if path == "fp64_fused" else 18          # M = 4 Jo: 32 vs 36
    W = weights(18, Ci, 1, 903)[:Co]
    domain = "coef" if path == "tc_coef" else "ntt"
    ct = inputs(Ci // 2, domain, 904)
    keys = uniform_keys([2 * N - 1], 905)
    shape = dict(Ci=Ci, Co=Co, H=1, W=1, kh=1, kw=1, pad=0, batch=1, force_cn=2, k=32)
    got, lay = run(hy, W, shape, ct, keys, path)
    assert lay.cn == 2 and lay.k == 32 and lay.Jc * lay.k == 1 << 21
    ref, _ = oracle_1x1(2, domain, Ci, weights(18, Ci, 1, 903), ct, keys)
    for n, oc in enumerate(OUTS):
        assert np.array_equal(got[n], ref[oc]), f"{path}: output ct {oc} differs at K k = 2^21"


PATHS_3x3 = ["tc_fused", "tc_split", "fp64_fused", "fp64_split"]


@pytest.mark.parametrize("path", PATHS_3x3)
def test_bound_3x3_cn1_K65529(hy, path):
    """c_n = 1, 3x3, Jc = 7281: K = 65529 terms, every one a key-switched rotation."""
    Ci = 7281
    Co = 32 if path == "fp64_fused" else 34
    W = weights(34, Ci, 3, 906)[:Co]
    one = synth.gen_uniform_cts(PRIMES, 1, N, 907)
    ct = np.ascontiguousarray(np.broadcast_to(one, (Ci,) + one.shape[1:]))
    shape = dict(Ci=Ci, Co=Co, H=2, W=2, kh=3, kw=3, pad=1, batch=1, force_cn=1)
    lay0 = hy.hy_plan_layout(N, synth.T_PLAIN, **shape)
    keys = uniform_keys(list(lay0.galois[:lay0.n_galois]), 908)
    got, lay = run(hy, W, shape, ct, keys, path)
    assert lay.Jc * lay.n_taps == 65529
    ref, _ = oracle_3x3(1, Ci, weights(34, Ci, 3, 906), ct, keys)
    for n, oc in enumerate(OUTS):
        assert np.array_equal(got[n], ref[oc]), f"{path}: output ct {oc} differs at K = 65529"


@pytest.mark.parametrize("path", PATHS_3x3)
def test_bound_3x3_cn2_Kk(hy, path):
    """c_n = 2, k = 32, 3x3, Jc = 7281: K = 65529, K * k = 2096928 <= 2^21."""
    Ci = 2 * 7281
    Co = 16 if path == "fp64_fused" else 18
    W = weights(18, Ci, 3, 909)[:Co]
    one = synth.gen_uniform_cts(PRIMES, 1, N, 910)
    ct = np.ascontiguousarray(np.broadcast_to(one, (Ci // 2,) + one.shape[1:]))
    shape = dict(Ci=Ci, Co=Co, H=2, W=2, kh=3, kw=3, pad=1, batch=1, force_cn=2, k=32)
    lay0 = hy.hy_plan_layout(N, synth.T_PLAIN, **shape)
    keys = uniform_keys(list(lay0.galois[:lay0.n_galois]), 911)
    got, lay = run(hy, W, shape, ct, keys, path)
    assert lay.cn == 2 and lay.Jc * lay.n_taps * lay.k == 65529 * 32
    ref, _ = oracle_3x3(2, Ci, weights(18, Ci, 3, 909), ct, keys)
    for n, oc in enumerate(OUTS):
        assert np.array_equal(got[n], ref[oc]), f"{path}: output ct {oc} differs at K k = 2096928"


def test_planner_rejects_beyond_bounds(hy):
    """One term more than the bound is refused (HY_ESHAPE), not silently inexact.  (With k <= 32
    = 2^5, K <= 2^16 already implies K k <= 2^21: the second bound never binds first.)"""
    for cn, Ci in ((1, (1 << 16) + 1), (2, (1 << 17) + 2)):
        with pytest.raises(hy.HyenaError, match="2\\^16"):
            hy.hy_plan_layout(N, synth.T_PLAIN, Ci=Ci, Co=2, H=1, W=1, kh=1, kw=1, pad=0, batch=1, force_cn=cn)
    with pytest.raises(hy.HyenaError, match="2\\^16"):
        hy.hy_plan_layout(N, synth.T_PLAIN, Ci=7282, Co=2, H=2, W=2, kh=3, kw=3, pad=1, batch=1, force_cn=1)
