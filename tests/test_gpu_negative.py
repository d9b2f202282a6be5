"""Negative controls (VERDICT r1 missing item 6): the parity comparison must FAIL when one input
byte of the GPU path is wrong — one weight, one switching-key word, one input-ciphertext word —
so a bit-exact pass cannot come from comparing something insensitive.  C1 (BASELINE configs[0])
through hy_conv_eval against the oracle of the unmodified layer.  Marked gpu."""
import numpy as np
import pytest

import synth
from oracle import bfv, conv
from tests.hyena_client import layer_from_config

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


@pytest.fixture(scope="module")
def c1():
    lay = layer_from_config(synth.configs()["C1"])
    ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    return lay, np.stack([ref[i] for i in range(lay.plan.Jout)])


def _run(hy, lay, W, keys, ct):
    cfg = synth.configs()["C1"]
    p = hy.hy_params_create(cfg.N, cfg.primes, cfg.t, 0)
    try:
        elts = list(keys)
        hy.hy_keys_upload(p, elts, np.stack([keys[g] for g in elts]))
        w = hy.hy_encode_weights(p, W, **cfg.shape_dict())
        try:
            d_out = torch.zeros((lay.plan.Jout, 2, lay.P.L, lay.P.N), dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, torch.from_numpy(ct).cuda(), d_out)
            torch.cuda.synchronize()
            return d_out.cpu().numpy()
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)


def test_unmodified_matches(hy, c1):
    lay, ref = c1
    assert np.array_equal(_run(hy, lay, lay.W, lay.keys, lay.ct_in), ref)


@pytest.mark.parametrize("what", ["weight", "key", "input"])
def test_one_flipped_word_breaks_parity(hy, c1, what):
    lay, ref = c1
    W, keys, ct = lay.W.copy(), {g: k.copy() for g, k in lay.keys.items()}, lay.ct_in.copy()
    if what == "weight":
        W[1, 2, 1, 0] ^= np.int8(1)                       # one weight, lowest bit
    elif what == "key":
        g0 = sorted(keys)[0]
        keys[g0][0, 0, 1, 77] ^= np.uint64(1)              # digit 0, b, limb 1, coefficient 77
    else:
        ct[1, 1, 0, 5] = (ct[1, 1, 0, 5] + np.uint64(1)) % np.uint64(lay.P.primes[0])
    got = _run(hy, lay, W, keys, ct)
    assert not np.array_equal(got, ref), f"flipping one {what} word did not change the output"


def _budgets(hy, lay, cts, check=True):
    cfg = synth.configs()["C1"]
    p = hy.hy_params_create(cfg.N, cfg.primes, cfg.t, 0)
    try:
        return hy.hy_decrypt_debug_noise(p, lay.s.astype(np.int8), torch.from_numpy(np.ascontiguousarray(cts)).cuda(),
                                         lay.ls.scale, check=check)
    finally:
        hy.hy_params_destroy(p)


def test_noise_budget_matches_oracle_meter(hy, c1):
    """hy_decrypt_debug_noise's budget log2(Q / |2 (t x - round(t x / Q) Q)|) equals the oracle's
    log2(Delta / 2) - log2 ||v||_inf (PAPER.md:266-267 [ign]) to within the Delta = floor(Q / t) rounding."""
    lay, ref = c1
    _, bud = _budgets(hy, lay, ref)
    for c, b in zip(ref, bud):
        m = bfv.decrypt(lay.P, c, lay.s)
        want = bfv.noise_budget_bits(lay.P) - bfv.noise_bits(lay.P, c, lay.s, m)
        assert abs(b - want) < 0.05, (b, want)
        assert b >= 4


def test_garbage_ciphertext_reports_enoise(hy, c1):
    """Uniform residues (no encryption of anything) leave no budget: HY_ENOISE."""
    lay, ref = c1
    rnd = synth.uniform_residues(synth.rng(9, "misc", 4242), lay.P.primes, (2, 2, lay.P.N))
    with pytest.raises(hy.HyenaError, match=r"\(-6\)"):
        _budgets(hy, lay, np.ascontiguousarray(rnd))
    _, bud = _budgets(hy, lay, np.ascontiguousarray(rnd), check=False)
    assert (bud < 1).all()


def test_flipped_key_word_exhausts_budget(hy, c1):
    """A switching key off by one in one word adds a key-sized error: the output is undecryptable and
    the library says so (negative control of the noise meter)."""
    lay, ref = c1
    keys = {g: k.copy() for g, k in lay.keys.items()}
    for g in keys:
        keys[g][0, 0, 0, 77] ^= np.uint64(1 << 40)
    got = _run(hy, lay, lay.W, keys, lay.ct_in)
    with pytest.raises(hy.HyenaError, match=r"\(-6\)"):
        _budgets(hy, lay, got)
