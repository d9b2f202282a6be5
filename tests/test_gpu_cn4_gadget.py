"""GPU parity of c_n = 4 Walsh-Hadamard packing and of the
sub-digit decomposition base (NEXT-4; PAPER.md:1470 [app]) against the oracle: ciphertext limbs bit
for bit and decryption = plain convolution mod t, including BASELINE C1 packed as ONE ciphertext.
Marked gpu."""
import numpy as np
import pytest

import synth
from oracle import bfv, conv
from oracle.params import ntt_primes
from synth import philox
from tests.hyena_client import check_decrypted, make_layer

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


def shape_of(lay):
    p = lay.plan
    return dict(Ci=p.Ci, Co=p.Co, H=p.H, W=p.W, kh=p.kh, kw=p.kw, pad=p.pad, depthwise=int(p.depthwise),
                batch=p.batch, k=lay.ls.k if p.cn == 2 else 0, force_cn=p.cn)


def run(hy, lay, path=None):
    p = hy.hy_params_create(lay.P.N, lay.P.primes, lay.P.t, 0, w_dcmp=lay.P.w)
    try:
        elts = list(lay.keys)
        if elts:
            hy.hy_keys_upload(p, elts, np.stack([lay.keys[g] for g in elts]))
        w = hy.hy_encode_weights(p, lay.W, **shape_of(lay))
        try:
            if path is not None:
                try:
                    hy.hy_weights_set_mac_path(w, path)
                except hy.HyenaError as e:
                    assert "not valid" in str(e)
                    pytest.skip(f"{path} does not apply")
            L = hy.hy_weights_layout(w)
            assert (L.J, L.Jout, L.cn, L.scale) == (lay.plan.J, lay.plan.Jout, lay.plan.cn, lay.ls.scale)
            assert sorted(L.galois[:L.n_galois]) == sorted(lay.ls.galois)
            out = torch.full((L.Jout, 2, lay.P.L, lay.P.N), 3, dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, torch.from_numpy(lay.ct_in).cuda(), out)
            torch.cuda.synchronize()
            dec = hy.hy_decrypt_debug(p, lay.s.astype(np.int8), out, L.scale)
            return out.cpu().numpy(), dec, hy.hy_weights_mac_path(w)
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)


def compare(lay, got, dec):
    ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    for i in range(lay.plan.Jout):
        assert np.array_equal(got[i], ref[i]), f"output ct {i} differs from the oracle"
    check_decrypted(lay, {i: got[i] for i in range(lay.plan.Jout)})
    assert np.array_equal(conv.unpack(lay.plan, dec.astype(np.int64)),
                          np.mod(conv.plain_conv(lay.x, lay.W, lay.plan.pad, lay.plan.depthwise), lay.P.t))


CN4 = {
    # fp64_fused (M = 16 Jo <= 32) with a ragged last channel group, and fp64_split (M > 32)
    "cn4_fused": dict(N=1024, bits=50, L=3, batch=3, Ci=6, Co=7, H=6, W=6, kh=3, kw=3, pad=1),
    "cn4_split": dict(N=1024, bits=50, L=3, batch=1, Ci=4, Co=12, H=5, W=5, kh=3, kw=3, pad=1),
    "cn4_1x1": dict(N=1024, bits=50, L=2, batch=2, Ci=8, Co=4, H=6, W=6, kh=1, kw=1, pad=0),
}


@pytest.mark.parametrize("w", [0, 20])
@pytest.mark.parametrize("name", sorted(CN4))
def test_cn4_bit_exact(hy, name, w):
    c = dict(CN4[name])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=1300 + sorted(CN4).index(name), force_cn=4, w=w,
                     xrange=(-128, 128), wrange=(-128, 128), **c)
    got, dec, path = run(hy, lay)
    assert path in ("fp64_fused", "fp64_split")
    compare(lay, got, dec)


def test_c1_in_one_ciphertext(hy):
    """BASELINE configs[0] (C1): 4 channels of 8 x 8 in ONE N = 4096 ciphertext (c_n = 4) with the
    2^25 sub-digit base the noise needs (tests/test_oracle_conv.py pins both)."""
    cfg = synth.configs()["C1"]
    lay = make_layer(cfg.N, cfg.primes, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad,
                     seed=cfg.index, force_cn=4, x=synth.gen_image(cfg), Wt=synth.gen_weights(cfg), w=25)
    assert (lay.plan.J, lay.plan.Jout) == (1, 1)
    got, dec, _ = run(hy, lay)
    compare(lay, got, dec)


GADGET = {
    "cn2_blocks": dict(N=1024, bits=50, L=2, batch=2, Ci=4, Co=4, H=5, W=5, kh=3, kw=3, pad=1),
    "cn1_bands": dict(N=1024, bits=50, L=3, batch=1, Ci=3, Co=2, H=20, W=20, kh=3, kw=3, pad=1),
    "dw_cn2": dict(N=1024, bits=50, L=2, batch=2, Ci=4, Co=4, H=6, W=6, kh=3, kw=3, pad=1, depthwise=True),
    "pw_cn2": dict(N=1024, bits=50, L=2, batch=2, Ci=4, Co=4, H=6, W=6, kh=1, kw=1, pad=0),
    "tc_rows70": dict(N=1024, bits=50, L=3, batch=17, Ci=3, Co=70, H=6, W=6, kh=3, kw=3, pad=1),
}


@pytest.mark.parametrize("path", [None, "tc_split", "fp64_split"])
@pytest.mark.parametrize("name", sorted(GADGET))
def test_subdigit_base_bit_exact(hy, name, path):
    """Every layout kind with a 2^20 sub-digit base (digits floor([c1]_{q_i} / 2^{20 v}) mod 2^20)."""
    c = dict(GADGET[name])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=1400 + sorted(GADGET).index(name), w=20, **c)
    assert lay.P.ND == 3 * L
    got, dec, _ = run(hy, lay, path)
    compare(lay, got, dec)


def test_gpu_keygen_with_subdigit_base(hy):
    N, primes = 1024, ntt_primes(1024, 50, 2)
    P = bfv.BFVParams(N, primes, synth.T_PLAIN, w=20)
    seed = 0x6A6
    p = hy.hy_params_create(N, primes, synth.T_PLAIN, 0, w_dcmp=20)
    try:
        s = philox.secret(seed, N)
        elts = [3, 2 * N - 1]
        kd = torch.zeros((2, P.ND, 2, len(primes), N), dtype=torch.uint64, device="cuda")
        hy.hy_keygen(p, seed, elts, kd, upload=False)
        got = kd.cpu().numpy()
        for n, g in enumerate(elts):
            ref = bfv.galois_keygen(P, s, g, philox.key_mask(seed, g, primes, N, P.ND),
                                    philox.key_error(seed, g, P.ND, N))
            assert np.array_equal(got[n], ref)
    finally:
        hy.hy_params_destroy(p)


def test_bad_bases_rejected(hy):
    primes = ntt_primes(1024, 50, 2)
    for w in (1, 3, 50, 64):
        with pytest.raises(hy.HyenaError, match="decomposition base"):
            hy.hy_params_create(1024, primes, synth.T_PLAIN, 0, w_dcmp=w)
