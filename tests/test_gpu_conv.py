"""GPU parity of the whole encrypted convolution (hy_conv_eval) vs the oracle (T2):
ciphertext limbs bit-exact, and decryption = plain convolution mod t.  Marked gpu."""
import numpy as np
import pytest

import synth
from oracle import bfv, conv
from oracle.params import ntt_primes
from tests.hyena_client import check_decrypted, layer_from_config, make_layer

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


def run_gpu(hy, lay, shape_kw, units=None, path=None):
    p = hy.hy_params_create(lay.P.N, lay.P.primes, lay.P.t, 0)
    try:
        elts = list(lay.keys)
        if elts:
            hy.hy_keys_upload(p, elts, np.stack([lay.keys[g] for g in elts]))
        w = hy.hy_encode_weights(p, lay.W, **shape_kw)
        try:
            if path is not None:
                try:
                    hy.hy_weights_set_mac_path(w, path)
                except hy.HyenaError as e:
                    assert "not valid" in str(e)
                    pytest.skip(f"MAC path {path} does not apply to this layout")
                assert hy.hy_weights_mac_path(w) == path
            L = hy.hy_weights_layout(w)
            assert (L.J, L.Jout, L.cn, L.k) == (lay.plan.J, lay.plan.Jout, lay.plan.cn, lay.ls.k)
            nu = L.U if units is None else units
            ct_in = torch.from_numpy(lay.ct_in[: nu * L.Jc]).cuda()
            ct_out = torch.full((nu * L.Jo, 2, lay.P.L, lay.P.N), 7, dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, ct_in, ct_out)
            torch.cuda.synchronize()
            got = ct_out.cpu().numpy()
            # library debug decryption of everything (checked against the plain conv below)
            dec = hy.hy_decrypt_debug(p, lay.s.astype(np.int8), ct_out, L.scale)
            # end-to-end host API gives the same bytes
            host_out = np.zeros_like(got)
            hy.hy_conv_eval_host(w, np.ascontiguousarray(lay.ct_in[: nu * L.Jc]), host_out)
            assert np.array_equal(host_out, got)
            return got, dec, L
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)


def shape_of(lay):
    p = lay.plan
    return dict(Ci=p.Ci, Co=p.Co, H=p.H, W=p.W, kh=p.kh, kw=p.kw, pad=p.pad, depthwise=int(p.depthwise),
                batch=p.batch, k=lay.ls.k if p.cn == 2 else 0, force_cn=p.cn)


def check_plain_from_library_decrypt(lay, dec):
    p = lay.plan
    got = conv.unpack(p, dec.astype(np.int64))
    from tests.hyena_client import expected_plain
    exp = expected_plain(lay)
    sel = (slice(None),) * 4
    assert np.array_equal(got, exp)


CASES = {
    "cn2_blocks": dict(N=1024, bits=50, L=2, batch=2, Ci=4, Co=4, H=5, W=5, kh=3, kw=3, pad=1),
    "cn2_k1": dict(N=1024, bits=50, L=2, batch=1, Ci=4, Co=6, H=6, W=6, kh=3, kw=3, pad=1, k=1),
    "cn2_odd_channels": dict(N=2048, bits=60, L=3, batch=1, Ci=3, Co=5, H=7, W=7, kh=3, kw=3, pad=1),
    "cn1_bands": dict(N=1024, bits=50, L=2, batch=1, Ci=3, Co=2, H=20, W=20, kh=3, kw=3, pad=1),
    "cn1_blocks_tail": dict(N=1024, bits=50, L=2, batch=5, Ci=2, Co=3, H=6, W=6, kh=3, kw=3, pad=1, force_cn=1),
    "dw_cn2": dict(N=1024, bits=50, L=2, batch=2, Ci=4, Co=4, H=6, W=6, kh=3, kw=3, pad=1, depthwise=True),
    "dw_cn1": dict(N=1024, bits=50, L=2, batch=9, Ci=3, Co=3, H=6, W=6, kh=3, kw=3, pad=1, depthwise=True),
    "pw_cn1": dict(N=1024, bits=50, L=2, batch=9, Ci=5, Co=4, H=6, W=6, kh=1, kw=1, pad=0),
    "pw_cn2": dict(N=1024, bits=50, L=2, batch=2, Ci=4, Co=4, H=6, W=6, kh=1, kw=1, pad=0),
    "k5x5": dict(N=2048, bits=50, L=2, batch=1, Ci=2, Co=2, H=8, W=8, kh=5, kw=5, pad=2),
    "wide_weights": dict(N=2048, bits=60, L=3, batch=1, Ci=8, Co=8, H=6, W=6, kh=3, kw=3, pad=1,
                         xrange=(-128, 128), wrange=(-128, 128)),
    # 64 .. 140 MAC rows (row padding to 128, two M tiles above 128), L = 2/3/5
    "tc_cn2_rows140": dict(N=1024, bits=50, L=2, batch=5, Ci=3, Co=70, H=6, W=6, kh=3, kw=3, pad=1,
                           xrange=(-128, 128), wrange=(-128, 128)),
    "tc_cn1_units": dict(N=1024, bits=50, L=3, batch=17, Ci=3, Co=70, H=6, W=6, kh=3, kw=3, pad=1,
                         xrange=(-128, 128), wrange=(-128, 128)),
    "tc_cn2": dict(N=2048, bits=60, L=3, batch=1, Ci=5, Co=34, H=6, W=6, kh=3, kw=3, pad=1,
                   xrange=(-128, 128), wrange=(-128, 128)),
    "tc_cn2_L5_rows130": dict(N=1024, bits=50, L=5, batch=2, Ci=2, Co=65, H=5, W=5, kh=3, kw=3, pad=1),
    "tc_pw_cn1": dict(N=1024, bits=50, L=3, batch=9, Ci=40, Co=66, H=6, W=6, kh=1, kw=1, pad=0),
    # degenerate layers: one channel of one pixel (c_n = 2 with an empty second slot row), a 1x1
    # single-channel layer, the largest kernel (7x7 = HY_MAX_TAPS taps) on a 3x3 image
    "one_pixel": dict(N=1024, bits=50, L=2, batch=1, Ci=1, Co=1, H=1, W=1, kh=3, kw=3, pad=1),
    "pw_one_channel": dict(N=1024, bits=50, L=2, batch=3, Ci=1, Co=1, H=5, W=5, kh=1, kw=1, pad=0),
    "k7x7": dict(N=1024, bits=50, L=2, batch=1, Ci=2, Co=3, H=3, W=3, kh=7, kw=7, pad=3),
    # the persistent warp-specialised kernel (Jc % 4 == 0): c_n = 1 with 2 epilogue warps (M <= 64) and
    # c_n = 2 with a ragged K (K = 36 -> 2 K steps of 32, the second 4 terms long)
    "tc_v2_cn1": dict(N=1024, bits=50, L=3, batch=17, Ci=4, Co=40, H=6, W=6, kh=3, kw=3, pad=1,
                      xrange=(-128, 128), wrange=(-128, 128)),
    "tc_v2_cn2_rows96": dict(N=1024, bits=50, L=2, batch=1, Ci=8, Co=48, H=6, W=6, kh=3, kw=3, pad=1,
                             xrange=(-128, 128), wrange=(-128, 128)),
    # K = Jc * 9 = 297 terms: 5 chunks of 64 with a ragged last K step; 128 rows exactly
    "tc_cn2_k297_rows128": dict(N=1024, bits=60, L=3, batch=1, Ci=66, Co=64, H=5, W=5, kh=3, kw=3, pad=1,
                                xrange=(-128, 128), wrange=(-128, 128)),
}


PATHS = ["default", "tc_fused", "tc_split", "fp64_fused", "fp64_split", "thin", "tc_coef"]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", sorted(CASES))
def test_conv_bit_exact_small(hy, name, path):
    """Every S2+S3 kernel path that applies to the layout gives the oracle's bits."""
    c = dict(CASES[name])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=500 + sorted(CASES).index(name), **c)
    got, dec, Lay = run_gpu(hy, lay, shape_of(lay), path=None if path == "default" else path)
    ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    for i in range(Lay.Jout):
        assert np.array_equal(got[i], ref[i]), f"output ct {i} differs"
    check_decrypted(lay, {i: got[i] for i in range(Lay.Jout)})
    check_plain_from_library_decrypt(lay, dec)


def test_conv_partial_units(hy):
    """hy_conv_eval on a prefix of the units (the sharding primitive) = the same outputs."""
    c = dict(CASES["cn1_blocks_tail"])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=550, **c)
    got, _, Lay = run_gpu(hy, lay, shape_of(lay), units=1)
    ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys, out_cts=list(range(Lay.Jo)))
    for i in range(Lay.Jo):
        assert np.array_equal(got[i], ref[i])


@pytest.mark.parametrize("batches", ["1", "2", "64"])
def test_host_path_batches(hy, monkeypatch, batches):
    """hy_conv_eval_host pipelined over several batches of units (HY_HOST_BATCHES forces the batch
    count; the default policy keeps >= 32 MiB per batch, i.e. one batch at test sizes) returns the
    device path's bytes; run_gpu compares host and device outputs."""
    monkeypatch.setenv("HY_HOST_BATCHES", batches)
    c = dict(CASES["cn1_blocks_tail"], batch=50)   # 4 units: batches of 4 / 2 / 1 units
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=551, **c)
    got, _, Lay = run_gpu(hy, lay, shape_of(lay))
    assert Lay.U == 4
    ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys, out_cts=[0, Lay.Jout - 1])
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[Lay.Jout - 1], ref[Lay.Jout - 1])


def test_c1_config_full(hy):
    """BASELINE configs[0] (C1) end to end: full ciphertext parity + decryption."""
    lay = layer_from_config(synth.configs()["C1"])
    got, dec, Lay = run_gpu(hy, lay, synth.configs()["C1"].shape_dict())
    ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    for i in range(Lay.Jout):
        assert np.array_equal(got[i], ref[i])
    check_plain_from_library_decrypt(lay, dec)


def test_shape_errors(hy):
    c = dict(CASES["cn2_blocks"])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=560, **c)
    p = hy.hy_params_create(N, lay.P.primes, 65537)
    try:
        w = hy.hy_encode_weights(p, lay.W, **shape_of(lay))
        try:
            x = torch.zeros((3, 2, L, N), dtype=torch.uint64, device="cuda")
            with pytest.raises(hy.HyenaError, match="multiple of Jc"):
                hy.hy_conv_eval(w, x, x)
            x2 = torch.zeros((2, 2, L, N), dtype=torch.uint64, device="cuda")
            with pytest.raises(hy.HyenaError, match="no Galois key"):
                hy.hy_conv_eval(w, x2, x2)
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)


def test_empty_and_misaligned_inputs(hy):
    """J = 0 and J not a multiple of Jc are rejected by both entry points, with no launch."""
    c = dict(CASES["cn1_blocks_tail"])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=570, **c)
    p = hy.hy_params_create(N, lay.P.primes, 65537)
    try:
        elts = list(lay.keys)
        hy.hy_keys_upload(p, elts, np.stack([lay.keys[g] for g in elts]))
        w = hy.hy_encode_weights(p, lay.W, **shape_of(lay))
        try:
            Lay = hy.hy_weights_layout(w)
            n0 = hy.hy_kernel_launches()
            x = torch.zeros((0, 2, L, N), dtype=torch.uint64, device="cuda")
            with pytest.raises(hy.HyenaError, match="positive multiple"):
                hy.hy_conv_eval(w, x, x)
            h = np.zeros((0, 2, L, N), dtype=np.uint64)
            with pytest.raises(hy.HyenaError, match="positive multiple"):
                hy.hy_conv_eval_host(w, h, h)
            if Lay.Jc > 1:
                h1 = np.zeros((Lay.Jc + 1, 2, L, N), dtype=np.uint64)
                with pytest.raises(hy.HyenaError, match="multiple of Jc"):
                    hy.hy_conv_eval_host(w, h1, np.zeros((Lay.Jo, 2, L, N), dtype=np.uint64))
            assert hy.hy_kernel_launches() == n0
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)


def test_streams_and_shared_params(hy):
    """ABI conventions (include/hyena.h): params and keys are shared by several weight handles; two
    layers evaluated concurrently on two non-default streams (stream-ordered, no host sync) give
    the oracle's bits; re-evaluating with the same handles is deterministic."""
    c1 = dict(CASES["cn2_blocks"])
    N, bits, L = c1.pop("N"), c1.pop("bits"), c1.pop("L")
    primes = ntt_primes(N, bits, L)
    lay1 = make_layer(N, primes, seed=580, **c1)
    c2 = dict(c1, Co=6)
    lay2 = make_layer(N, primes, seed=580, **c2)  # same seed: same secret and keys, other weights
    assert sorted(lay1.keys) == sorted(lay2.keys)
    p = hy.hy_params_create(N, primes, 65537)
    try:
        elts = list(lay1.keys)
        hy.hy_keys_upload(p, elts, np.stack([lay1.keys[g] for g in elts]))
        w1 = hy.hy_encode_weights(p, lay1.W, **shape_of(lay1))
        w2 = hy.hy_encode_weights(p, lay2.W, **shape_of(lay2))
        try:
            outs = {}
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
            for name, w, lay, st in (("a", w1, lay1, s1), ("b", w2, lay2, s2)):
                Lw = hy.hy_weights_layout(w)
                ct_in = torch.from_numpy(lay.ct_in).cuda()
                ct_out = torch.zeros((Lw.Jout, 2, L, N), dtype=torch.uint64, device="cuda")
                torch.cuda.synchronize()
                with torch.cuda.stream(st):
                    hy.hy_conv_eval(w, ct_in, ct_out, stream=st.cuda_stream)
                outs[name] = (ct_in, ct_out, lay, Lw)
            torch.cuda.synchronize()
            for name, (ct_in, ct_out, lay, Lw) in outs.items():
                ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
                got = ct_out.cpu().numpy()
                for i in range(Lw.Jout):
                    assert np.array_equal(got[i], ref[i]), f"layer {name} ct {i}"
            # second evaluation of layer a (buffers reused): bit-identical
            ct_in, ct_out, lay, Lw = outs["a"]
            again = torch.zeros_like(ct_out)
            hy.hy_conv_eval(w1, ct_in, again)
            torch.cuda.synchronize()
            assert torch.equal(again, ct_out)
        finally:
            hy.hy_weights_destroy(w1)
            hy.hy_weights_destroy(w2)
    finally:
        hy.hy_params_destroy(p)


def test_key_reupload_rebinds(hy):
    """Uploading new switching keys after hy_encode_weights is picked up by the next evaluation
    (the weights' tap-key table is rebound), and the result matches the oracle with the new keys."""
    c = dict(CASES["cn1_blocks_tail"])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    primes = ntt_primes(N, bits, L)
    lay = make_layer(N, primes, seed=590, **c)
    p = hy.hy_params_create(N, primes, 65537)
    try:
        elts = list(lay.keys)
        junk = {g: synth.gen_uniform_keys(primes, 1, N, 99, stream=n)[0] for n, g in enumerate(elts)}
        hy.hy_keys_upload(p, elts, np.stack([junk[g] for g in elts]))
        w = hy.hy_encode_weights(p, lay.W, **shape_of(lay))
        try:
            Lw = hy.hy_weights_layout(w)
            ct_in = torch.from_numpy(lay.ct_in).cuda()
            ct_out = torch.zeros((Lw.Jout, 2, L, N), dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, ct_in, ct_out)              # with the junk keys
            hy.hy_keys_upload(p, elts, np.stack([lay.keys[g] for g in elts]))
            hy.hy_conv_eval(w, ct_in, ct_out)              # must use the real keys now
            torch.cuda.synchronize()
            ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
            got = ct_out.cpu().numpy()
            for i in range(Lw.Jout):
                assert np.array_equal(got[i], ref[i])
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)
