"""Pins for oracle/conv.py: decrypt(HE-conv(enc(x))) = plain conv mod t on tiny layers (P8),
layout pins (Table 2/3, P4/P5), lazy = eager reduction (P10), plain conv vs brute force — CPU."""
import itertools
import json
import os

import numpy as np
import pytest

import synth
from oracle import bfv, conv, costmodel, ring
from oracle.params import ntt_primes
from tests.hyena_client import check_decrypted, layer_from_config, make_layer

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_plain_conv_bruteforce():
    g = np.random.default_rng(0)
    x = g.integers(-5, 5, (2, 3, 5, 4))
    W = g.integers(-3, 3, (2, 3, 3, 3))
    y = conv.plain_conv(x, W, 1)
    for b, o, yy, xx in itertools.product(range(2), range(2), range(5), range(4)):
        acc = 0
        for c, dy, dx in itertools.product(range(3), range(3), range(3)):
            iy, ix = yy + dy - 1, xx + dx - 1
            if 0 <= iy < 5 and 0 <= ix < 4:
                acc += W[o, c, dy, dx] * x[b, c, iy, ix]
        assert y[b, o, yy, xx] == acc
    Wd = g.integers(-3, 3, (3, 3, 3))
    yd = conv.plain_conv(x, Wd, 1, depthwise=True)
    Wfull = np.zeros((3, 3, 3, 3), dtype=np.int64)
    for c in range(3):
        Wfull[c, c] = Wd[c]
    assert (yd == conv.plain_conv(x, Wfull, 1)).all()


def test_config_plans():
    """Layouts of BASELINE.json configs."""
    cf = synth.configs()
    p = lambda c: conv.plan(c.N, c.batch, c.Ci, c.Co, c.H, c.W, c.kh, c.kw, c.pad, c.depthwise, c.force_cn)
    c1 = p(cf["C1"]); assert (c1.Wp, c1.cn, c1.J, c1.Jout) == (16, 2, 2, 2)
    c2 = p(cf["C2"]); assert (c2.Wp, c2.cn, c2.J, c2.Jout, c2.per_row) == (64, 2, 8, 8, 1)
    c3a = p(cf["C3a"]); assert (c3a.Wp, c3a.per_row, c3a.cn, c3a.J, c3a.Jout) == (16, 16, 2, 32, 32)
    c3b = p(cf["C3b"]); assert (c3b.Wp, c3b.per_row, c3b.G, c3b.cn, c3b.J, c3b.Jout) == (32, 4, 4, 1, 64, 128)
    c4 = p(cf["C4"])
    assert (c4.mode, c4.Wp, c4.Hb, c4.Hv, c4.bands, c4.G, c4.cn, c4.J, c4.Jout) == \
        ("bands", 256, 16, 14, 16, 128, 1, 4096, 4096)
    for N, cn, J in ((4096, 1, 1024), (8192, 1, 512), (16384, 2, 256)):
        d = p(cf[f"C5dw_{N}"]); assert (d.cn, d.J, d.Jout) == (cn, J, J)
        w = p(cf[f"C5pw_{N}"]); assert (w.cn, w.J, w.Jout, w.Wp) == (cn, J, J, 16)


def test_table2_and_table3_accounting():
    """Pow2 padding + ceil(C Wp^2 / n) packing reproduce Table 2's input-ct and model columns
     and Table 3's communication."""
    MB = 2**20
    for r in GOLD["table2_rows"]["rows"]:
        assert costmodel.input_ct_bytes(r["Ci"], r["H"], r["n"]) / MB == pytest.approx(r["input_ct_MB"], rel=1e-9)
        assert round(costmodel.model_bytes_proposed(r["Ci"], r["Co"], 3) / MB, 2) == pytest.approx(
            r["model_MB"], abs=0.011)
    for r in GOLD["table3_comm"]["rows"]:
        assert round(costmodel.comm_bytes(r["H"], r["Ci"], r["Co"], r["f"], r["n"]) / MB) == r["comm_MB"]
    # 2x3x3 kernel at n = 2048: 16.1 KB vs 288 KB
    assert round(costmodel.storage_proposed_bytes(18, 2048) / 1024, 1) == GOLD["storage_2x3x3_n2048_proposed_KB"]["value"]
    assert costmodel.storage_conventional_bytes(18, 2048) / 1024 == GOLD["storage_2x3x3_n2048_conventional_KB"]["value"]


def test_pack_unpack_identity():
    """A 1x1 identity kernel through pack/unpack returns x in every layout mode."""
    for (N, batch, C, H, pad) in [(64, 3, 2, 2, 0), (256, 2, 3, 10, 0)]:
        p = conv.plan(N, batch, C, C, H, H, 1, 1, pad)
        x = np.arange(batch * C * H * H).reshape(batch, C, H, H) % 65537
        s = conv.pack(p, x, 65537)
        assert (conv.unpack(p, s) == x).all()


PRIMES64 = ntt_primes(64, 50, 3)


@pytest.mark.parametrize("case", [
    dict(batch=2, Ci=4, Co=4, H=2, W=2, k=0),                       # c_n = 2, 2 images / slot row, k = 32
    dict(batch=2, Ci=4, Co=4, H=2, W=2, k=1),                       # k = 1
    dict(batch=1, Ci=3, Co=5, H=3, W=3, k=0),                       # odd channel counts (zero rows)
    dict(batch=1, Ci=2, Co=3, H=6, W=6, k=0),                       # c_n = 1: bands with halos (Wp=8, Hb=4)
    dict(batch=3, Ci=2, Co=2, H=2, W=2, k=0, force_cn=1),           # c_n = 1 blocks, odd group tail
    dict(batch=2, Ci=4, Co=4, H=2, W=2, k=0, depthwise=True),       # depthwise c_n = 2
    dict(batch=1, Ci=2, Co=2, H=6, W=6, k=0, depthwise=True),       # depthwise c_n = 1 bands
    dict(batch=2, Ci=4, Co=4, H=3, W=3, k=0, kh=1, kw=1, pad=0),    # 1x1 conv, c_n = 2
])
def test_he_conv_decrypts_to_plain_conv(case):
    """P8: decrypt(HE-conv(enc x)) * (c_n k)^{-1} = plain conv mod t at every valid position."""
    case = dict(case)
    kh = case.pop("kh", 3); kw = case.pop("kw", 3); pad = case.pop("pad", 1)
    lay = make_layer(64, PRIMES64, kh=kh, kw=kw, pad=pad, seed=60, **case)
    out = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    n = check_decrypted(lay, out)
    assert n == lay.x.shape[0] * (lay.W.shape[0]) * lay.plan.Hout * lay.plan.Wout
    if lay.plan.cn == 2:
        assert lay.ls.scale == 2 * lay.ls.k


def test_noise_margin_small_primes_fails():
    """With too small a modulus the same layer decrypts WRONG: the noise meter matters (P8/P12)."""
    lay = make_layer(64, ntt_primes(64, 30, 2), batch=2, Ci=4, Co=4, H=2, W=2, kh=3, kw=3, pad=1,
                     xrange=(-128, 128), wrange=(-128, 128), seed=61)
    out = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    with pytest.raises(AssertionError):
        check_decrypted(lay, out)


def test_lazy_equals_eager():
    """P10: reducing the unreduced wide sum once equals reducing every term."""
    q = PRIMES64[0]
    g = np.random.default_rng(2)
    R = g.integers(0, q, (600, 64), dtype=np.uint64)
    w = g.integers(-128, 128, 600)
    lazy = [sum(int(w[n]) * int(R[n, k]) for n in range(600)) % q for k in range(64)]
    eager = [0] * 64
    for n in range(600):
        for k in range(64):
            eager[k] = (eager[k] + (int(w[n]) * int(R[n, k])) % q) % q
    assert lazy == eager
    # the oracle's lincomb (30-bit split, int64) agrees with both
    cts = [np.stack([np.stack([R[n]] * 1)] * 2) for n in range(600)]
    P = bfv.BFVParams(64, [q], 65537)
    out = conv._lincomb(P, [(int(w[n]), cts[n]) for n in range(600)])
    assert list(out[0, 0]) == lazy


def test_c1_config_end_to_end():
    """BASELINE configs[0] (C1) through the oracle: exact decryption + >= 4 bits noise margin."""
    lay = layer_from_config(synth.configs()["C1"])
    out = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    check_decrypted(lay, out)
    budget = bfv.noise_budget_bits(lay.P)
    from oracle.encoding import encode
    for i, ct in out.items():
        dec = bfv.decrypt(lay.P, ct, lay.s)
        assert budget - bfv.noise_bits(lay.P, ct, lay.s, dec) >= 4


# ---------------------------------------------------------------------------------------------
# c_n = 4 Walsh-Hadamard channel packing (reading R11)
# ---------------------------------------------------------------------------------------------
def test_sylvester_hadamard():
    """H_n H_n^T = n I with +/-1 entries; H_4's rows are the paper's c_n = 4 basis with the garbled
    duplicate row replaced by [1, -1, 1, -1] (reading R11)."""
    for n in (1, 2, 4, 8):
        H = conv.hadamard(n)
        assert set(np.unique(H)) <= {-1, 1}
        assert np.array_equal(H @ H.T, n * np.eye(n, dtype=np.int64))
    rows = {tuple(r) for r in conv.hadamard(4)}
    assert rows == {(1, 1, 1, 1), (1, -1, 1, -1), (1, 1, -1, -1), (1, -1, -1, 1)}


def test_hadamard_row_plaintexts_decode_to_patterns():
    """The row-r plaintexts hold H_4[r][c] in every slot of group c (decoding = evaluation)."""
    from oracle.encoding import decode
    N = 64
    P = bfv.BFVParams(N, ntt_primes(N, 50, 2), 65537)
    p = conv.plan(N, 1, 4, 4, 2, 2, 3, 3, 1, False, 4)
    H = conv.hadamard(4)
    polys = conv.hadamard_row_polys(P, p)
    for r in (1, 2, 3):
        q = P.primes[0]
        m = [conv.centered(int(x) if int(x) < q // 2 else int(x) - q, 65537) for x in polys[r - 1][0]]
        slots = decode(np.mod(np.array(m, dtype=np.int64), 65537), 65537, N)
        for c in range(4):
            b = conv._group_base(p, c)
            assert set(slots[b:b + N // 4].tolist()) == {H[r][c] % 65537}


@pytest.mark.parametrize("w", [0, 20])
def test_cn4_toy_decrypts_to_plain_conv(w):
    """decrypt(HE-conv(enc x)) * 4^{-1} = plain conv mod t with 4 channels per ciphertext, for
    the one-digit-per-limb gadget and a 2^20 sub-digit base."""
    lay = make_layer(64, ntt_primes(64, 50, 3), batch=1, Ci=8, Co=5, H=2, W=2, kh=3, kw=3, pad=1,
                     xrange=(-128, 128), wrange=(-128, 128), seed=71, force_cn=4, w=w)
    assert (lay.plan.cn, lay.plan.J, lay.plan.Jout, lay.ls.scale) == (4, 2, 2, 4)
    out = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    check_decrypted(lay, out)


def test_c1_in_one_ciphertext():
    """BASELINE configs[0] (C1) packed as ONE ciphertext (c_n = 4; reading R19 superseded): needs the
    sub-digit base for noise (dense Hadamard-row plaintexts multiply the key-switching noise by up
    to N t / 2); with w = 20 it decrypts exactly with >= 4 bits of margin."""
    cfg = synth.configs()["C1"]
    lay = make_layer(cfg.N, cfg.primes, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad,
                     seed=cfg.index, force_cn=4, x=synth.gen_image(cfg), Wt=synth.gen_weights(cfg), w=20)
    assert (lay.plan.J, lay.plan.Jout) == (1, 1)
    out = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    check_decrypted(lay, out)
    budget = bfv.noise_budget_bits(lay.P)
    for ct in out.values():
        assert budget - bfv.noise_bits(lay.P, ct, lay.s, bfv.decrypt(lay.P, ct, lay.s)) >= 4


def test_c1_one_ciphertext_fails_without_subdigits():
    """Negative control for the decomposition base: with one digit per 50-bit limb the c_n = 4 C1
    layer's noise reaches Delta/2 and decryption is wrong (why NEXT-4's smaller base is needed)."""
    cfg = synth.configs()["C1"]
    lay = make_layer(cfg.N, cfg.primes, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad,
                     seed=cfg.index, force_cn=4, x=synth.gen_image(cfg), Wt=synth.gen_weights(cfg), w=0)
    out = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
    with pytest.raises(AssertionError):
        check_decrypted(lay, out)
