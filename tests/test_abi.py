"""C-ABI checks that need no GPU: the library builds/loads, exports every symbol include/hyena.h
declares, and its host-only layout planner agrees with the oracle's (independent implementations)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import synth
from oracle import conv
from oracle.params import find_k, h_pn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hy():
    from paper_2311_12519_b200 import build
    build.build()
    import paper_2311_12519_b200 as pkg
    pkg.load_library()
    return pkg


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "hyena.h")).read()
    return sorted(set(re.findall(r"^\s*(?:hy_status|void|uint64_t|const char\*)\s+(hy_\w+)\s*\(", txt, re.M)))


def test_exports_every_declared_symbol(hy):
    names = declared_symbols()
    assert len(names) >= 14
    lib = ctypes.CDLL(hy.library_path())
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(hy.EXPORTED) == names
    out = subprocess.run(["nm", "-D", "--defined-only", hy.library_path()], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_sm100a_code_in_library(hy):
    out = subprocess.run(["cuobjdump", "--list-elf", hy.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


CFGS = synth.configs()


@pytest.mark.parametrize("name", sorted(CFGS))
def test_planner_matches_oracle(hy, name):
    c = CFGS[name]
    lay = hy.hy_plan_layout(c.N, c.t, **c.shape_dict())
    p = conv.plan(c.N, c.batch, c.Ci, c.Co, c.H, c.W, c.kh, c.kw, c.pad, c.depthwise, c.force_cn)
    got = (lay.Wp, lay.Hp, lay.mode, lay.per_row, lay.Hb, lay.Hv, lay.bands, lay.G, lay.cn, lay.U, lay.Jc, lay.Jo,
           lay.J, lay.Jout, lay.Hout, lay.Wout)
    exp = (p.Wp, p.Hp, 0 if p.mode == "blocks" else 1, p.per_row, p.Hb, p.Hv, p.bands, p.G, p.cn, p.U, p.Jc, p.Jo,
           p.J, p.Jout, p.Hout, p.Wout)
    assert got == exp
    assert list(lay.tap_step[:lay.n_taps]) == [s for _, _, s in p.taps]
    ls = conv.setup(p, c.t)
    assert list(lay.galois[:lay.n_galois]) == ls.galois
    assert (lay.k, lay.scale, lay.sign_coeff) == (ls.k, ls.scale, ls.sign_coeff)


def test_library_h_and_k_match_oracle(hy):
    """The library's closed-form h (-(w + w^3)/2) equals the oracle's by-encoding h."""
    for N in (1024, 4096, 16384):
        lay = hy.hy_plan_layout(N, 65537, Ci=2, Co=2, H=4, W=4, kh=3, kw=3, pad=1, batch=1)
        assert lay.h == h_pn(65537, N)
        assert lay.k == find_k(65537, lay.h)


def test_planner_rejects_bad_shapes(hy):
    with pytest.raises(hy.HyenaError, match="stride"):
        hy.hy_plan_layout(4096, 65537, Ci=2, Co=2, H=4, W=4, kh=3, kw=3, pad=1, batch=1, stride=2)
    with pytest.raises(hy.HyenaError, match="empty"):
        hy.hy_plan_layout(4096, 65537, Ci=0, Co=2, H=4, W=4, kh=3, kw=3, pad=1, batch=1)
    with pytest.raises(hy.HyenaError, match="prime"):
        hy.hy_plan_layout(4096, 65539, Ci=2, Co=2, H=4, W=4, kh=3, kw=3, pad=1, batch=1)
    with pytest.raises(hy.HyenaError, match="k must"):
        hy.hy_plan_layout(4096, 65537, Ci=2, Co=2, H=4, W=4, kh=3, kw=3, pad=1, batch=1, k=33)
    with pytest.raises(hy.HyenaError, match="exceeds a slot row"):
        hy.hy_plan_layout(1024, 65537, Ci=2, Co=2, H=4, W=1000, kh=3, kw=3, pad=1, batch=1)


def test_params_create_validation_without_gpu(hy):
    """Argument validation happens before any device call."""
    with pytest.raises(hy.HyenaError, match="not prime"):
        hy.hy_params_create(4096, [2**59 + 1], 65537)
    with pytest.raises(hy.HyenaError, match="1 mod 2N"):
        hy.hy_params_create(4096, [2147483647], 65537)            # 2^31-1: prime, not 1 mod 8192
    with pytest.raises(hy.HyenaError, match=r"\(2\^20, 2\^60\)"):
        hy.hy_params_create(4096, [2305843009213693951], 65537)   # 2^61-1: prime but too large


def test_layout_accounting_matches_paper_tables(hy):
    """hy_layout_accounting (host only) reproduces PAPER.md Table 2's input-ct and model columns and
    the :561-562 storage example with one 60-bit prime (the paper's setting, L = 1), and agrees with
    the oracle's cost model; the library's own layout counts its J / Jout ciphertexts."""
    import json
    from oracle import costmodel
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_values.json")))
    MB = 1 << 20
    for r in gold["table2_rows"]["rows"]:
        H, n = r["H"], r["n"]
        t = 65537
        shape = dict(Ci=r["Ci"], Co=r["Co"], H=H - 2, W=H - 2, kh=3, kw=3, pad=1, batch=1, force_cn=1)
        lay = hy.hy_plan_layout(n, t, **shape)
        acc = hy.hy_layout_accounting(lay, 1, **shape)
        assert acc["input_ct_bytes_paper"] == costmodel.input_ct_bytes(r["Ci"], H, n)
        assert round(acc["input_ct_bytes_paper"] / MB) == r["input_ct_MB"]
        assert acc["model_bytes_paper"] == costmodel.model_bytes_proposed(r["Ci"], r["Co"], 3)
        assert abs(acc["model_bytes_paper"] / MB - r["model_MB"]) <= 0.01 * r["model_MB"] + 0.005
    # a 2 x 3 x 3 kernel at n = 2048, c_n = 2: 16.1 KB vs 288 KB
    shape = dict(Ci=2, Co=1, H=8, W=8, kh=3, kw=3, pad=1, batch=1, force_cn=2)
    lay = hy.hy_plan_layout(2048, 65537, **shape)
    acc = hy.hy_layout_accounting(lay, 1, **shape)
    assert acc["model_bytes_paper"] == costmodel.storage_proposed_bytes(18, 2048) == 16528
    assert acc["model_bytes_conventional"] == costmodel.storage_conventional_bytes(18, 2048) == 288 * 1024
    # C4 with this library's layout: bands of 14 valid rows -> 4096 input and output cts
    import synth
    cfg = synth.configs()["C4"]
    lay = hy.hy_plan_layout(cfg.N, cfg.t, **cfg.shape_dict())
    acc = hy.hy_layout_accounting(lay, 3, **cfg.shape_dict())
    assert acc["input_ct_bytes"] == acc["output_ct_bytes"] == 4096 * 2 * 3 * 8192 * 8
    assert acc["rotations"] == 4096 * 8 and acc["n_keys"] == 8
    assert acc["coef_macs"] == 64 * 64 * 576 * 2 * 3 * 8192


def test_noise_model_tracks_the_oracle(hy):
    """The base-selection noise model (hy_noise_estimate) against the oracle's noise meter on C1 with
    c_n = 2 and with c_n = 4 at two sub-digit bases: within 3 bits; hy_select_dcmp_base picks one
    digit per limb for c_n = 2 and the 2^25 base (2 sub-digits per limb) for c_n = 4, which the oracle
    confirms decrypts with >= 4 bits of margin (tests/test_oracle_conv.py: w = 20, 25; w = 0 fails)."""
    from oracle import bfv
    from tests.hyena_client import layer_from_config, make_layer
    cfg = synth.configs()["C1"]
    for cn, w in ((2, 0), (4, 25), (4, 20)):
        if cn == 2:
            lay = layer_from_config(cfg)
        else:
            lay = make_layer(cfg.N, cfg.primes, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad,
                             seed=cfg.index, force_cn=4, x=synth.gen_image(cfg), Wt=synth.gen_weights(cfg), w=w)
        out = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
        measured = max(bfv.noise_bits(lay.P, c, lay.s, bfv.decrypt(lay.P, c, lay.s)) for c in out.values())
        shape = dict(cfg.shape_dict(), force_cn=cn)
        est, budget = hy.hy_noise_estimate(cfg.N, cfg.primes, cfg.t, w_dcmp=w, w_max=8, **shape)
        assert abs(est - measured) <= 3, (cn, w, est, measured)
        assert abs(budget - bfv.noise_budget_bits(lay.P)) < 0.01
    assert hy.hy_select_dcmp_base(cfg.N, cfg.primes, cfg.t, 4.0, 8, **cfg.shape_dict()) == 0
    assert hy.hy_select_dcmp_base(cfg.N, cfg.primes, cfg.t, 4.0, 8, **dict(cfg.shape_dict(), force_cn=4)) == 25
