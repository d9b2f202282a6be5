"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times (T2).

Every config runs through hy_conv_eval over ALL its input ciphertexts (the bench workload);
the oracle then recomputes a sample of output ciphertexts one by one and they must agree
bit for bit.  To keep the oracle's schoolbook products affordable at N = 8192/16384 the
input ciphertexts have SPARSE c1 (a few nonzero coefficients per limb, same positions in
every limb): the oracle's product skips zero coefficients of its first operand
(oracle/negacyclic.c), and the hoisted digits d_i = [c1]_{q_i} inherit the sparsity.  The
library does not know (its kernels do the same work on any input).  c0 and the switching keys
are dense uniform.  A second test encrypts real images (with sparse masks: insecure but
exact BFV) for the units it samples and checks the decryptions against the plain
convolution mod t.  Marked gpu.
"""
import numpy as np
import pytest

import synth
from oracle import bfv, conv
from tests.hyena_client import encrypt_slots, keygen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FULL = ["C2", "C3a", "C3b", "C4", "C5dw_8192", "C5pw_8192", "C5dw_4096", "C5pw_4096", "C5dw_16384",
        "C5pw_16384"]


@pytest.fixture(scope="module")
def hy():
    import paper_2311_12519_b200 as pkg
    from paper_2311_12519_b200 import build
    build.build()
    pkg.load_library()
    assert torch.cuda.is_available()
    return pkg


def sparse_c1_cts(primes, n, N, seed, nz=12):
    """[n][2][L][N]: c0 dense uniform, c1 with nz nonzero coefficients (shared positions)."""
    g = synth.rng(seed, "ct", 7)
    ct = np.zeros((n, 2, len(primes), N), dtype=np.uint64)
    for l, q in enumerate(primes):
        ct[:, 0, l] = g.integers(0, q, size=(n, N), dtype=np.uint64)
    for i in range(n):
        pos = g.choice(N, size=nz, replace=False)
        for l, q in enumerate(primes):
            ct[i, 1, l, pos] = g.integers(1, q, size=nz, dtype=np.uint64)
    return ct


def sample_outputs(p):
    """First and last output ct of the first and last unit (deduplicated)."""
    outs = {0, p.Jo - 1, (p.U - 1) * p.Jo, p.Jout - 1}
    return sorted(outs)


def run_full(hy, cfg, ct_in, keys):
    p = hy.hy_params_create(cfg.N, cfg.primes, cfg.t, 0)
    try:
        elts = sorted(keys)
        if elts:                                   # a 1x1 layer needs no switching key
            hy.hy_keys_upload(p, elts, np.stack([keys[g] for g in elts]))
        w = hy.hy_encode_weights(p, synth.gen_weights(cfg), **cfg.shape_dict())
        try:
            lay = hy.hy_weights_layout(w)
            assert lay.J == len(ct_in)
            d_in = torch.from_numpy(ct_in).cuda()
            d_out = torch.full((lay.Jout, 2, len(cfg.primes), cfg.N), 3, dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, d_in, d_out)
            torch.cuda.synchronize()
            return d_out.cpu().numpy(), lay
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)


@pytest.mark.parametrize("name", FULL)
def test_fullsize_ciphertext_parity(hy, name):
    cfg = synth.configs()[name]
    P = bfv.BFVParams(cfg.N, cfg.primes, cfg.t)
    plan = conv.plan(cfg.N, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad, cfg.depthwise,
                     cfg.force_cn)
    ls = conv.setup(plan, cfg.t, cfg.k)
    ct_in = sparse_c1_cts(cfg.primes, plan.J, cfg.N, cfg.index)
    kk = synth.gen_uniform_keys(cfg.primes, len(ls.galois), cfg.N, cfg.index)
    keys = {g: kk[n] for n, g in enumerate(ls.galois)}
    got, lay = run_full(hy, cfg, ct_in, keys)
    assert (lay.J, lay.Jout, lay.cn, lay.k) == (plan.J, plan.Jout, plan.cn, ls.k)
    outs = sample_outputs(plan)
    ref = conv.he_conv(P, ls, synth.gen_weights(cfg), ct_in, keys, out_cts=outs)
    for oc in outs:
        assert np.array_equal(got[oc], ref[oc]), f"{name}: output ct {oc} differs from the oracle"
    # every output ciphertext is canonical (all written, residues < q_l)
    q = np.array(cfg.primes, dtype=np.uint64)[None, None, :, None]
    assert (got < q).all()


@pytest.mark.parametrize("name", FULL)
def test_fullsize_decrypts_to_plain_conv(hy, name):
    """Real BFV encryptions (DENSE uniform masks a, CBD errors, dense Galois keys: the real
    noise of the key switching) of the sampled units' inputs, uniform junk elsewhere: the
    sampled outputs decrypt to scale * conv mod t at every valid position, and the noise meter
    (SURVEY §5, P12; PAPER.md:266-267 [ign], :318) shows >= 4 bits of margin below Delta/2."""
    cfg = synth.configs()[name]
    P = bfv.BFVParams(cfg.N, cfg.primes, cfg.t)
    plan = conv.plan(cfg.N, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad, cfg.depthwise,
                     cfg.force_cn)
    ls = conv.setup(plan, cfg.t, cfg.k)
    x = synth.gen_image(cfg)
    Wt = synth.gen_weights(cfg)
    s = synth.gen_secret(cfg)
    slots = conv.pack(plan, x, cfg.t)
    outs = sample_outputs(plan)
    units = sorted({oc // plan.Jo for oc in outs})
    need = [u * plan.Jc + c for u in units for c in range(plan.Jc)]
    if plan.depthwise:          # a depthwise output reads only its own channel
        need = sorted({oc // plan.Jo * plan.Jc + oc % plan.Jo for oc in outs})
    ct_in = sparse_c1_cts(cfg.primes, plan.J, cfg.N, cfg.index + 50)
    ct_in[need] = encrypt_slots(P, s, slots[need], cfg.index)
    keys = keygen(P, s, ls.galois, cfg.index)
    got, lay = run_full(hy, cfg, ct_in, keys)
    dec = conv.decrypt_outputs(P, ls, {oc: got[oc] for oc in outs}, s)
    full = np.zeros((plan.Jout, plan.N), dtype=np.int64)
    mask = np.zeros((plan.Jout, plan.N), dtype=np.int64)
    for oc, v in dec.items():
        full[oc] = v
        mask[oc] = 1
    have = conv.unpack(plan, mask).astype(bool)
    got_px = conv.unpack(plan, full)
    exp = np.mod(conv.plain_conv(x, Wt, plan.pad, plan.depthwise), cfg.t)
    assert have.sum() > 0
    bad = np.argwhere(have & (got_px != exp))
    assert bad.size == 0, f"{name}: {len(bad)} mismatches, first {bad[:5].tolist()}"
    budget = bfv.noise_budget_bits(P)
    margins = {oc: budget - bfv.noise_bits(P, got[oc], s, bfv.decrypt(P, got[oc], s)) for oc in outs}
    print(f"{name}: noise margin bits (log2(Delta/2) - log2 ||v||) = "
          + ", ".join(f"ct {oc}: {m:.1f}" for oc, m in margins.items()))
    assert min(margins.values()) >= 4, f"{name}: noise margin {margins}"


def encrypt_sparse(P, s, slots, seed, nz=12):
    """Symmetric BFV encryption with a sparse uniform mask a: exact, cheap for the
    oracle's schoolbook product (zero coefficients of the first operand are skipped)."""
    from oracle.encoding import encode_batch
    polys = encode_batch(slots, P.t, P.N)
    out = np.empty((len(slots), 2, P.L, P.N), dtype=np.uint64)
    g = synth.rng(seed, "a", 900)
    for j, m in enumerate(polys):
        a = np.zeros((P.L, P.N), dtype=np.uint64)
        pos = g.choice(P.N, size=nz, replace=False)
        for l, q in enumerate(P.primes):
            a[l, pos] = g.integers(1, q, size=nz, dtype=np.uint64)
        e = synth.cbd(synth.rng(seed, "e", 900 + j), P.N)
        out[j] = bfv.encrypt(P, m, s, a, e)
    return out


@pytest.mark.parametrize("name", ["C3b", "C4"])
def test_fullsize_host_pipeline_matches_device(hy, name):
    """hy_conv_eval_host (uploads / downloads pipelined over batches of units on the library's
    copy streams) returns exactly the device path's ciphertexts at full size."""
    cfg = synth.configs()[name]
    full = hy.hy_plan_layout(cfg.N, cfg.t, **cfg.shape_dict())
    elts = list(full.galois[:full.n_galois])
    ct = synth.gen_uniform_cts(cfg.primes, full.J, cfg.N, cfg.index, stream=3)
    p = hy.hy_params_create(cfg.N, cfg.primes, cfg.t, 0)
    try:
        hy.hy_keys_upload(p, elts, synth.gen_uniform_keys(cfg.primes, len(elts), cfg.N, cfg.index))
        w = hy.hy_encode_weights(p, synth.gen_weights(cfg), **cfg.shape_dict())
        try:
            lay = hy.hy_weights_layout(w)
            d_out = torch.empty((lay.Jout, 2, len(cfg.primes), cfg.N), dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, torch.from_numpy(ct).cuda(), d_out)
            torch.cuda.synchronize()
            dev = d_out.cpu().numpy()
            del d_out
            host = np.zeros_like(dev)
            hy.hy_conv_eval_host(w, ct, host)
            assert np.array_equal(host, dev)
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)
