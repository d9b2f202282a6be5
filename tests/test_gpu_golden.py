"""Full-size ciphertext parity of EVERY output ciphertext: C1, C2, C3a, C3b
whole, and two whole units of C4 (units 0 and U-1), on dense uniform inputs and keys, through
hy_conv_eval over the whole layer in the bench launch configuration.  The expected values are
SHA-256 digests of the ORACLE's output ciphertexts written by tools/make_golden.py (which calls
only oracle/ and synth/); the input digests are checked first so a generator change cannot
silently break the comparison.  Marked gpu."""
import hashlib
import json
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_sha256.json")))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def hy():
    import paper_2311_12519_b200 as pkg
    from paper_2311_12519_b200 import build
    build.build()
    pkg.load_library()
    assert torch.cuda.is_available()
    return pkg


@pytest.mark.parametrize("name", [n for n in ["C1", "C2", "C3a", "C3b", "C4"] if n in GOLD])
def test_fullsize_every_output_matches_oracle_digest(hy, name):
    g = GOLD[name]
    cfg = synth.configs()[name]
    full = hy.hy_plan_layout(cfg.N, cfg.t, **cfg.shape_dict())
    elts = list(full.galois[:full.n_galois])
    ct = synth.gen_uniform_cts(cfg.primes, full.J, cfg.N, cfg.index, stream=11)
    kk = synth.gen_uniform_keys(cfg.primes, max(1, len(elts)), cfg.N, cfg.index)
    W = synth.gen_weights(cfg)
    assert (full.J, full.Jout) == (g["J"], g["Jout"])
    assert sha(ct) == g["ct_in_sha256"] and sha(kk) == g["keys_sha256"]
    assert hashlib.sha256(W.tobytes()).hexdigest() == g["weights_sha256"]
    p = hy.hy_params_create(cfg.N, cfg.primes, cfg.t, 0)
    try:
        hy.hy_keys_upload(p, elts, kk[: len(elts)])
        w = hy.hy_encode_weights(p, W, **cfg.shape_dict())
        try:
            d_in = torch.from_numpy(ct).cuda()
            del ct
            d_out = torch.full((full.Jout, 2, len(cfg.primes), cfg.N), 5, dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, d_in, d_out)
            torch.cuda.synchronize()
            del d_in
            bad = []
            for oc, want in g["outputs"].items():
                if sha(d_out[int(oc)].cpu().numpy()) != want:
                    bad.append(int(oc))
            assert not bad, f"{name}: {len(bad)} of {len(g['outputs'])} output cts differ, first {bad[:8]}"
            q = torch.tensor(cfg.primes, dtype=torch.int64, device="cuda").view(1, 1, -1, 1)
            assert bool((d_out.view(torch.int64) < q).all()), "non-canonical output residues"
        finally:
            hy.hy_weights_destroy(w)
    finally:
        hy.hy_params_destroy(p)
