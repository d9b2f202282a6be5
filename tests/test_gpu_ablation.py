"""The Fig. 4 ablations on this library's kernels:
  * HY_MAC_EAGER  -- lazy reduction OFF (reduce after every product and addition): the same residues
    as the lazy MAC (P10), so bit-exact against the oracle's (hoisted) layer;
  * HY_MAC_DIRECT -- hoisting OFF (every rotation decomposes the rotated c1 again): bit-exact
    against the oracle's layer built from bfv.rotate_direct rotations (reading R6: direct and
    hoisted HRot differ in their bits, not in their decryption).
Marked gpu."""
import numpy as np
import pytest

from oracle import conv
from oracle.params import ntt_primes
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


CASES = {
    "cn2_blocks": dict(N=1024, bits=50, L=2, batch=2, Ci=4, Co=6, H=5, W=5, kh=3, kw=3, pad=1),
    "cn1_bands": dict(N=1024, bits=50, L=3, batch=1, Ci=3, Co=2, H=20, W=20, kh=3, kw=3, pad=1),
    "cn1_rows70": dict(N=1024, bits=50, L=3, batch=17, Ci=3, Co=70, H=6, W=6, kh=3, kw=3, pad=1,
                       xrange=(-128, 128), wrange=(-128, 128)),
    "cn2_wide": dict(N=2048, bits=60, L=3, batch=1, Ci=8, Co=8, H=6, W=6, kh=3, kw=3, pad=1,
                     xrange=(-128, 128), wrange=(-128, 128)),
}


def shape_of(lay):
    p = lay.plan
    return dict(Ci=p.Ci, Co=p.Co, H=p.H, W=p.W, kh=p.kh, kw=p.kw, pad=p.pad, depthwise=int(p.depthwise),
                batch=p.batch, k=lay.ls.k if p.cn == 2 else 0, force_cn=p.cn)


@pytest.mark.parametrize("w", [0, 20])
@pytest.mark.parametrize("path", ["eager", "direct"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_ablation_paths_bit_exact(hy, name, path, w):
    c = dict(CASES[name])
    N, bits, L = c.pop("N"), c.pop("bits"), c.pop("L")
    lay = make_layer(N, ntt_primes(N, bits, L), seed=1500 + sorted(CASES).index(name), w=w, **c)
    p = hy.hy_params_create(N, lay.P.primes, lay.P.t, 0, w_dcmp=w)
    try:
        elts = list(lay.keys)
        hy.hy_keys_upload(p, elts, np.stack([lay.keys[g] for g in elts]))
        wt = hy.hy_encode_weights(p, lay.W, **shape_of(lay))
        try:
            hy.hy_weights_set_mac_path(wt, path)
            Lw = hy.hy_weights_layout(wt)
            out = torch.full((Lw.Jout, 2, L, N), 5, dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(wt, torch.from_numpy(lay.ct_in).cuda(), out)
            torch.cuda.synchronize()
            got = out.cpu().numpy()
        finally:
            hy.hy_weights_destroy(wt)
    finally:
        hy.hy_params_destroy(p)
    R = conv.rotations(lay.P, lay.plan, lay.ct_in, lay.keys, hoisted=(path != "direct"))
    ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys, R=R)
    for i in range(Lw.Jout):
        assert np.array_equal(got[i], ref[i]), f"{path}: output ct {i} differs from the oracle"
    check_decrypted(lay, {i: got[i] for i in range(Lw.Jout)})
