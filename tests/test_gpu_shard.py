"""1-GPU "fake shard" check of the multi-GPU partition:
for world = 2, 4, 8 every rank's slice chosen by shard.plan_shard (units, output channels with
c_n = 2 channel pairs, depthwise channel pairs with their own input ciphertexts) goes through
hy_encode_weights / hy_conv_eval on cuda:0 exactly as bench.py --mode shard sends it; the slices
assembled by out_index must equal the unsharded layer byte for byte, and the unsharded layer the
oracle.  This also covers hy_conv_eval on a unit subset on the tc_fused, tc_coef, thin and
fp64_fused paths.  Marked gpu."""
import numpy as np
import pytest

from oracle import conv
from oracle.params import ntt_primes
from paper_2311_12519_b200 import shard as sh
from tests.hyena_client import make_layer

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = {
    # units when U >= world, channels otherwise (tc_fused: 32 < M <= 128)
    "units_tc": dict(N=1024, batch=64, Ci=3, Co=40, H=6, W=6, kh=3, kw=3, pad=1, wrange=(-128, 128)),
    # 1x1 c_n = 1 (tc_coef): units
    "units_pw": dict(N=1024, batch=64, Ci=20, Co=36, H=6, W=6, kh=1, kw=1, pad=0),
    # c_n = 2, one unit: output channel pairs (fp64_fused)
    "channels_cn2": dict(N=1024, batch=1, Ci=4, Co=16, H=6, W=6, kh=3, kw=3, pad=1),
    # depthwise c_n = 2: channel pairs with their own input cts (thin)
    "dw_cn2": dict(N=1024, batch=1, Ci=16, Co=16, H=6, W=6, kh=3, kw=3, pad=1, depthwise=True),
    # depthwise c_n = 1 with units
    "dw_units": dict(N=1024, batch=40, Ci=3, Co=3, H=6, W=6, kh=3, kw=3, pad=1, depthwise=True),
}


@pytest.fixture(scope="module")
def hy():
    import paper_2311_12519_b200 as pkg
    from paper_2311_12519_b200 import build
    build.build()
    pkg.load_library()
    assert torch.cuda.is_available()
    return pkg


def _shape(lay):
    p = lay.plan
    return dict(Ci=p.Ci, Co=p.Co, H=p.H, W=p.W, kh=p.kh, kw=p.kw, pad=p.pad, depthwise=int(p.depthwise),
                batch=p.batch, k=lay.ls.k if p.cn == 2 else 0, force_cn=0)


def _eval(hy, p, W, shape, ct, n_out):
    w = hy.hy_encode_weights(p, W, **shape)
    try:
        lay = hy.hy_weights_layout(w)
        d_in = torch.from_numpy(np.ascontiguousarray(ct)).cuda()
        d_out = torch.full((n_out, 2, ct.shape[2], ct.shape[3]), 11, dtype=torch.uint64, device="cuda")
        hy.hy_conv_eval(w, d_in, d_out)
        torch.cuda.synchronize()
        return d_out.cpu().numpy(), hy.hy_weights_mac_path(w)
    finally:
        hy.hy_weights_destroy(w)


@pytest.mark.parametrize("name", sorted(CASES))
def test_fake_shard_equals_unsharded(hy, name):
    c = dict(CASES[name])
    N = c.pop("N")
    primes = ntt_primes(N, 50, 2)
    lay = make_layer(N, primes, seed=1200 + sorted(CASES).index(name), **c)
    p = hy.hy_params_create(N, primes, lay.P.t, 0)
    try:
        elts = list(lay.keys)
        if elts:
            hy.hy_keys_upload(p, elts, np.stack([lay.keys[g] for g in elts]))
        shape = _shape(lay)
        full = hy.hy_plan_layout(N, lay.P.t, **shape)
        ref, path = _eval(hy, p, lay.W, shape, lay.ct_in, full.Jout)
        oracle = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
        for i in range(full.Jout):
            assert np.array_equal(ref[i], oracle[i]), f"unsharded output {i} differs from the oracle"
        kinds = set()
        for world in (2, 4, 8):
            got = np.zeros_like(ref)
            seen = np.zeros(full.Jout, dtype=bool)
            for rank in range(world):
                s = sh.plan_shard(hy.layout_dict(full), shape, world, rank)
                kinds.add(s.kind)
                if s.empty:
                    continue
                out, _ = _eval(hy, p, sh.slice_weights(lay.W, s), s.shape, lay.ct_in[s.in_index],
                               len(s.out_index))
                got[s.out_index] = out
                assert not seen[s.out_index].any(), "two ranks produced the same output ct"
                seen[s.out_index] = True
            assert seen.all(), f"world {world}: outputs not covered"
            assert np.array_equal(got, ref), f"world {world}: assembled shards differ from the unsharded layer"
        print(name, path, sorted(kinds))
    finally:
        hy.hy_params_destroy(p)
