"""Multi-rank sharding on CPU: world_size 2 over gloo.  Every rank
evaluates its shard of a tiny layer (with the ORACLE standing in for its GPU — the GPU side
runs the same slices through hy_conv_eval in bench.py --mode shard), rank 0 gathers with
shard.gather_outputs, and the assembled ciphertexts must equal the unsharded oracle layer bit
for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bfv, conv
from oracle.params import ntt_primes
from paper_2311_12519_b200 import shard as sh
from tests.hyena_client import make_layer

CASES = {
    # name: make_layer kwargs (N small so the oracle is fast)
    "units_cn1": dict(N=128, batch=5, Ci=2, Co=3, H=4, W=4, kh=3, kw=3, pad=1),
    "channels_cn2": dict(N=128, batch=1, Ci=4, Co=6, H=4, W=4, kh=3, kw=3, pad=1),
    "channels_cn1": dict(N=128, batch=2, Ci=2, Co=3, H=4, W=4, kh=3, kw=3, pad=1, force_cn=1),
    "dw_cn2": dict(N=128, batch=1, Ci=6, Co=6, H=4, W=4, kh=3, kw=3, pad=1, depthwise=True),
    "dw_units": dict(N=128, batch=5, Ci=3, Co=3, H=4, W=4, kh=3, kw=3, pad=1, depthwise=True),
}


def _layer(name):
    c = dict(CASES[name])
    N = c.pop("N")
    return make_layer(N, ntt_primes(N, 50, 2), seed=800 + sorted(CASES).index(name), **c)


def _layout(lay):
    p = lay.plan
    return dict(U=p.U, Jc=p.Jc, Jo=p.Jo, cn=p.cn, J=p.J, Jout=p.Jout)


def _shape(lay):
    p = lay.plan
    return dict(Ci=p.Ci, Co=p.Co, H=p.H, W=p.W, kh=p.kh, kw=p.kw, pad=p.pad, depthwise=int(p.depthwise),
                batch=p.batch, k=lay.ls.k if p.cn == 2 else 0, force_cn=0)


def _eval_shard(lay, s):
    """The rank's slice as its own layer (what hy_encode_weights + hy_conv_eval get)."""
    if s.empty:
        return np.zeros((0, 2, lay.P.L, lay.P.N), dtype=np.uint64)
    shp = s.shape
    p2 = conv.plan(lay.P.N, shp["batch"], shp["Ci"], shp["Co"], shp["H"], shp["W"], shp["kh"], shp["kw"],
                   shp["pad"], bool(shp["depthwise"]), shp["force_cn"])
    ls2 = conv.setup(p2, lay.P.t, lay.ls.k if p2.cn == 2 else 0)
    ct = lay.ct_in[s.in_index]
    n_local = len(s.out_index)
    res = conv.he_conv(lay.P, ls2, sh.slice_weights(lay.W, s), ct, lay.keys, out_cts=list(range(n_local)))
    return np.stack([res[i] for i in range(n_local)])


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = _layer(name)
        s = sh.plan_shard(_layout(lay), _shape(lay), world, rank)
        local = torch.from_numpy(_eval_shard(lay, s))
        out = sh.gather_outputs(local, s, lay.plan.Jout)
        if rank == 0:
            ref = conv.he_conv(lay.P, lay.ls, lay.W, lay.ct_in, lay.keys)
            got = out.numpy()
            ok = all(np.array_equal(got[i], ref[i]) for i in range(lay.plan.Jout))
            q.put((s.kind, ok))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.parametrize("name", sorted(CASES))
def test_sharded_equals_single(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(2, _free_port(), name, q), nprocs=2, join=True, start_method="spawn")
    kind, ok = q.get(timeout=60)
    assert ok, f"{name} ({kind}): sharded outputs differ from the single-rank layer"
    expect = "units" if name.endswith("units") or name == "units_cn1" else "channels"
    assert kind == expect


def test_plan_covers_every_output_once():
    for name in CASES:
        lay = _layer(name)
        for world in (1, 2, 3, 4, 8):
            outs = []
            for r in range(world):
                outs += sh.plan_shard(_layout(lay), _shape(lay), world, r).out_index
            assert sorted(outs) == list(range(lay.plan.Jout)), (name, world)
