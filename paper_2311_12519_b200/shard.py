"""Multi-GPU sharding of one encrypted convolution layer.

Host logic only (no arithmetic of the method): which slice of the layer each rank evaluates
with its own hy_conv_eval, and the gather of the output ciphertexts to rank 0 — the only
collective of the path (north_star: "NCCL over NVLink only to gather output ciphertexts").

Independent pieces of a layer:
  * units (slot-row groups: batch images / halo bands, hy_layout.U): disjoint input and output
    ciphertexts, no shared work -> split units when there are at least as many as ranks;
  * output channels (c_n = 2: channel pairs = output ciphertexts; c_n = 1: channels): every
    rank needs all input ciphertexts and recomputes their rotations (O(Ci f^2), cheap next to
    the O(Ci Co f^2) MAC) and evaluates the layer restricted to its output channels, i.e. the
    weights W[o_lo:o_hi];
  * depthwise layers: channels (pairs for c_n = 2) with their own input ciphertexts.
A rank's slice is itself a valid layer for hy_encode_weights (same N, t, layout, c_n forced),
so sharding needs no library support beyond hy_conv_eval on a unit prefix.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import numpy as np


def _split(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split of range(n) (sizes differ by at most one)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class Shard:
    rank: int
    world: int
    kind: str                      # "units" | "channels"
    shape: Dict[str, int]          # hy_conv_shape fields of this rank's layer (force_cn fixed)
    w_slice: Tuple[int, int]       # slice of the weights' first axis (Co, or C for depthwise)
    in_index: List[int] = field(default_factory=list)   # global input ct indices, in order
    out_index: List[int] = field(default_factory=list)  # global output ct index of each local output

    @property
    def empty(self) -> bool:
        return len(self.out_index) == 0


def plan_shard(layout: Dict[str, int], shape: Dict[str, int], world: int, rank: int) -> Shard:
    """layout: hy_layout fields (U, Jc, Jo, cn, ...) of the FULL layer; shape: its hy_conv_shape.
    Returns what `rank` of `world` evaluates."""
    U, Jc, Jo, cn = layout["U"], layout["Jc"], layout["Jo"], layout["cn"]
    dw = bool(shape.get("depthwise", 0))
    sh = dict(shape)
    sh["force_cn"] = cn
    Co = shape["Ci"] if dw else shape["Co"]
    if U >= world:
        u0, u1 = _split(U, world, rank)
        return Shard(rank, world, "units", sh, (0, Co),
                     [u * Jc + c for u in range(u0, u1) for c in range(Jc)],
                     [u * Jo + o for u in range(u0, u1) for o in range(Jo)])
    # fewer units than ranks: split output ciphertexts of every unit by channel groups
    per = 2 if cn == 2 else 1                      # channels per output ct
    g0, g1 = _split(Jo, world, rank)
    c0, c1 = g0 * per, min(g1 * per, Co)
    if g1 <= g0:
        return Shard(rank, world, "channels", sh, (0, 0), [], [])
    if dw:
        sh["Ci"] = sh["Co"] = c1 - c0
        ins = [u * Jc + j for u in range(U) for j in range(g0, g1)]
    else:
        sh["Co"] = c1 - c0
        ins = list(range(U * Jc))
    outs = [u * Jo + g for u in range(U) for g in range(g0, g1)]
    return Shard(rank, world, "channels", sh, (c0, c1), ins, outs)


def slice_weights(W: np.ndarray, shard: Shard) -> np.ndarray:
    return np.ascontiguousarray(W[shard.w_slice[0]:shard.w_slice[1]])


def gather_outputs(local, shard: Shard, n_out: int, group=None):
    """Gather every rank's output ciphertexts (tensor [n_local][2][L][N], uint64 or int64) into
    a [n_out][2][L][N] tensor on rank 0 (global order); other ranks return None.  One padded
    torch.distributed.gather (NCCL on GPUs, gloo on CPU tests)."""
    import torch
    import torch.distributed as dist

    world = shard.world
    n_local = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    n_max = max(sizes)
    tail = tuple(local.shape[1:])
    buf = torch.zeros((n_max,) + tail, dtype=torch.int64, device=local.device)
    if local.shape[0]:
        buf[: local.shape[0]] = local.view(torch.int64)
    idx = torch.full((n_max,), -1, dtype=torch.int64, device=local.device)
    idx[: len(shard.out_index)] = torch.tensor(shard.out_index, dtype=torch.int64)
    if shard.rank == 0:
        bufs = [torch.empty_like(buf) for _ in range(world)]
        idxs = [torch.empty_like(idx) for _ in range(world)]
    else:
        bufs = idxs = None
    dist.gather(buf, bufs, dst=0, group=group)
    dist.gather(idx, idxs, dst=0, group=group)
    if shard.rank != 0:
        return None
    out = torch.empty((n_out,) + tail, dtype=torch.int64, device=local.device)
    seen = torch.zeros(n_out, dtype=torch.bool)
    for r in range(world):
        ir = idxs[r][: sizes[r]].cpu()
        assert (ir >= 0).all()
        out[ir.to(local.device)] = bufs[r][: sizes[r]]
        seen[ir] = True
    assert bool(seen.all()), "some output ciphertexts were not produced by any rank"
    return out.view(local.dtype) if local.dtype != torch.int64 else out
