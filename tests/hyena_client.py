"""Client-side test harness (TEST INFRASTRUCTURE): plays the PI client of PAPER.md:883-884 —
encrypts inputs and generates Galois keys with the ORACLE — and checks server outputs.

Used by the oracle pins (CPU) and the GPU parity tests; the GPU path receives only the
ciphertexts, keys and int8 weights this module produces.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

import synth
from oracle import bfv, conv


@dataclass
class Layer:
    P: bfv.BFVParams
    plan: conv.Plan
    ls: conv.LayerSetup
    x: np.ndarray
    W: np.ndarray
    s: np.ndarray
    ct_in: np.ndarray                    # [J][2][L][N] uint64
    keys: Dict[int, np.ndarray]          # galois elt -> [L][2][L][N] uint64
    seed: int


def keygen(P: bfv.BFVParams, s, elts: List[int], seed: int) -> Dict[int, np.ndarray]:
    keys = {}
    for n, g in enumerate(elts):
        a = synth.uniform_residues(synth.rng(seed, "a", 100000 + n), P.primes, (P.ND, P.N))
        e = synth.cbd(synth.rng(seed, "e", 100000 + n), (P.ND, P.N))
        keys[g] = bfv.galois_keygen(P, s, g, a, e)
    return keys


def encrypt_slots(P: bfv.BFVParams, s, slots: np.ndarray, seed: int) -> np.ndarray:
    """Encrypt each slot vector (rows of `slots`) with a fresh seeded mask a and error e."""
    from oracle.encoding import encode_batch
    polys = encode_batch(slots, P.t, P.N)
    out = np.empty((len(slots), 2, P.L, P.N), dtype=np.uint64)
    for j, m in enumerate(polys):
        e = synth.cbd(synth.rng(seed, "e", j), P.N)
        a = synth.uniform_residues(synth.rng(seed, "a", j), P.primes, (P.N,))
        out[j] = bfv.encrypt(P, m, s, a, e)
    return out


def make_layer(N: int, primes: List[int], batch: int, Ci: int, Co: int, H: int, W: int, kh: int, kw: int,
               pad: int, depthwise: bool = False, xrange=(-8, 8), wrange=(-8, 8), seed: int = 50,
               force_cn: int = 0, k: int = 0, t: int = synth.T_PLAIN, x=None, Wt=None, w: int = 0) -> Layer:
    P = bfv.BFVParams(N, list(primes), t, w=w)
    p = conv.plan(N, batch, Ci, Co, H, W, kh, kw, pad, depthwise, force_cn)
    ls = conv.setup(p, t, k)
    if x is None:
        x = synth.uniform_int(synth.rng(seed, "x"), xrange[0], xrange[1], (batch, Ci, H, W))
    if Wt is None:
        shape = (Ci, kh, kw) if depthwise else (Co, Ci, kh, kw)
        Wt = synth.uniform_int(synth.rng(seed, "W"), wrange[0], wrange[1], shape).astype(np.int8)
    s = synth.ternary(synth.rng(seed, "sk"), N)
    slots = conv.pack(p, x, t)
    ct_in = encrypt_slots(P, s, slots, seed)
    keys = keygen(P, s, ls.galois, seed)
    return Layer(P, p, ls, x, Wt, s, ct_in, keys, seed)


def layer_from_config(cfg: synth.ConvConfig) -> Layer:
    return make_layer(cfg.N, cfg.primes, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad,
                      cfg.depthwise, seed=cfg.index, force_cn=cfg.force_cn, k=cfg.k, t=cfg.t,
                      x=synth.gen_image(cfg), Wt=synth.gen_weights(cfg))


def expected_plain(layer: Layer) -> np.ndarray:
    """Plain convolution mod t."""
    y = conv.plain_conv(layer.x, layer.W, layer.plan.pad, layer.plan.depthwise)
    return np.mod(y, layer.P.t)


def check_decrypted(layer: Layer, out_cts: Dict[int, np.ndarray]) -> int:
    """Decrypt the given output cts (oracle), unscale, compare every valid position they hold
    against the plain convolution mod t.  Returns the number of positions compared."""
    p = layer.plan
    dec = conv.decrypt_outputs(layer.P, layer.ls, out_cts, layer.s)
    slots = np.zeros((p.Jout, p.N), dtype=np.int64)
    mask = np.zeros((p.Jout, p.N), dtype=bool)
    for i, v in dec.items():
        slots[i] = v
        mask[i] = True
    got = conv.unpack(p, slots)
    have = conv.unpack(p, mask.astype(np.int64)).astype(bool)
    exp = expected_plain(layer)
    bad = np.argwhere(have & (got != exp))
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"
    return int(have.sum())
