"""Write tests/golden/fullsize_sha256.json: SHA-256 of every output ciphertext the ORACLE computes
for full-size BASELINE configs on seeded dense uniform inputs (test infrastructure; calls only
oracle/ and synth/, never the CUDA path).

  python tools/make_golden.py [C1 C2 C3a C3b C4]      # multi-process over input / output cts

Inputs (regenerated identically by tests/test_gpu_golden.py):
  ct_in = synth.gen_uniform_cts(primes, J, N, cfg.index, stream=11)   dense uniform [J][2][L][N]
  keys  = synth.gen_uniform_keys(primes, n_galois, N, cfg.index)       dense uniform, layout order
  W     = synth.gen_weights(cfg)
Outputs covered: every output ct of C1, C2, C3a, C3b; units 0 and U-1 of C4 (64 + 64 of 4096).
"""
from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import synth
from oracle import bfv, conv

OUT = os.path.join(ROOT, "tests", "golden", "fullsize_sha256.json")
STREAM = 11
G = {}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def _rot(ci):
    return conv.rotations(G["P"], G["p"], G["ct"], G["keys"], cts=[ci])


def _out(oc):
    res = conv.he_conv(G["P"], G["ls"], G["W"], G["ct"], G["keys"], out_cts=[oc], R=G["R"])
    return oc, sha(res[oc])


def setup(cfg):
    P = bfv.BFVParams(cfg.N, cfg.primes, cfg.t)
    p = conv.plan(cfg.N, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad, cfg.depthwise,
                  cfg.force_cn)
    ls = conv.setup(p, cfg.t, cfg.k)
    ct = synth.gen_uniform_cts(cfg.primes, p.J, cfg.N, cfg.index, stream=STREAM)
    kk = synth.gen_uniform_keys(cfg.primes, max(1, len(ls.galois)), cfg.N, cfg.index)
    keys = {g: kk[n] for n, g in enumerate(ls.galois)}
    return P, p, ls, ct, kk, keys


def golden(name: str, procs: int):
    cfg = synth.configs()[name]
    P, p, ls, ct, kk, keys = setup(cfg)
    units = [0, p.U - 1] if name == "C4" else list(range(p.U))
    units = sorted(set(units))
    in_cts = [u * p.Jc + c for u in units for c in range(p.Jc)]
    out_cts = [u * p.Jo + o for u in units for o in range(p.Jo)]
    G.update(P=P, p=p, ls=ls, ct=ct, keys=keys, W=synth.gen_weights(cfg))
    t0 = time.time()
    with mp.get_context("fork").Pool(procs) as pool:
        R = {}
        for r in pool.imap_unordered(_rot, in_cts, chunksize=1):
            R.update(r)
    G["R"] = R
    t1 = time.time()
    with mp.get_context("fork").Pool(procs) as pool:
        hashes = dict(pool.imap_unordered(_out, out_cts, chunksize=1))
    t2 = time.time()
    print(f"{name}: {len(in_cts)} input cts rotated in {t1 - t0:.0f} s, {len(out_cts)} outputs in {t2 - t1:.0f} s",
          flush=True)
    return {"J": p.J, "Jout": p.Jout, "units": units, "ct_in_sha256": sha(ct), "keys_sha256": sha(kk),
            "weights_sha256": hashlib.sha256(synth.gen_weights(cfg).tobytes()).hexdigest(),
            "inputs": f"synth.gen_uniform_cts(primes, {p.J}, {cfg.N}, {cfg.index}, stream={STREAM}); "
                      f"synth.gen_uniform_keys(primes, {len(ls.galois)}, {cfg.N}, {cfg.index}); synth.gen_weights",
            "outputs": {str(k): hashes[k] for k in sorted(hashes)}}


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3a", "C3b", "C4"]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "_source": "tools/make_golden.py (oracle/ only): SHA-256 of oracle output ciphertexts, little-endian u64 "
                   "[2][L][N]"}
    for n in names:
        data[n] = golden(n, os.cpu_count() or 1)
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
