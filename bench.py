#!/usr/bin/env python
"""Benchmark of the Hyena encrypted-convolution hot path on B200 (contract: see DESIGN.md §Measurement).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A step = one hy_conv_eval of the configured layer (all of SURVEY §8(a): PermDecomp, PermAuto fused
with the lazy MAC + WHT + reduction + sign PMult, row-swap alignment, INTT) on synthetic
ciphertexts already resident in HBM.  Default workload: BASELINE.json configs[3] (C4, the VGG-16
early layer Ci = Co = 64 at 224 x 224, batch 8, N = 8192, L = 3): the metric names only N = 8192, so
the workload is the largest single-GPU N = 8192 configuration; the other configs (--config) are
parity-test cases and secondary lines.
Multi-GPU (torchrun), --mode replica (default): every rank evaluates its own layer instance on
its own images (weak scaling, no data-path collective); --mode shard: the ranks split ONE layer
(units or output channels, paper_2311_12519_b200/shard.py) and rank 0 gathers the output
ciphertexts with NCCL (strong scaling; the gather is inside the timed step).  The time is the
max over ranks of CUDA-event time.

Inputs are uniformly random ciphertexts and switching keys (synth/): under RLWE a real
encryption is indistinguishable from uniform, and the kernels' work does not depend on the values.
bench.py never runs the oracle except in the cpu_baseline leg (rank 0, N = 1) and --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

import synth

METRIC = "encrypted conv layers/sec (ct×pt MAC GOps/s) at N=8192; % of HBM/INT roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
INT_PEAKS_PATH = os.path.join(ROOT, "profiles", "int_peaks.json")
SM_COUNT = 148
DFMA_PER_CLK_SM = 64     # FP64 pipe: 16 lanes/clk/SMSP x 4 (tools/intbench measured 58/clk/SM at 1965 MHz nominal)
IMAD_PER_CLK_SM = 64


def load_peaks():
    """MEASURED_PEAKS.json (driver-written: HBM copy GB/s, bf16 TF/s) + profiles/int_peaks.json
    (tools/peaks.py on a B200: Shoup modmul, DFMA and tcgen05 int8 throughput)."""
    out = {}
    for path in (PEAKS_PATH, INT_PEAKS_PATH):
        try:
            out.update(json.load(open(path)))
        except Exception:
            pass
    return out


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML while the timed region runs."""

    def __init__(self, dev: int = 0, period: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.dev = period, dev
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------------------------
STAGES = ["S1_permdecomp", "S2S3_ksmac_wht", "S4S5_align_intt"]


def run_gpu(args, cfg, rank, world):
    import torch
    import paper_2311_12519_b200 as hy
    from paper_2311_12519_b200 import build
    from paper_2311_12519_b200 import shard as shard_mod

    if rank == 0 or not os.path.exists(hy.library_path()):
        build.build()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    device = f"cuda:{dev}"
    L, N = len(cfg.primes), cfg.N
    full = hy.hy_plan_layout(cfg.N, cfg.t, **cfg.shape_dict())
    W_full = synth.gen_weights(cfg)
    shard = None
    if args.mode == "shard" and world > 1:
        shard = shard_mod.plan_shard(hy.layout_dict(full), cfg.shape_dict(), world, rank)
        shape, W = shard.shape, shard_mod.slice_weights(W_full, shard)
        ct_full = synth.gen_uniform_cts(cfg.primes, full.J, cfg.N, cfg.index, stream=0)
        ct_host = np.ascontiguousarray(ct_full[shard.in_index])
    else:                   # replica: this rank's own images through the whole layer
        shape, W = cfg.shape_dict(), W_full
        ct_host = synth.gen_uniform_cts(cfg.primes, full.J, cfg.N, cfg.index, stream=rank)
    p = hy.hy_params_create(cfg.N, cfg.primes, cfg.t, dev)
    elts = list(full.galois[:full.n_galois])
    if elts:
        hy.hy_keys_upload(p, elts, synth.gen_uniform_keys(cfg.primes, len(elts), cfg.N, cfg.index))
    w = None
    empty = shard is not None and shard.empty
    if not empty:
        w = hy.hy_encode_weights(p, W, **shape)
        lay = hy.hy_weights_layout(w)
        # a units shard keeps the full layer's shape and evaluates its own units only
        n_out = len(shard.out_index) if shard is not None else lay.Jout
        assert len(ct_host) == n_out // lay.Jo * lay.Jc
        ct_in = torch.from_numpy(ct_host).to(device)
        ct_out = torch.empty((n_out, 2, L, cfg.N), dtype=torch.uint64, device=device)
    else:
        lay = None
        ct_out = torch.empty((0, 2, L, cfg.N), dtype=torch.uint64, device=device)
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=device)  # > 126 MB L2

    def step():
        if not empty:
            hy.hy_conv_eval(w, ct_in, ct_out)
        if shard is not None:
            shard_mod.gather_outputs(ct_out, shard, full.Jout)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    mac_path = None
    if w is not None:
        if args.mac_path:
            hy.hy_weights_set_mac_path(w, args.mac_path)
        mac_path = hy.hy_weights_mac_path(w)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    step_ms, stage_ms, mac_ms, mac_n = [], [[] for _ in range(3)], [], 0
    launches0 = hy.hy_kernel_launches()
    # timed steps: no events inside the step (they would serialise the programmatic-dependent
    # launches between the library's kernels)
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.zero_()                       # L2 flushed between timed iterations (untimed)
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            t0.record()
            step()
            t1.record()
            t1.synchronize()
            step_ms.append(t0.elapsed_time(t1))
    torch.cuda.synchronize()
    launches = hy.hy_kernel_launches() - launches0
    # per-stage / per-MAC-launch breakdown (rooflines): the same steps with the library's stage and
    # MAC-launch events enabled, timed separately
    if w is not None:
        hy.hy_weights_set_stage_events(w, ev)
        for it in range(min(args.steps, 10) + 1):
            flush.zero_()
            torch.cuda.synchronize()
            step()
            torch.cuda.synchronize()
            if it == 0:
                continue                        # first run with events: warm-up
            for i in range(3):
                stage_ms[i].append(ev[i].elapsed_time(ev[i + 1]))
            m, n = hy.hy_weights_mac_time(w)      # the MAC kernel's own launches
            mac_ms.append(m)
            mac_n += n
    total_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([total_ms, float(launches)], dtype=torch.float64, device=device)
        tl = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(tl, t)
        total_ms = max(float(x[0].item()) for x in tl)          # max over ranks
        launches = int(sum(float(x[1].item()) for x in tl))     # all ranks' kernels
        dist.barrier()

    # end-to-end through the public host API: H2D of the inputs and D2H of the outputs inside
    # the timed region, every step (hy_conv_eval_host synchronises its stream)
    e2e_s, e2e_steps = None, max(3, min(args.steps, 50))
    if w is not None:
        hy.hy_weights_set_stage_events(w, [])
        pin_in = torch.from_numpy(ct_host).pin_memory().numpy()
        pin_out = torch.empty(tuple(ct_out.shape), dtype=torch.uint64).pin_memory().numpy()
        for _ in range(2):
            hy.hy_conv_eval_host(w, pin_in, pin_out)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    tt = time.perf_counter()
    for _ in range(e2e_steps):
        if w is not None:
            hy.hy_conv_eval_host(w, pin_in, pin_out)
        if shard is not None:      # the gather runs on device buffers of the host call's outputs
            shard_mod.gather_outputs(torch.from_numpy(pin_out).to(device) if w is not None else ct_out,
                                     shard, full.Jout)
    e2e_s = time.perf_counter() - tt
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    if w is not None:
        hy.hy_weights_destroy(w)
    hy.hy_params_destroy(p)
    return dict(total_ms=total_ms, step_ms=step_ms, mac_path=mac_path,
                stage_ms=[statistics.mean(s) if s else 0.0 for s in stage_ms],
                mac_ms=statistics.mean(mac_ms) if mac_ms else 0.0, mac_launches=mac_n,
                launches=launches, clocks=clk.summary(), lay=lay, full=full, e2e_s=e2e_s, e2e_steps=e2e_steps,
                in_bytes=len(ct_host) * 2 * L * N * 8, out_bytes=int(ct_out.shape[0]) * 2 * L * N * 8)


def layer_work(cfg, lay):
    """Algorithmic work of one hy_conv_eval on layout `lay`.
    coef_macs: coefficient-MACs of S3 (M MAC rows x K terms x 2LN columns per unit; c_n = 2 has
    4 rows per output ct = 2 diagonals x 2 slot rows).  Modular products
    ("modmul" = one 64-bit Shoup product, the unit of the INT roofline) per stage:
      S1: (L^2 + L) forward NTTs per input ct, N/2 log2 N butterflies each;
      S2: 2 L^2 N key-switching products per (input ct, non-identity tap) (hoisted PermAuto);
      S4+S5: c_n = 2 non-depthwise: per output ct L INTT + L(L-1) NTT + 2 L^2 N key switching +
             2L INTT (row swap, then coefficient form); otherwise 2L INTT per output ct."""
    L, N, T = len(cfg.primes), cfg.N, lay.n_taps
    ctw = 2 * L * N
    if cfg.depthwise:
        M, K, units = (2 if lay.cn == 2 else 1), T, lay.U * lay.Jc
    else:
        M, K, units = (4 * lay.Jo if lay.cn == 2 else lay.Jo), lay.Jc * T, lay.U
    mac = M * K * ctw * units
    ntap = sum(1 for s in lay.tap_step[:T] if s % (N // 2))
    rot = lay.J * ntap
    swaps = lay.Jout if (lay.cn == 2 and not cfg.depthwise) else 0
    bfly = N // 2 * int(np.log2(N))
    s1 = lay.J * (L * L + L) * bfly
    s2 = rot * 2 * L * L * N
    s45 = swaps * ((L + L * (L - 1)) * bfly + 2 * L * L * N) + lay.Jout * 2 * L * bfly
    return dict(coef_macs=mac, dfma=2 * mac, rotations=rot, rowswaps=swaps, M=M, K=K, units=units,
                modmul={"S1_permdecomp": s1, "S2S3_ksmac_wht": s2, "S4S5_align_intt": s45},
                r_bytes=K * ctw * 8 * units, in_bytes=lay.J * ctw * 8, out_bytes=lay.Jout * ctw * 8)


def traffic_for(cfg_name, kernel):
    """dram bytes per launch of `kernel` from the committed ncu capture (profiles/traffic.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[cfg_name][kernel]
    except Exception:
        return None


MODMUL_PER_CLK_SM = 4.0   # 64-bit Shoup product = 6 IMAD.WIDE (2 issue slots) + 4 IMAD on 64 lanes/clk/SM
I8_PER_BF16 = 2.0         # dense int8 / bf16 tensor throughput, nominal (B200_PROFILING.md: 4.5 vs 2.25 P)
MAC_KERNEL = {"thin": "ksmac_thin_kernel (fused S2+S3, FP64 MAC)",
              "tc_fused": "ksmac_v2_kernel (persistent fused S2+S3: key switching + tcgen05 int8 MAC; HY_KSMAC=1 selects round 1's ksmac_tc_kernel)",
              "tc_split": "mac_tc_kernel (S3 tcgen05 int8 MAC over stored R)",
              "fp64_fused": "ksmac_gemm_kernel (fused S2+S3, FP64 MAC)",
              "fp64_split": "mac_gemm_kernel (S3 FP64 MAC over stored R)",
              "tc_coef": "ksmac_tc_kernel (1x1: tcgen05 int8 MAC on the coefficient-form input cts, no key switching)",
              "eager": "mac_eager_kernel (ablation: lazy reduction off, one Shoup product per coefficient-MAC)",
              "direct": "mac_tc_kernel after per-rotation decompositions (ablation: hoisting off)"}


def roofline(cfg, res, peaks, steps):
    """Roofline of the dominant kernel of the step.  Stage times come from CUDA events
    the library records on its stream; the MAC kernel's own launches are timed separately.
      - INT-bound kernels (NTTs, key switching fused into the MAC): achieved = algorithmic 64-bit
        modular products / time; peak = MODMUL_PER_CLK_SM x 148 SMs x max SM clock (unit count
        derived in DESIGN.md §4, measured by tools/intbench).
      - tc_split MAC: HBM-bound streaming of the stored rotated inputs R (algorithmic bytes = R read
        + outputs written) against the measured HBM copy bandwidth.
      - FP64 MAC variants: 2 exact DFMA per coefficient-MAC against 64 DFMA/clk/SM."""
    lay = res["lay"]
    w = layer_work(cfg, lay)
    st = dict(zip(STAGES, res["stage_ms"]))
    path = res.get("mac_path", "tc_fused")
    clk_mhz = res["clocks"].get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    mm_clk = peaks.get("modmul_per_clk_sm", MODMUL_PER_CLK_SM)            # measured (tools/peaks.py)
    dfma_clk = peaks.get("dfma_per_clk_sm", DFMA_PER_CLK_SM)
    int_peak = mm_clk * SM_COUNT * clk_mhz * 1e6 / 1e9                    # Gmodmul/s
    mac_ms = res["mac_ms"] or st["S2S3_ksmac_wht"]
    per_step = max(1, res["mac_launches"] // max(1, min(steps, 10)))
    dom = max(st, key=st.get)
    kernels = {}
    if path == "tc_coef":           # 1x1 coefficient-domain MAC: no S1; c_n = 2 keeps the row swap
        L, N = len(cfg.primes), cfg.N
        bfly = N // 2 * int(np.log2(N))
        w["modmul"]["S1_permdecomp"] = 0
        w["modmul"]["S4S5_align_intt"] = (lay.Jout * ((L * L + L) * bfly + 2 * L * L * N + 2 * L * bfly)
                                          if lay.cn == 2 else 0)
    for stage in ("S1_permdecomp", "S4S5_align_intt"):
        if w["modmul"][stage] == 0:   # empty stage (1x1 coefficient-domain path)
            kernels[stage] = {"bound": "none", "achieved": 0.0, "peak": int_peak, "unit": "Gmodmul/s", "frac": 0.0,
                              "ms": st[stage], "note": "empty stage (no NTT in this stage of the 1x1 path)"}
            continue
        a = w["modmul"][stage] / (st[stage] * 1e-3) / 1e9 if st[stage] > 0 else 0.0
        kernels[stage] = {"bound": "alu", "achieved": a, "peak": int_peak, "unit": "Gmodmul/s",
                          "frac": a / int_peak, "ms": st[stage]}
    if path == "eager":             # one modular product per coefficient-MAC (the ablation's bound)
        a = w["coef_macs"] / (mac_ms * 1e-3) / 1e9
        mac = {"bound": "alu", "achieved": a, "peak": int_peak, "unit": "Gmodmul/s", "frac": a / int_peak}
    elif path in ("tc_fused", "thin"):
        a = w["modmul"]["S2S3_ksmac_wht"] / (mac_ms * 1e-3) / 1e9
        mac = {"bound": "alu", "achieved": a, "peak": int_peak, "unit": "Gmodmul/s", "frac": a / int_peak}
    elif path in ("tc_split", "tc_coef", "direct"):
        hbm = peaks.get("hbm_gbs", 6546.6)
        a = (w["r_bytes"] + w["out_bytes"] * (2 if lay.cn == 2 and not cfg.depthwise else 1)) / (mac_ms * 1e-3) / 1e9
        mac = {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm}
    else:
        pk = dfma_clk * SM_COUNT * clk_mhz * 1e6 / 1e12
        a = w["dfma"] / (mac_ms * 1e-3) / 1e12
        mac = {"bound": "alu", "achieved": a, "peak": pk, "unit": "TDFMA/s", "frac": a / pk}
    mac.update(kernel=MAC_KERNEL[path], ms=mac_ms, launches_per_step=per_step)
    if path.startswith("tc"):
        i8 = 2 * 8 * w["coef_macs"] / (mac_ms * 1e-3) / 1e12                # 8 byte planes
        i8_peak = peaks.get("i8_tensor_tops") or peaks.get("bf16_tflops", 2250.0) * I8_PER_BF16
        mac["tensor_int8"] = {"achieved": i8, "peak": i8_peak, "unit": "TOP/s", "frac": i8 / i8_peak,
                              "peak_source": "profiles/int_peaks.json (tcgen05 kind::i8 microbench)"
                              if peaks.get("i8_tensor_tops") else "bf16 measured x nominal int8/bf16 ratio 2"}
    kernels["S2S3_ksmac_wht"] = mac
    top = dict(kernels[dom])
    top.setdefault("kernel", {"S1_permdecomp": "ntt_fwd_kernel<PermDecompJob> (S1)",
                              "S4S5_align_intt": "S4+S5 stage (row-swap key switching, NTT/INTT)"}.get(dom, dom))
    top["dominant_stage"] = dom
    top["share_of_step"] = st[dom] / max(1e-9, sum(st.values()))
    top["traffic"] = traffic_for(cfg.name, dom)
    src = "measured, profiles/int_peaks.json" if "modmul_per_clk_sm" in peaks else "unit-count nominal"
    top["peak_note"] = (f"INT: {mm_clk:g} Shoup modmul/clk/SM ({src}) x {SM_COUNT} SMs x {clk_mhz:.0f} MHz; "
                        "HBM: MEASURED_PEAKS.json hbm_gbs")
    top["stages"] = kernels
    return top


# --------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference)
# --------------------------------------------------------------------------------------------
def oracle_sample(cfg):
    """Time the oracle AS IT STANDS on a bounded, exact 1/J share of the layer (J = input cts):
    its work is one PermDecomp + hoisted rotation per (input ct, non-identity tap) and one MAC
    (+ WHT, sign PMult and row-swap HRot for c_n = 2) per output ct, identical for every input /
    output ct, so the sample = one input ct's rotations (conv.rotations) + Jout/J output cts'
    evaluation from those rotations (conv.he_conv with R given) is 1/J of a layer.
    Returns (layers per sample, seconds, description)."""
    from oracle import bfv, conv
    P = bfv.BFVParams(cfg.N, cfg.primes, cfg.t)
    p = conv.plan(cfg.N, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad, cfg.depthwise,
                  cfg.force_cn)
    ls = conv.setup(p, cfg.t, cfg.k)
    ct = synth.gen_uniform_cts(cfg.primes, 1, cfg.N, cfg.index, stream=9)
    kk = synth.gen_uniform_keys(cfg.primes, max(1, len(ls.galois)), cfg.N, cfg.index)
    keys = {g: kk[n] for n, g in enumerate(ls.galois)}
    W = synth.gen_weights(cfg)
    n_out = max(1, p.Jout // p.J)
    t0 = time.perf_counter()
    R1 = conv.rotations(P, p, ct, keys, cts=[0])                  # one input ct, every tap
    # every output ct of unit 0 reads R[(c, tau)] for all its input cts: the same rotated ct
    # stands in for each (values do not change the oracle's work)
    R = {(c, tau): R1[(0, tau)] for c in range(max(p.Jc, n_out)) for tau in range(len(p.taps))}
    conv.he_conv(P, ls, W, ct, keys, out_cts=list(range(n_out)), R=R)
    dt = time.perf_counter() - t0
    n_rot = sum(1 for _, _, s in p.taps if s % (cfg.N // 2))
    desc = (f"exact 1/J = 1/{p.J} share of the layer: 1 input ct's PermDecomp + {n_rot} hoisted rotations and "
            f"{n_out} output ct(s)' MAC over {p.Jc if not p.depthwise else 1}x{len(p.taps)} terms"
            + (" + WHT/sign PMult/row-swap HRot" if p.cn == 2 else "") + f" ({dt:.2f} s); single thread")
    return 1.0 / p.J, dt, desc


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    secs, desc, frac = [], "", 1.0
    for i in range(args.warmup + args.steps):
        frac, dt, desc = oracle_sample(cfg)
        if i >= args.warmup:
            secs.append(dt)
    sec = sum(secs)
    v = frac * len(secs) / sec
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "layers/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", 1)), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec / len(secs), "layers_per_step": frac, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "int (Python/NumPy + C schoolbook)", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "N": cfg.N, "L": len(cfg.primes)},
            "cpu_baseline": {"value": v, "unit": "layers/s", "cores": 1, "kind": "oracle", "sample": desc,
                             "host": host_info()},
            "e2e": {"value": v, "unit": "layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def host_info():
    import platform
    model = platform.processor()
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count()}


def workload_name(cfg):
    return (f"{cfg.name}: Ci={cfg.Ci} Co={cfg.Co} H=W={cfg.H} {cfg.kh}x{cfg.kw} pad={cfg.pad} batch={cfg.batch} "
            f"depthwise={cfg.depthwise} N={cfg.N} L={len(cfg.primes)} (BASELINE.json configs)")


# --------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 50; 10 for --impl reference, whose steps take seconds)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="hyena", choices=["hyena", "reference"])
    ap.add_argument("--mode", default="replica", choices=["replica", "shard"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mac-path", default=None, help="A/B: force an S2+S3 kernel path (hyena.MAC_PATHS)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 10 if getattr(args, "impl", None) == "reference" else 50
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    cfg = synth.configs()[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{int(os.environ.get('LOCAL_RANK', 0))}"))
    res = run_gpu(args, cfg, rank, world)
    if rank == 0:
        peaks = load_peaks()
        full, lay = res["full"], res["lay"]
        work = layer_work(cfg, full)
        ms = res["total_ms"] / args.steps
        shard = args.mode == "shard" and world > 1
        layers_per_step = 1 if shard else world
        layers_s = layers_per_step * args.steps / (res["total_ms"] * 1e-3)
        e2e = layers_per_step * res["e2e_steps"] / res["e2e_s"]
        line = {
            "metric": METRIC, "value": layers_s, "unit": "layers/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if shard else "weak", "vs_baseline": None,
            "dtype": "u64",
            "data": "synthetic (uniform ciphertexts + keys: RLWE-indistinguishable from real encryptions; "
                    "int8 weights uniform in the config's range)",
            "config": {"workload": workload_name(cfg),
                       "N": cfg.N, "L": len(cfg.primes), "t": cfg.t, "c_n": full.cn, "k": full.k, "J": full.J,
                       "Jout": full.Jout, "rotations": work["rotations"], "rowswaps": work["rowswaps"],
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "parallelism": (f"shard x{world} (units/output channels + NCCL gather to rank 0)" if shard
                                       else f"replica x{world} (independent images per GPU)")},
            "ct_mac_gops": layers_s * work["coef_macs"] / 1e9,
            "stages_ms": dict(zip(STAGES, res["stage_ms"])),
            "mac_path": res["mac_path"],
            "roofline": roofline(cfg, res, peaks, args.steps) if lay is not None else None,
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
            "e2e": {"value": e2e, "unit": "layers/s", "h2d_bytes_per_step": res["in_bytes"],
                    "d2h_bytes_per_step": res["out_bytes"]},
        }
        if world == 1 and not args.no_cpu_baseline:
            frac, dt, desc = oracle_sample(cfg)
            line["cpu_baseline"] = {"value": frac / dt, "unit": "layers/s", "cores": 1, "kind": "oracle",
                                    "sample": desc, "host": host_info()}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
