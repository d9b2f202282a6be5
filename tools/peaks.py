"""Run tools/intbench on the GPU and write profiles/int_peaks.json: the MEASURED denominators of
bench.py's "alu" and int8-tensor rooflines (64-bit Shoup modmul, IMAD, IMAD.WIDE, DFMA and the
tcgen05 kind::i8 UMMA throughput), per clock per SM and at the max SM clock.

  python tools/peaks.py          # on a B200 (gpurun)
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = os.path.join(ROOT, "tools", "intbench")


def main():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", "intbench",
                           "intbench.cu"], cwd=D)
    out = subprocess.check_output([os.path.join(D, "intbench")], cwd=D, text=True)
    ops = {}
    for ln in out.splitlines():
        if ln.startswith("{"):
            r = json.loads(ln)
            ops[r["op"]] = r
    try:
        smi = subprocess.check_output(["nvidia-smi", "--query-gpu=name,clocks.max.sm,clocks.sm",
                                       "--format=csv,noheader,nounits"], text=True).strip()
    except Exception:
        smi = ""
    res = {
        "how": "tools/intbench/intbench.cu: 148 SMs x 8 CTAs x 256 threads, 8 independent chains per thread "
               "(tcgen05: 1 CTA/SM issuing back-to-back kind::i8 M=128 N=256 K=32 UMMAs), CUDA events, "
               "per_clk_per_sm = ops/s / (148 x cudaDevAttrClockRate)",
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "nvidia_smi": smi,
        "ops": ops,
        "modmul_per_clk_sm": ops["shoup_modmul64"]["per_clk_per_sm_at_maxclk"],
        "dfma_per_clk_sm": ops["dfma"]["per_clk_per_sm_at_maxclk"],
        "imad_per_clk_sm": ops["imad_s32"]["per_clk_per_sm_at_maxclk"],
        "imad_wide_per_clk_sm": ops["imad_wide_s32"]["per_clk_per_sm_at_maxclk"],
        "i8_tensor_tops": ops["tcgen05_i8_ops"]["ops_per_s"] / 1e12,
    }
    path = os.path.join(ROOT, "profiles", "int_peaks.json")
    json.dump(res, open(path, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    sys.exit(main())
