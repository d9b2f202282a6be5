"""Copy the evidence of a GPU run from gpurun_out/ into profiles/ (tracked): bench JSON lines,
ncu launch lists with per-kernel shares, and the per-kernel counters of the ncu --set full
captures (duration, DRAM bytes, pipe utilisation, registers) + profiles/traffic.json.
Usage: python tools/gpu/mkprofiles.py r01"""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs("profiles", exist_ok=True)
out_md = [f"# Profiles {tag}\n", "All numbers from B200 runs through `gpurun` (commands in tools/gpu/). ncu launch times "
          "are cold-cache and serialised: compare shares, not absolutes.\n"]

# bench lines
bench = {}
for f in sorted(glob.glob("gpurun_out/bench_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            name = os.path.basename(f)[6:-4]
            bench[name] = d
json.dump(bench, open(f"profiles/{tag}_bench.json", "w"), indent=1)
out_md.append("## bench.py lines\n\n| run | value | ms/step | MAC path | S1 ms | S2+S3 ms | S4+S5 ms | dominant stage: kernel, achieved / peak (frac) | e2e | clocks |\n|---|---|---|---|---|---|---|---|---|---|")
for n, d in bench.items():
    if "roofline" not in d:
        out_md.append(f"| {n} (reference arm) | {d['value']:.4g} {d['unit']} | {d['ms_per_step']:.1f} | | | | | | | |")
        continue
    st = d["stages_ms"]
    r = d["roofline"] or {}
    out_md.append(f"| {n} | {d['value']:.1f} {d['unit']} | {d['ms_per_step']:.3f} | {d.get('mac_path')} | "
                  f"{st['S1_permdecomp']:.3f} | {st['S2S3_ksmac_wht']:.3f} | {st['S4S5_align_intt']:.3f} | "
                  f"{r.get('dominant_stage')}: {r.get('kernel', '')[:40]}, {r.get('achieved', 0):.1f} / {r.get('peak', 0):.1f} "
                  f"{r.get('unit', '')} ({r.get('frac', 0):.3f}) | {d['e2e']['value']:.1f} | {d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']} |")

# launch lists
for f in sorted(glob.glob("gpurun_out/launches_*.csv")):
    cfg = os.path.basename(f)[9:-4]
    rows = [r for r in csv.reader(open(f)) if len(r) > 5]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows:
        agg.setdefault(r[ki].split("(")[0][:90], []).append(float(r[vi].replace(",", "")) / 1000)
    tot = sum(sum(v) for v in agg.values())
    os.system(f"cp {f} profiles/{tag}_launches_{cfg}.csv")
    out_md.append(f"\n## ncu launch list {cfg} ({len(rows)} launches, gpu__time_duration.sum)\n\n| share | launches | avg µs | kernel |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out_md.append(f"| {sum(v) / tot * 100:.1f}% | {len(v)} | {sum(v) / len(v):.2f} | `{k}` |")

# full captures
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
traffic = {}
for f in sorted(glob.glob("gpurun_out/prof_*_full.ncu-rep")):
    cfg = os.path.basename(f).split("_")[1]
    raw = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out_md.append(f"\n## ncu --set full, {cfg} (`{f}`)\n")
    cols = [w for w in want if w in hdr]
    out_md.append("| kernel | " + " | ".join(c.replace("avg.pct_of_peak_sustained_", "%") for c in cols) + " |")
    out_md.append("|---" * (len(cols) + 1) + "|")
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        vals = []
        for c in cols:
            i = hdr.index(c)
            vals.append(f"{r[i]} {units[i]}".strip())
        out_md.append(f"| `{name[:60]}` | " + " | ".join(vals) + " |")
        stage = ("S2S3_ksmac_wht" if "mac" in name else "S1_permdecomp" if "PermDecomp" in name else
                 "S4S5_align_intt" if any(k in name for k in ("OutInv", "StridedInv", "DigitLift", "ks_apply")) else None)
        if stage:   # dram bytes per launch, summed over the stage's kernels (one launch of each captured)
            i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = float(r[i_r].replace(",", "")) * scale.get(units[i_r], 1) + \
                float(r[i_w].replace(",", "")) * scale.get(units[i_w], 1)
            traffic.setdefault(cfg, {}).setdefault(stage, {})[name.split("::")[-1][:40]] = b
    os.system(f"cp {f} profiles/{tag}_{os.path.basename(f)[5:]}")
if traffic:
    traffic = {c: {st: sum(v.values()) for st, v in d.items()} for c, d in traffic.items()}
    json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)
open(f"profiles/{tag}_summary.md", "w").write("\n".join(out_md) + "\n")
print("\n".join(out_md))
