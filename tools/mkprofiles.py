"""Copy the evidence of round-`tag` GPU runs from gpurun_out/ into profiles/ (tracked):
  * gpurun_out/{tag}_bench.json, {tag}_ablation.json   (tools/sweep.py)       -> tables
  * gpurun_out/launches_<cfg>.csv                       (ncu gpu__time_duration launch lists) -> shares
  * gpurun_out/{tag}_<kernel>_<cfg>.ncu-rep             (ncu --set full)       -> counters + traffic.json
  * gpurun_out/int_peaks.json, san_*.log                                       -> peaks, sanitizer verdicts
Usage: python tools/mkprofiles.py r02"""
import collections
import csv
import glob
import json
import os
import re
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
os.makedirs("profiles", exist_ok=True)
md = [f"# Profiles {tag}\n",
      "B200 runs through `gpurun` (commands: tools/sweep.py, tools/peaks.py, ncu as in B200_PROFILING.md). ncu "
      "launch times are cold-cache and serialised: compare shares, not absolutes. Peaks: profiles/int_peaks.json "
      "(measured: Shoup modmul 4.08/clk/SM = 1186.5 Gmodmul/s at 1965 MHz, DFMA 58.4/clk/SM, tcgen05 kind::i8 4545 "
      "TOP/s) and MEASURED_PEAKS.json (HBM 6546.6 GB/s).\n"]


def bench_table(path, title):
    if not os.path.exists(path):
        return
    data = json.load(open(path))
    json.dump(data, open(f"profiles/{os.path.basename(path)}", "w"), indent=1)
    md.append(f"## {title}\n\n| run | layers/s | ms/step | MAC path | S1 ms (frac) | S2+S3 ms (frac) | S4+S5 ms (frac) | "
              "e2e layers/s | clocks |\n|---|---|---|---|---|---|---|---|---|")
    for n, d in data.items():
        if "error" in d or "roofline" not in d:
            md.append(f"| {n} | error | | | | | | | |")
            continue
        st, rs = d["stages_ms"], d["roofline"]["stages"]
        cell = lambda k: f"{st[k]:.3f} ({rs[k]['frac']:.3f})"
        md.append(f"| {n} | {d['value']:.1f} | {d['ms_per_step']:.3f} | {d['mac_path']} | {cell('S1_permdecomp')} | "
                  f"{cell('S2S3_ksmac_wht')} | {cell('S4S5_align_intt')} | {d['e2e']['value']:.1f} | "
                  f"{d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']} |")
    md.append("")


bench_table(f"gpurun_out/{tag}_bench.json", "bench.py, every BASELINE config (tools/sweep.py)")
bench_table(f"gpurun_out/{tag}_ablation.json", "Fig. 4 ablations on this library (PAPER.md:778-787): default vs "
            "lazy reduction off (eager) vs hoisting off (direct)")

for f in sorted(glob.glob("gpurun_out/launches_*.csv")):
    cfg = os.path.basename(f)[9:-4]
    rows = [r for r in csv.reader(open(f)) if len(r) > 5]
    if not rows:
        continue
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows:
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else v * 1000 if r[ui] == "ms" else v
        agg.setdefault(r[ki].split("(")[0][:90], []).append(v)
    tot = sum(sum(v) for v in agg.values())
    os.system(f"cp {f} profiles/{tag}_launches_{cfg}.csv")
    md.append(f"## ncu launch list {cfg} ({len(rows)} launches, gpu__time_duration.sum, µs)\n\n"
              "| share | launches | avg µs | kernel |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        md.append(f"| {sum(v) / tot * 100:.1f}% | {len(v)} | {sum(v) / len(v):.2f} | `{k}` |")
    md.append("")

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic = json.load(open("profiles/traffic.json")) if os.path.exists("profiles/traffic.json") else {}
# ncu --set full captures, exported on the GPU box to CSV (tools/gpu_prof.sh: {tag}_full_<cfg>_raw.csv)
for f in sorted(glob.glob(f"gpurun_out/{tag}_full_*_raw.csv")):
    base = os.path.basename(f)[len(tag) + 1:-8]
    cfg = base.split("_")[-1]
    os.system(f"cp {f} profiles/")
    rows = list(csv.reader(open(f).read().splitlines()))
    if len(rows) < 3:
        continue
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [w for w in want if w in hdr]
    md.append(f"## ncu --set full: {base}\n\n| kernel | " +
              " | ".join(c.replace(".avg.pct_of_peak_sustained_", " %").replace("smsp__average_warps_issue_", "")
                         for c in cols) + " |")
    md.append("|---" * (len(cols) + 1) + "|")
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        md.append(f"| `{name[:70]}` | " + " | ".join(f"{r[hdr.index(c)]} {units[hdr.index(c)]}".strip() for c in cols)
                  + " |")
        stage = ("S2S3_ksmac_wht" if "mac" in name else "S1_permdecomp" if "PermDecomp" in name else
                 "S4S5_align_intt" if "OutInv" in name else None)
        stage = stage if stage else None
        if stage:  # dram bytes per launch of the stage's dominant kernel
            i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            b = float(r[i_r].replace(",", "")) * scale.get(units[i_r], 1) + \
                float(r[i_w].replace(",", "")) * scale.get(units[i_w], 1)
            traffic.setdefault(cfg, {})[stage] = b
    md.append("")
json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)

if os.path.exists("gpurun_out/int_peaks.json"):
    os.system("cp gpurun_out/int_peaks.json profiles/int_peaks.json")
for f in sorted(glob.glob("gpurun_out/san_*.log")):
    txt = open(f).read()
    summ = re.findall(r"ERROR SUMMARY: \d+ errors?|RACECHECK SUMMARY: .*|\d+ passed.*", txt)
    md.append(f"## {os.path.basename(f)}: " + ("; ".join(summ) if summ else "(no summary line)"))
    os.system(f"cp {f} profiles/{tag}_{os.path.basename(f)}")
open(f"profiles/{tag}_summary.md", "w").write("\n".join(md) + "\n")
print("\n".join(md))
