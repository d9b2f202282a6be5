"""Opcode histogram + stall summary of one kernel in an ncu report (local helper).
Usage: python tools/gpu/sass_hist.py gpurun_out/x.ncu-rep [top-lines]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
si, ei, smp = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
tot = 0; ops = collections.Counter(); samples = collections.Counter(); lines = []
for r in rows[2:]:
    try: n = int(r[ei]); s = int(r[smp])
    except Exception: continue
    toks = r[si].split()
    op = toks[1] if toks and toks[0].startswith('@') else (toks[0] if toks else '')
    ops[op.split('.')[0]] += n; tot += n; samples[op.split('.')[0]] += s
    lines.append((s, n, r[si]))
print('total warp instr', tot, 'samples', sum(samples.values()))
for op, n in ops.most_common(22): print(f'{op:10s} {n:14d} {n/tot*100:5.1f}%  samples {samples[op]}')
if top:
    for s, n, t in sorted(lines, reverse=True)[:top]: print(f'{s:7d} {n:12d}  {t}')
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh, vv = rr[0], rr[2]
st = []
for i, k in enumerate(hh):
    if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued'):
        try: st.append((float(vv[i].replace(',', '')), k.split('stalled_')[1]))
        except Exception: pass
print('stalls:', ', '.join(f'{k}={v:.0f}' for v, k in sorted(st, reverse=True)[:8]))
for k in ('gpu__time_duration.sum', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
          'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
          'sm__issue_active.avg.pct_of_peak_sustained_elapsed', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
          'lts__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active'):
    if k in hh: print(k, vv[hh.index(k)])
