"""Summarise bench JSON lines and ncu launch lists under gpurun_out/ (local helper)."""
import collections, csv, glob, json, sys

for f in sorted(glob.glob('gpurun_out/bench_*.log')):
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            if 'roofline' not in d:
                print(f"{f[16:-4]:12s} reference {d['value']:.4g} {d['unit']}")
                continue
            r = d['roofline']
            print(f"{f[16:-4]:12s} {d['value']:10.2f} {d['unit']} ms={d['ms_per_step']:.3f} path={d.get('mac_path')} "
                  f"stages={ {k: round(v, 3) for k, v in d['stages_ms'].items()} } clk={d['clocks']['sm_mhz']} "
                  f"e2e={d['e2e']['value']:.2f}")
            for k, v in r.get('stages', {}).items():
                print(f"      {k:18s} {v['bound']} {v['achieved']:.1f}/{v['peak']:.1f} {v['unit']} frac={v['frac']:.3f}"
                      + (f" tc={v['tensor_int8']['frac']:.3f}" if 'tensor_int8' in v else ''))
for f in sorted(glob.glob('gpurun_out/launches*.csv')):
    rows = [r for r in csv.reader(open(f)) if len(r) > 5]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
    agg = collections.OrderedDict()
    for r in rows:
        agg.setdefault(r[ki][:80], []).append(float(r[vi].replace(',', '')) / 1000)
    tot = sum(sum(v) for v in agg.values())
    print(f, 'launches', len(rows), 'total us', round(tot, 1))
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f'  {sum(v) / tot * 100:5.1f}%  n={len(v):4d} avg={sum(v) / len(v):10.2f}us  {k}')
