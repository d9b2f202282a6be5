timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_bounds.py tests/test_gpu_golden.py tests/test_gpu_guard.py -x -q -p no:cacheprovider > gpurun_out/t4.log 2>&1; tail -n 3 gpurun_out/t4.log
for C in C4 C3a C3b; do timeout 300 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench4_$C.log 2>&1; python -c "
import json,sys; d=json.loads([l for l in open('gpurun_out/bench4_$C.log') if l.startswith('{')][-1]); print('$C', d['value'], d['stages_ms'])"; done
timeout 600 ncu --set full -f --clock-control none --import-source on -k 'regex:ksmac_v2' -c 1 -o /tmp/v2 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/v2.ncu-rep --page raw --csv > gpurun_out/v2_raw.csv; ncu -i /tmp/v2.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/v2_sass.csv.gz
