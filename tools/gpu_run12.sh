timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t12.log 2>&1; tail -n 5 gpurun_out/t12.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 300 python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench12.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench12.log') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"
