mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for c in C2 C1 C3a C3b C5pw_8192 C5dw_8192 C4; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 300 $B --config C4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B --config C4 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu2 rc=$?"
