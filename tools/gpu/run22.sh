mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log gpurun_out/launches_*.csv
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "C2 or C1" > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest full rc=$?"; tail -2 gpurun_out/pytest_gpu_full.log
for c in C1 C2; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv $B --config C2 --steps 3 > gpurun_out/ncu_launch_c2.log 2>&1; echo "ncu c2 rc=$?"
