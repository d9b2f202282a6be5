mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider -k "default" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for c in C2 C3b C4 C5dw_8192; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
