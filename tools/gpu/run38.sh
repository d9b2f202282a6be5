mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 1500 python -m pytest tests/test_gpu_conv.py tests/test_gpu_stages.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "parity and (C3b or C4 or C5pw_8192)" > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest full rc=$?"; tail -1 gpurun_out/pytest_gpu_full.log
for c in C3a C3b C4 C5pw_8192; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
