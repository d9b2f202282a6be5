mkdir -p gpurun_out
rm -f gpurun_out/bench_r*.log
timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider -k "default or ntt or poly or rotat" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for r in 1 2 3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --config C2 > gpurun_out/bench_r$r.log 2>&1; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config C4 > gpurun_out/bench_r4.log 2>&1
