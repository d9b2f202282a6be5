# APX check: v2-path parity + bench C4, then profile
timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu_bounds.py tests/test_gpu_golden.py tests/test_gpu_guard.py -x -q -p no:cacheprovider --durations=15 > gpurun_out/t3.log 2>&1; tail -n 25 gpurun_out/t3.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C4_apx.log 2>&1; tail -c 600 gpurun_out/bench_C4_apx.log
bash tools/gpu_prof.sh r02 nosweep
