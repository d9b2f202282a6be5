timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_bounds.py tests/test_gpu_golden.py tests/test_gpu_guard.py tests/test_gpu_shard.py -x -q -p no:cacheprovider > gpurun_out/t11.log 2>&1; tail -n 3 gpurun_out/t11.log
CFGS="C3a C3b C2" bash tools/gpu_ab.sh
