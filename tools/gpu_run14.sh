timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_bounds.py tests/test_gpu_golden.py tests/test_gpu_guard.py tests/test_gpu_shard.py tests/test_gpu_negative.py -x -q -p no:cacheprovider > gpurun_out/t14.log 2>&1; tail -n 2 gpurun_out/t14.log
bash tools/gpu_prof.sh r02
