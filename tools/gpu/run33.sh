mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu_stages.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
