timeout 300 python -m pytest tests/test_gpu_negative.py -x -q -p no:cacheprovider > gpurun_out/neg.log 2>&1; tail -n 3 gpurun_out/neg.log
bash tools/gpu_prof.sh r02 nosweep
