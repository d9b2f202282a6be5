mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
for t in 0 2 8; do HY_FP64_TILE=$t timeout 300 $B --config C2 > gpurun_out/bench_t${t}_C2.log 2>&1; echo "t $t rc=$?"; done
HY_FP64_TILE=8 timeout 300 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider -k "fp64_fused" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
