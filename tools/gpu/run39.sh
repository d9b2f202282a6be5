mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --config C2"
for r in 1 2 3; do timeout 300 $B > gpurun_out/bench_new$r.log 2>&1; done
cp tools/ab/kernels.cu paper_2311_12519_b200/csrc/kernels.cu; cp tools/ab/ntt.cuh paper_2311_12519_b200/csrc/ntt.cuh
python -c "import sys; sys.path.insert(0,'.'); from paper_2311_12519_b200 import build; build.build(force=True)"
for r in 1 2 3; do timeout 300 $B > gpurun_out/bench_old$r.log 2>&1; done
echo done
