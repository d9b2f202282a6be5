mkdir -p gpurun_out
rm -f gpurun_out/bench_r*.log
for r in 1 2 3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --config C2 > gpurun_out/bench_r$r.log 2>&1; done
cp tools/ab/kernels.cu paper_2311_12519_b200/csrc/kernels.cu
python -c "import sys; sys.path.insert(0,'.'); from paper_2311_12519_b200 import build; build.build(force=True)"
for r in 4 5 6; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --config C2 > gpurun_out/bench_r$r.log 2>&1; done
