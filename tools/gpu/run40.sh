mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --config C2"
for r in 1 2; do timeout 300 $B > gpurun_out/bench_fp$r.log 2>&1; timeout 300 $B --mac-path tc_fused > gpurun_out/bench_tc$r.log 2>&1; done
echo done
