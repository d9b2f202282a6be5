mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for d in 0 6 14 22 30 31; do HY_DEBUG_KSMAC=$d timeout 300 $B --config C4 > gpurun_out/bench_dbg${d}_C4.log 2>&1; echo "dbg $d rc=$?"; done
