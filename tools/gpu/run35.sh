mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for d in 0 1 8 9 16; do HY_DEBUG_KSMAC=$d timeout 300 $B --config C5pw_8192 > gpurun_out/bench_dbg${d}_C5pw.log 2>&1; echo "dbg $d rc=$?"; done
