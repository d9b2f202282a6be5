mkdir -p gpurun_out
set -x
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
for c in C1 C3a C3b C5pw_8192 C5dw_8192 C4; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 300 $B --config C4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B --config C4 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu2 rc=$?"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mac_kernel|permauto|ntt_fwd" -s 12 -c 6 -o gpurun_out/prof_c2 $B > gpurun_out/ncu_full.log 2>&1; echo "ncu3 rc=$?"
