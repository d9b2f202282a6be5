mkdir -p gpurun_out
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=12 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/pytest_gpu.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for c in C2 C4; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
rm -f gpurun_out/launches_*.csv
timeout 300 $B --config C2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B --config C2 > gpurun_out/ncu_launch_c2.log 2>&1; echo "ncu1 rc=$?"
timeout 300 $B --config C4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksmac_gemm|ntt_fwd_kernel<13, .*PermDecomp" -s 1 -c 2 -o gpurun_out/prof_c4_ksmac3 $B --config C4 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu2 rc=$?"
