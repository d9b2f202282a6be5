mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default rc=$?"; tail -c 600 gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "bench ref rc=$?"; tail -c 600 gpurun_out/bench_reference.log
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
for c in C1 C3a C3b C4 C5pw_4096 C5dw_4096 C5pw_8192 C5dw_8192 C5pw_16384 C5dw_16384; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
rm -f gpurun_out/launches_*.csv
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1; echo "ncu1 rc=$?"
timeout 300 $B --config C4 --steps 3 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $B --config C4 --steps 3 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu2 rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksmac|ntt_|ks_apply" -s 20 -c 8 -o gpurun_out/prof_C2_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu3 rc=$?"
timeout 300 $B --config C4 --steps 3 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksmac|ntt_" -s 10 -c 3 -o gpurun_out/prof_C4_full $B --config C4 --steps 3 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu4 rc=$?"
