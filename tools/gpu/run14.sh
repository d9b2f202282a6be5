mkdir -p gpurun_out
set -x
timeout 600 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "parity and (C4 or C3a or C3b or C5pw_16384 or C5pw_4096)" > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest-full rc=$?"; tail -3 gpurun_out/pytest_gpu_full.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for c in C2 C3a C3b C4 C5pw_8192 C5pw_16384; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
for c in C4 C3a; do HY_SPLIT_TC=1 timeout 300 $B --config $c > gpurun_out/bench_split_$c.log 2>&1; echo "split $c rc=$?"; done
rm -f gpurun_out/launches_*.csv
timeout 300 $B --config C4 --steps 3 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $B --config C4 --steps 3 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu1 rc=$?"
timeout 300 $B --config C4 --steps 3 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksmac_tc" -s 2 -c 1 -o gpurun_out/prof_C4_ksmactc $B --config C4 --steps 3 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu3 rc=$?"
