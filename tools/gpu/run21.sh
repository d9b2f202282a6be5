mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log gpurun_out/launches_*.csv
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "C5pw or C2 or C3b" > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest full rc=$?"; tail -2 gpurun_out/pytest_gpu_full.log
for c in C2 C3a C3b C4 C5pw_4096 C5pw_8192; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv $B --config C2 --steps 3 > gpurun_out/ncu_launch_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksmac_tc" -s 2 -c 1 -o gpurun_out/prof_C3a_ksmactc $B --config C3a --steps 3 > gpurun_out/ncu_full_c3a.log 2>&1; echo "ncu full c3a rc=$?"
