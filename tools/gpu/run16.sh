mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"
for c in C1 C3a C3b C4 C5dw_4096 C5dw_8192 C5dw_16384 C5pw_4096 C5pw_8192 C5pw_16384; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 300 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
rm -f gpurun_out/launches_*.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv $B --steps 3 > gpurun_out/ncu_launch_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $B --config C4 --steps 3 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mac_tc|permauto|ntt_" -s 20 -c 6 -o gpurun_out/prof_C4_full $B --config C4 --steps 3 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu full c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -s 30 -c 12 -o gpurun_out/prof_C2_full $B --steps 3 > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu full c2 rc=$?"
