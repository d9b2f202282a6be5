mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log gpurun_out/launches_*.csv
set -x
(cd tools/intbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o intbench intbench.cu && ./intbench) > gpurun_out/intbench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for c in C2 C1 C3a C3b C4; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
for c in C2 C4; do timeout 300 $B --config $c --mac-path tc_split > gpurun_out/bench_split_$c.log 2>&1; echo "split $c rc=$?"; done
timeout 300 $B --config C2 --mac-path fp64_fused > gpurun_out/bench_fp64_C2.log 2>&1; echo "fp64 C2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $B --config C4 --steps 3 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksmac_tc" -s 3 -c 1 -o gpurun_out/prof_C4_ksmactc $B --config C4 --steps 3 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu full c4 rc=$?"
