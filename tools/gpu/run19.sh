mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log gpurun_out/launches_*.csv
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -p no:cacheprovider -k "tc_fused or default or tc_split" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in C2 C4; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksmac_tc" -s 3 -c 1 -o gpurun_out/prof_C4_ksmactc $B --config C4 --steps 3 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu full c4 rc=$?"
