# round evidence run: parity, smoke, bench lines of every config, reference arm, ncu launch lists + full captures
mkdir -p gpurun_out
rm -f gpurun_out/bench_*.log gpurun_out/launches_*.csv gpurun_out/prof_*_full.ncu-rep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for c in C1 C3a C3b C4 C5dw_4096 C5dw_8192 C5dw_16384 C5pw_4096 C5pw_8192 C5pw_16384; do timeout 300 $B --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv $B --config C2 --steps 3 > gpurun_out/ncu_launch_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $B --config C4 --steps 3 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ksmac|PermDecomp|OutInv|StridedInv|DigitLift|ks_apply" -s 12 -c 6 -o gpurun_out/prof_C2_full $B --config C2 --steps 3 > gpurun_out/ncu_full_c2.log 2>&1; echo "ncu full c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ksmac_tc|PermDecomp|OutInv" -s 3 -c 3 -o gpurun_out/prof_C4_full $B --config C4 --steps 3 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu full c4 rc=$?"
