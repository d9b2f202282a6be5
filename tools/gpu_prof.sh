# Round profiling pass on one B200 (run through gpurun): every config's bench line, the ncu launch list of
# C4 and C2, and one `ncu --set full` capture of the C4 and C2 kernels.  Usage: bash tools/gpu_prof.sh r02
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --out gpurun_out/${TAG}_bench.json > gpurun_out/sweep.log 2>&1
for C in C4 C2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$C.csv \
    python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$C.log 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:ksmac|ntt2|ntt_' -c 4 \
  -o gpurun_out/${TAG}_full_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_C4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ksmac|ntt|ks_|mac" -c 8 \
  -o gpurun_out/${TAG}_full_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_C2.log 2>&1
tail -2 gpurun_out/ncu_full_C4.log gpurun_out/ncu_full_C2.log; cat gpurun_out/sweep.log
