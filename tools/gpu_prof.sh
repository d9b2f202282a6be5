# Round profiling pass on one B200 (run through gpurun): every config's bench line, the ncu launch list of
# C4 and C2, and one `ncu --set full` capture of the C4 and C2 kernels, exported to CSV on the box
# (the .ncu-rep files are too large to bring back).  Usage: bash tools/gpu_prof.sh r02 [nosweep]
TAG=${1:-r02}
mkdir -p gpurun_out /tmp/ncu
if [ "$2" != "nosweep" ]; then
  timeout 900 python tools/sweep.py --out gpurun_out/${TAG}_bench.json > gpurun_out/sweep.log 2>&1
fi
for C in C4 C2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$C.csv \
    python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$C.log 2>&1
done
timeout 1200 ncu --set full -f --clock-control none --import-source on -k 'regex:ksmac_v2|ntt2_' -c 3 \
  -o /tmp/ncu/${TAG}_full_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_C4.log 2>&1
timeout 900 ncu --set full -f --clock-control none --import-source on -k 'regex:ksmac|PermDecomp|OutInv|StridedInv|DigitLift|ks_apply' -c 6 \
  -o /tmp/ncu/${TAG}_full_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_C2.log 2>&1
for C in C4 C2; do
  R=/tmp/ncu/${TAG}_full_$C.ncu-rep
  [ -f $R ] || continue
  ncu -i $R --page raw --csv > gpurun_out/${TAG}_full_${C}_raw.csv 2>/dev/null
  ncu -i $R --page details --csv > gpurun_out/${TAG}_full_${C}_details.csv 2>/dev/null
  ncu -i $R --page source --csv --print-source sass > gpurun_out/${TAG}_full_${C}_sass.csv 2>/dev/null
  ls -la $R
done
gzip -f gpurun_out/*_sass.csv 2>/dev/null
tail -n 2 gpurun_out/ncu_full_C4.log gpurun_out/ncu_full_C2.log; cat gpurun_out/sweep.log 2>/dev/null; du -sh gpurun_out
