mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C4"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"PermDecomp|OutInv" -s 2 -c 2 -o gpurun_out/prof_C4_ntt $B > gpurun_out/ncu_c4ntt.log 2>&1; echo "ncu rc=$?"
