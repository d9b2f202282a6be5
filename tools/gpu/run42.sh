mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C4"
HY_DEBUG_KSMAC=31 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ksmac_tc" -s 3 -c 1 -o gpurun_out/prof_C4_skel $B > gpurun_out/ncu_skel.log 2>&1; echo "ncu rc=$?"
