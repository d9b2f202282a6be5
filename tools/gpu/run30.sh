mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C2"
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on --kernel-name-base demangled -k regex:"StridedInv|PermDecomp" -s 2 -c 2 -o gpurun_out/prof_C2_ntt $B > gpurun_out/ncu_c2ntt.log 2>&1; echo "ncu rc=$?"
