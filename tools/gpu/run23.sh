mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C2"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ksmac_gemm|StridedInv|PermDecomp" -s 6 -c 3 -o gpurun_out/prof_C2_k $B > gpurun_out/ncu_c2k.log 2>&1; echo "ncu rc=$?"
