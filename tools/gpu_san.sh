# compute-sanitizer pass over small layers on every MAC path (one tool per gpurun call):
#   bash tools/gpu_san.sh memcheck|racecheck|synccheck
T=${1:-memcheck}
mkdir -p gpurun_out
K="test_conv_bit_exact_small and (tc_v2_cn1 or tc_v2_cn2_rows96 or cn2_blocks or dw_cn1 or pw_cn1 or one_pixel or tc_cn2_rows140)"
timeout 2400 compute-sanitizer --tool $T --target-processes all --print-limit 20 \
  python -m pytest tests/test_gpu_conv.py -k "$K" -x -q -p no:cacheprovider > gpurun_out/san_$T.log 2>&1
echo "rc=$?" >> gpurun_out/san_$T.log
tail -n 6 gpurun_out/san_$T.log
