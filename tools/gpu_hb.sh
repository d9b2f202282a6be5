# host-path batch-count sweep (HY_HOST_BATCHES) with ab/libhyena_$1.so: e2e layers/s per batch count
V=${1:-pre1}
for HB in ${HBS:-8 16 32 64}; do
  HY_HOST_BATCHES=$HB HYENA_LIB=ab/libhyena_$V.so timeout 300 python bench.py --config ${CFG:-C4} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/hb_$HB.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/hb_$HB.log') if l.startswith('{')][-1]); print('HB', $HB, round(d['ms_per_step'],3), d['e2e'])" || tail -n 3 gpurun_out/hb_$HB.log
done
