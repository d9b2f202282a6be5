# A/B: bench.py with each ab/libhyena_*.so (HYENA_LIB), interleaved twice, configs in $CFGS (default C4)
for C in ${CFGS:-C4}; do for rep in 1 2; do for v in $(ls ab/ | sed 's/libhyena_\(.*\).so/\1/'); do
  HYENA_LIB=ab/libhyena_$v.so timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/ab_$v.log') if l.startswith('{')][-1]); print('$C', '$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})" || tail -n 3 gpurun_out/ab_$v.log
done; done; done
