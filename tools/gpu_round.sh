# One round-end-style GPU pass through gpurun: the whole -m gpu suite, smoke(), then the profiling pass
# (tools/gpu_prof.sh: every config's bench line, ncu launch lists and full captures).
#   gpurun --timeout 5400 -- 'bash tools/gpu_round.sh r02 [notests] [nosweep]'
TAG=${1:-r02}
mkdir -p gpurun_out
if [ "$2" != "notests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/gputests_$TAG.log; tail -n 3 gpurun_out/gputests_$TAG.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -n 1 gpurun_out/smoke_$TAG.log
fi
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default_$TAG.log
tail -n 2 gpurun_out/bench_default_$TAG.log | cut -c1-400
bash tools/gpu_prof.sh $TAG $3
