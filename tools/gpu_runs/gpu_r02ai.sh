# round-2 GPU batch ai: bench.py's N > 1 leg end to end on the one B200 (HX_BENCH_SHARED_GPU=1: ranks
# time-share cuda:0 over gloo) -- checks the multi-rank bench path, not a number
for n in 2 4; do
  HX_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus $n --workload tiny --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r2ai_bench_shared_n$n.log 2>&1; echo rc=$? >> gpurun_out/r2ai_bench_shared_n$n.log
done
