# round-2 GPU batch ax: LayerNorm backward v5 (bulk-copied row ring, whole rows per warp, fused
# gain / bias sums) vs the v1 pair at h <= 2048: LN kernel tests both ways, timings, parity, bench A/B
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k layernorm > gpurun_out/r2ax_kern.log 2>&1; echo rc=$? >> gpurun_out/r2ax_kern.log
HX_LN_BWD5=0 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k layernorm >> gpurun_out/r2ax_kern.log 2>&1; echo rc_v1=$? >> gpurun_out/r2ax_kern.log
if grep -q "^rc=0" gpurun_out/r2ax_kern.log; then
  for rep in 1 2; do for v in 0 1; do
    HX_LN_BWD5=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 | sed "s/^/v5=$v 1.3b /" >> gpurun_out/r2ax_ln.txt
    HX_LN_BWD5=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 --workload tiny | sed "s/^/v5=$v tiny /" >> gpurun_out/r2ax_ln.txt
  done; done
  timeout 900 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/r2ax_parity.log 2>&1; echo rc=$? >> gpurun_out/r2ax_parity.log
  timeout 1800 python tools/bench_ab.py v1=HX_LN_BWD5=0 v5=HX_LN_BWD5=1 --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2ax_ab.txt 2>&1
fi
