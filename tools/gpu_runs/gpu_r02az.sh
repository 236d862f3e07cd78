# round-2 GPU batch az: LayerNorm forward v5 with 15 consumer warps vs v2
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k layernorm > gpurun_out/r2az_kern.log 2>&1; echo rc=$? >> gpurun_out/r2az_kern.log
if grep -q "^rc=0" gpurun_out/r2az_kern.log; then
  for rep in 1 2; do for v in 0 1; do
    HX_LN_FWD5=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 | sed "s/^/fwd5=$v 1.3b /" >> gpurun_out/r2az_ln.txt
    HX_LN_FWD5=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 --workload gpt3b_64k | sed "s/^/fwd5=$v 3b /" >> gpurun_out/r2az_ln.txt
  done; done
fi
