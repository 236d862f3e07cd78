# round-2 GPU batch bn: LayerNorm backward v5 with warp pairs per row at h = 4096 (vs v2), and the
# h <= 2048 path re-checked after the generalisation
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k layernorm > gpurun_out/r2bn_kern.log 2>&1; echo rc=$? >> gpurun_out/r2bn_kern.log
if grep -q "^rc=0" gpurun_out/r2bn_kern.log; then
  for rep in 1 2; do for v in 0 1; do
    HX_LN_BWD5=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 --workload gpt3b_64k | sed "s/^/v5=$v 3b /" >> gpurun_out/r2bn_ln.txt
    HX_LN_BWD5=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 | sed "s/^/v5=$v 1.3b /" >> gpurun_out/r2bn_ln.txt
  done; done
  timeout 1500 python -m pytest tests/test_fullsize_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/r2bn_parity.log 2>&1; echo rc=$? >> gpurun_out/r2bn_parity.log
fi
