# round-2 GPU batch ar: LayerNorm backward v4 (one pass, fused column sums, h <= 2048) vs the v1 pair
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k layernorm > gpurun_out/r2ar_kern.log 2>&1; echo rc=$? >> gpurun_out/r2ar_kern.log
HX_LN_BWD=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k layernorm >> gpurun_out/r2ar_kern.log 2>&1; echo rc_v1=$? >> gpurun_out/r2ar_kern.log
if grep -q "^rc=0" gpurun_out/r2ar_kern.log; then
  for rep in 1 2; do for v in 1 4; do
    HX_LN_BWD=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 | sed "s/^/bwd$v 1.3b /" >> gpurun_out/r2ar_ln.txt
  done; done
  timeout 900 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/r2ar_parity.log 2>&1; echo rc=$? >> gpurun_out/r2ar_parity.log
  timeout 1800 python tools/bench_ab.py v1=HX_LN_BWD=1 v4=HX_LN_BWD=4 --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2ar_ab.txt 2>&1
fi
