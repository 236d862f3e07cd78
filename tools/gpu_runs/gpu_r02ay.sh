# round-2 GPU batch ay: LayerNorm forward v5 (bulk-copied row ring) vs v2 at h <= 2048
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k layernorm > gpurun_out/r2ay_kern.log 2>&1; echo rc=$? >> gpurun_out/r2ay_kern.log
if grep -q "^rc=0" gpurun_out/r2ay_kern.log; then
  for rep in 1 2; do for v in 0 1; do
    HX_LN_FWD5=$v timeout 120 python tools/kernel_bench.py --only ln --reps 20 | sed "s/^/fwd5=$v 1.3b /" >> gpurun_out/r2ay_ln.txt
  done; done
  timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/r2ay_parity.log 2>&1; echo rc=$? >> gpurun_out/r2ay_parity.log
  timeout 1800 python tools/bench_ab.py v2=HX_LN_FWD5=0 v5=HX_LN_FWD5=1 --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2ay_ab.txt 2>&1
fi
