# round-2 GPU batch am: L2 prefetch of the epilogue aux chunks at tile start (HX_GEMM_AUX_PREFETCH 0 / 1)
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm or linear" > gpurun_out/r2am_kern.log 2>&1; echo rc=$? >> gpurun_out/r2am_kern.log
if grep -q "rc=0" gpurun_out/r2am_kern.log; then
  for rep in 1 2 3; do
    for v in 0 1; do
      HX_GEMM_AUX_PREFETCH=$v timeout 300 python tools/kernel_bench.py --only gemm --reps 10 | grep -E "dgelu|o_proj|w1_gelu" | sed "s/^/pf$v /" >> gpurun_out/r2am_gemm.txt
    done
  done
  timeout 1800 python tools/bench_ab.py pf0=HX_GEMM_AUX_PREFETCH=0 pf1=HX_GEMM_AUX_PREFETCH=1 --rounds 3 -- --steps 3 --warmup 2 > gpurun_out/r2am_ab.txt 2>&1
fi
