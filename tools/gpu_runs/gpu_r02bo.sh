# round-2 GPU batch bo: GeLU / GeLU' epilogue math on FFMA2 / FMUL2 pairs -- epilogue tests (incl. the
# bf16-ulp test), GEMM shape timings, in-step bench A/B against the scalar epilogue (previous commit)
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm or gelu" > gpurun_out/r2bo_kern.log 2>&1; echo rc=$? >> gpurun_out/r2bo_kern.log
if grep -q "^rc=0" gpurun_out/r2bo_kern.log; then
  for rep in 1 2; do timeout 300 python tools/kernel_bench.py --only gemm --reps 10 > gpurun_out/r2bo_gemm_$rep.txt 2>&1; done
  timeout 1800 python tools/bench_ab.py pair=HX_LIB=paper_2507_00394_b200/libhx.so scalar=HX_LIB=lib_scalar_ab.so --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2bo_ab.txt 2>&1
fi
