# round-2 GPU batch al: pair-GEMM accumulator hand-back as one cta-scope remote arrive per epilogue warp
# (was: every epilogue thread, .release.cluster = MEMBAR.ALL.GPU per thread per tile); A/B against the
# previous build (build/epi_old/libhx.so)
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm or linear" > gpurun_out/r2al_kern.log 2>&1; echo rc=$? >> gpurun_out/r2al_kern.log
if grep -q "rc=0" gpurun_out/r2al_kern.log; then
  for rep in 1 2; do
    for v in old new; do
      if [ $v = old ]; then L=build/epi_old/libhx.so; else L=paper_2507_00394_b200/libhx.so; fi
      HX_LIB=$L timeout 300 python tools/kernel_bench.py --only gemm --reps 10 | sed "s/^/$v /" >> gpurun_out/r2al_gemm.txt
    done
  done
  timeout 1800 python tools/bench_ab.py old=HX_LIB=build/epi_old/libhx.so new=HX_LIB=paper_2507_00394_b200/libhx.so --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2al_ab.txt 2>&1
fi
