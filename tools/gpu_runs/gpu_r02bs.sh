# round-2 GPU batch bs: with the cheaper packed GeLU math, 4 vs 8 epilogue warps for the GeLU GEMM
# (HX_GEMM_GELU_WARPS) and for all pair GEMMs (HX_GEMM_EPI_WARPS): shape timings, then in-step A/B
for v in 8 4; do
  HX_GEMM_GELU_WARPS=$v timeout 300 python tools/kernel_bench.py --only gemm --reps 10 | sed "s/^/gelu_ew=$v /" >> gpurun_out/r2bs_gemm.txt 2>&1
done
HX_GEMM_EPI_WARPS=4 timeout 300 python tools/kernel_bench.py --only gemm --reps 10 | sed "s/^/all_ew=4 /" >> gpurun_out/r2bs_gemm.txt 2>&1
timeout 2400 python tools/bench_ab.py ew8=HX_GEMM_GELU_WARPS=8 ew4=HX_GEMM_GELU_WARPS=4 --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2bs_ab.txt 2>&1
