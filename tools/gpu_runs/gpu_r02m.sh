# round-2 GPU batch m: GELU epilogue warps A/B; ncu --set full of the top kernels
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k gemm > gpurun_out/r2m_kern.log 2>&1; echo rc=$? >> gpurun_out/r2m_kern.log
timeout 1800 python tools/bench_ab.py g4=HX_GEMM_GELU_WARPS=4 g8=HX_GEMM_GELU_WARPS=8 --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2m_ab.txt 2>&1
HX_GEMM_GELU_WARPS=8 timeout 300 python tools/kernel_bench.py --only gemm --reps 10 > gpurun_out/r2m_gemm8.txt 2>&1
timeout 300 python tools/kernel_bench.py --only gemm --reps 10 > gpurun_out/r2m_gemm4.txt 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_kernel|attn_bwd_fused|gemm_2sm|ln_fwd_v2|ln_bwd|ce_loss" -c 40 -o gpurun_out/prof_r02 python tools/kernel_bench.py --reps 1 > gpurun_out/r2m_ncu.log 2>&1
