# round-2 GPU batch au: GEMM epilogue aux two chunks ahead (unrolled chunk loop)
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/r2au_kern.log 2>&1; echo rc=$? >> gpurun_out/r2au_kern.log
for rep in 1 2; do timeout 300 python tools/kernel_bench.py --only gemm --reps 10 > gpurun_out/r2au_gemm_$rep.txt 2>&1; done
timeout 900 python bench.py > gpurun_out/r2au_bench.json 2> gpurun_out/r2au_bench.err; echo rc=$? >> gpurun_out/r2au_bench.err
