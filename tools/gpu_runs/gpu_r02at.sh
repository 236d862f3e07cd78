# round-2 GPU batch at: GeLU / GeLU' epilogues with bare MUFU rcp / ex2 (no __frcp_rn slow-path CALLs,
# no __expf denormal guard): kernel tests, GEMM shape timings, bench A/B vs the previous build
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/r2at_kern.log 2>&1; echo rc=$? >> gpurun_out/r2at_kern.log
for rep in 1 2; do timeout 300 python tools/kernel_bench.py --only gemm --reps 10 > gpurun_out/r2at_gemm_$rep.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_2sm -c 2 \
  -o gpurun_out/r2at_epi python tools/epi_gemm_probe.py > gpurun_out/r2at_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2at_ncu.log
timeout 900 python bench.py > gpurun_out/r2at_bench.json 2> gpurun_out/r2at_bench.err; echo rc=$? >> gpurun_out/r2at_bench.err
