# round-2 GPU batch as (re-entry): smoke on the restored tree, GEMM shapes incl. the GeLU /
# GeLU' epilogues next to the plain store, ncu --set full of the two heavy-epilogue GEMMs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2as_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2as_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2as_smoke.log
for rep in 1 2; do timeout 300 python tools/kernel_bench.py --only gemm --reps 10 --cublas > gpurun_out/r2as_gemm_$rep.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_2sm -c 2 \
  -o gpurun_out/r2as_epi python tools/epi_gemm_probe.py > gpurun_out/r2as_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2as_ncu.log
