# round-2 GPU batch ba: final-build evidence -- bench (default), the reference arm, the ncu launch list
# of the bench command (every launch; cold-cache, serialised: shares, not absolutes), ncu --set full
# of the two heavy-epilogue GEMMs and of the LayerNorm backward v5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/r2ba_smi.txt
timeout 900 python bench.py > gpurun_out/r2ba_bench.json 2> gpurun_out/r2ba_bench.err; echo rc=$? >> gpurun_out/r2ba_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2ba_ref.json 2> gpurun_out/r2ba_ref.err; echo rc=$? >> gpurun_out/r2ba_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2ba_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no > gpurun_out/r2ba_ncu_bench.log 2>&1; echo rc=$? >> gpurun_out/r2ba_ncu_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_2sm|ln_bwd_v5" -c 3 \
  -o gpurun_out/r2ba_kern python tools/epi_gemm_probe.py --ln > gpurun_out/r2ba_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2ba_ncu.log
