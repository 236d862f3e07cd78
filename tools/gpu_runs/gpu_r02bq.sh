# round-2 GPU batch bq: final-build validation -- full GPU suite, smoke, bench (default), reference arm,
# ncu launch list of the bench command, ncu --set full of the GeLU GEMMs
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2bq_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2bq_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bq_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bq_smoke.log
timeout 900 python bench.py > gpurun_out/r2bq_bench.json 2> gpurun_out/r2bq_bench.err; echo rc=$? >> gpurun_out/r2bq_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2bq_ref.json 2> gpurun_out/r2bq_ref.err; echo rc=$? >> gpurun_out/r2bq_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2bq_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no > gpurun_out/r2bq_ncu_bench.log 2>&1; echo rc=$? >> gpurun_out/r2bq_ncu_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_2sm" -c 2 \
  -o gpurun_out/r2bq_epi python tools/epi_gemm_probe.py > gpurun_out/r2bq_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2bq_ncu.log
