# round-2 GPU batch h: LM tests, bench (GEMM shapes), ncu launch list of our kernels, 7B probes
timeout 600 python -m pytest tests/test_lm_gpu.py -q -x -rA > gpurun_out/r2h_lm.log 2>&1; echo rc=$? >> gpurun_out/r2h_lm.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2h_bench.log 2>&1
timeout 900 ncu --kernel-name regex:hx:: --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no > gpurun_out/r2h_ncu_bench.log 2>&1
P="timeout 1500 python tools/stage_probe.py"
$P --workload gpt7b_128k --p 8 --stage 0 --method helix_twofold_rc --mlp-chunk 16384 --regen-pre-x --stash-budget-gb 140 >> gpurun_out/r2h_probe.jsonl 2>>gpurun_out/r2h_probe.err
$P --workload gpt7b_128k --p 8 --stage 0 --method 1f1b_rc --mlp-chunk 16384 --stash-budget-gb 140 >> gpurun_out/r2h_probe.jsonl 2>>gpurun_out/r2h_probe.err
