# round-2 GPU batch g: tests, bench, ncu launch list, probes for the p=8 predictions
timeout 1500 python -m pytest tests -m gpu -q -x -rA > gpurun_out/r2g_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2g_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2g_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no > gpurun_out/r2g_ncu_bench.log 2>&1
P="timeout 1200 python tools/stage_probe.py"
$P --workload gpt3b_64k --p 8 --stage 0 --method 1f1b >> gpurun_out/r2g_probe.jsonl 2>>gpurun_out/r2g_probe.err
$P --workload gpt3b_64k --p 8 --stage 0 --method helix_twofold_rc --mlp-chunk 8192 >> gpurun_out/r2g_probe.jsonl 2>>gpurun_out/r2g_probe.err
$P --workload gpt3b_64k --p 8 --stage 0 --method helix_twofold --mlp-chunk 8192 --stash-budget-gb 140 >> gpurun_out/r2g_probe.jsonl 2>>gpurun_out/r2g_probe.err
