# round-2 GPU batch: tests, LN A/B, probe, bench
timeout 1500 python -m pytest tests -m gpu -q -x -rA > gpurun_out/r2e_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2e_pytest.log
for v in 1 2 3; do for wl in gpt1.3b_32k gpt3b_64k; do HX_LN=$v timeout 120 python tools/kernel_bench.py --workload $wl --only ln --reps 20 | sed "s/^/HX_LN=$v $wl /" >> gpurun_out/r2e_ln.txt 2>&1; done; done
timeout 600 python tools/stage_probe.py --workload gpt3b_64k --p 8 --stage 0 --method helix_twofold_rc --mlp-chunk 8192 >> gpurun_out/r2e_probe.jsonl 2>>gpurun_out/r2e_probe.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2e_bench.log 2>&1
