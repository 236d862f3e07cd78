# round-2 GPU batch j
timeout 600 python tools/config1_profile.py > gpurun_out/r2j_config1.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2j_bench.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 --lm-vocab 50257 --no-cpu-baseline --no-config1 > gpurun_out/r2j_bench_lm.log 2>&1
P="timeout 1500 python tools/stage_probe.py"
$P --workload gpt7b_128k --L 8 --p 8 --stage 0 --method 1f1b_rc --mlp-chunk 16384 >> gpurun_out/r2j_probe.jsonl 2>>gpurun_out/r2j_probe.err
$P --workload gpt7b_128k --L 8 --p 8 --stage 0 --method helix_twofold_rc --mlp-chunk 16384 --regen-pre-x >> gpurun_out/r2j_probe.jsonl 2>>gpurun_out/r2j_probe.err
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2j_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2j_pytest.log
