# round-2 GPU batch i: GEMM epilogue (8 warps + aux prefetch) A/B, tests, bench, 7B probes
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/r2i_kern.log 2>&1; echo rc=$? >> gpurun_out/r2i_kern.log
for ew in 4 8 4 8; do HX_GEMM_EPI_WARPS=$ew timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('EW=$ew', round(d['value']), d['clocks']['sm_mhz'], round(d['kernel_share']['gemm']['ms_per_step'],1), [(g['layout'],g['M'],g['N'],g['K'],g['epilogue'],round(g['tflops'])) for g in d['gemm_shapes']][:6])" >> gpurun_out/r2i_ew.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2i_pytest.log
P="timeout 1500 python tools/stage_probe.py"
$P --workload gpt7b_128k --p 8 --stage 0 --method helix_twofold_rc --mlp-chunk 16384 --regen-pre-x --stream-inputs --stash-budget-gb 100 >> gpurun_out/r2i_probe.jsonl 2>>gpurun_out/r2i_probe.err
$P --workload gpt7b_128k --p 8 --stage 0 --method 1f1b_rc --mlp-chunk 16384 --stream-inputs --stash-budget-gb 100 >> gpurun_out/r2i_probe.jsonl 2>>gpurun_out/r2i_probe.err
$P --workload gpt3b_64k --p 8 --stage 0 --method 1f1b_rc --mlp-chunk 8192 >> gpurun_out/r2i_probe.jsonl 2>>gpurun_out/r2i_probe.err
