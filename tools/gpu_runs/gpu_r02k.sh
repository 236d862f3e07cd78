# round-2 GPU batch k: TMA-store epilogue tests + A/B, full tests
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k gemm > gpurun_out/r2k_kern.log 2>&1; echo rc=$? >> gpurun_out/r2k_kern.log
for t in 0 1 0 1; do HX_GEMM_TMA_STORE=$t timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('TMA=$t', round(d['value']), d['clocks']['sm_mhz'], round(d['kernel_share']['gemm']['ms_per_step'],1), [(g['layout'],g['M'],g['N'],g['K'],g['epilogue'],round(g['tflops'])) for g in d['gemm_shapes']])" >> gpurun_out/r2k_ab.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2k_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2k_pytest.log
