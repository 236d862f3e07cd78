# round-2 GPU batch z: dQ partials by red.global.add.v2 from 16x256b TMEM loads (HX_ATTN_DQ=red) vs smem staging + TMA reduce-add
HX_ATTN_DQ=red timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_backward or attn_bwd" > gpurun_out/r2z_kern.log 2>&1; echo rc=$? >> gpurun_out/r2z_kern.log
if grep -q "rc=0" gpurun_out/r2z_kern.log; then
  for v in tma red tma red; do HX_ATTN_DQ=$v timeout 120 python tools/kernel_bench.py --only attn --reps 10 | sed "s/^/$v /" >> gpurun_out/r2z_attn.txt; done
  HX_ATTN_DQ=red timeout 600 python -m pytest tests/test_fullsize_gpu.py -q -x > gpurun_out/r2z_full.log 2>&1; echo rc=$? >> gpurun_out/r2z_full.log
  timeout 1500 python tools/bench_ab.py tma=HX_ATTN_DQ=tma red=HX_ATTN_DQ=red --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2z_ab.txt 2>&1
fi
