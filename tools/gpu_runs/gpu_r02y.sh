# round-2 GPU batch y: one-tile-per-CTA forward with double-buffered S (HX_ATTN_FWD=2)
HX_ATTN_FWD=2 timeout 180 python -m pytest tests/test_kernels_gpu.py -q -x -k attention_forward > gpurun_out/r2y_kern.log 2>&1; echo rc=$? >> gpurun_out/r2y_kern.log
if grep -q "rc=0" gpurun_out/r2y_kern.log; then
  for v in 1 2 1 2; do HX_ATTN_FWD=$v timeout 120 python tools/kernel_bench.py --only attn --reps 10 | head -1 | sed "s/^/fwd$v /" >> gpurun_out/r2y_attn.txt; done
  for v in 1 2; do HX_ATTN_FWD=$v timeout 300 python tools/kernel_bench.py --workload gpt7b_128k --only attn --reps 2 | head -1 | sed "s/^/7b fwd$v /" >> gpurun_out/r2y_attn.txt; done
  HX_ATTN_FWD=2 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/r2y_parity.log 2>&1; echo rc=$? >> gpurun_out/r2y_parity.log
  timeout 1800 python tools/bench_ab.py f1=HX_ATTN_FWD=1 f2=HX_ATTN_FWD=2 --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2y_ab.txt 2>&1
fi
