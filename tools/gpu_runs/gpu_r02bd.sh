# round-2 GPU batch bd: our forward / backward next to cuDNN's under ncu at s=8k (clock, instructions,
# pipe utilisation), and the SM clock + power during the isolated kernels (nvidia-smi sampling)
timeout 600 ncu --set full --clock-control none -k regex:"attn_fwd_kernel|attn_bwd_fused|cudnn" -c 6 \
  -o gpurun_out/r2bd_attn python tools/cudnn_attn_ref.py 8192 16 128 > gpurun_out/r2bd_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2bd_ncu.log
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 50 > gpurun_out/r2bd_smi.txt) &
SMI=$!
timeout 300 python tools/kernel_bench.py --only attn --reps 40 > gpurun_out/r2bd_kb.txt 2>&1
kill $SMI
