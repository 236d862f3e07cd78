# round-2 GPU batch bi: forward attention source-level stall sampling (s=8k) for the softmax loop
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^attn_fwd_kernel" -c 1 \
  -o gpurun_out/r2bi_fwd python tools/cudnn_attn_ref.py 8192 16 128 > gpurun_out/r2bi_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2bi_ncu.log
