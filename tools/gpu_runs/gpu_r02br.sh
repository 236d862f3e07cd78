# round-2 GPU batch br: cuDNN's sm100 backward next to attn_bwd_fused_kernel under ncu at s=8k
timeout 600 ncu --set full --clock-control none -k regex:"cudnn.*bprop|^attn_bwd_fused_kernel" -c 8 \
  -o gpurun_out/r2br_bwd python tools/cudnn_attn_ref.py 8192 16 128 > gpurun_out/r2br_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2br_ncu.log
