# round-2 GPU batch be: our attention kernels under ncu at s=8k (compare r2bd's cuDNN capture)
timeout 600 ncu --set full --clock-control none -k regex:"^attn_(fwd|bwd_fused)_kernel" -c 2 \
  -o gpurun_out/r2be_attn python tools/cudnn_attn_ref.py 8192 16 128 > gpurun_out/r2be_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2be_ncu.log
