# round-2 GPU batch aw: what cuDNN's sm100 causal forward looks like under ncu (structure hints:
# block size, registers, smem, cluster, tensor / MUFU / issue utilisation) next to attn_fwd_kernel
timeout 300 ncu --metrics gpu__time_duration.sum,launch__block_size,launch__grid_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,launch__cluster_dim_x --clock-control none --csv \
  python tools/cudnn_attn_ref.py 8192 16 128 > gpurun_out/r2aw_launches.csv 2> gpurun_out/r2aw_launches.err
timeout 600 ncu --set full --clock-control none -k regex:"cudnn|fmha|fprop|flash|sm100|attn_fwd" -c 4 \
  -o gpurun_out/r2aw_cudnn python tools/cudnn_attn_ref.py 8192 16 128 > gpurun_out/r2aw_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2aw_ncu.log
