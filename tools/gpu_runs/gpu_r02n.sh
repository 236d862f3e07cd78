# round-2 GPU batch n: ncu --set full of the top kernels (report kept in /tmp, summary copied back)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_kernel|attn_bwd_fused|gemm_2sm|ln_fwd_v2|ln_bwd|attn_bwd_pre" -c 40 -o /tmp/prof_r02 python tools/kernel_bench.py --reps 1 > gpurun_out/r2n_ncu.log 2>&1
python tools/ncu_summary.py /tmp/prof_r02.ncu-rep --out gpurun_out/ncu_summary_r02.json --tag r02 > gpurun_out/r2n_summary.txt 2>&1
ncu -i /tmp/prof_r02.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size > gpurun_out/r2n_raw.csv 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2n_bench.log 2>&1
