# round-2 GPU batch ae: per-SASS-instruction source counters of the attention forward
timeout 600 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none \
  -k regex:"attn_fwd_kernel" -c 1 -f -o /tmp/fwd_src python tools/kernel_bench.py --only attn --reps 1 > gpurun_out/r2ae_ncu.log 2>&1
ncu -i /tmp/fwd_src.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/r2ae_fwd_sass.csv.gz
