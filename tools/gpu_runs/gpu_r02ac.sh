# round-2 GPU batch ac: per-SASS-instruction source counters of the attention backward (shared wavefronts, stalls)
timeout 600 ncu --section SourceCounters --section WarpStateStats --section MemoryWorkloadAnalysis_Tables \
  --import-source on --clock-control none -k regex:"attn_bwd_fused_kernel" -c 1 -f -o /tmp/attn_src \
  python tools/kernel_bench.py --only attn --reps 1 > gpurun_out/r2ac_ncu.log 2>&1
ncu -i /tmp/attn_src.ncu-rep --page source --csv --print-source sass > /tmp/attn_sass.csv 2>&1
python - <<'PY'
import csv, io, os
raw = open('/tmp/attn_sass.csv').read()
os.makedirs('gpurun_out', exist_ok=True)
open('gpurun_out/r2ac_attn_sass_head.txt', 'w').write(raw[:4000])
# keep the file if it is small enough; else gzip it
import gzip
with gzip.open('gpurun_out/r2ac_attn_sass.csv.gz', 'wt') as f:
    f.write(raw)
PY
ncu -i /tmp/attn_src.ncu-rep --page details --print-details all > gpurun_out/r2ac_details.txt 2>&1
ls -la gpurun_out/r2ac* >> gpurun_out/r2ac_ncu.log
