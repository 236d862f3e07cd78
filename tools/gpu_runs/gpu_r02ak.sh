# round-2 GPU batch ak: per-SASS source counters of the two heavy-epilogue GEMMs (W1 + GeLU, W2^T + GeLU')
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --import-source on \
  --clock-control none -k regex:gemm_2sm -c 2 -f -o /tmp/epi_src python tools/epi_gemm_probe.py > gpurun_out/r2ak_ncu.log 2>&1
ncu -i /tmp/epi_src.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/r2ak_epi_sass.csv.gz
ncu -i /tmp/epi_src.ncu-rep --page details > gpurun_out/r2ak_details.txt 2>&1
