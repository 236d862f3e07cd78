# round-2 GPU batch bh: forward pipeline trace at polynomial shares 1/4 and 1/2 (vs bg's 1/16)
for v in 4 2; do HX_POLY_EVERY=$v timeout 600 python tools/fwd_trace.py > gpurun_out/r2bh_fwd_trace_poly$v.txt 2>&1; done
