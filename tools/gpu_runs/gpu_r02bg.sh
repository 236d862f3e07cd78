# round-2 GPU batch bg: forward pipeline trace on the current build (HX_POLY_EVERY=16 as shipped)
HX_POLY_EVERY=16 timeout 600 python tools/fwd_trace.py > gpurun_out/r2bg_fwd_trace.txt 2>&1; echo rc=$? >> gpurun_out/r2bg_fwd_trace.txt
