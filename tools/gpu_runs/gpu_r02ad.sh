# round-2 GPU batch ad: backward pipeline traces (default, no reduce, MMA only)
timeout 400 python tools/bwd_trace.py > gpurun_out/r2ad_trace_default.txt 2>&1
HX_TRACE_FLAGS="-DHX_BWD_NOREDUCE" timeout 400 python tools/bwd_trace.py > gpurun_out/r2ad_trace_noreduce.txt 2>&1
HX_TRACE_FLAGS="-DHX_BWD_NOCOMPUTE -DHX_BWD_NOREDUCE" timeout 400 python tools/bwd_trace.py > gpurun_out/r2ad_trace_mmaonly.txt 2>&1
