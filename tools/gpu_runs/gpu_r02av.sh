# round-2 GPU batch av: full GPU suite + smoke on the current tree
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2av_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2av_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2av_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2av_smoke.log
