# round-2 GPU batch bx: validation of the final tree -- full GPU suite, smoke, bench
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2bx_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2bx_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bx_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bx_smoke.log
timeout 900 python bench.py > gpurun_out/r2bx_bench.json 2> gpurun_out/r2bx_bench.err; echo rc=$? >> gpurun_out/r2bx_bench.err
