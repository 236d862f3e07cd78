# round-2 GPU batch f: new dQ protocol + LN v2 prefetch + streamer A/B
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention or layernorm" > gpurun_out/r2f_kern.log 2>&1; echo rc=$? >> gpurun_out/r2f_kern.log
timeout 1500 python -m pytest tests -m gpu -q -x -rA > gpurun_out/r2f_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2f_pytest.log
for v in 1 2 3; do for wl in gpt1.3b_32k gpt3b_64k; do HX_LN=$v timeout 120 python tools/kernel_bench.py --workload $wl --only ln --reps 20 | sed "s/^/HX_LN=$v $wl /" >> gpurun_out/r2f_ln.txt 2>&1; done; done
timeout 300 python tools/kernel_bench.py --only attn --reps 10 > gpurun_out/r2f_attn.txt 2>&1
timeout 600 python tools/stream_ab.py 8 > gpurun_out/r2f_stream.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench.log 2>&1
