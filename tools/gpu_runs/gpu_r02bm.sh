# round-2 GPU batch bm: LM-mode bench (V=50257, tied head, CE in the backward) on the current build
timeout 900 python bench.py --lm-vocab 50257 --steps 3 --warmup 2 --no-cpu-baseline --no-config1 > gpurun_out/r2bm_lm.json 2> gpurun_out/r2bm_lm.err; echo rc=$? >> gpurun_out/r2bm_lm.err
