# round-2 GPU batch bl: final-build evidence -- full GPU suite, smoke, long-sequence benches
# (3B/64k helix rc, 7B/128k helix rc + offload) and the LM-mode bench on the current tree
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2bl_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2bl_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bl_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bl_smoke.log
timeout 1500 python bench.py --workload gpt3b_64k --method helix_twofold_rc --mlp-chunk 8192 --steps 3 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r2bl_3b.json 2> gpurun_out/r2bl_3b.err
timeout 900 python bench.py --lm --steps 3 --warmup 2 --no-cpu-baseline --no-config1 > gpurun_out/r2bl_lm.json 2> gpurun_out/r2bl_lm.err
timeout 2700 python bench.py --workload gpt7b_128k --method helix_twofold_rc --mlp-chunk 16384 --steps 2 --warmup 3 --no-cpu-baseline --no-config1 --no-e2e > gpurun_out/r2bl_7b.json 2> gpurun_out/r2bl_7b.err
