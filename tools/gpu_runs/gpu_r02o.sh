# round-2 GPU batch o: long-sequence single-GPU benches + seq sweep with the round-2 kernels
timeout 1200 python bench.py --workload gpt3b_64k --method helix_twofold_rc --mlp-chunk 8192 --steps 3 --warmup 2 --no-cpu-baseline --no-config1 > gpurun_out/r2o_3b.log 2>&1
timeout 1800 python bench.py --workload gpt7b_128k --method helix_twofold_rc --mlp-chunk 16384 --steps 2 --warmup 2 --no-cpu-baseline --no-config1 --no-e2e > gpurun_out/r2o_7b.log 2>&1
timeout 2400 python tools/seq_sweep.py --out gpurun_out/r02_seq_sweep.json --config1-off > gpurun_out/r2o_sweep.log 2>&1 || timeout 2400 python tools/seq_sweep.py --out gpurun_out/r02_seq_sweep.json > gpurun_out/r2o_sweep.log 2>&1
