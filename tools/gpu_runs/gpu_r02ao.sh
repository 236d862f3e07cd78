# round-2 GPU batch ao: large configs on the current build + the ncu launch list of the bench command
timeout 1200 python bench.py --workload gpt3b_64k --method helix_twofold_rc --mlp-chunk 8192 --steps 3 --warmup 3 --no-cpu-baseline --no-config1 > gpurun_out/r2ao_3b.log 2>&1
timeout 2400 python bench.py --workload gpt7b_128k --method helix_twofold_rc --mlp-chunk 16384 --steps 2 --warmup 3 --no-cpu-baseline --no-config1 --no-e2e > gpurun_out/r2ao_7b.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r2ao_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no > gpurun_out/r2ao_ncu_bench.log 2>&1
