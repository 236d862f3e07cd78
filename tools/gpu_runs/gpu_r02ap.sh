# round-2 GPU batch ap: the ncu launch list of the bench command on the final build (per-launch times,
# cold-cache and serialised: shares, not absolutes)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2ap_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-config1 --compare-1f1b no > gpurun_out/r2ap_ncu_bench.log 2>&1
