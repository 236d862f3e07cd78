# round-2 GPU batch x: rank-0 stage probes for the sequence sweep (BASELINE config 5), GPT-3B p=8
P="timeout 1200 python tools/stage_probe.py --workload gpt3b_64k --p 8 --stage 0 --mlp-chunk 8192"
for s in 16384 32768 98304 131072; do
  $P --seq $s --method helix_twofold_rc >> gpurun_out/r2x_probe.jsonl 2>>gpurun_out/r2x_probe.err
  $P --seq $s --method 1f1b_rc >> gpurun_out/r2x_probe.jsonl 2>>gpurun_out/r2x_probe.err
done
for s in 16384 32768; do $P --seq $s --method 1f1b >> gpurun_out/r2x_probe.jsonl 2>>gpurun_out/r2x_probe.err; done
