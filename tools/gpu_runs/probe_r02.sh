set -x
P="timeout 900 python tools/stage_probe.py"
$P --workload gpt3b_64k --p 8 --stage 0 --method 1f1b >> gpurun_out/r2d_probe.jsonl 2>>gpurun_out/r2d_probe.err
$P --workload gpt3b_64k --p 8 --stage 0 --method 1f1b_rc --mlp-chunk 8192 >> gpurun_out/r2d_probe.jsonl 2>>gpurun_out/r2d_probe.err
$P --workload gpt3b_64k --p 8 --stage 0 3 --method helix_twofold_rc --mlp-chunk 8192 >> gpurun_out/r2d_probe.jsonl 2>>gpurun_out/r2d_probe.err
$P --workload gpt7b_128k --L 8 --p 8 --stage 0 3 --method helix_twofold_rc --mlp-chunk 16384 --regen-pre-x >> gpurun_out/r2d_probe.jsonl 2>>gpurun_out/r2d_probe.err
$P --workload gpt7b_128k --L 8 --p 8 --stage 3 --method helix_twofold_rc --mlp-chunk 16384 >> gpurun_out/r2d_probe.jsonl 2>>gpurun_out/r2d_probe.err
