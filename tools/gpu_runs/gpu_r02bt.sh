# round-2 GPU batch bt: split-softmax forward (HX_ATTN_FWD=3: MUFU half + polynomial half per row on two
# warps): kernel tests with it, same-process timing against the default (HX_ATTN_FWD is read once per
# process, so two processes alternate)
HX_ATTN_FWD=3 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_forward" > gpurun_out/r2bt_kern.log 2>&1; echo rc=$? >> gpurun_out/r2bt_kern.log
if grep -q "^rc=0" gpurun_out/r2bt_kern.log; then
  for rep in 1 2 3; do for v in 1 3; do
    HX_ATTN_FWD=$v timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/fwd=$v /" >> gpurun_out/r2bt_kb.txt
  done; done
fi
