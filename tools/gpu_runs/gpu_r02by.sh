# round-2 GPU batch by: is the one-tile forward (HX_ATTN_FWD=2) shared-memory bound? Same kernel with the
# K/V loads dropped after the ring's first fill (debug-only -DHX_FWD_NOKV, results wrong) vs normal, and
# the two-tile default for reference
bash tools/build_variant.sh nokv -DHX_POLY_EVERY=16 -DHX_FWD_NOKV > gpurun_out/r2by_build.log 2>&1
for rep in 1 2; do
  HX_ATTN_FWD=2 HX_LIB=build/variants/nokv/libhx.so timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/fwd1_nokv /" >> gpurun_out/r2by_kb.txt
  HX_ATTN_FWD=2 timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/fwd1 /" >> gpurun_out/r2by_kb.txt
  HX_ATTN_FWD=1 HX_LIB=build/variants/nokv/libhx.so timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/fwd_nokv /" >> gpurun_out/r2by_kb.txt
  HX_ATTN_FWD=1 timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/fwd /" >> gpurun_out/r2by_kb.txt
done
