# round-2 GPU batch bv: split-softmax forward with both halves on MUFU (-DHX_FWDS_POLY=0) vs the
# MUFU/poly split and the default kernel
bash tools/build_variant.sh mufu -DHX_POLY_EVERY=16 -DHX_FWDS_POLY=0 > gpurun_out/r2bv_build.log 2>&1
for rep in 1 2; do
  HX_ATTN_FWD=3 HX_LIB=build/variants/mufu/libhx.so timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/split_mufu /" >> gpurun_out/r2bv_kb.txt
  HX_ATTN_FWD=3 timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/split_poly /" >> gpurun_out/r2bv_kb.txt
  HX_ATTN_FWD=1 timeout 120 python tools/kernel_bench.py --only attn --reps 20 | grep attn_fwd | sed "s/^/default /" >> gpurun_out/r2bv_kb.txt
done
