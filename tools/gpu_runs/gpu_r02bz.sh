# round-2 GPU batch bz: backward Q/dO-stream probe in alternating processes (cf. by for the forward)
bash tools/build_variant.sh noqdo -DHX_POLY_EVERY=16 -DHX_BWD_NOQDO > gpurun_out/r2bz_build.log 2>&1
for rep in 1 2; do
  HX_LIB=build/variants/noqdo/libhx.so timeout 120 python tools/kernel_bench.py --only attn --reps 10 | grep attn_bwd | sed "s/^/bwd_noqdo /" >> gpurun_out/r2bz_kb.txt
  timeout 120 python tools/kernel_bench.py --only attn --reps 10 | grep attn_bwd | sed "s/^/bwd /" >> gpurun_out/r2bz_kb.txt
done
