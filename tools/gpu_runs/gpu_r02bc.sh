# round-2 GPU batch bc: what bounds the forward softmax -- the same kernel with no exponentials
# (debug-only -DHX_FWD_NOEXP, results wrong) and with every / every 2nd / 4th exponential pair on
# the FMA-pipe polynomial, each against the default build in one process
bash tools/build_variant.sh base -DHX_POLY_EVERY=16 > gpurun_out/r2bc_build.log 2>&1
bash tools/build_variant.sh noexp -DHX_FWD_NOEXP -DHX_POLY_EVERY=16 >> gpurun_out/r2bc_build.log 2>&1
for v in 1 2 4 8; do bash tools/build_variant.sh poly$v -DHX_POLY_EVERY=$v >> gpurun_out/r2bc_build.log 2>&1; done
for v in noexp poly1 poly2 poly4 poly8; do
  timeout 600 python tools/ab_attn.py build/variants/$v/libhx.so build/variants/base/libhx.so --rounds 7 --only fwd >> gpurun_out/r2bc_ab.txt 2>&1
done
echo rc=$? >> gpurun_out/r2bc_ab.txt
