# round-2 GPU batch bj: forward softmax with P stored 8 pairs at a time (HX_FWD_CHUNK_ST=1: in-order
# tcgen05.st sinks keep ptxas from hoisting all polynomial pairs ahead of a back-to-back MUFU tail),
# at polynomial shares 1/16, 1/8, 1/4, 1/3, same-process A/B against the shipped build
bash tools/build_variant.sh base -DHX_POLY_EVERY=16 > gpurun_out/r2bj_build.log 2>&1
for v in 16 8 4 3; do bash tools/build_variant.sh c$v -DHX_POLY_EVERY=$v -DHX_FWD_CHUNK_ST=1 >> gpurun_out/r2bj_build.log 2>&1; done
for v in 16 8 4 3; do
  timeout 600 python tools/ab_attn.py build/variants/c$v/libhx.so build/variants/base/libhx.so --rounds 9 --only fwd >> gpurun_out/r2bj_ab.txt 2>&1
done
echo rc=$? >> gpurun_out/r2bj_ab.txt
