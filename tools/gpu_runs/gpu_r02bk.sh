# round-2 GPU batch bk: forward with self-issued MMAs (HX_FWD_SELF_ISSUE=1): kernel tests on that build,
# same-process A/B against the shipped build at 32k and 128k, pipeline trace
bash tools/build_variant.sh si -DHX_POLY_EVERY=16 -DHX_FWD_SELF_ISSUE=1 > gpurun_out/r2bk_build.log 2>&1
bash tools/build_variant.sh base -DHX_POLY_EVERY=16 >> gpurun_out/r2bk_build.log 2>&1
HX_LIB=build/variants/si/libhx.so timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_forward" > gpurun_out/r2bk_kern.log 2>&1; echo rc=$? >> gpurun_out/r2bk_kern.log
if grep -q "^rc=0" gpurun_out/r2bk_kern.log; then
  timeout 600 python tools/ab_attn.py build/variants/si/libhx.so build/variants/base/libhx.so --rounds 11 --only fwd > gpurun_out/r2bk_ab.txt 2>&1
  timeout 600 python tools/ab_attn.py build/variants/si/libhx.so build/variants/base/libhx.so --rounds 3 --only fwd --seq 131072 --heads 32 >> gpurun_out/r2bk_ab.txt 2>&1
fi
