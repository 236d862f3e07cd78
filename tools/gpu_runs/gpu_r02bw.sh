# round-2 GPU batch bw: cheaper polynomial exp2 (f = x - n by one FFMA2): forward kernel tests at shares
# 1/4 and the default 1/16, then shares 1/16, 1/8, 1/4 against the previous polynomial (HEAD build)
for v in 16 8 4; do bash tools/build_variant.sh new$v -DHX_POLY_EVERY=$v >> gpurun_out/r2bw_build.log 2>&1; done
HX_LIB=build/variants/new4/libhx.so timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_forward" > gpurun_out/r2bw_kern.log 2>&1; echo rc=$? >> gpurun_out/r2bw_kern.log
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" >> gpurun_out/r2bw_kern.log 2>&1; echo rc16=$? >> gpurun_out/r2bw_kern.log
for v in 16 8 4; do
  timeout 600 python tools/ab_attn.py build/variants/new$v/libhx.so $GRAFT_REPO_ROOT/lib_head_ab.so --rounds 9 --only fwd >> gpurun_out/r2bw_ab.txt 2>&1
done
