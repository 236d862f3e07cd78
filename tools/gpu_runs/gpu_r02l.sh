# round-2 GPU batch l: fast-erf GeLU epilogues A/B vs libm erff; cuDNN attention yardstick
mkdir -p /tmp/v && nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -DHX_POLY_EVERY=16 -DHX_EXACT_ERF -shared -o /tmp/v/libhx_exact.so paper_2507_00394_b200/csrc/*.cu
cp paper_2507_00394_b200/libhx.so /tmp/v/libhx_fast.so
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > gpurun_out/r2l_kern.log 2>&1; echo rc=$? >> gpurun_out/r2l_kern.log
timeout 1800 python tools/bench_ab.py fast=HX_LIB=/tmp/v/libhx_fast.so exact=HX_LIB=/tmp/v/libhx_exact.so --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2l_ab.txt 2>&1
timeout 600 python tools/cudnn_attn_ref.py > gpurun_out/r2l_cudnn.txt 2>&1
timeout 600 python tools/cudnn_attn_ref.py 131072 32 128 >> gpurun_out/r2l_cudnn.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2l_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2l_pytest.log
