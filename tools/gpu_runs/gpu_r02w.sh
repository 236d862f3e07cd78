# round-2 GPU batch w: GeLU' epilogue with A&S erf sharing the density's exp (A/B)
mkdir -p /tmp/v
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -DHX_POLY_EVERY=16 -DHX_DGELU_AS -shared -o /tmp/v/libhx_as.so paper_2507_00394_b200/csrc/*.cu
HX_LIB=/tmp/v/libhx_as.so timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > gpurun_out/r2w_kern.log 2>&1; echo rc=$? >> gpurun_out/r2w_kern.log
for r in 1 2; do for v in cur as; do lib=paper_2507_00394_b200/libhx.so; [ $v = as ] && lib=/tmp/v/libhx_as.so
HX_LIB=$lib timeout 300 python tools/kernel_bench.py --only gemm --reps 20 | grep -E "dgelu" | sed "s/^/$v /" >> gpurun_out/r2w_gemm.txt; done; done
timeout 1800 python tools/bench_ab.py cur=HX_LIB=paper_2507_00394_b200/libhx.so as=HX_LIB=/tmp/v/libhx_as.so --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2w_ab.txt 2>&1
