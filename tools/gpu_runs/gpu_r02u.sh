# round-2 GPU batch u: TMA aux loads in the pair GEMM epilogue (vs the previous build)
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k gemm > gpurun_out/r2u_kern.log 2>&1; echo rc=$? >> gpurun_out/r2u_kern.log
for r in 1 2; do for v in prev cur; do lib=paper_2507_00394_b200/libhx.so; [ $v = prev ] && lib=paper_2507_00394_b200/libhx_prev.so
HX_LIB=$lib timeout 300 python tools/kernel_bench.py --only gemm --reps 20 | grep -E "dgelu|w1_gelu|fwd_o_proj|fwd_mlp_w2" | sed "s/^/$v /" >> gpurun_out/r2u_gemm.txt; done; done
timeout 1800 python tools/bench_ab.py prev=HX_LIB=paper_2507_00394_b200/libhx_prev.so cur=HX_LIB=paper_2507_00394_b200/libhx.so --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2u_ab.txt 2>&1
