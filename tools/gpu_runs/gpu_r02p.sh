# round-2 GPU batch p: forward exp-offload share A/B on the current build; offload+regen test
timeout 900 python -m pytest tests/test_offload_gpu.py -q -x > gpurun_out/r2p_offload.log 2>&1; echo rc=$? >> gpurun_out/r2p_offload.log
mkdir -p /tmp/v
for n in 0 4 8 32; do nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -DHX_POLY_EVERY=$n -shared -o /tmp/v/libhx_p$n.so paper_2507_00394_b200/csrc/*.cu; done
cp paper_2507_00394_b200/libhx.so /tmp/v/libhx_p16.so
for n in 0 4 8 16 32; do HX_LIB=/tmp/v/libhx_p$n.so timeout 120 python tools/kernel_bench.py --only attn --reps 10 | head -1 | sed "s/^/p$n /" >> gpurun_out/r2p_fwd.txt; done
timeout 2400 python tools/bench_ab.py p16=HX_LIB=/tmp/v/libhx_p16.so p8=HX_LIB=/tmp/v/libhx_p8.so p4=HX_LIB=/tmp/v/libhx_p4.so p0=HX_LIB=/tmp/v/libhx_p0.so --rounds 2 -- --steps 3 --warmup 2 > gpurun_out/r2p_ab.txt 2>&1
