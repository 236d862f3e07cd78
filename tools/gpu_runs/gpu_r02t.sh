# round-2 GPU batch t: what bounds the GeLU' epilogue (aux traffic vs math), isolated
mkdir -p /tmp/v
for pr in 1 2; do nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -DHX_POLY_EVERY=16 -DHX_EPI_PROBE=$pr -shared -o /tmp/v/libhx_probe$pr.so paper_2507_00394_b200/csrc/*.cu; done
for r in 1 2 3; do
for v in base probe1 probe2; do
  lib=paper_2507_00394_b200/libhx.so; [ $v = probe1 ] && lib=/tmp/v/libhx_probe1.so; [ $v = probe2 ] && lib=/tmp/v/libhx_probe2.so
  HX_LIB=$lib timeout 300 python tools/kernel_bench.py --only gemm --reps 20 | grep -E "dgelu|w1_gelu|dx_mlp_w2\"|fwd_o_proj" | sed "s/^/$v /" >> gpurun_out/r2t.txt
done; done
