# round-2 GPU batch af: exp2 FMA-pipe share (HX_POLY_EVERY 16 / 4 / 3 / 2) for the two-tile forward and the
# one-tile double-buffered-S forward (HX_ATTN_FWD=2), where the softmax is the critical path
for n in 16 4 3 2; do
  mkdir -p build/poly$n
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude -DHX_POLY_EVERY=$n -shared -o build/poly$n/libhx.so paper_2507_00394_b200/csrc/*.cu &
done
wait
for rep in 1 2; do
  for n in 16 4 3 2; do
    for v in 1 2; do
      HX_LIB=build/poly$n/libhx.so HX_ATTN_FWD=$v timeout 120 python tools/kernel_bench.py --only attn --reps 10 | head -1 | sed "s/^/poly$n fwd$v /" >> gpurun_out/r2af_poly.txt
    done
  done
done
