// Measures L2 fp32 reduce-add throughput of bulk async copies
// (cp.reduce.async.bulk .add.f32, shared::cta -> global) in the access pattern
// a fused flash-attention backward would use for dQ: CTA = one 128-row key
// tile of one head, iterating query tiles from the diagonal to the end and
// reducing a 128 x D fp32 partial dQ tile per query tile (as NCHUNK contiguous
// chunks) into a tile-blocked fp32 dQ accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2507_00394_b200/csrc tools/reduce_probe.cu -o reduce_probe
#include <cstdio>
#include <cstdlib>

#include "hx_common.cuh"

using namespace hx;

constexpr int ROWS = 128;

template <int CHUNK_COLS, int NBUF>
__global__ void __launch_bounds__(128, 1) probe(float* acc, int nq, int D, int spin_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CHUNK_BYTES = ROWS * CHUNK_COLS * 4;
  const int kt = blockIdx.x, bh = blockIdx.y;
  const int nchunk = D / CHUNK_COLS;
  float* sbuf = reinterpret_cast<float*>(smem);
  int k = 0;
  for (int qt = kt; qt < nq; ++qt) {
    if (spin_ns > 0) {
      const uint64_t t0 = global_ns();
      while (global_ns() - t0 < static_cast<uint64_t>(spin_ns)) {
      }
    }
    for (int c = 0; c < nchunk; ++c, ++k) {
      const int b = k % NBUF;
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
      __syncthreads();
      float* dst = sbuf + b * (CHUNK_BYTES / 4);
      for (int i = threadIdx.x; i < CHUNK_BYTES / 4; i += 128) dst[i] = 1.0f;
      fence_proxy_async();
      __syncthreads();
      if (threadIdx.x == 0) {
        float* g = acc + ((static_cast<int64_t>(bh) * nq + qt) * nchunk + c) * (CHUNK_BYTES / 4);
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(g),
            "r"(smem_u32(dst)), "r"(CHUNK_BYTES)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int CC, int NB>
void run(float* acc, int nq, int heads, int D, int spin) {
  const int smem = NB * ROWS * CC * 4;
  cudaFuncSetAttribute(probe<CC, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(nq, heads);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe<CC, NB><<<grid, 128, smem>>>(acc, nq, D, spin);
  cudaEventRecord(a);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) probe<CC, NB><<<grid, 128, smem>>>(acc, nq, D, spin);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double pairs = static_cast<double>(heads) * nq * (nq + 1) / 2;
  const double bytes = pairs * ROWS * D * 4;
  printf("chunk_cols=%d nbuf=%d spin=%dns: %.3f ms, %.2f GB reduced, %.0f GB/s, %.2f us per tile pair per CTA-slot\n",
         CC, NB, spin, ms, bytes / 1e9, bytes / ms / 1e6, ms * 1e3 / (pairs / 148.0));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
}

int main(int argc, char** argv) {
  const int s = argc > 1 ? atoi(argv[1]) : 32768;
  const int heads = argc > 2 ? atoi(argv[2]) : 16;
  const int D = 128;
  const int nq = s / ROWS;
  float* acc;
  cudaMalloc(&acc, static_cast<size_t>(heads) * s * D * 4);
  cudaMemset(acc, 0, static_cast<size_t>(heads) * s * D * 4);
  run<32, 2>(acc, nq, heads, D, 0);
  run<32, 4>(acc, nq, heads, D, 0);
  run<64, 2>(acc, nq, heads, D, 0);
  run<128, 1>(acc, nq, heads, D, 0);
  run<32, 4>(acc, nq, heads, D, 1000);
  run<32, 4>(acc, nq, heads, D, 1500);
  run<32, 4>(acc, nq, heads, D, 2000);
  // correctness of the accumulated count: every element of q tile qt got (qt+1) adds per rep
  float h[4];
  cudaMemcpy(h, acc, 16, cudaMemcpyDeviceToHost);
  printf("acc[0] = %.0f\n", h[0]);
  return 0;
}
