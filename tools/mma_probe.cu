// Measures sustained tcgen05.mma throughput on one SM per CTA for the operand
// forms used by libhx: SS (A and B from smem) and TS (A from TMEM), M = 128,
// N in {64, 128, 256}, bf16 -> fp32, K = 16 per instruction.  Prints cycles per
// MMA and the implied dense TFLOP/s at the measured clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include \
//        -I../paper_2507_00394_b200/csrc tools/mma_probe.cu -o mma_probe
#include <cstdio>

#include "hx_common.cuh"

using namespace hx;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16(128, N, false, false);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t db = sw128_desc(sb + (kk & 3) * 32, 16, 1024);
        if (TS)
          umma_f16_ts(tmem, tmem + 256 + kk * 8, db, id, 1);
        else
          umma_f16_ss(tmem, sw128_desc(sa + (kk & 3) * 32, 16, 1024), db, id, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, bool TS>
void run(int sms) {
  const int iters = 4096;
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<N, TS><<<sms, 128, 64 * 1024>>>(16, d);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<N, TS><<<sms, 128, 64 * 1024>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long c0 = 0;
  cudaMemcpy(&c0, d, sizeof(long long), cudaMemcpyDeviceToHost);
  const double mmas = 8.0 * iters;
  const double flops = 2.0 * 128 * N * 16 * mmas * sms;
  printf("{\"form\": \"%s\", \"M\": 128, \"N\": %d, \"cycles_per_mma\": %.2f, \"tflops\": %.1f, \"ideal_cycles\": %d}\n",
         TS ? "TS" : "SS", N, c0 / mmas, flops / (ms * 1e-3) / 1e12, 128 * N / 256);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>(sms);
  run<128, false>(sms);
  run<256, false>(sms);
  run<64, true>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
