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

// SS with MN-major operands (the dQ = dS K form of the fused backward: A and B
// both MN-major, K = 128 rows, two 64-element atoms per operand).
template <int N, bool AMN, bool BMN, bool TSA = false>
__global__ void __launch_bounds__(128, 1) probe_mn(int iters, long long* cycles) {
  static_assert(!(TSA && AMN), "TS A is TMEM");
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
    constexpr uint32_t id = idesc_bf16(128, N, AMN, BMN);
    const uint32_t sa = smem_u32(smem), sb = sa + 32768;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t da = AMN ? sw128_desc(sa + kk * 2048, 128 * 128, 1024) : sw128_desc(sa + (kk & 3) * 32, 16, 1024);
        const uint64_t db = BMN ? sw128_desc(sb + kk * 2048, 128 * 128, 1024) : sw128_desc(sb + (kk & 3) * 32, 16, 1024);
        if (TSA)
          umma_f16_ts(tmem, tmem + 256 + kk * 8, db, id, 1);
        else
          umma_f16_ss(tmem, da, db, id, 1);
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

template <int N, bool AMN, bool BMN, bool TSA = false>
void run_mn(int sms) {
  const int iters = 4096;
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaFuncSetAttribute(probe_mn<N, AMN, BMN, TSA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe_mn<N, AMN, BMN, TSA><<<sms, 128, 64 * 1024>>>(16, d);
  probe_mn<N, AMN, BMN, TSA><<<sms, 128, 64 * 1024>>>(iters, d);
  cudaDeviceSynchronize();
  long long c0 = 0;
  cudaMemcpy(&c0, d, sizeof(long long), cudaMemcpyDeviceToHost);
  printf("{\"form\": \"%s a_mn=%d b_mn=%d\", \"M\": 128, \"N\": %d, \"cycles_per_mma\": %.2f, \"ideal_cycles\": %d}\n",
         TSA ? "TS" : "SS", AMN, BMN, N, c0 / (8.0 * iters), 128 * N / 256);
  cudaFree(d);
}

// SS MMAs (N=128, K-major) on thread 0 while warps 1..3 stream 16-byte smem
// stores (ST=1) or loads (ST=2) into a separate region: does other smem traffic
// slow the tensor core's operand reads?
template <int ST>
__global__ void __launch_bounds__(128, 1) probe_contend(int iters, long long* cycles, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    stop = 0;
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16(128, 128, false, false);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_f16_ss(tmem, sw128_desc(sa + (kk & 3) * 32, 16, 1024), sw128_desc(sb + (kk & 3) * 32, 16, 1024), id, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
    atomicExch(&stop, 1);
  } else if (warp > 0 && ST == 4) {
    // TMEM writes of columns 256.. by warps 1..3
    long long n = 0;
    const long long c0 = clock64();
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = i;
    while (!*reinterpret_cast<volatile int*>(&stop)) {
      tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 256 + (n & 7) * 32, r);
      tmem_wait_st();
      ++n;
    }
    if (threadIdx.x == 32 && blockIdx.x == 0) { sink[0] = static_cast<int>(n); sink[1] = static_cast<int>(clock64() - c0); }
  } else if (warp == 1 && ST == 5) {
    // bulk smem -> global copies (TMA engine reading smem), 16 KB each, 2 in flight
    long long n = 0;
    const long long c0 = clock64();
    float* g = reinterpret_cast<float*>(sink) + 64 + blockIdx.x * 8192;
    if (lane_id() == 0) {
      while (!*reinterpret_cast<volatile int*>(&stop)) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(g),
                     "r"(smem_u32(smem + 32768 + (n & 1) * 16384))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        ++n;
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      if (blockIdx.x == 0) { sink[0] = static_cast<int>(n); sink[1] = static_cast<int>(clock64() - c0); }
    }
  } else if (warp > 0 && ST == 3) {
    // TMEM reads of columns 256.. (not touched by the MMA) by warps 1..3
    long long n = 0;
    const long long c0 = clock64();
    uint32_t acc = 0;
    while (!*reinterpret_cast<volatile int*>(&stop)) {
      uint32_t r[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 256 + (n & 7) * 32, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= r[i];
      ++n;
    }
    if (threadIdx.x == 32 && blockIdx.x == 0) { sink[0] = static_cast<int>(n); sink[1] = static_cast<int>(clock64() - c0); }
    if (acc == 12345) sink[2] = 1;
  } else if (warp > 0 && ST > 0) {
    uint4* reg = reinterpret_cast<uint4*>(smem + 32768);  // 64 KB region
    const int t = threadIdx.x - 32;
    uint4 acc = make_uint4(0, 0, 0, 0);
    long long n = 0;
    const long long c0 = clock64();
    while (!*reinterpret_cast<volatile int*>(&stop)) {
#pragma unroll 8
      for (int i = 0; i < 64; ++i) {
        if (ST == 1) reg[(i * 96 + t) & 4095] = make_uint4(i, n, t, 1);
        else {
          uint32_t a, b, c, e;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(e)
                       : "r"(smem_u32(reg + ((i * 96 + t) & 4095))));
          acc.x ^= a ^ b ^ c ^ e;
        }
      }
      n += 64;
    }
    if (t == 0 && blockIdx.x == 0) { sink[0] = static_cast<int>(n); sink[1] = static_cast<int>(clock64() - c0); }
    if (acc.x == 12345) sink[2] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int ST>
void run_contend(int sms) {
  const int iters = 2048;
  long long* d;
  int* sink;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaMalloc(&sink, 256 + 148 * 8192 * 4);
  cudaFuncSetAttribute(probe_contend<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  probe_contend<ST><<<sms, 128, 96 * 1024>>>(16, d, sink);
  probe_contend<ST><<<sms, 128, 96 * 1024>>>(iters, d, sink);
  cudaDeviceSynchronize();
  long long c0 = 0;
  int hs[2] = {0, 0};
  cudaMemcpy(&c0, d, sizeof(long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(hs, sink, 8, cudaMemcpyDeviceToHost);
  const double bytes_per_clk = ST == 3 || ST == 4 ? 3.0 * 32 * 128 * hs[0] / hs[1]
                             : ST == 5 ? 16384.0 * hs[0] / hs[1] : ST ? 96.0 * 16 * hs[0] / hs[1] : 0.0;
  printf("{\"form\": \"SS N=128 + %s\", \"cycles_per_mma\": %.2f, \"other_smem_B_per_clk\": %.1f}\n",
         ST == 0 ? "idle" : ST == 1 ? "96 threads STS.128" : ST == 2 ? "96 threads LDS.128" : ST == 3 ? "3 warps tcgen05.ld x32" : ST == 4 ? "3 warps tcgen05.st x32" : "bulk smem->global 16KB x2", c0 / (8.0 * iters), bytes_per_clk);
  cudaFree(d);
  cudaFree(sink);
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
  run_mn<128, false, false>(sms);
  run_mn<128, false, true>(sms);
  run_mn<128, true, false>(sms);
  run_mn<128, true, true>(sms);
  run_mn<128, false, true, true>(sms);
  run_contend<0>(sms);
  run_contend<1>(sms);
  run_contend<2>(sms);
  run_contend<3>(sms);
  run_contend<4>(sms);
  run_contend<5>(sms);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
