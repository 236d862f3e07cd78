// Throughput probe for the softmax instruction mix on B200: MUFU.EX2, FFMA2,
// and the FMA-pipe exp2 polynomial.  Each thread runs independent chains so
// the numbers are pipe throughput, not latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mufu_probe tools/mufu_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;      // independent chains per thread
constexpr int ITERS = 4096;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ex2(float* out, float seed) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c) * 1e-9f;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = ex2(v[c]) - 1.0f;
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float seed) {
  uint64_t v[CH];
  const uint64_t a = 0x3f8000003f800000ull, b = 0x3a83126f3a83126full;
  for (int c = 0; c < CH; ++c) v[c] = static_cast<uint64_t>(__float_as_uint(seed * c)) * 0x100000001ull;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = ffma2(v[c], a, b);
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 12345) out[0] = 1;
}

__global__ void k_ffma(float* out, float seed) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = seed * c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = fmaf(v[c], 1.0001f, 1e-3f);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
}

__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// bf16x2 by integer round-half-up and a byte permute (ALU pipe only)
__device__ __forceinline__ uint32_t alu_bf16x2(float lo, float hi) {
  const uint32_t a = __float_as_uint(lo) + 0x8000u, b = __float_as_uint(hi) + 0x8000u;
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// one F2FP per inner op (LOP3 feeds the next input)
__global__ void k_f2fp(float* out, float seed) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c);
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __uint_as_float(cvt_bf16x2(v[c], v[c]) ^ 0x1u);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_alupack(float* out, float seed) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c);
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __uint_as_float(alu_bf16x2(v[c], v[c]) ^ 0x1u);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
}
// one EX2 + one F2FP per inner op: if they share the XU pipe this takes ~2x k_ex2
__global__ void k_ex2_f2fp(float* out, float seed) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c) * 1e-9f;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __uint_as_float(cvt_bf16x2(ex2(v[c]), v[c]) & 0x3fff3fffu);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
}

// packed exponentials: two results per MUFU instruction if the unit is 2-wide
__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__global__ void k_ex2_f16x2(float* out, float seed) {
  uint32_t v[CH];
  for (int c = 0; c < CH; ++c) v[c] = 0xb800b800u + threadIdx.x + c;  // ~ -0.5 halves
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = ex2_f16x2(v[c]) ^ 0x80008000u;
  uint32_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 12345) out[0] = 1;
}
__global__ void k_ex2_bf16x2(float* out, float seed) {
  uint32_t v[CH];
  for (int c = 0; c < CH; ++c) v[c] = 0xbf00bf00u + threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = ex2_bf16x2(v[c]) ^ 0x80008000u;
  uint32_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 12345) out[0] = 1;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 4;
  auto run = [&](const char* name, void (*k)(float*, float), double ops_per_inner) {
    k<<<blocks, threads>>>(out, 1.0f);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double total = double(blocks) * threads * ITERS * CH * ops_per_inner;
    const double per_ns = total / (ms * 1e6);
    // lanes per clock per SM at the nominal max clock (khz)
    printf("{\"probe\": \"%s\", \"ms\": %.4f, \"lane_ops_per_ns\": %.1f, \"per_clk_per_sm_at_max\": %.2f}\n", name, ms,
           per_ns, per_ns / (clk * 1e-6) / sms);
  };
  run("mufu_ex2", k_ex2, 1.0);
  run("ffma2_lanes", k_ffma2, 2.0);
  run("ffma", k_ffma, 1.0);
  run("f2fp_bf16x2", k_f2fp, 1.0);
  run("alu_bf16x2", k_alupack, 1.0);
  run("ex2+f2fp (pairs)", k_ex2_f2fp, 1.0);
  run("ex2_f16x2 (elements)", k_ex2_f16x2, 2.0);
  run("ex2_bf16x2 (elements)", k_ex2_bf16x2, 2.0);
  printf("{\"sms\": %d, \"max_clock_mhz\": %d, \"err\": \"%s\"}\n", sms, clk / 1000,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
