// HBM-bound kernels of the helix components: LayerNorm forward / backward
// (+ residual add, + gain/bias gradient accumulation), the synthetic MSE loss,
// fp32 accumulation.  All vectorised 16-byte accesses, one warp per row.
//
// Roofline: LN fwd reads x and writes y (2*T*h*2 B); LN bwd
// reads dy, x, dres and writes dx (4*T*h*2 B); loss reads z, writes dz.
#include "hx_common.cuh"
#include "hx_gemm.h"

namespace hx {

constexpr float LN_EPS = 1e-5f;

template <int NV>  // NV = 16-byte vectors (8 bf16) per lane
__global__ void __launch_bounds__(256) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const float* __restrict__ gain,
                                                      const float* __restrict__ bias,
                                                      __nv_bfloat16* __restrict__ y, int rows,
                                                      int h) {
  const int row = blockIdx.x * 8 + warp_id();
  if (row >= rows) return;
  const int lane = lane_id();
  const int nvec = h / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(row) * h);
  float v[NV][8];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      uint4 u = xr[c];
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = unpack_bf16(w[j]);
        v[i][2 * j] = f.x;
        v[i][2 * j + 1] = f.y;
        sum += f.x + f.y;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mu = sum / h;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (lane + 32 * i < nvec)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = v[i][j] - mu;
        sq += d * d;
      }
#pragma unroll
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rstd = rsqrtf(sq / h + LN_EPS);
  uint4* yr = reinterpret_cast<uint4*>(y + static_cast<int64_t>(row) * h);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      const float4 g0 = reinterpret_cast<const float4*>(gain)[2 * c];
      const float4 g1 = reinterpret_cast<const float4*>(gain)[2 * c + 1];
      const float4 b0 = reinterpret_cast<const float4*>(bias)[2 * c];
      const float4 b1 = reinterpret_cast<const float4*>(bias)[2 * c + 1];
      const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mu) * rstd * g[j] + bb[j];
      yr[c] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                         pack_bf16(o[6], o[7]));
    }
  }
}

// LN backward, input-gradient half: one warp per row, row data in registers,
// dx = rstd*(dy*g - mean(dy*g) - xhat*mean(dy*g*xhat)) (+ dres).  Also stores
// the row's (mean, rstd) for the column-reduction kernel below.
template <int NV>
__global__ void __launch_bounds__(256) ln_bwd_dx_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ gain, const __nv_bfloat16* __restrict__ dres,
    __nv_bfloat16* __restrict__ dx, float2* __restrict__ stats, int rows, int h) {
  const int row = blockIdx.x * 8 + warp_id();
  if (row >= rows) return;
  const int lane = lane_id();
  const int nvec = h / 8;
  const int64_t off = static_cast<int64_t>(row) * h;
  float xv[NV][8], gv[NV][8];
  float sx = 0.f, sxx = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      const uint4 ux = reinterpret_cast<const uint4*>(x + off)[c];
      const uint4 ud = reinterpret_cast<const uint4*>(dy + off)[c];
      const float4 g0 = reinterpret_cast<const float4*>(gain)[2 * c];
      const float4 g1 = reinterpret_cast<const float4*>(gain)[2 * c + 1];
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const uint32_t wx[4] = {ux.x, ux.y, ux.z, ux.w}, wd[4] = {ud.x, ud.y, ud.z, ud.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fx = unpack_bf16(wx[j]), fd = unpack_bf16(wd[j]);
        xv[i][2 * j] = fx.x;
        xv[i][2 * j + 1] = fx.y;
        gv[i][2 * j] = fd.x * gg[2 * j];  // dxhat = dy * gain
        gv[i][2 * j + 1] = fd.y * gg[2 * j + 1];
        sx += fx.x + fx.y;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
  const float mu = sx / h;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (lane + 32 * i < nvec)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = xv[i][j] - mu;
        sxx += d * d;
      }
#pragma unroll
  for (int o = 16; o; o >>= 1) sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
  const float rstd = rsqrtf(sxx / h + LN_EPS);
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (lane + 32 * i < nvec)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        xv[i][j] = (xv[i][j] - mu) * rstd;
        s1 += gv[i][j];
        s2 += gv[i][j] * xv[i][j];
      }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const float m1 = s1 / h, m2 = s2 / h;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = rstd * (gv[i][j] - m1 - xv[i][j] * m2);
      if (dres) {
        const uint4 ur = reinterpret_cast<const uint4*>(dres + off)[c];
        const uint32_t wr[4] = {ur.x, ur.y, ur.z, ur.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16(wr[j]);
          o[2 * j] += f.x;
          o[2 * j + 1] += f.y;
        }
      }
      reinterpret_cast<uint4*>(dx + off)[c] =
          make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
    }
  }
  if (lane == 0) stats[row] = make_float2(mu, rstd);
}

// LN backward, weight half: dgain += sum_rows dy*xhat, dbias += sum_rows dy.
// Block = 256 threads over 256 columns (8 per thread) x a chunk of rows; each
// warp takes every 8th row, the 8 warps combine in smem, one fp32 atomic per
// column per block.  Coalesced 512-byte row segments per warp.
constexpr int LN_COL_ROWS = 256;
__global__ void __launch_bounds__(256) ln_bwd_dgdb_kernel(const __nv_bfloat16* __restrict__ dy,
                                                          const __nv_bfloat16* __restrict__ x,
                                                          const float2* __restrict__ stats,
                                                          float* __restrict__ dgain, float* __restrict__ dbias,
                                                          int rows, int h) {
  __shared__ float red[8][2][256 + 8];
  const int lane = lane_id(), w = warp_id();
  const int col = blockIdx.x * 256 + lane * 8;
  const int r0 = blockIdx.y * LN_COL_ROWS;
  const int r1 = min(rows, r0 + LN_COL_ROWS);
  float ag[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ab[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (col < h) {
    for (int r = r0 + w; r < r1; r += 8) {
      const float2 st = stats[r];
      const uint4 ux = *reinterpret_cast<const uint4*>(x + static_cast<int64_t>(r) * h + col);
      const uint4 ud = *reinterpret_cast<const uint4*>(dy + static_cast<int64_t>(r) * h + col);
      const uint32_t wx[4] = {ux.x, ux.y, ux.z, ux.w}, wd[4] = {ud.x, ud.y, ud.z, ud.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fx = unpack_bf16(wx[j]), fd = unpack_bf16(wd[j]);
        ag[2 * j] += fd.x * (fx.x - st.x) * st.y;
        ag[2 * j + 1] += fd.y * (fx.y - st.x) * st.y;
        ab[2 * j] += fd.x;
        ab[2 * j + 1] += fd.y;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[w][0][lane * 8 + j] = ag[j];
    red[w][1][lane * 8 + j] = ab[j];
  }
  __syncthreads();
  const int t = threadIdx.x;  // one column per thread
  const int c = blockIdx.x * 256 + t;
  if (c < h) {
    float sg = 0.f, sb = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      sg += red[k][0][t];
      sb += red[k][1][t];
    }
    atomicAdd(&dgain[c], sg);
    atomicAdd(&dbias[c], sb);
  }
}

__global__ void __launch_bounds__(256) mse_loss_kernel(const __nv_bfloat16* __restrict__ z, int64_t n,
                                                        __nv_bfloat16* __restrict__ dz,
                                                        double* __restrict__ sumsq) {
  const float scale = static_cast<float>(2.0 / static_cast<double>(n));
  float acc = 0.f;
  const int64_t nvec = n / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nvec;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4 u = reinterpret_cast<const uint4*>(z)[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = unpack_bf16(w[j]);
      acc += f.x * f.x + f.y * f.y;
      o[j] = pack_bf16(f.x * scale, f.y * scale);
    }
    reinterpret_cast<uint4*>(dz)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ float part[8];
  if (lane_id() == 0) part[warp_id()] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < blockDim.x / 32; ++w) s += part[w];
    atomicAdd(sumsq, s);
  }
}

__global__ void axpy_f32_kernel(float* __restrict__ y, const float* __restrict__ x, int64_t n) {
  const int64_t nv = n / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(y)[i];
    const float4 b = reinterpret_cast<const float4*>(x)[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    reinterpret_cast<float4*>(y)[i] = a;
  }
  const int64_t tail = nv * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (blockIdx.x == 0 && tail < n) y[tail] += x[tail];
}

// ------------------------------------------------------------------ launchers

#define HX_NV_DISPATCH(h, F)            \
  do {                                  \
    const int nv_ = ((h) / 8 + 31) / 32; \
    if (nv_ <= 1) { F(1); }             \
    else if (nv_ <= 2) { F(2); }        \
    else if (nv_ <= 4) { F(4); }        \
    else if (nv_ <= 8) { F(8); }        \
    else if (nv_ <= 16) { F(16); }      \
    else if (nv_ <= 32) { F(32); }      \
    else return cudaErrorInvalidValue;  \
  } while (0)

cudaError_t ln_fwd_launch(const void* x, const float* g, const float* b, void* y, int rows, int h,
                          cudaStream_t st) {
  const int grid = (rows + 7) / 8;
#define L(NV)                                                                          \
  ln_fwd_kernel<NV><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), g, b, \
                                          static_cast<__nv_bfloat16*>(y), rows, h)
  HX_NV_DISPATCH(h, L);
#undef L
  return cudaGetLastError();
}

cudaError_t ln_bwd_launch(const void* dy, const void* x, const float* g, const void* dres, void* dx,
                          float* dg, float* db, float* stats, int rows, int h, cudaStream_t st) {
  const int grid = (rows + 7) / 8;
  float2* st2 = reinterpret_cast<float2*>(stats);
#define L(NV)                                                                                   \
  ln_bwd_dx_kernel<NV><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(dy),            \
                                             static_cast<const __nv_bfloat16*>(x), g,           \
                                             static_cast<const __nv_bfloat16*>(dres),           \
                                             static_cast<__nv_bfloat16*>(dx), st2, rows, h)
  HX_NV_DISPATCH(h, L);
#undef L
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 cg((h + 255) / 256, (rows + LN_COL_ROWS - 1) / LN_COL_ROWS);
  ln_bwd_dgdb_kernel<<<cg, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(dy),
                                         static_cast<const __nv_bfloat16*>(x), st2, dg, db, rows, h);
  return cudaGetLastError();
}

cudaError_t mse_loss_launch(const void* z, int64_t n, void* dz, double* sumsq, cudaStream_t st) {
  int64_t nvec = n / 8;
  int grid = static_cast<int>((nvec + 255) / 256);
  if (grid > num_sms() * 8) grid = num_sms() * 8;
  if (grid < 1) grid = 1;
  mse_loss_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(z), n,
                                        static_cast<__nv_bfloat16*>(dz), sumsq);
  return cudaGetLastError();
}

cudaError_t axpy_f32_launch(float* y, const float* x, int64_t n, cudaStream_t st) {
  int64_t nv = n / 4;
  int grid = static_cast<int>((nv + 255) / 256);
  if (grid > num_sms() * 8) grid = num_sms() * 8;
  if (grid < 1) grid = 1;
  axpy_f32_kernel<<<grid, 256, 0, st>>>(y, x, n);
  return cudaGetLastError();
}

}  // namespace hx
