// HBM-bound kernels of the helix components: LayerNorm forward / backward
// (+ residual add, + gain/bias gradient accumulation), the synthetic MSE loss,
// fp32 accumulation.  All vectorised 16-byte accesses, one warp per row.
//
// Roofline: LN fwd reads x and writes y (2*T*h*2 B); LN bwd
// reads dy, x, dres and writes dx (4*T*h*2 B); loss reads z, writes dz.
#include "hx_common.cuh"
#include "hx_gemm.h"

#ifndef HX_LN_PERSISTENT
#define HX_LN_PERSISTENT 1
#endif

namespace hx {

constexpr float LN_EPS = 1e-5f;

// One warp per row, two passes over the row: pass 1 reads it from HBM and
// accumulates the row sums (sum and sum of squares in one sweep), pass 2
// re-reads it (an L1/L2 hit) to write the output.  Nothing row-sized stays live
// across the warp reductions, so registers stay low and enough warps per SM
// keep HBM busy.  var = E[x^2] - mu^2 in fp32 over bf16 inputs: the
// cancellation error is ~1e-7 * mu^2/var relative, far below bf16 output rounding.
HX_DEVICE void unpack8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = unpack_bf16(w[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
HX_DEVICE void load_gain8(const float* __restrict__ g, int c, float (&f)[8]) {
  const float4 a = reinterpret_cast<const float4*>(g)[2 * c];
  const float4 b = reinterpret_cast<const float4*>(g)[2 * c + 1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
HX_DEVICE float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NV>  // NV = 16-byte vectors (8 bf16) per lane
__global__ void __launch_bounds__(256) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const float* __restrict__ gain,
                                                      const float* __restrict__ bias,
                                                      __nv_bfloat16* __restrict__ y, int rows,
                                                      int h) {
  const int lane = lane_id();
  const int nvec = h / 8;
  // persistent warps (grid sized to the resident slots): no partial last wave
  for (int row = blockIdx.x * 8 + warp_id(); row < rows; row += gridDim.x * 8) {
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(row) * h);
  float sum = 0.f, sq = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      float f[8];
      unpack8(xr[c], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sum += f[j];
        sq = fmaf(f[j], f[j], sq);
      }
    }
  }
  sum = warp_sum(sum);
  sq = warp_sum(sq);
  const float mu = sum / h;
  const float rstd = rsqrtf(fmaxf(sq / h - mu * mu, 0.f) + LN_EPS);
  uint4* yr = reinterpret_cast<uint4*>(y + static_cast<int64_t>(row) * h);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      float f[8], g[8], bb[8], o[8];
      unpack8(xr[c], f);
      load_gain8(gain, c, g);
      load_gain8(bias, c, bb);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (f[j] - mu) * rstd * g[j] + bb[j];
      yr[c] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                         pack_bf16(o[6], o[7]));
    }
  }
  }
}

// LN backward, input-gradient half: one warp per row,
// dx = rstd*(dy*g - mean(dy*g) - xhat*mean(dy*g*xhat)) (+ dres).  Pass 1 gathers
// sum x, sum x^2, sum dy*g, sum dy*g*x in one sweep; pass 2 re-reads x, dy and
// writes dx.  Also stores the row's (mean, rstd) for the column reduction below.
template <int NV>
__global__ void __launch_bounds__(256) ln_bwd_dx_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ gain, const __nv_bfloat16* __restrict__ dres,
    __nv_bfloat16* __restrict__ dx, float2* __restrict__ stats, int rows, int h) {
  const int lane = lane_id();
  const int nvec = h / 8;
  for (int row = blockIdx.x * 8 + warp_id(); row < rows; row += gridDim.x * 8) {
  const int64_t off = static_cast<int64_t>(row) * h;
  const uint4* xr = reinterpret_cast<const uint4*>(x + off);
  const uint4* dr = reinterpret_cast<const uint4*>(dy + off);
  float sx = 0.f, sxx = 0.f, sg = 0.f, sgx = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      float f[8], d[8], g[8];
      unpack8(xr[c], f);
      unpack8(dr[c], d);
      load_gain8(gain, c, g);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float gd = d[j] * g[j];  // dxhat = dy * gain
        sx += f[j];
        sxx = fmaf(f[j], f[j], sxx);
        sg += gd;
        sgx = fmaf(gd, f[j], sgx);
      }
    }
  }
  sx = warp_sum(sx);
  sxx = warp_sum(sxx);
  sg = warp_sum(sg);
  sgx = warp_sum(sgx);
  const float mu = sx / h;
  const float rstd = rsqrtf(fmaxf(sxx / h - mu * mu, 0.f) + LN_EPS);
  const float m1 = sg / h;                          // mean(dxhat)
  const float m2 = (sgx / h - mu * m1) * rstd;      // mean(dxhat * xhat)
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      float f[8], d[8], g[8], o[8];
      unpack8(xr[c], f);
      unpack8(dr[c], d);
      load_gain8(gain, c, g);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = rstd * (d[j] * g[j] - m1 - (f[j] - mu) * rstd * m2);
      if (dres) {
        float r[8];
        unpack8(reinterpret_cast<const uint4*>(dres + off)[c], r);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += r[j];
      }
      reinterpret_cast<uint4*>(dx + off)[c] =
          make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
    }
  }
  if (lane == 0) stats[row] = make_float2(mu, rstd);
  }
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

// ------------------------------------------------------------------ LayerNorm v2
// Column-sliced blocks (round 2).  A block of 8 warps owns a contiguous range of
// rows and walks it R rows at a time; lane (w, l) owns the 16-byte column
// vectors (32w + l) + 256i, i < VPL, so every warp reads whole 512-byte
// segments of a row and each thread's LayerNorm gain / bias (and, backward,
// its gain / bias gradient partials) stay in registers for the whole block.
// Per-row statistics are combined across the 8 warps through shared memory.
// Each row is read from HBM exactly once (the row-per-warp v1 re-read it for
// the second pass), and the backward fuses the gain / bias column reduction
// (v1 re-read dy and x in a second kernel): LN forward moves 2*T*h*2 bytes and
// LN backward 4*T*h*2 (dy, x, dres in; dx out), the algorithmic minimum.
template <int VPL, int R, int MINB>
__global__ void __launch_bounds__(256, MINB) ln_fwd_v2_kernel(const __nv_bfloat16* __restrict__ x,
                                                         const float* __restrict__ gain,
                                                         const float* __restrict__ bias,
                                                         __nv_bfloat16* __restrict__ y, int rows, int h,
                                                         int rows_per_block) {
  __shared__ float2 part[2][R][8];
  const int lane = lane_id(), w = warp_id();
  const int nvec = h / 8;
  const int base = 32 * w + lane;
  float g[VPL][8], bb[VPL][8];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = base + 256 * i;
#pragma unroll
    for (int k = 0; k < 8; ++k) g[i][k] = bb[i][k] = 0.f;
    if (c < nvec) {
      load_gain8(gain, c, g[i]);
      load_gain8(bias, c, bb[i]);
    }
  }
  const int r_begin = blockIdx.x * rows_per_block;
  const int r_end = min(rows, r_begin + rows_per_block);
  uint4 u[R][VPL], nx[R][VPL];
  auto load = [&](uint4 (&dst)[R][VPL], int r0) {
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = base + 256 * i;
        if (r0 + j < r_end && c < nvec)
          dst[j][i] = __ldcs(reinterpret_cast<const uint4*>(x + static_cast<int64_t>(r0 + j) * h) + c);
        else
          dst[j][i] = make_uint4(0, 0, 0, 0);
      }
  };
  load(u, r_begin);
  int buf = 0;
  for (int r0 = r_begin; r0 < r_end; r0 += R, buf ^= 1) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      float sum = 0.f, sq = 0.f;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        float f[8];
        unpack8(u[j][i], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          sum += f[k];
          sq = fmaf(f[k], f[k], sq);
        }
      }
      sum = warp_sum(sum);
      sq = warp_sum(sq);
      if (lane == 0) part[buf][j][w] = make_float2(sum, sq);
    }
    // double-buffered partials: one barrier per batch (the next batch writes the other buffer)
    __syncthreads();
    load(nx, r0 + R);  // the next batch's loads fly during this batch's normalise / store
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (r0 + j >= r_end) break;
      float sum = 0.f, sq = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 t = part[buf][j][k];
        sum += t.x;
        sq += t.y;
      }
      const float mu = sum / h;
      const float rstd = rsqrtf(fmaxf(sq / h - mu * mu, 0.f) + LN_EPS);
      uint4* yr = reinterpret_cast<uint4*>(y + static_cast<int64_t>(r0 + j) * h);
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = base + 256 * i;
        if (c < nvec) {
          float f[8], o[8];
          unpack8(u[j][i], f);
#pragma unroll
          for (int k = 0; k < 8; ++k) o[k] = (f[k] - mu) * rstd * g[i][k] + bb[i][k];
          yr[c] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                             pack_bf16(o[6], o[7]));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int i = 0; i < VPL; ++i) u[j][i] = nx[j][i];
  }
}

template <int VPL, int R, int MINB>
__global__ void __launch_bounds__(256, MINB) ln_bwd_v2_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const float* __restrict__ gain,
    const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx, float* __restrict__ dgain,
    float* __restrict__ dbias, int rows, int h, int rows_per_block) {
  __shared__ float4 part[2][R][8];
  const int lane = lane_id(), w = warp_id();
  const int nvec = h / 8;
  const int base = 32 * w + lane;
  float g[VPL][8], adg[VPL][8], adb[VPL][8];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = base + 256 * i;
#pragma unroll
    for (int k = 0; k < 8; ++k) g[i][k] = adg[i][k] = adb[i][k] = 0.f;
    if (c < nvec) load_gain8(gain, c, g[i]);
  }
  const int r_begin = blockIdx.x * rows_per_block;
  const int r_end = min(rows, r_begin + rows_per_block);
  uint4 ux[R][VPL], ud[R][VPL], nxx[R][VPL], nxd[R][VPL];
  auto load = [&](uint4 (&dx_)[R][VPL], uint4 (&dd_)[R][VPL], int r0) {
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = base + 256 * i;
        const int64_t off = static_cast<int64_t>(r0 + j) * h;
        if (r0 + j < r_end && c < nvec) {
          dx_[j][i] = __ldcs(reinterpret_cast<const uint4*>(x + off) + c);
          dd_[j][i] = __ldcs(reinterpret_cast<const uint4*>(dy + off) + c);
        } else {
          dx_[j][i] = dd_[j][i] = make_uint4(0, 0, 0, 0);
        }
      }
  };
  load(ux, ud, r_begin);
  int buf = 0;
  for (int r0 = r_begin; r0 < r_end; r0 += R, buf ^= 1) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      float sx = 0.f, sxx = 0.f, sg = 0.f, sgx = 0.f;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        float f[8], d[8];
        unpack8(ux[j][i], f);
        unpack8(ud[j][i], d);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float gd = d[k] * g[i][k];
          sx += f[k];
          sxx = fmaf(f[k], f[k], sxx);
          sg += gd;
          sgx = fmaf(gd, f[k], sgx);
        }
      }
      sx = warp_sum(sx);
      sxx = warp_sum(sxx);
      sg = warp_sum(sg);
      sgx = warp_sum(sgx);
      if (lane == 0) part[buf][j][w] = make_float4(sx, sxx, sg, sgx);
    }
    __syncthreads();
    load(nxx, nxd, r0 + R);  // next batch in flight during this batch's dx / column sums
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (r0 + j >= r_end) break;
      float4 t = part[buf][j][0];
#pragma unroll
      for (int k = 1; k < 8; ++k) {
        const float4 q = part[buf][j][k];
        t.x += q.x;
        t.y += q.y;
        t.z += q.z;
        t.w += q.w;
      }
      const float mu = t.x / h;
      const float rstd = rsqrtf(fmaxf(t.y / h - mu * mu, 0.f) + LN_EPS);
      const float m1 = t.z / h;                       // mean(dxhat)
      const float m2 = (t.w / h - mu * m1) * rstd;    // mean(dxhat * xhat)
      const int64_t off = static_cast<int64_t>(r0 + j) * h;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = base + 256 * i;
        if (c < nvec) {
          float f[8], d[8], o[8];
          unpack8(ux[j][i], f);
          unpack8(ud[j][i], d);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float xh = (f[k] - mu) * rstd;
            o[k] = rstd * (d[k] * g[i][k] - m1) - xh * rstd * m2;
            adg[i][k] = fmaf(d[k], xh, adg[i][k]);
            adb[i][k] += d[k];
          }
          if (dres) {
            float r[8];
            unpack8(__ldcs(reinterpret_cast<const uint4*>(dres + off) + c), r);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] += r[k];
          }
          reinterpret_cast<uint4*>(dx + off)[c] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]),
                                                             pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        ux[j][i] = nxx[j][i];
        ud[j][i] = nxd[j][i];
      }
  }
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = base + 256 * i;
    if (c < nvec && r_begin < r_end) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        atomicAdd(&dgain[8 * c + k], adg[i][k]);
        atomicAdd(&dbias[8 * c + k], adb[i][k]);
      }
    }
  }
}

// ------------------------------------------------------------------ LayerNorm backward v5
// For h <= 2048 (h % 256 == 0), where v2's column-sliced 2-row batches are
// barrier-bound and v1 re-reads x and dy for the gain / bias sums.  Rows stream
// through a shared-memory ring filled by 1-D bulk copies (cp.async.bulk, the
// TMA engine) from a producer warp: each slot holds one row of x, dy (and the
// residual gradient), so up to 16 rows per SM (h = 2048) are in flight without a
// register holding them.  Each of the 7 consumer warps owns whole rows (warp
// shuffles for the row statistics, no block barrier in the loop) and keeps its
// lanes' gain / bias gradient partials in registers across all its rows; the
// block combines them once at the end.  HBM traffic is the algorithmic
// 4*T*h*2 bytes (3*T*h*2 without a residual gradient), each row read once.
// 7 consumers + the producer = 8 warps, so the per-SMSP register file allows 255
// registers (9 warps capped ptxas at 168 and spilled the 128 gradient partials).
constexpr int LN5_CONSUMERS = 7;
constexpr int LN5_THREADS = 32 * (LN5_CONSUMERS + 1);
constexpr int LN5_RING_BYTES = 192 * 1024;

HX_DEVICE void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int NV>  // 16-byte vectors per lane per row: h = 256 * NV
__global__ void __launch_bounds__(LN5_THREADS, 1) ln_bwd_v5_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const float* __restrict__ gain,
    const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx, float* __restrict__ dgain,
    float* __restrict__ dbias, int rows, int h, int rows_per_block) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int nt = dres ? 3 : 2;
  const uint32_t row_bytes = static_cast<uint32_t>(h) * 2;
  const int slot_bytes = nt * static_cast<int>(row_bytes);
  const int nslot = LN5_RING_BYTES / slot_bytes;
  float* sgain = reinterpret_cast<float*>(smem + LN5_RING_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sgain + h);
  uint64_t* empty = full + nslot;
  const int lane = lane_id(), w = warp_id();
  const int r_begin = blockIdx.x * rows_per_block;
  const int n = min(rows, r_begin + rows_per_block) - r_begin;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslot; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  for (int c = threadIdx.x; c < h; c += LN5_THREADS) sgain[c] = gain[c];
  __syncthreads();

  if (w == LN5_CONSUMERS) {  // ---------------- producer: rows into the ring
    if (lane == 0) {
      for (int k = 0; k < n; ++k) {
        const int sl = k % nslot;
        mbar_wait(&empty[sl], ((k / nslot) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[sl], slot_bytes);
        uint8_t* dst = smem + sl * slot_bytes;
        const int64_t off = static_cast<int64_t>(r_begin + k) * h;
        bulk_g2s(dst, x + off, row_bytes, &full[sl]);
        bulk_g2s(dst + row_bytes, dy + off, row_bytes, &full[sl]);
        if (dres) bulk_g2s(dst + 2 * row_bytes, dres + off, row_bytes, &full[sl]);
      }
    }
    __syncwarp();
  } else {  // ---------------- consumers: whole rows, warp k % 8 takes row k
    float ag[NV][8], ab[NV][8];
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) ag[i][j] = ab[i][j] = 0.f;
    const float inv_h = 1.0f / static_cast<float>(h);
    for (int k = w; k < n; k += LN5_CONSUMERS) {
      const int sl = k % nslot;
      mbar_wait(&full[sl], (k / nslot) & 1);
      const uint4* sx = reinterpret_cast<const uint4*>(smem + sl * slot_bytes);
      const uint4* sd = sx + h / 8;
      const uint4* sr = sd + h / 8;
      float s_x = 0.f, s_xx = 0.f, s_g = 0.f, s_gx = 0.f;
      // (unrolled by 2 only: fully unrolled, ptxas hoists every vector's shared loads
      // next to the 16 * NV gradient partials and spills at NV >= 6)
#pragma unroll 2
      for (int i = 0; i < NV; ++i) {
        const int c = lane + 32 * i;
        float f[8], d[8], g[8];
        unpack8(sx[c], f);
        unpack8(sd[c], d);
        load_gain8(sgain, c, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float gd = d[j] * g[j];
          s_x += f[j];
          s_xx = fmaf(f[j], f[j], s_xx);
          s_g += gd;
          s_gx = fmaf(gd, f[j], s_gx);
        }
      }
      s_x = warp_sum(s_x);
      s_xx = warp_sum(s_xx);
      s_g = warp_sum(s_g);
      s_gx = warp_sum(s_gx);
      const float mu = s_x * inv_h;
      const float rstd = rsqrtf(fmaxf(s_xx * inv_h - mu * mu, 0.f) + LN_EPS);
      const float m1 = s_g * inv_h;                      // mean(dxhat)
      const float m2 = (s_gx * inv_h - mu * m1) * rstd;  // mean(dxhat * xhat)
      const int64_t off = static_cast<int64_t>(r_begin + k) * h;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = lane + 32 * i;
        float f[8], d[8], g[8], o[8];
        unpack8(sx[c], f);
        unpack8(sd[c], d);
        load_gain8(sgain, c, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (f[j] - mu) * rstd;
          o[j] = rstd * (d[j] * g[j] - m1) - xh * rstd * m2;
          ag[i][j] = fmaf(d[j], xh, ag[i][j]);
          ab[i][j] += d[j];
        }
        if (dres) {
          float r[8];
          unpack8(sr[c], r);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += r[j];
        }
        reinterpret_cast<uint4*>(dx + off)[c] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]),
                                                           pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    }
    __syncthreads();  // (A) every consumer is past the ring; the producer waits here too
    float* red = reinterpret_cast<float*>(smem);  // [8 warps][2][h] over the drained ring
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + 32 * i;
      float4* pg = reinterpret_cast<float4*>(red + (2 * w) * h + 8 * c);
      float4* pb = reinterpret_cast<float4*>(red + (2 * w + 1) * h + 8 * c);
      pg[0] = make_float4(ag[i][0], ag[i][1], ag[i][2], ag[i][3]);
      pg[1] = make_float4(ag[i][4], ag[i][5], ag[i][6], ag[i][7]);
      pb[0] = make_float4(ab[i][0], ab[i][1], ab[i][2], ab[i][3]);
      pb[1] = make_float4(ab[i][4], ab[i][5], ab[i][6], ab[i][7]);
    }
  }
  if (w == LN5_CONSUMERS) __syncthreads();  // (A) for the producer warp
  __syncthreads();                          // (B) partials written
  if (n > 0) {
    const float* red = reinterpret_cast<const float*>(smem);
    for (int c = threadIdx.x; c < h; c += LN5_THREADS) {
      float tg = 0.f, tb = 0.f;
#pragma unroll
      for (int q = 0; q < LN5_CONSUMERS; ++q) {
        tg += red[(2 * q) * h + c];
        tb += red[(2 * q + 1) * h + c];
      }
      atomicAdd(&dgain[c], tg);
      atomicAdd(&dbias[c], tb);
    }
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

// Persistent row loops: at most as many blocks of 8 warps as fit on the GPU at
// once (occupancy of the kernel), so the grid has no partial last wave.
template <typename K>
static int ln_blocks_per_sm(K kernel) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return per_sm;
}
static int ln_grid(int per_sm, int rows) {
  const int blocks = (rows + 7) / 8;
  if (!HX_LN_PERSISTENT) return blocks;
  const int resident = num_sms() * per_sm;
  return blocks < resident ? blocks : resident;
}

// LN v2 (default; the backward only for h > 2048) / v1 (HX_LN=1, kept for A/B runs).
// Measured alone (tools/kernel_bench.py, B200): forward T=32k h=2048 0.058 ms
// (4.66 TB/s) vs v1 0.070; T=64k h=4096 0.197 ms (5.45 TB/s, 83%) vs 0.263.
static int ln_version() {
  static const int v = getenv("HX_LN") ? atoi(getenv("HX_LN")) : 2;
  return v;
}
// (2: 2 blocks of 8 warps per SM, small row batches; 3: 1 block, larger batches)

// Persistent grid for the v2 kernels: the blocks that fit at once, each owning
// an equal contiguous share of the rows (a multiple of R).
template <typename K>
static void ln_v2_grid(K kernel, int rows, int R, int* grid, int* per_block) {
  static int per_sm_cache = 0;
  (void)per_sm_cache;
  const int per_sm = ln_blocks_per_sm(kernel);
  int blocks = num_sms() * per_sm;
  const int batches = (rows + R - 1) / R;
  if (blocks > batches) blocks = batches;
  const int per = (batches + blocks - 1) / blocks;
  *per_block = per * R;
  *grid = (rows + *per_block - 1) / *per_block;
}

// (VPL, R) per width: R rows per batch keep the row data of a batch (R * VPL
// 16-byte vectors per tensor and lane) in registers without spills at 2
// blocks per SM (ptxas -v: no stack for any instance)
#define HX_VPL_DISPATCH(h, F, R1, R2, R4)    \
  do {                                       \
    const int vpl_ = ((h) / 8 + 255) / 256;  \
    if (vpl_ <= 1) { F(1, R1); }             \
    else if (vpl_ <= 2) { F(2, R2); }        \
    else if (vpl_ <= 4) { F(4, R4); }        \
    else return cudaErrorInvalidValue;       \
  } while (0)

cudaError_t ln_fwd_launch(const void* x, const float* g, const float* b, void* y, int rows, int h,
                          cudaStream_t st) {
  if (ln_version() >= 2) {
#define LF(VPL, R, MB)                                                                                    \
  {                                                                                                       \
    int grid, per;                                                                                        \
    ln_v2_grid(ln_fwd_v2_kernel<VPL, R, MB>, rows, R, &grid, &per);                                       \
    ln_fwd_v2_kernel<VPL, R, MB><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), g, b,         \
                                                       static_cast<__nv_bfloat16*>(y), rows, h, per);    \
  }
#define L2(VPL, R) LF(VPL, R, 2)
#define L3(VPL, R) LF(VPL, R, 1)
    if (ln_version() == 3) {
      HX_VPL_DISPATCH(h, L3, 8, 4, 2);
    } else {
      HX_VPL_DISPATCH(h, L2, 4, 2, 1);
    }
#undef L2
#undef L3
#undef LF
    return cudaGetLastError();
  }
#define L(NV)                                                                          \
  static const int per_sm_##NV = ln_blocks_per_sm(ln_fwd_kernel<NV>);                    \
  ln_fwd_kernel<NV><<<ln_grid(per_sm_##NV, rows), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), g, b, \
                                          static_cast<__nv_bfloat16*>(y), rows, h)
  HX_NV_DISPATCH(h, L);
#undef L
  return cudaGetLastError();
}

cudaError_t ln_bwd_launch(const void* dy, const void* x, const float* g, const void* dres, void* dx,
                          float* dg, float* db, float* stats, int rows, int h, cudaStream_t st) {
  // v2 (one pass, gain / bias sums fused) wins from h = 4096 (0.47 vs 0.59 ms at
  // T = 64k); at h <= 2048 its 2-row batches are barrier-bound and the row-per-warp
  // v1 pair is faster (0.142 vs 0.170 ms at T = 32k), tools/kernel_bench.py
  if (ln_version() >= 2 && (ln_version() > 2 || h > 2048)) {
#define LB(VPL, R, MB)                                                                                      \
  {                                                                                                         \
    int grid, per;                                                                                          \
    ln_v2_grid(ln_bwd_v2_kernel<VPL, R, MB>, rows, R, &grid, &per);                                         \
    ln_bwd_v2_kernel<VPL, R, MB><<<grid, 256, 0, st>>>(                                                     \
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), g,                     \
        static_cast<const __nv_bfloat16*>(dres), static_cast<__nv_bfloat16*>(dx), dg, db, rows, h, per);    \
  }
#define L2(VPL, R) LB(VPL, R, 2)
#define L3(VPL, R) LB(VPL, R, 1)
    if (ln_version() == 3) {
      HX_VPL_DISPATCH(h, L3, 4, 2, 1);
    } else {
      HX_VPL_DISPATCH(h, L2, 2, 1, 1);
    }
#undef L2
#undef L3
#undef LB
    return cudaGetLastError();
  }
  // v5 (ring of bulk-copied rows, whole rows per warp, fused gain / bias sums) for
  // h <= 2048; HX_LN_BWD5=0 keeps the v1 pair for A/B runs
  static const int v5 = getenv("HX_LN_BWD5") ? atoi(getenv("HX_LN_BWD5")) : 1;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(x) |
                         reinterpret_cast<uintptr_t>(dres)) & 15) == 0;
  if (v5 && ln_version() >= 2 && h % 256 == 0 && h <= 2048 && aligned) {
    const int smem = LN5_RING_BYTES + h * 4 + 2 * 8 * (LN5_RING_BYTES / (2 * h * 2));
#define L5(NV)                                                                                            \
  {                                                                                                       \
    static bool set_##NV = false;                                                                         \
    if (!set_##NV) {                                                                                      \
      cudaError_t e5 = cudaFuncSetAttribute(ln_bwd_v5_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                            LN5_RING_BYTES + 2048 * 4 + 2 * 8 * (LN5_RING_BYTES / 1024));  \
      if (e5 != cudaSuccess) return e5;                                                                   \
      set_##NV = true;                                                                                    \
    }                                                                                                     \
    const int grid = rows < num_sms() ? (rows > 0 ? rows : 1) : num_sms();                                \
    const int per = (rows + grid - 1) / grid;                                                             \
    ln_bwd_v5_kernel<NV><<<grid, LN5_THREADS, smem, st>>>(                                                 \
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), g,                     \
        static_cast<const __nv_bfloat16*>(dres), static_cast<__nv_bfloat16*>(dx), dg, db, rows, h, per);    \
    return cudaGetLastError();                                                                            \
  }
    switch (h / 256) {
      case 1: L5(1)
      case 2: L5(2)
      case 3: L5(3)
      case 4: L5(4)
      case 5: L5(5)
      case 6: L5(6)
      case 7: L5(7)
      case 8: L5(8)
      default: break;
    }
#undef L5
  }
  float2* st2 = reinterpret_cast<float2*>(stats);
#define L(NV)                                                                                   \
  static const int per_sm_##NV = ln_blocks_per_sm(ln_bwd_dx_kernel<NV>);                         \
  ln_bwd_dx_kernel<NV><<<ln_grid(per_sm_##NV, rows), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(dy),            \
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
