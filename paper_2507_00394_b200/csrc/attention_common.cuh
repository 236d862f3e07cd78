// Shared pieces of the causal flash-attention kernels (forward / backward).
//
// Tile layouts: a [rows x D] bf16 tile of one head is D/64 swizzle atoms of
// [rows x 64] (rows*128 bytes each), written by TMA with SWIZZLE_128B.  The same
// physical tile is a K-major UMMA operand (K = the 64-column atoms) or an
// MN-major one (K = rows), so no transposed copies exist anywhere.
// TMEM A operands ("packed"): lane = row, 32-bit column c holds K elements
// (2c, 2c+1) as bf16x2.
#pragma once

#include "hx_common.cuh"
#include "hx_gemm.h"

namespace hx {

constexpr int AT_TILE = 128;  // rows of a resident (M-side) tile
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

template <int D>
struct Tile {  // [128 x D]
  static constexpr int BYTES = AT_TILE * D * 2;
};

struct AttnParams {
  int s, b, heads, h;
  float scale_log2;  // log2(e) / sqrt(d)
  float scale;       // 1 / sqrt(d)
  __nv_bfloat16* o;  // forward output [s*b, ld_o]
  int ld_o;
  float* lse;          // [b, heads, s], natural log
  const float* delta;  // [b, heads, s], rowsum(dO * O)
  __nv_bfloat16* dqkv;
  int ld_dqkv;
  int band;            // (batch, head)s per band of the CTA order (band_order)
};

// Smem descriptors for K-step kk (16 elements) of a tile with `rows` rows.
HX_DEVICE uint64_t kdesc(uint32_t base, int kk, int rows) {  // K along the 64-col atoms
  return sw128_desc(base + (kk >> 2) * rows * 128 + (kk & 3) * 32, 16, 1024);
}
HX_DEVICE uint64_t mndesc(uint32_t base, int kk, int rows) {  // K along rows, N/M along atoms
  return sw128_desc(base + kk * 2048, rows * 128, 1024);
}

// [rows x D] tile of head columns col0.. for tokens s0.. of batch bi (3-D map {cols, b, s}).
template <int D>
HX_DEVICE void tma_tile_rows(void* dst, const CUtensorMap* map, uint64_t* bar, int col0, int bi, int s0,
                             int rows) {
#pragma unroll
  for (int a = 0; a < D / 64; ++a)
    tma_load_3d(static_cast<uint8_t*>(dst) + a * rows * 128, map, bar, col0 + 64 * a, bi, s0);
}

// CTA order of the attention grids: blocks enumerate bands of `band` (batch, head)
// pairs; inside a band the work index w (0 = heaviest) is the slow coordinate, so
// every head of the band starts its heaviest tile before any lighter one.  Wide
// bands shorten the grid's tail; narrow bands keep the concurrently streamed
// per-head data (K/V, the fp32 dQ accumulator) in L2.  Under the B200's power
// cap the DRAM traffic costs clock: see attn_band() in the launchers.
HX_DEVICE void band_order(int blk, int nwork, int nbh, int band, int& bh, int& w) {
  band = band < 1 ? 1 : (band > nbh ? nbh : band);
  const int b0 = blk / (band * nwork) * band;
  const int r = blk - b0 * nwork;
  const int bsz = min(band, nbh - b0);
  w = r / bsz;
  bh = b0 + r % bsz;
}

HX_DEVICE float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (no MUFU): x = n + f, f in [0,1); 2^f by a degree-3
// minimax polynomial (max rel. error ~9e-5, below bf16's 2^-9 rounding of P);
// 2^n added to the exponent field.  Valid for x <= 0 (softmax arguments);
// clamped at -127 so the result flushes to ~0.  Used for a fraction of the
// elements so the 16/clk/SM MUFU unit stops being the softmax floor (FA4).
HX_DEVICE float exp2_poly(float x) {
  x = fmaxf(x, -127.0f);
  const float n = floorf(x);
  const float f = x - n;
  float p = fmaf(f, 0.0794402384f, 0.2244943373f);
  p = fmaf(f, p, 0.6960656422f);
  p = fmaf(f, p, 1.0f);
  return __int_as_float(__float_as_int(p) + (static_cast<int>(n) << 23));
}

// Exponential of element k of an unrolled softmax row: every HX_POLY_EVERY-th
// one is computed on the FMA pipe, the rest on MUFU (k is a compile-time
// constant after unrolling, so the choice costs nothing).
#ifndef HX_POLY_EVERY
#define HX_POLY_EVERY 16
#endif
HX_DEVICE float exp2_mixed(float x, int k) {
  if constexpr (HX_POLY_EVERY > 0) {
    constexpr int every = HX_POLY_EVERY > 0 ? HX_POLY_EVERY : 1;
    if (k % every == every - 1) return exp2_poly(x);
  }
  return fast_exp2(x);
}

// (packed two-wide fp32 helpers f2pack / ffma2 / fadd2 / fmul2: hx_common.cuh)
HX_DEVICE float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// bf16x2 of exp2 of a packed pair
HX_DEVICE uint32_t exp2_pack(uint64_t x2, float& s0, float& s1) {
  const float2 x = f2unpack(x2);
  s0 = fast_exp2(x.x);
  s1 = fast_exp2(x.y);
  return pack_bf16(s0, s1);
}

// exp2 of a packed pair on the FMA pipe (no MUFU): n = round(x) via the 1.5*2^23
// magic add, f = x - n in [-0.5, 0.5], 2^f by a degree-3 relative-minimax
// polynomial (max rel. error 7.5e-5, far below bf16's 2^-9 rounding of P), 2^n
// added to the exponent field.  x <= 0 (softmax arguments); clamped at -125 so
// the exponent sum never wraps (2^f can sit just below 1 with n = -125).
HX_DEVICE uint32_t exp2_pack_poly(uint64_t x2, float& s0, float& s1) {
  const float2 xu = f2unpack(x2);
  const uint64_t x = f2pack(fmaxf(xu.x, -125.f), fmaxf(xu.y, -125.f));
  constexpr float MAGIC = 12582912.f;
  const uint64_t j = fadd2(x, f2pack(MAGIC, MAGIC));
  // f = x - n with n = j - MAGIC (exact): one FADD2 + one FFMA2 (was two FADD2 and
  // two LOP3 sign flips)
  const uint64_t f = ffma2(fadd2(j, f2pack(-MAGIC, -MAGIC)), f2pack(-1.f, -1.f), x);
  uint64_t q = ffma2(f, f2pack(0.0551716536f, 0.0551716536f), f2pack(0.242611155f, 0.242611155f));
  q = ffma2(f, q, f2pack(0.693260968f, 0.693260968f));
  q = ffma2(f, q, f2pack(0.999928057f, 0.999928057f));
  const float2 qf = f2unpack(q), jf = f2unpack(j);
  s0 = __int_as_float(__float_as_int(qf.x) + (__float_as_int(jf.x) << 23));
  s1 = __int_as_float(__float_as_int(qf.y) + (__float_as_int(jf.y) << 23));
  return pack_bf16(s0, s1);
}

// Pair i of an unrolled softmax row: every HX_POLY_EVERY-th pair on the FMA pipe.
// (i is a compile-time constant after unrolling, so the choice costs nothing.)
HX_DEVICE uint32_t exp2_pack_mixed(uint64_t x2, int i, float& s0, float& s1) {
#ifdef HX_FWD_NOEXP  // debug-only probe: no exponentials at all (results wrong)
  {
    const float2 xu = f2unpack(x2);
    s0 = xu.x * 0.5f;
    s1 = xu.y * 0.5f;
    return pack_bf16(s0, s1);
  }
#endif
  if constexpr (HX_POLY_EVERY > 0) {
    constexpr int every = HX_POLY_EVERY > 0 ? HX_POLY_EVERY : 1;
    if (i % every == every - 1) return exp2_pack_poly(x2, s0, s1);
  }
  return exp2_pack(x2, s0, s1);
}

HX_DEVICE void named_barrier_sync(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

HX_DEVICE uint4 bf16x8(const float* f) {
  return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}

// Copy NB bf16 values of one global row into packed TMEM columns (NB/2 of them).
template <int NB>
HX_DEVICE void row_to_tmem(uint32_t taddr, const __nv_bfloat16* src, bool valid) {
  static_assert(NB == 16 || NB == 32 || NB == 64, "row chunk");
  uint32_t w[NB / 2];
#pragma unroll
  for (int v = 0; v < NB / 8; ++v) {
    const uint4 a = valid ? reinterpret_cast<const uint4*>(src)[v] : make_uint4(0, 0, 0, 0);
    w[4 * v] = a.x; w[4 * v + 1] = a.y; w[4 * v + 2] = a.z; w[4 * v + 3] = a.w;
  }
  if constexpr (NB == 64) {
    tmem_st32(taddr, w);
  } else if constexpr (NB == 32) {
    tmem_st16(taddr, w);
  } else {
    tmem_st8(taddr, w);
  }
}

// Read NC fp32 accumulator columns of this thread's row, scale, store bf16 to global.
template <int NC>
HX_DEVICE void tmem_row_to_global(uint32_t taddr, __nv_bfloat16* dst, float scale, bool valid) {
  static_assert(NC == 16 || NC == 32, "row chunk");
  uint32_t r[NC];
  if constexpr (NC == 32) tmem_ld32(taddr, r);
  else tmem_ld16(taddr, r);
  tmem_wait_ld();
  if (!valid) return;
#pragma unroll
  for (int v = 0; v < NC / 8; ++v) {
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[v * 8 + i]) * scale;
    reinterpret_cast<uint4*>(dst)[v] = bf16x8(f);
  }
}

}  // namespace hx
