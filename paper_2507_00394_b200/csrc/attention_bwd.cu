// Causal flash attention backward on tcgen05 / TMEM / TMA (sm_100a).
// Replaces P/runtime/mathops.py:103-116:
//   dV = P^T dO, dP = dO V^T, dS = P (dP - D), dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d)
// with D = rowsum(dO * O) (pre-pass) and P rebuilt from the forward's LSE.
//
// Default (v10): one fused pass per 128-row key tile, dK / dV resident in TMEM,
// dQ partials reduced into an fp32 accumulator by TMA bulk reduce-adds (see the
// "fused (v10)" section).  HX_ATTN_BWD=9 selects the deterministic, atomic-free
// split kernels (v9: a dK/dV kernel per key tile and a dQ kernel per query tile).
#include "attention_common.cuh"

namespace hx {

// Packed TMEM A-operand address of K-step kk when warpgroup g owns columns
// [CW*g, CW*g+CW) of a 64-wide tile and packs them at region + CW*g.
template <int CW>
HX_DEVICE uint32_t packed_kstep(uint32_t region, int kk) {
  return region + CW * ((16 * kk) / CW) + ((16 * kk) % CW) / 2;
}

// dK / dV epilogue / dQ epilogue: columns [g*D/NWG, (g+1)*D/NWG) of one row.
template <int D, int NWG>
HX_DEVICE void acc_row_out(uint32_t tacc, int g, __nv_bfloat16* dst, float scale, bool valid) {
  constexpr int W = D / NWG;
  constexpr int NC = W < 32 ? W : 32;
#pragma unroll
  for (int ch = 0; ch < W / NC; ++ch)
    tmem_row_to_global<NC>(tacc + g * W + ch * NC, dst + g * W + ch * NC, scale, valid);
}

// =====================================================================================
// v9: 128-wide streamed tiles (every MMA at N >= 128, the full-rate shapes on B200:
// a measured 64 cycles per 128x128x16 MMA, vs 45-48 for 128x64x16 instead of 32)
// =====================================================================================
//
// dK/dV: CTA = 128-row key tile; streams 128-row query tiles.
//   S^T(i) = K Q^T  SS -> 256 | dP^T(i) = V dO^T  SS -> 384 |
//   [P^T packed over S^T] dV += P^T dO  TS | [dS^T packed over dP^T] dK += dS^T Q  TS
//   The softmax of tile i overlaps dP^T(i); dS^T overlaps dV.
//   TMEM: dK 0 | dV 128 | S^T 256 | dP^T 384.   smem: K, V + Q/dO x 2 stages.
// dQ: CTA = 128-row query tile; streams 128-row key tiles.
//   S(j) = Q K^T TS -> 0 | dP(j) = dO V^T TS -> 128 | [dS packed over dP] dQ += dS K TS
//   S(j+1) is issued as soon as the softmax has read S(j), so it runs under dS(j).
//   TMEM: S 0 | dP 128 | dQ 256 | Q 384 | dO 384+D/2.   smem: K/V x 3 stages.

template <int D>
struct KV9Smem {
  static constexpr int STAGES = 2;
  static constexpr int K = 0;
  static constexpr int V = K + Tile<D>::BYTES;
  static constexpr int Q = V + Tile<D>::BYTES;              // STAGES x [128 x D]
  static constexpr int DO = Q + STAGES * Tile<D>::BYTES;    // STAGES x [128 x D]
  static constexpr int STAT = DO + STAGES * Tile<D>::BYTES;  // [2][lse2 | delta][128]
  static constexpr int BAR = STAT + 2 * 2 * AT_TILE * 4;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_dkdv9_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                          const AttnParams p) {
  using L = KV9Smem<D>;
  constexpr int ST = L::STAGES;
  constexpr int NT = 256;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* qdo_full = bars;              // ST
  uint64_t* qdo_empty = bars + ST;        // ST
  uint64_t* kv_full = bars + 2 * ST;
  uint64_t* s_full = bars + 2 * ST + 1;
  uint64_t* dp_full = bars + 2 * ST + 2;
  uint64_t* p_full = bars + 2 * ST + 3;   // NT arrivals
  uint64_t* ds_full = bars + 2 * ST + 4;  // NT arrivals
  uint64_t* acc_full = bars + 2 * ST + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 6);
  constexpr int NBARS = 2 * ST + 6;
  float* stat = reinterpret_cast<float*>(smem + L::STAT);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int kt = static_cast<int>(blockIdx.x);  // heaviest key tiles first
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;
  const int n_it = nq - kt;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    for (int i = 0; i < NBARS; ++i) mbar_init(&bars[i], (i == 2 * ST + 3 || i == 2 * ST + 4) ? NT : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDK = tmem, tDV = tmem + 128, tS = tmem + 256, tDP = tmem + 384;

  if (warp == 8) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * Tile<D>::BYTES);
      tma_tile_rows<D>(smem + L::K, &tm_qkv, kv_full, kcol, bi, kt * AT_TILE, AT_TILE);
      tma_tile_rows<D>(smem + L::V, &tm_qkv, kv_full, vcol, bi, kt * AT_TILE, AT_TILE);
      for (int it = 0; it < n_it; ++it) {
        const int st = it % ST, q0 = (kt + it) * AT_TILE;
        mbar_wait(&qdo_empty[st], ((it / ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&qdo_full[st], 2 * Tile<D>::BYTES);
        tma_tile_rows<D>(smem + L::Q + st * Tile<D>::BYTES, &tm_qkv, &qdo_full[st], qcol, bi, q0, AT_TILE);
        tma_tile_rows<D>(smem + L::DO + st * Tile<D>::BYTES, &tm_do, &qdo_full[st], head * D, bi, q0, AT_TILE);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_sp = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_kv = idesc_bf16(128, D, false, true);
      const uint32_t sk = smem_u32(smem + L::K), sv = smem_u32(smem + L::V);
      auto sq = [&](int it) { return smem_u32(smem + L::Q + (it % ST) * Tile<D>::BYTES); };
      auto sdo = [&](int it) { return smem_u32(smem + L::DO + (it % ST) * Tile<D>::BYTES); };
      auto issue_s = [&](int it) {  // S^T(it): the S region is free once dV(it-1) was issued
        mbar_wait(&qdo_full[it % ST], (it / ST) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tS, kdesc(sk, kk, AT_TILE), kdesc(sq(it), kk, AT_TILE), id_sp, kk > 0);
        umma_commit(s_full);
      };
      auto issue_dp = [&](int it) {  // dP^T(it): the dP region is free once dK(it-1) was issued
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tDP, kdesc(sv, kk, AT_TILE), kdesc(sdo(it), kk, AT_TILE), id_sp, kk > 0);
        umma_commit(dp_full);
      };
      mbar_wait(kv_full, 0);
      issue_s(0);
      issue_dp(0);
      // Stream: dV(i) | S^T(i+1) | dK(i) | dP^T(i+1).  S^T(i+1) only waits for P^T(i)
      // (consumed by dV(i)), so the next softmax starts while dK(i) and dP^T(i+1) run.
      for (int it = 0; it < n_it; ++it) {
        mbar_wait(p_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts(tDV, packed_kstep<64>(tS, kk), mndesc(sdo(it), kk, AT_TILE), id_kv, it > 0 || kk > 0);
        if (it + 1 < n_it) issue_s(it + 1);
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts(tDK, packed_kstep<64>(tDP, kk), mndesc(sq(it), kk, AT_TILE), id_kv, it > 0 || kk > 0);
        umma_commit(&qdo_empty[it % ST]);
        if (it + 1 < n_it) issue_dp(it + 1);
      }
      umma_commit(acc_full);
    }
  } else {
    // compute: thread = key row c, query columns [64g, 64g + 64)
    const int g = warp >> 2, quad = warp & 3;
    const int c = quad * 32 + lane;
    const int qoff = 64 * g;
    const int ct = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row_base = static_cast<int64_t>(bh) * p.s;
    const int kv_row = kt * AT_TILE + c;
    float nxt = 0.f;
    auto fetch = [&](int it) {  // thread ct < 128: lse2 of query ct, else delta of query ct-128
      const int qi = ct & (AT_TILE - 1), q = (kt + it) * AT_TILE + qi;
      nxt = q >= p.s ? 0.f : (ct < AT_TILE ? p.lse[row_base + q] * LOG2E : p.delta[row_base + q]);
    };
    fetch(0);
    for (int it = 0; it < n_it; ++it) {
      const int q0 = (kt + it) * AT_TILE;
      float* s_lse = stat + (it & 1) * 2 * AT_TILE;
      float* s_del = s_lse + AT_TILE;
      (ct < AT_TILE ? s_lse : s_del)[ct & (AT_TILE - 1)] = nxt;
      named_barrier_sync(1, NT);
      if (it + 1 < n_it) fetch(it + 1);
      const bool need_mask = it == 0 || q0 + AT_TILE > p.s;
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      uint32_t raw[64];
      tmem_ld32(tS + lane_off + qoff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tS + lane_off + qoff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      float pv[64];
#pragma unroll
      for (int v = 0; v < 16; ++v) {
        const float4 l4 = reinterpret_cast<const float4*>(s_lse + qoff)[v];
        pv[4 * v] = exp2_mixed(fmaf(__uint_as_float(raw[4 * v]), p.scale_log2, -l4.x), 0);
        pv[4 * v + 1] = exp2_mixed(fmaf(__uint_as_float(raw[4 * v + 1]), p.scale_log2, -l4.y), 1);
        pv[4 * v + 2] = exp2_mixed(fmaf(__uint_as_float(raw[4 * v + 2]), p.scale_log2, -l4.z), 2);
        pv[4 * v + 3] = exp2_mixed(fmaf(__uint_as_float(raw[4 * v + 3]), p.scale_log2, -l4.w), 3);
      }
      if (need_mask) {  // diagonal tile (query < key) and the sequence tail
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (q0 + qoff + j < kv_row || q0 + qoff + j >= p.s) pv[j] = 0.f;
      }
      {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) pk[j] = pack_bf16(pv[2 * j], pv[2 * j + 1]);
        tmem_st32(tS + lane_off + qoff, pk);  // P^T over this warpgroup's S^T columns
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
      mbar_wait(dp_full, it & 1);
      tc_fence_after();
      tmem_ld32(tDP + lane_off + qoff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tDP + lane_off + qoff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      {
        uint32_t pk[32];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float4 d4 = reinterpret_cast<const float4*>(s_del + qoff)[v];
          pk[2 * v] = pack_bf16(pv[4 * v] * (__uint_as_float(raw[4 * v]) - d4.x),
                                pv[4 * v + 1] * (__uint_as_float(raw[4 * v + 1]) - d4.y));
          pk[2 * v + 1] = pack_bf16(pv[4 * v + 2] * (__uint_as_float(raw[4 * v + 2]) - d4.z),
                                    pv[4 * v + 3] * (__uint_as_float(raw[4 * v + 3]) - d4.w));
        }
        tmem_st32(tDP + lane_off + qoff, pk);  // dS^T over this warpgroup's dP^T columns
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int64_t kv_tok = static_cast<int64_t>(kv_row) * p.b + bi;
    __nv_bfloat16* dst = p.dqkv + kv_tok * p.ld_dqkv + head * D;
    acc_row_out<D, 2>(tDK + lane_off, g, dst + p.h, p.scale, kv_row < p.s);
    acc_row_out<D, 2>(tDV + lane_off, g, dst + 2 * p.h, 1.f, kv_row < p.s);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
struct Q9Smem {
  static constexpr int STAGES = 3;
  static constexpr int KV = 0;  // STAGES x (K, V) [128 x D]
  static constexpr int BAR = KV + STAGES * 2 * Tile<D>::BYTES;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_dq9_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __nv_bfloat16* __restrict__ qkv, int ld_qkv,
                        const __nv_bfloat16* __restrict__ d_o, int ld_o, const AttnParams p) {
  using L = Q9Smem<D>;
  constexpr int ST = L::STAGES;
  constexpr int NT = 256;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* kv_full = bars;                 // ST
  uint64_t* kv_empty = bars + ST;           // ST
  uint64_t* s_full = bars + 2 * ST;
  uint64_t* s_free = bars + 2 * ST + 1;     // NT arrivals
  uint64_t* dp_full = bars + 2 * ST + 2;
  uint64_t* ds_full = bars + 2 * ST + 3;    // NT arrivals
  uint64_t* qdo_ready = bars + 2 * ST + 4;  // NT arrivals
  uint64_t* dq_done = bars + 2 * ST + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 6);
  constexpr int NBARS = 2 * ST + 6;

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int qt = nq - 1 - static_cast<int>(blockIdx.x);  // heaviest query tiles first
  const int nkv = qt + 1;
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    for (int i = 0; i < NBARS; ++i)
      mbar_init(&bars[i], (i == 2 * ST + 1 || i == 2 * ST + 3 || i == 2 * ST + 4) ? NT : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tDP = tmem + 128, tDQ = tmem + 256, tQ = tmem + 384, tDO = tmem + 384 + D / 2;

  if (warp == 8) {
    if (lane == 0) {
      for (int j = 0; j < nkv; ++j) {
        const int st = j % ST;
        mbar_wait(&kv_empty[st], ((j / ST) & 1) ^ 1);
        uint8_t* kb = smem + L::KV + st * 2 * Tile<D>::BYTES;
        mbar_arrive_expect_tx(&kv_full[st], 2 * Tile<D>::BYTES);
        tma_tile_rows<D>(kb, &tm_qkv, &kv_full[st], kcol, bi, j * AT_TILE, AT_TILE);
        tma_tile_rows<D>(kb + Tile<D>::BYTES, &tm_qkv, &kv_full[st], vcol, bi, j * AT_TILE, AT_TILE);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_sp = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_q = idesc_bf16(128, D, false, true);
      auto skv = [&](int j) { return smem_u32(smem + L::KV + (j % ST) * 2 * Tile<D>::BYTES); };
      auto issue_s = [&](int j) {
        mbar_wait(&kv_full[j % ST], (j / ST) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) umma_f16_ts(tS, tQ + kk * 8, kdesc(skv(j), kk, AT_TILE), id_sp, kk > 0);
        umma_commit(s_full);
      };
      auto issue_dp = [&](int j) {
        const uint32_t sv = skv(j) + Tile<D>::BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) umma_f16_ts(tDP, tDO + kk * 8, kdesc(sv, kk, AT_TILE), id_sp, kk > 0);
        umma_commit(dp_full);
      };
      mbar_wait(qdo_ready, 0);
      tc_fence_after();
      issue_s(0);
      issue_dp(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) {
          mbar_wait(s_free, j & 1);  // the softmax has read S(j)
          issue_s(j + 1);
        }
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts(tDQ, packed_kstep<64>(tDP, kk), mndesc(skv(j), kk, AT_TILE), id_q, j > 0 || kk > 0);
        umma_commit(&kv_empty[j % ST]);
        if (j + 1 < nkv) issue_dp(j + 1);
      }
      umma_commit(dq_done);
    }
  } else {
    // compute: thread = query row r, key columns [64g, 64g + 64)
    const int g = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const int koff = 64 * g;
    const int q = qt * AT_TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t tok = static_cast<int64_t>(q) * p.b + bi;
    row_to_tmem<D / 2>(tQ + lane_off + g * (D / 4), qkv + tok * ld_qkv + head * D + g * (D / 2), q < p.s);
    row_to_tmem<D / 2>(tDO + lane_off + g * (D / 4), d_o + tok * ld_o + head * D + g * (D / 2), q < p.s);
    tmem_wait_st();
    tc_fence_before();
    mbar_arrive(qdo_ready);
    const int64_t row = static_cast<int64_t>(bh) * p.s + q;
    const float lse2 = q < p.s ? p.lse[row] * LOG2E : 0.f;
    const float dlt = q < p.s ? p.delta[row] : 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      uint32_t raw[64];
      tmem_ld32(tS + lane_off + koff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tS + lane_off + koff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_free);
      float pv[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) pv[i] = exp2_mixed(fmaf(__uint_as_float(raw[i]), p.scale_log2, -lse2), i);
      if (j == qt) {  // diagonal tile
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (koff + i > r) pv[i] = 0.f;
      }
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
      tmem_ld32(tDP + lane_off + koff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tDP + lane_off + koff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        pk[i] = pack_bf16(pv[2 * i] * (__uint_as_float(raw[2 * i]) - dlt),
                          pv[2 * i + 1] * (__uint_as_float(raw[2 * i + 1]) - dlt));
      tmem_st32(tDP + lane_off + koff, pk);  // dS over this warpgroup's dP columns
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    acc_row_out<D, 2>(tDQ + lane_off, g, p.dqkv + tok * p.ld_dqkv + head * D, p.scale, q < p.s);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ fused (v10)
// One pass, CTA = one 128-row key tile of one (batch, head); streams 128-row
// query tiles i from the diagonal to the end.  dK and dV stay in TMEM for the
// CTA's lifetime; the partial dQ(i) = dS(i) K of every tile is reduced into an
// fp32 accumulator in global memory by TMA bulk reduce-adds (L2 does the adds),
// so the score / dP matmuls and the exponentials are done once (5 MMAs per tile
// pair instead of the split kernels' 7).  MMA stream per tile:
//   dV(i) += P^T dO | dP^T(i) = V dO^T | S^T(i+1) = K Q^T | dK += dS^T Q | dQ(i) = dS K
//   (P^T written over S^T, dS^T over dP^T in TMEM; dS also to smem as dQ's A operand.)
// TMEM (D=128): dK 0 | dV 128 | S^T 256 | dP^T 384, dQ(i) over dP^T once dK(i)
//   has read dS^T (the tensor pipe runs in issue order); the reduce warpgroup
//   drains dQ(i) while dV(i+1) runs.  D=64: dQ gets its own columns at 384.
// Warps: 0-7 compute (thread = key row, warpgroup g owns query columns 64g..),
//   8 TMA, 9 MMA, 10-11 idle, 12-15 dQ reduce (thread = query row).
// Debug-only ablations for pipeline analysis (tools/bwd_trace.py): skip the
// softmax math (NOCOMPUTE) or the dQ staging / reduce-add (NOREDUCE).
#ifdef HX_BWD_NOCOMPUTE
constexpr bool kNoCompute = true;
#else
constexpr bool kNoCompute = false;
#endif
#ifdef HX_BWD_NOREDUCE
constexpr bool kNoReduce = true;
#else
constexpr bool kNoReduce = false;
#endif

#ifdef HX_BWD_TRACE
// Debug build only: clock64 per event and iteration for CTA (0, 0) (the key tile
// with the most query tiles), read back with hx_debug_bwd_trace (tools/bwd_trace.py).
__device__ long long g_bwd_trace[16][512];
#define HX_BT(slot, idx) \
  if (blockIdx.x == 0 && (idx) < 512) g_bwd_trace[slot][idx] = clock64()
#else
#define HX_BT(slot, idx)
#endif

template <int D>
struct FusedSmem {
  static constexpr int K = 0;
  static constexpr int V = K + Tile<D>::BYTES;
  static constexpr int Q = V + Tile<D>::BYTES;               // 2 x [128 x D]
  static constexpr int DO = Q + 2 * Tile<D>::BYTES;          // [128 x D]
  static constexpr int DS = DO + Tile<D>::BYTES;             // [128 keys x 128 q], MN-major A of dQ
  static constexpr int STG = DS + AT_TILE * AT_TILE * 2;     // 2 x [128 x 32] fp32 reduce staging
  static constexpr int STAT = STG + 2 * AT_TILE * 32 * 4;    // [2][-lse2 | -delta][128]
  static constexpr int BAR = STAT + 2 * 2 * AT_TILE * 4;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(512, 1)
    attn_bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_dq, const AttnParams p) {
  using L = FusedSmem<D>;
  constexpr int NT = 256;  // compute threads
  constexpr bool DQ_SHARES_DP = 2 * D + 256 + D > 512;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;        // 2
  uint64_t* q_empty = bars + 2;   // 2
  uint64_t* kv_full = bars + 4;
  uint64_t* do_full = bars + 5;
  uint64_t* do_empty = bars + 6;
  uint64_t* s_full = bars + 7;
  uint64_t* p_full = bars + 8;    // NT arrivals
  uint64_t* dp_full = bars + 9;
  uint64_t* ds_full = bars + 10;  // NT arrivals
  uint64_t* dq_full = bars + 11;
  uint64_t* dq_empty = bars + 12; // 128 arrivals
  uint64_t* acc_full = bars + 13;
  [[maybe_unused]] uint64_t* dv_done = bars + 14;  // trace builds only: completion of dV / dK groups
  [[maybe_unused]] uint64_t* dk_done = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  constexpr int NBARS = 16;
  float* stat = reinterpret_cast<float*>(smem + L::STAT);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  // 1-D grid in bands of p.band (batch, head)s, key-tile-major inside a band:
  // heaviest key tiles first (attention_common.cuh band_order)
  int bh, kt;
  band_order(static_cast<int>(blockIdx.x), nq, p.b * p.heads, p.band, bh, kt);
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;
  const int n_it = nq - kt;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    for (int i = 0; i < NBARS; ++i) mbar_init(&bars[i], (i == 8 || i == 10) ? NT : (i == 12 ? 128 : 1));
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDK = tmem, tDV = tmem + D, tS = tmem + 2 * D, tDP = tmem + 2 * D + 128;
  const uint32_t tDQ = DQ_SHARES_DP ? tDP : tmem + 2 * D + 256;

  // Each role ends the kernel itself (no code shared after the role branches,
  // so ptxas can allocate each branch under its own setmaxnreg budget).
  auto finish = [&]() {
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
      tc_fence_after();
      tmem_dealloc(tmem, 512);
    }
  };
  if (warp >= 8 && warp < 12) {
    regs_dec<120>();
    if (warp == 8 && lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * Tile<D>::BYTES);
      tma_tile_rows<D>(smem + L::K, &tm_qkv, kv_full, kcol, bi, kt * AT_TILE, AT_TILE);
      tma_tile_rows<D>(smem + L::V, &tm_qkv, kv_full, vcol, bi, kt * AT_TILE, AT_TILE);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1, q0 = (kt + it) * AT_TILE;
        mbar_wait(&q_empty[st], ((it >> 1) & 1) ^ 1);
#ifdef HX_BWD_NOQDO  // debug-only probe: no Q / dO traffic after the first two tiles (wrong results)
        if (it >= 2) {
          mbar_arrive(&q_full[st]);
          mbar_wait(do_empty, (it & 1) ^ 1);
          mbar_arrive(do_full);
          continue;
        }
#endif
        mbar_arrive_expect_tx(&q_full[st], Tile<D>::BYTES);
        tma_tile_rows<D>(smem + L::Q + st * Tile<D>::BYTES, &tm_qkv, &q_full[st], qcol, bi, q0, AT_TILE);
        mbar_wait(do_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(do_full, Tile<D>::BYTES);
        tma_tile_rows<D>(smem + L::DO, &tm_do, do_full, head * D, bi, q0, AT_TILE);
      }
    }
#ifdef HX_BWD_TRACE
    else if (warp == 10 && lane == 0) {  // observer: completion time of every MMA group
      for (int it = 0; it < n_it; ++it) {
        mbar_wait(dp_full, it & 1);
        HX_BT(16, it);
        mbar_wait(dv_done, it & 1);
        HX_BT(17, it);
        if (it + 1 < n_it) {
          mbar_wait(s_full, (it + 1) & 1);
          HX_BT(18, it);
        }
        mbar_wait(dk_done, it & 1);
        HX_BT(19, it);
        mbar_wait(dq_full, it & 1);
        HX_BT(20, it);
      }
    }
#endif
    else if (warp == 9) {
      // The whole warp runs the issue loop (warp-uniform descriptors on the uniform
      // datapath); one elected lane issues each tcgen05 instruction.  Fully unrolled
      // chains: the tensor pipe's queue is shallow, so per-MMA issue cost must stay
      // well below the 64-cycle MMA time.
      constexpr uint32_t id_s = idesc_bf16(128, 128, false, false);  // S^T, dP^T: K-major x K-major
      constexpr uint32_t id_kv = idesc_bf16(128, D, false, true);    // dV, dK: TMEM A x MN-major B
      constexpr uint32_t id_dq = idesc_bf16(128, D, true, true);     // dQ: MN-major dS x MN-major K
      const uint32_t sk = smem_u32(smem + L::K), sv = smem_u32(smem + L::V);
      const uint32_t sdo = smem_u32(smem + L::DO), sds = smem_u32(smem + L::DS);
      auto sq = [&](int it) { return smem_u32(smem + L::Q + (it & 1) * Tile<D>::BYTES); };
      auto mma_kk = [&](uint32_t d, uint32_t a_smem, uint32_t b_smem, uint32_t id) {
        // K-major x K-major over K = D: per 64-column atom, four 16-wide steps (+32 B)
        const uint64_t da = sw128_desc(a_smem, 16, 1024), db = sw128_desc(b_smem, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * AT_TILE * 128 + (kk & 3) * 32) >> 4;
          umma_f16_ss_e(d, da + off, db + off, id, kk > 0);
        }
      };
      auto mma_ts_mn = [&](uint32_t d, uint32_t a_tmem, uint32_t b_smem, uint32_t id, bool acc) {
        // TMEM A (packed, 64-column groups) x MN-major B over K = 128 rows (+2048 B per step)
        const uint64_t db = sw128_desc(b_smem, AT_TILE * 128, 1024);
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts_e(d, a_tmem + 64 * (kk >> 2) + 8 * (kk & 3), db + 128 * kk, id, acc || kk > 0);
      };
      auto issue_s = [&](int it) {
        mbar_wait(&q_full[it & 1], (it >> 1) & 1);
        tc_fence_after();
        mma_kk(tS, sk, sq(it), id_s);
        umma_commit_e(s_full);
      };
      auto issue_dp = [&]() {
        mma_kk(tDP, sv, sdo, id_s);
        umma_commit_e(dp_full);
      };
      // Stream per tile: dP^T(i) was issued at the end of tile i-1 (as soon as dQ(i-1)
      // left the shared TMEM columns), so it runs while the softmax builds P^T(i):
      //   dV(i) | S^T(i+1) | dK(i) | dQ(i) | dP^T(i+1)
      mbar_wait(kv_full, 0);
      issue_s(0);
      mbar_wait(do_full, 0);
      tc_fence_after();
      issue_dp();
      const uint64_t dq_a = sw128_desc(sds, AT_TILE * 128, 1024), dq_b = sw128_desc(sk, AT_TILE * 128, 1024);
      for (int it = 0; it < n_it; ++it) {
        mbar_wait(p_full, it & 1);
        tc_fence_after();
        HX_BT(0, it);
        mma_ts_mn(tDV, tS, sdo, id_kv, it > 0);
#ifdef HX_BWD_TRACE
        umma_commit_e(dv_done);
#endif
        umma_commit_e(do_empty);  // dO(it) read by dP^T(it) and dV(it)
        if (it + 1 < n_it) issue_s(it + 1);
        HX_BT(2, it);
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
        HX_BT(3, it);
        mma_ts_mn(tDK, tDP, sq(it), id_kv, it > 0);
#ifdef HX_BWD_TRACE
        umma_commit_e(dk_done);
#endif
        umma_commit_e(&q_empty[it & 1]);
        if (!DQ_SHARES_DP && it > 0) {
          mbar_wait(dq_empty, (it - 1) & 1);
          tc_fence_after();
        }
        HX_BT(4, it);
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk) umma_f16_ss_e(tDQ, dq_a + 128 * kk, dq_b + 128 * kk, id_dq, kk > 0);
        umma_commit_e(dq_full);
        if (it + 1 < n_it) {
          mbar_wait(do_full, (it + 1) & 1);
          if (DQ_SHARES_DP) mbar_wait(dq_empty, it & 1);  // dQ(it) drained from the dP columns
          tc_fence_after();
          HX_BT(1, it + 1);
          issue_dp();
        }
      }
      umma_commit_e(acc_full);
    }
    finish();
    return;
  } else if (warp >= 12) {
    // dQ reduce: thread = query row r of the current tile; TMEM -> registers ->
    // swizzled smem staging -> TMA reduce-add into the fp32 accumulator.
    regs_inc<136>();
    const int quad = warp & 3, r = quad * 32 + lane, rt = threadIdx.x - 384;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    uint8_t* stg = smem + L::STG;
    int k = 0;
    for (int it = 0; it < n_it; ++it) {
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      if (rt == 0) HX_BT(9, it);
      uint32_t v[D];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) tmem_ld32(tDQ + lane_off + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(dq_empty);
      if (rt == 0) HX_BT(10, it);
      const int q0 = (kt + it) * AT_TILE;
      if (kNoReduce) continue;
#pragma unroll
      for (int c = 0; c < D / 32; ++c, ++k) {
        uint8_t* buf = stg + (k & 1) * (AT_TILE * 128);
        if (rt == 0) bulk_wait_read<1>();
        named_barrier_sync(2, 128);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(buf + r * 128 + ((j ^ (r & 7)) << 4)) =
              make_uint4(v[32 * c + 4 * j], v[32 * c + 4 * j + 1], v[32 * c + 4 * j + 2], v[32 * c + 4 * j + 3]);
        fence_proxy_async();
        named_barrier_sync(2, 128);
        if (rt == 0) {
          tma_reduce_add_3d(&tm_dq, buf, 32 * c, q0, bh);
          bulk_commit();
        }
      }
      if (rt == 0) HX_BT(11, it);
    }
    if (rt == 0) bulk_wait_all();
    finish();
    return;
  } else {
    // compute: thread = key row c, query columns [64g, 64g + 64)
    // (compute warpgroups keep the launch budget of 128 registers)
    const int g = warp >> 2, quad = warp & 3;
    const int c = quad * 32 + lane;
    const int qoff = 64 * g;
    const int ct = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row_base = static_cast<int64_t>(bh) * p.s;
    const int kv_row = kt * AT_TILE + c;
    uint8_t* sds_row = smem + L::DS + g * (AT_TILE * 128) + c * 128;
    const uint64_t scale2 = f2pack(p.scale_log2, p.scale_log2);
    // Statistics of the next query tile: thread ct < 128 loads lse of query ct, the
    // others delta of query ct-128.  The raw value is only consumed (scaled, negated,
    // stored to smem) one iteration later, so the global-load latency is hidden.
    const float* stat_src = (ct < AT_TILE ? p.lse : p.delta) + row_base + (ct & (AT_TILE - 1));
    const float stat_mul = ct < AT_TILE ? -LOG2E : -1.f;
    float nxt = 0.f;
    auto fetch = [&](int it) {
      const int q = (kt + it) * AT_TILE + (ct & (AT_TILE - 1));
      nxt = q < p.s ? __ldg(stat_src + (kt + it) * AT_TILE) : 0.f;
    };
    fetch(0);
    for (int it = 0; it < n_it; ++it) {
      const int q0 = (kt + it) * AT_TILE;
      float* s_nl = stat + (it & 1) * 2 * AT_TILE;
      float* s_nd = s_nl + AT_TILE;
      (ct < AT_TILE ? s_nl : s_nd)[ct & (AT_TILE - 1)] = nxt * stat_mul;
      named_barrier_sync(1, NT);
      if (ct == 0) HX_BT(12, it);
      if (it + 1 < n_it) fetch(it + 1);
      const bool need_mask = it == 0 || q0 + AT_TILE > p.s;
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      if (ct == 0) HX_BT(5, it);
      if (ct == 224) HX_BT(14, it);
      uint32_t raw[32];
      if (kNoCompute) {
        tc_fence_before();
        mbar_arrive(p_full);
        mbar_wait(dp_full, it & 1);
        tc_fence_before();
        mbar_arrive(ds_full);
        continue;
      }
      // Both phases run in 32-column halves (TMEM -> registers -> TMEM), so only
      // P (64 fp32) stays live across the phases: no register spills at 136.
      float pv[64];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        tmem_ld32(tS + lane_off + qoff + 32 * hh, *reinterpret_cast<uint32_t(*)[32]>(raw));
        tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float2 l2 = reinterpret_cast<const float2*>(s_nl + qoff + 32 * hh)[v];
          const float2 x = f2unpack(ffma2(f2pack(__uint_as_float(raw[2 * v]), __uint_as_float(raw[2 * v + 1])),
                                          scale2, f2pack(l2.x, l2.y)));
          pv[32 * hh + 2 * v] = fast_exp2(x.x);
          pv[32 * hh + 2 * v + 1] = fast_exp2(x.y);
        }
        if (need_mask) {  // diagonal tile (query < key) and the sequence tail
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int q = q0 + qoff + 32 * hh + j;
            if (q < kv_row || q >= p.s) pv[32 * hh + j] = 0.f;
          }
        }
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(pv[32 * hh + 2 * j], pv[32 * hh + 2 * j + 1]);
        tmem_st16(tS + lane_off + qoff + 16 * hh, pk);  // P^T over S^T columns already read
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
      if (ct == 0) HX_BT(6, it);
      mbar_wait(dp_full, it & 1);
      tc_fence_after();
      if (ct == 0) HX_BT(7, it);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        tmem_ld32(tDP + lane_off + qoff + 32 * hh, *reinterpret_cast<uint32_t(*)[32]>(raw));
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float2 d2 = reinterpret_cast<const float2*>(s_nd + qoff + 32 * hh)[v];
          const float2 ds = f2unpack(fmul2(fadd2(f2pack(__uint_as_float(raw[2 * v]), __uint_as_float(raw[2 * v + 1])),
                                                 f2pack(d2.x, d2.y)),
                                           f2pack(pv[32 * hh + 2 * v], pv[32 * hh + 2 * v + 1])));
          pk[v] = pack_bf16(ds.x, ds.y);
        }
        tmem_st16(tDP + lane_off + qoff + 16 * hh, pk);  // dS^T over dP^T columns already read
#pragma unroll
        for (int j = 0; j < 4; ++j)  // dS^T row c, query columns 64g + 32hh + 8j.. (SW128 atom g)
          *reinterpret_cast<uint4*>(sds_row + (((4 * hh + j) ^ (c & 7)) << 4)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      }
      fence_proxy_async();
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full);
      if (ct == 0) HX_BT(8, it);
      if (ct == 224) HX_BT(13, it);
      if (ct == 224) HX_BT(13, it);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int64_t kv_tok = static_cast<int64_t>(kv_row) * p.b + bi;
    __nv_bfloat16* dst = p.dqkv + kv_tok * p.ld_dqkv + head * D;
    acc_row_out<D, 2>(tDK + lane_off, g, dst + p.h, p.scale, kv_row < p.s);
    acc_row_out<D, 2>(tDV + lane_off, g, dst + 2 * p.h, 1.f, kv_row < p.s);
    finish();
  }
}

// dq (bf16, into dqkv's q columns) = scale * fp32 accumulator [b*heads][s][D].
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_dq_convert_kernel(const float* __restrict__ acc, AttnParams p) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;  // 8 columns each
  constexpr int VPR = D / 8;
  const int64_t total = static_cast<int64_t>(p.b) * p.heads * p.s * VPR;
  if (idx >= total) return;
  const int v = static_cast<int>(idx % VPR);
  const int64_t row = idx / VPR;  // (bh, q)
  const int q = static_cast<int>(row % p.s);
  const int bh = static_cast<int>(row / p.s);
  const int bi = bh / p.heads, head = bh % p.heads;
  const float4 a = reinterpret_cast<const float4*>(acc + row * D)[2 * v];
  const float4 b = reinterpret_cast<const float4*>(acc + row * D)[2 * v + 1];
  const float sc = p.scale;
  const uint4 o = make_uint4(pack_bf16(a.x * sc, a.y * sc), pack_bf16(a.z * sc, a.w * sc), pack_bf16(b.x * sc, b.y * sc),
                             pack_bf16(b.z * sc, b.w * sc));
  *reinterpret_cast<uint4*>(p.dqkv + (static_cast<int64_t>(q) * p.b + bi) * p.ld_dqkv + head * D + 8 * v) = o;
}

// ------------------------------------------------------------------ pre-pass

// D = rowsum(dO * O) per (batch, head, query): one warp per token.
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ o,
                                                           const __nv_bfloat16* __restrict__ d_o, int ld_o,
                                                           float* __restrict__ delta, int s, int b, int heads) {
  const int tok = blockIdx.x * 8 + warp_id();  // token = s_idx * b + bi
  if (tok >= s * b) return;
  const int si = tok / b, bi = tok % b;
  const int lane = lane_id();
  constexpr int VPH = D / 8;  // 16-byte vectors per head
  const int nvec = heads * VPH;
  for (int v0 = 0; v0 < nvec; v0 += 32) {
    const int v = v0 + lane;
    float acc = 0.f;
    if (v < nvec) {
      const uint4 a = reinterpret_cast<const uint4*>(o + static_cast<int64_t>(tok) * ld_o)[v];
      const uint4 gg = reinterpret_cast<const uint4*>(d_o + static_cast<int64_t>(tok) * ld_o)[v];
      const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wg[4] = {gg.x, gg.y, gg.z, gg.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fa = unpack_bf16(wa[j]), fg = unpack_bf16(wg[j]);
        acc += fa.x * fg.x + fa.y * fg.y;
      }
    }
#pragma unroll
    for (int off = VPH / 2; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (v < nvec && v % VPH == 0)
      delta[(static_cast<int64_t>(bi) * heads + v / VPH) * s + si] = acc;
  }
}

// ------------------------------------------------------------------ host side

template <int D>
static cudaError_t bwd9_launch(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o,
                               const AttnParams& p, cudaStream_t st) {
  CUtensorMap tq, tdo;
  cudaError_t e = make_tma_3d_rows(&tq, qkv, 3 * p.h, p.b, p.s, ld_qkv, 64, AT_TILE);
  if (e == cudaSuccess) e = make_tma_3d_rows(&tdo, d_o, p.h, p.b, p.s, ld_o, 64, AT_TILE);
  if (e != cudaSuccess) return e;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(attn_bwd_dkdv9_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             KV9Smem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq9_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q9Smem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int tokens = p.s * p.b;
  if (o != nullptr)  // else delta already holds D (hx_attn_bwd_delta on the post stage)
    attn_bwd_pre_kernel<D><<<(tokens + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                             static_cast<const __nv_bfloat16*>(d_o), ld_o,
                                                             const_cast<float*>(p.delta), p.s, p.b, p.heads);
  dim3 grid((p.s + AT_TILE - 1) / AT_TILE, p.b * p.heads);
  attn_bwd_dkdv9_kernel<D><<<grid, 320, KV9Smem<D>::TOTAL, st>>>(tq, tdo, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  attn_bwd_dq9_kernel<D><<<grid, 320, Q9Smem<D>::TOTAL, st>>>(tq, static_cast<const __nv_bfloat16*>(qkv), ld_qkv,
                                                               static_cast<const __nv_bfloat16*>(d_o), ld_o, p);
  return cudaGetLastError();
}

template <int D>
static cudaError_t fused_launch(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o, float* dq_acc,
                                const AttnParams& p, cudaStream_t st) {
  CUtensorMap tq, tdo, tdq;
  cudaError_t e = make_tma_3d_rows(&tq, qkv, 3 * p.h, p.b, p.s, ld_qkv, 64, AT_TILE);
  if (e == cudaSuccess) e = make_tma_3d_rows(&tdo, d_o, p.h, p.b, p.s, ld_o, 64, AT_TILE);
  if (e == cudaSuccess) e = make_tma_f32_3d(&tdq, dq_acc, D, p.s, static_cast<uint64_t>(p.b) * p.heads, 32, AT_TILE);
  if (e != cudaSuccess) return e;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(attn_bwd_fused_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FusedSmem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int tokens = p.s * p.b;
  e = cudaMemsetAsync(dq_acc, 0, static_cast<size_t>(tokens) * p.h * sizeof(float), st);
  if (e != cudaSuccess) return e;
  if (o != nullptr)  // else delta already holds D (hx_attn_bwd_delta on the post stage)
    attn_bwd_pre_kernel<D><<<(tokens + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                             static_cast<const __nv_bfloat16*>(d_o), ld_o,
                                                             const_cast<float*>(p.delta), p.s, p.b, p.heads);
  const int grid = ((p.s + AT_TILE - 1) / AT_TILE) * p.b * p.heads;
  attn_bwd_fused_kernel<D><<<grid, 512, FusedSmem<D>::TOTAL, st>>>(tq, tdo, tdq, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t vecs = static_cast<int64_t>(tokens) * p.h / 8;
  attn_bwd_dq_convert_kernel<D><<<static_cast<unsigned>((vecs + 255) / 256), 256, 0, st>>>(dq_acc, p);
  return cudaGetLastError();
}

cudaError_t attn_bwd_delta_launch(const void* o, const void* d_o, int ld_o, float* delta, int s, int b, int heads,
                                  int d, cudaStream_t st) {
  const int tokens = s * b;
  if (d == 128)
    attn_bwd_pre_kernel<128><<<(tokens + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                               static_cast<const __nv_bfloat16*>(d_o), ld_o, delta,
                                                               s, b, heads);
  else if (d == 64)
    attn_bwd_pre_kernel<64><<<(tokens + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                              static_cast<const __nv_bfloat16*>(d_o), ld_o, delta,
                                                              s, b, heads);
  else
    return cudaErrorNotSupported;
  return cudaGetLastError();
}

cudaError_t attn_bwd_launch(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o,
                            const float* lse, float* delta, float* dq_acc, void* dqkv,
                            int ld_dqkv, int s, int b, int heads, int d, cudaStream_t st) {
  AttnParams p{};
  p.s = s;
  p.b = b;
  p.heads = heads;
  p.h = heads * d;
  p.scale = 1.0f / sqrtf(static_cast<float>(d));
  p.scale_log2 = p.scale * LOG2E;
  // Backward band: one head at a time (its fp32 dQ accumulator, s * d * 4 bytes,
  // and Q / dO stay in L2).  In the GPT-1.3B/32k bench step: 10.45-10.47 ms per
  // call with 1 head, 10.54 with 4, 10.64-10.66 with 8, 10.79-10.80 with all 16
  // (9x the DRAM traffic of 1 head: 11.9 GB per call, and lower clocks under the
  // power cap), although all 16 measured 4% faster in isolation.
  static const int forced_band = getenv("HX_ATTN_BWD_BAND") ? atoi(getenv("HX_ATTN_BWD_BAND")) : 0;
  p.band = forced_band > 0 ? forced_band : 1;
  p.lse = const_cast<float*>(lse);
  p.delta = delta;
  p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  p.ld_dqkv = ld_dqkv;
  // Default: the fused one-pass kernel (v10).  HX_ATTN_BWD=9 selects the split
  // atomic-free dK/dV + dQ kernels (deterministic dq; also for A/B runs).
  static const int variant = getenv("HX_ATTN_BWD") ? atoi(getenv("HX_ATTN_BWD")) : 10;
  if (variant == 10) {
    if (d == 128) return fused_launch<128>(qkv, ld_qkv, o, d_o, ld_o, dq_acc, p, st);
    if (d == 64) return fused_launch<64>(qkv, ld_qkv, o, d_o, ld_o, dq_acc, p, st);
    return cudaErrorNotSupported;
  }
  if (d == 128) return bwd9_launch<128>(qkv, ld_qkv, o, d_o, ld_o, p, st);
  if (d == 64) return bwd9_launch<64>(qkv, ld_qkv, o, d_o, ld_o, p, st);
  return cudaErrorNotSupported;
}

}  // namespace hx

#ifdef HX_BWD_TRACE
extern "C" HX_API int hx_debug_bwd_trace(long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, hx::g_bwd_trace, sizeof(hx::g_bwd_trace)));
}
#endif
