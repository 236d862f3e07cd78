// Causal flash attention, forward and backward, on tcgen05 / TMEM / TMA (sm_100a).
//
// Replaces the reference's whole-matrix fp64 attention (P/runtime/mathops.py:83-116):
//   forward : O = softmax(Q K^T / sqrt(d) + causal mask) V, plus LSE per row
//   backward: dV = P^T dO, dP = dO V^T, dS = P (dP - D), dQ = dS K / sqrt d,
//             dK = dS^T Q / sqrt d, with D = rowsum(dO * O) and P rebuilt from LSE
//
// Tiles are 128 x 128 (queries x keys).  Every operand tile lives in shared
// memory in the UMMA 128B-swizzled layout written by TMA (or by the softmax
// threads for P / dS), so one physical layout serves both K-major and MN-major
// reads (a [rows][64-col atom] tile is K-major with K = cols, or MN-major with
// K = rows).  Accumulators live in TMEM; one thread per TMEM lane (row).
//
// Forward CTA   = one 128-row query tile of one (batch, head); walks key tiles
//                 0..diag.  Warps 0-3 softmax/epilogue, warp 4 TMA, warp 5 MMA.
// Backward CTA  = one 128-row key tile; walks query tiles diag..end, keeps dK,
//                 dV in TMEM, adds dQ tiles into an fp32 workspace with
//                 vector atomics.  Warps 0-3 compute, warp 4 TMA, warp 5 MMA.
#include "hx_common.cuh"
#include "hx_gemm.h"

namespace hx {

constexpr int AT_TILE = 128;
constexpr int AT_THREADS = 192;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// A [128 rows x D cols] bf16 tile = D/64 swizzle atoms of 16 KB.
template <int D>
struct Tile {
  static constexpr int ATOMS = D / 64;
  static constexpr int BYTES = AT_TILE * D * 2;
};

// Descriptor for K-step kk (16 elements) of a K-major tile whose K extent spans atoms.
HX_DEVICE uint64_t kmajor_desc(uint32_t base, int kk) {
  return sw128_desc(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
}
// Descriptor for K-step kk (16 rows) of an MN-major tile (rows = K, 64-col atoms = MN).
HX_DEVICE uint64_t mnmajor_desc(uint32_t base, int kk) {
  return sw128_desc(base + kk * 2048, 16384, 1024);
}

// Byte offset of element (row, col) inside a swizzled [128 x (64*atoms)] bf16 tile,
// for a 16-byte chunk starting at col (col % 8 == 0).
HX_DEVICE uint32_t swz_off(int row, int col) {
  const int atom = col >> 6;
  const int chunk = (col >> 3) & 7;
  return atom * 16384 + row * 128 + ((chunk ^ (row & 7)) << 4);
}

// Load a [128 x D] tile of head columns `col0` for rows (tokens) s0.. of batch bi.
template <int D>
HX_DEVICE void tma_tile(void* dst, const CUtensorMap* map, uint64_t* bar, int col0, int bi, int s0) {
#pragma unroll
  for (int a = 0; a < D / 64; ++a)
    tma_load_3d(static_cast<uint8_t*>(dst) + a * 16384, map, bar, col0 + 64 * a, bi, s0);
}

struct AttnParams {
  int s, b, heads, h;
  float scale_log2;  // log2(e) / sqrt(d)
  float scale;       // 1 / sqrt(d)
  __nv_bfloat16* o;  // fwd output
  int ld_o;
  float* lse;        // [b, heads, s]
  // backward
  const float* delta;  // [b, heads, s]
  float* dq_acc;       // [b*heads, s, d]
  __nv_bfloat16* dqkv;
  int ld_dqkv;
};

// =====================================================================================
// forward
// =====================================================================================
template <int D>
struct FwdSmem {
  static constexpr int Q = 0;
  static constexpr int KV = Q + Tile<D>::BYTES;          // 2 stages x (K, V)
  static constexpr int P = KV + 4 * Tile<D>::BYTES;
  static constexpr int BAR = P + AT_TILE * AT_TILE * 2;
  static constexpr int TOTAL = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnParams p) {
  using L = FwdSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* v_full = bars + 3;   // [2]
  uint64_t* kv_empty = bars + 5; // [2]
  uint64_t* s_full = bars + 7;
  uint64_t* p_full = bars + 8;
  uint64_t* o_full = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int qt = nq - 1 - static_cast<int>(blockIdx.x);  // longest rows first
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int nkv = qt + 1;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 4 && lane == 0) {
    tma_prefetch(&tm_qkv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 4) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_arrive_expect_tx(q_full, Tile<D>::BYTES);
      tma_tile<D>(smem + L::Q, &tm_qkv, q_full, qcol, bi, qt * AT_TILE);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* kb = smem + L::KV + st * 2 * Tile<D>::BYTES;
        mbar_arrive_expect_tx(&k_full[st], Tile<D>::BYTES);
        tma_tile<D>(kb, &tm_qkv, &k_full[st], kcol, bi, j * AT_TILE);
        mbar_arrive_expect_tx(&v_full[st], Tile<D>::BYTES);
        tma_tile<D>(kb + Tile<D>::BYTES, &tm_qkv, &v_full[st], vcol, bi, j * AT_TILE);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t id_s = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_o = idesc_bf16(128, D, false, true);
      const uint32_t sq = smem_u32(smem + L::Q), sp = smem_u32(smem + L::P);
      mbar_wait(q_full, 0);
      for (int j = 0; j <= nkv; ++j) {
        if (j > 0) {  // O += P(j-1) V(j-1) once softmax has published P(j-1)
          const int st = (j - 1) & 1;
          mbar_wait(p_full, (j - 1) & 1);
          mbar_wait(&v_full[st], ((j - 1) >> 1) & 1);
          tc_fence_after();
          const uint32_t sv = smem_u32(smem + L::KV + st * 2 * Tile<D>::BYTES + Tile<D>::BYTES);
#pragma unroll
          for (int kk = 0; kk < AT_TILE / 16; ++kk)
            umma_f16_ss(tO, kmajor_desc(sp, kk), mnmajor_desc(sv, kk), id_o, (j > 1 || kk > 0));
          umma_commit(&kv_empty[st]);
        }
        if (j < nkv) {  // S = Q K(j)^T
          const int st = j & 1;
          mbar_wait(&k_full[st], (j >> 1) & 1);
          tc_fence_after();
          const uint32_t sk = smem_u32(smem + L::KV + st * 2 * Tile<D>::BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            umma_f16_ss(tS, kmajor_desc(sq, kk), kmajor_desc(sk, kk), id_s, kk > 0);
          umma_commit(s_full);
        }
      }
      umma_commit(o_full);
    }
  } else {
    // ---------------- softmax / epilogue: thread = query row
    const int r = warp * 32 + lane;
    const int qrow = qt * AT_TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    uint8_t* ps = smem + L::P;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      float sv[AT_TILE];
#pragma unroll
      for (int c = 0; c < AT_TILE / 32; ++c) {
        uint32_t raw[32];
        tmem_ld32(tS + lane_off + c * 32, raw);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(raw[i]) * p.scale_log2;
      }
      if (j == qt) {  // diagonal tile: key index > query index is masked
#pragma unroll
        for (int i = 0; i < AT_TILE; ++i)
          if (i > r) sv[i] = -INFINITY;
      }
      float mx = m_run;
#pragma unroll
      for (int i = 0; i < AT_TILE; ++i) mx = fmaxf(mx, sv[i]);
      const float alpha = exp2f(m_run - mx);  // 0 on the first tile (m_run = -inf)
      // Rescale the running O only if some row of this warp raised its max.
      if (j > 0 && __any_sync(0xffffffffu, mx > m_run)) {
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t o16[16];
          tmem_ld16(tO + lane_off + c * 16, o16);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o16[i] = __float_as_uint(__uint_as_float(o16[i]) * alpha);
          tmem_st16(tO + lane_off + c * 16, o16);
        }
        tmem_wait_st();
      }
      m_run = mx;
      float rs = 0.f;
#pragma unroll
      for (int c8 = 0; c8 < AT_TILE / 8; ++c8) {
        float e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          e[i] = exp2f(sv[c8 * 8 + i] - mx);
          rs += e[i];
        }
        *reinterpret_cast<uint4*>(ps + swz_off(r, c8 * 8)) =
            make_uint4(pack_bf16(e[0], e[1]), pack_bf16(e[2], e[3]), pack_bf16(e[4], e[5]),
                       pack_bf16(e[6], e[7]));
      }
      l_run = l_run * alpha + rs;
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(o_full, 0);
    tc_fence_after();
    const float inv_l = 1.f / l_run;
    __nv_bfloat16* orow = p.o + (static_cast<int64_t>(qrow) * p.b + bi) * p.ld_o + head * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t raw[32];
      tmem_ld32(tO + lane_off + c * 32, raw);
      tmem_wait_ld();
      if (qrow < p.s) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(raw[v * 8 + i]) * inv_l;
          *reinterpret_cast<uint4*>(orow + c * 32 + v * 8) =
              make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]),
                         pack_bf16(f[6], f[7]));
        }
      }
    }
    if (qrow < p.s) p.lse[static_cast<int64_t>(bh) * p.s + qrow] = (m_run + log2f(l_run)) * LN2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// =====================================================================================
// backward
// =====================================================================================
template <int D>
struct BwdSmem {
  static constexpr int K = 0;
  static constexpr int V = K + Tile<D>::BYTES;
  static constexpr int Q = V + Tile<D>::BYTES;
  static constexpr int DO = Q + Tile<D>::BYTES;
  static constexpr int PT = DO + Tile<D>::BYTES;       // P^T  [kv x q]
  static constexpr int DST = PT + AT_TILE * AT_TILE * 2;  // dS^T [kv x q]
  static constexpr int LSE = DST + AT_TILE * AT_TILE * 2;
  static constexpr int DEL = LSE + AT_TILE * 4;
  static constexpr int BAR = DEL + AT_TILE * 4;
  static constexpr int TOTAL = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const AttnParams p) {
  using L = BwdSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;
  uint64_t* qdo_empty = bars + 2;
  uint64_t* sp_full = bars + 3;
  uint64_t* ds_full = bars + 4;
  uint64_t* dq_full = bars + 5;
  uint64_t* dq_free = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  float* s_lse = reinterpret_cast<float*>(smem + L::LSE);
  float* s_del = reinterpret_cast<float*>(smem + L::DEL);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int kt = static_cast<int>(blockIdx.x);   // key tile; work = nq - kt query tiles
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;
  const int n_it = nq - kt;

  if (warp == 4 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    for (int i = 0; i < 7; ++i) mbar_init(&bars[i], (i == 4 || i == 6) ? 128 : 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 256 + D;
  const uint32_t tDQ = tS;  // dQ reuses the S columns once P / dS are out

  if (warp == 4) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_arrive_expect_tx(kv_full, 2 * Tile<D>::BYTES);
      tma_tile<D>(smem + L::K, &tm_qkv, kv_full, kcol, bi, kt * AT_TILE);
      tma_tile<D>(smem + L::V, &tm_qkv, kv_full, vcol, bi, kt * AT_TILE);
      for (int it = 0; it < n_it; ++it) {
        const int qtile = kt + it;
        mbar_wait(qdo_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(qdo_full, 2 * Tile<D>::BYTES);
        tma_tile<D>(smem + L::Q, &tm_qkv, qdo_full, qcol, bi, qtile * AT_TILE);
        tma_tile<D>(smem + L::DO, &tm_do, qdo_full, head * D, bi, qtile * AT_TILE);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t id_sp = idesc_bf16(128, 128, false, false);  // S^T, dP^T
      constexpr uint32_t id_kv = idesc_bf16(128, D, false, true);      // dV, dK: A K-major, B MN
      constexpr uint32_t id_q = idesc_bf16(128, D, true, true);        // dQ: A (dS) MN-major
      const uint32_t sk = smem_u32(smem + L::K), sv = smem_u32(smem + L::V);
      const uint32_t sq = smem_u32(smem + L::Q), sdo = smem_u32(smem + L::DO);
      const uint32_t spt = smem_u32(smem + L::PT), sdst = smem_u32(smem + L::DST);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        mbar_wait(qdo_full, it & 1);
        if (it > 0) mbar_wait(dq_free, (it - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tS, kmajor_desc(sk, kk), kmajor_desc(sq, kk), id_sp, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tDP, kmajor_desc(sv, kk), kmajor_desc(sdo, kk), id_sp, kk > 0);
        umma_commit(sp_full);
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk) {
          umma_f16_ss(tDV, kmajor_desc(spt, kk), mnmajor_desc(sdo, kk), id_kv, it > 0 || kk > 0);
          umma_f16_ss(tDK, kmajor_desc(sdst, kk), mnmajor_desc(sq, kk), id_kv, it > 0 || kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ss(tDQ, mnmajor_desc(sdst, kk), mnmajor_desc(sk, kk), id_q, kk > 0);
        umma_commit(dq_full);
        umma_commit(qdo_empty);
      }
    }
  } else {
    // ---------------- compute warps: thread = key row for S^T / dP^T, query row for dQ
    const int c = warp * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    uint8_t* pt = smem + L::PT;
    uint8_t* dst = smem + L::DST;
    const int64_t row_base = static_cast<int64_t>(bh) * p.s;
    for (int it = 0; it < n_it; ++it) {
      const int qtile = kt + it;
      const int q0 = qtile * AT_TILE;
      // stage LSE (log2 domain) and D of this query tile
      named_barrier_sync_compute();
      {
        const int q = q0 + c;
        s_lse[c] = q < p.s ? p.lse[row_base + q] * LOG2E : 0.f;
        s_del[c] = q < p.s ? p.delta[row_base + q] : 0.f;
      }
      named_barrier_sync_compute();
      mbar_wait(sp_full, it & 1);
      tc_fence_after();
      const bool diag = (qtile == kt);
#pragma unroll 1
      for (int ch = 0; ch < AT_TILE / 32; ++ch) {
        uint32_t rs[32], rdp[32];
        tmem_ld32(tS + lane_off + ch * 32, rs);
        tmem_ld32(tDP + lane_off + ch * 32, rdp);
        tmem_wait_ld();
        float pv[32], dsv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int qi = ch * 32 + i;
          float pr = exp2f(__uint_as_float(rs[i]) * p.scale_log2 - s_lse[qi]);
          if ((diag && qi < c) || q0 + qi >= p.s) pr = 0.f;
          pv[i] = pr;
          dsv[i] = pr * (__uint_as_float(rdp[i]) - s_del[qi]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t off = swz_off(c, ch * 32 + v * 8);
          *reinterpret_cast<uint4*>(pt + off) =
              make_uint4(pack_bf16(pv[v * 8], pv[v * 8 + 1]), pack_bf16(pv[v * 8 + 2], pv[v * 8 + 3]),
                         pack_bf16(pv[v * 8 + 4], pv[v * 8 + 5]), pack_bf16(pv[v * 8 + 6], pv[v * 8 + 7]));
          *reinterpret_cast<uint4*>(dst + off) =
              make_uint4(pack_bf16(dsv[v * 8], dsv[v * 8 + 1]), pack_bf16(dsv[v * 8 + 2], dsv[v * 8 + 3]),
                         pack_bf16(dsv[v * 8 + 4], dsv[v * 8 + 5]), pack_bf16(dsv[v * 8 + 6], dsv[v * 8 + 7]));
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
      // dQ tile: TMEM lane = query row
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      const int q = q0 + c;
      float* dq = p.dq_acc + (row_base + q) * D;
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch) {
        uint32_t raw[32];
        tmem_ld32(tDQ + lane_off + ch * 32, raw);
        tmem_wait_ld();
        if (q < p.s) {
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            float4 val = make_float4(__uint_as_float(raw[4 * v]) * p.scale, __uint_as_float(raw[4 * v + 1]) * p.scale,
                                     __uint_as_float(raw[4 * v + 2]) * p.scale, __uint_as_float(raw[4 * v + 3]) * p.scale);
            atomicAdd(reinterpret_cast<float4*>(dq + ch * 32 + 4 * v), val);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(dq_free);
    }
    // dK, dV epilogue: wait for the last MMA batch (dq_full of the last iteration
    // commits after every dV/dK MMA, and they complete in order).
    const int krow = kt * AT_TILE + c;
    tc_fence_after();
    __nv_bfloat16* dk = p.dqkv + (static_cast<int64_t>(krow) * p.b + bi) * p.ld_dqkv + p.h + head * D;
    __nv_bfloat16* dv = p.dqkv + (static_cast<int64_t>(krow) * p.b + bi) * p.ld_dqkv + 2 * p.h + head * D;
#pragma unroll
    for (int ch = 0; ch < D / 32; ++ch) {
      uint32_t rk[32], rv[32];
      tmem_ld32(tDK + lane_off + ch * 32, rk);
      tmem_ld32(tDV + lane_off + ch * 32, rv);
      tmem_wait_ld();
      if (krow < p.s) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float fk[8], fv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            fk[i] = __uint_as_float(rk[v * 8 + i]) * p.scale;
            fv[i] = __uint_as_float(rv[v * 8 + i]);
          }
          *reinterpret_cast<uint4*>(dk + ch * 32 + v * 8) =
              make_uint4(pack_bf16(fk[0], fk[1]), pack_bf16(fk[2], fk[3]), pack_bf16(fk[4], fk[5]), pack_bf16(fk[6], fk[7]));
          *reinterpret_cast<uint4*>(dv + ch * 32 + v * 8) =
              make_uint4(pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// D = rowsum(dO * O) per (batch, head, query); also zeroes the dQ accumulator.
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ o,
                                                           const __nv_bfloat16* __restrict__ d_o, int ld_o,
                                                           float* __restrict__ delta, float* __restrict__ dq_acc,
                                                           int s, int b, int heads) {
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
      uint4 a = reinterpret_cast<const uint4*>(o + static_cast<int64_t>(tok) * ld_o)[v];
      uint4 g = reinterpret_cast<const uint4*>(d_o + static_cast<int64_t>(tok) * ld_o)[v];
      const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 fa = unpack_bf16(wa[j]), fg = unpack_bf16(wg[j]);
        acc += fa.x * fg.x + fa.y * fg.y;
      }
    }
#pragma unroll
    for (int off = VPH / 2; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (v < nvec) {
      const int head = v / VPH, sub = v % VPH;
      const int64_t row = (static_cast<int64_t>(bi) * heads + head) * s + si;
      if (sub == 0) delta[row] = acc;
      reinterpret_cast<uint4*>(dq_acc + row * D)[sub * 2] = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint4*>(dq_acc + row * D)[sub * 2 + 1] = make_uint4(0, 0, 0, 0);
    }
  }
}

// dqkv[:, head*D + c] = bf16(dq_acc)
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_post_kernel(const float* __restrict__ dq_acc,
                                                            __nv_bfloat16* __restrict__ dqkv, int ld,
                                                            int s, int b, int heads) {
  const int64_t n8 = static_cast<int64_t>(s) * b * heads * D / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = i * 8;
    const int c = static_cast<int>(e % D);
    const int64_t row = e / D;  // (bi*heads + head) * s + si
    const int si = static_cast<int>(row % s);
    const int bhh = static_cast<int>(row / s);
    const int head = bhh % heads, bi = bhh / heads;
    const float4 a = reinterpret_cast<const float4*>(dq_acc + e)[0];
    const float4 c2 = reinterpret_cast<const float4*>(dq_acc + e)[1];
    *reinterpret_cast<uint4*>(dqkv + (static_cast<int64_t>(si) * b + bi) * ld + head * D + c) =
        make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(c2.x, c2.y), pack_bf16(c2.z, c2.w));
  }
}

// ------------------------------------------------------------------ host side

static cudaError_t make_qkv_map(CUtensorMap* map, const void* ptr, int s, int b, int cols, int ld) {
  return make_tma_3d_rows(map, ptr, cols, b, s, ld, 64, AT_TILE);
}

template <int D>
static cudaError_t fwd_launch(const void* qkv, int ld_qkv, const AttnParams& p, cudaStream_t st) {
  CUtensorMap tm;
  cudaError_t e = make_qkv_map(&tm, qkv, p.s, p.b, 3 * p.h, ld_qkv);
  if (e != cudaSuccess) return e;
  auto k = attn_fwd_kernel<D>;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  dim3 grid((p.s + AT_TILE - 1) / AT_TILE, p.b * p.heads);
  k<<<grid, AT_THREADS, FwdSmem<D>::TOTAL, st>>>(tm, p);
  return cudaGetLastError();
}

template <int D>
static cudaError_t bwd_launch(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o,
                              const AttnParams& p, cudaStream_t st) {
  CUtensorMap tq, tdo;
  cudaError_t e = make_qkv_map(&tq, qkv, p.s, p.b, 3 * p.h, ld_qkv);
  if (e != cudaSuccess) return e;
  e = make_qkv_map(&tdo, d_o, p.s, p.b, p.h, ld_o);
  if (e != cudaSuccess) return e;
  const int tokens = p.s * p.b;
  attn_bwd_pre_kernel<D><<<(tokens + 7) / 8, 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(d_o), ld_o,
      const_cast<float*>(p.delta), p.dq_acc, p.s, p.b, p.heads);
  auto k = attn_bwd_kernel<D>;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdSmem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  dim3 grid((p.s + AT_TILE - 1) / AT_TILE, p.b * p.heads);
  k<<<grid, AT_THREADS, BwdSmem<D>::TOTAL, st>>>(tq, tdo, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n8 = static_cast<int64_t>(tokens) * p.heads * D / 8;
  int g = static_cast<int>((n8 + 255) / 256);
  if (g > num_sms() * 8) g = num_sms() * 8;
  attn_bwd_post_kernel<D><<<g, 256, 0, st>>>(p.dq_acc, p.dqkv, p.ld_dqkv, p.s, p.b, p.heads);
  return cudaGetLastError();
}

static AttnParams make_params(int s, int b, int heads, int d) {
  AttnParams p{};
  p.s = s;
  p.b = b;
  p.heads = heads;
  p.h = heads * d;
  p.scale = 1.0f / sqrtf(static_cast<float>(d));
  p.scale_log2 = p.scale * LOG2E;
  return p;
}

cudaError_t attn_fwd_launch(const void* qkv, int ld_qkv, void* o, int ld_o, float* lse, int s, int b,
                            int heads, int d, cudaStream_t st) {
  AttnParams p = make_params(s, b, heads, d);
  p.o = static_cast<__nv_bfloat16*>(o);
  p.ld_o = ld_o;
  p.lse = lse;
  if (d == 128) return fwd_launch<128>(qkv, ld_qkv, p, st);
  if (d == 64) return fwd_launch<64>(qkv, ld_qkv, p, st);
  return cudaErrorNotSupported;
}

cudaError_t attn_bwd_launch(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o,
                            const float* lse, float* delta, float* dq_acc, void* dqkv, int ld_dqkv,
                            int s, int b, int heads, int d, cudaStream_t st) {
  AttnParams p = make_params(s, b, heads, d);
  p.lse = const_cast<float*>(lse);
  p.delta = delta;
  p.dq_acc = dq_acc;
  p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  p.ld_dqkv = ld_dqkv;
  if (d == 128) return bwd_launch<128>(qkv, ld_qkv, o, d_o, ld_o, p, st);
  if (d == 64) return bwd_launch<64>(qkv, ld_qkv, o, d_o, ld_o, p, st);
  return cudaErrorNotSupported;
}

}  // namespace hx
