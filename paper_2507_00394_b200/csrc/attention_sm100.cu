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
// forward v2: two query tiles per CTA, ping-pong softmax, P in TMEM
// =====================================================================================
//
// CTA = query tiles (2t, 2t+1) of one (batch, head).  Two softmax warpgroups
// (warps 0-3 -> tile A, 4-7 -> tile B) alternate with the tensor core: while
// group A exponentiates S_A(j), the tensor core runs O_B += P_B(j-1) V(j-1) and
// S_B(j) = Q_B K(j)^T, and vice versa.  P is written back as bf16 into the
// first 64 columns of its own S region and consumed from TMEM by the
// PV tcgen05.mma (A operand in TMEM), so P never touches shared memory.
// O is rescaled only when a row's running max grows by more than 2^8
// (exponents stay <= 256, exact in fp32), which makes rescales rare.
//
// TMEM (512 columns): S_A 0-127 | S_B 128-255 | O_A 256-383 | O_B 384-511.

constexpr int FWD2_THREADS = 320;  // 8 softmax warps + TMA warp + MMA warp

template <int D>
struct Fwd2Smem {
  static constexpr int QA = 0;
  static constexpr int QB = QA + Tile<D>::BYTES;
  static constexpr int KV = QB + Tile<D>::BYTES;  // 2 stages x (K, V)
  static constexpr int BAR = KV + 4 * Tile<D>::BYTES;
  static constexpr int TOTAL = BAR + 256 + 1024;
};

HX_DEVICE float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D>
__global__ void __launch_bounds__(FWD2_THREADS, 1)
    attn_fwd2_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnParams p) {
  using L = Fwd2Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;          // 1
  uint64_t* k_full = bars + 1;      // 2
  uint64_t* v_full = bars + 3;      // 2
  uint64_t* kv_empty = bars + 5;    // 2
  uint64_t* s_full = bars + 7;      // 2 (per group)
  uint64_t* p_full = bars + 9;      // 2
  uint64_t* o_full = bars + 11;     // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int npairs = (nq + 1) / 2;
  const int t = npairs - 1 - static_cast<int>(blockIdx.x);  // heaviest pairs first
  const int qtile[2] = {2 * t, 2 * t + 1};
  const bool has_b = qtile[1] < nq;
  const int last[2] = {qtile[0], has_b ? qtile[1] : -1};
  const int nkv = has_b ? qtile[1] + 1 : qtile[0] + 1;
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    for (int i = 0; i < 13; ++i) mbar_init(&bars[i], (i == 9 || i == 10) ? 128 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_arrive_expect_tx(q_full, (has_b ? 2 : 1) * Tile<D>::BYTES);
      tma_tile<D>(smem + L::QA, &tm_qkv, q_full, qcol, bi, qtile[0] * AT_TILE);
      if (has_b) tma_tile<D>(smem + L::QB, &tm_qkv, q_full, qcol, bi, qtile[1] * AT_TILE);
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
  } else if (warp == 9) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t id_s = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_o = idesc_bf16(128, D, false, true);
      const uint32_t sq[2] = {smem_u32(smem + L::QA), smem_u32(smem + L::QB)};
      bool pending[2] = {false, false};
      int pcount[2] = {0, 0};
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int g, int jt) {
        mbar_wait(&p_full[g], pcount[g] & 1);
        ++pcount[g];
        mbar_wait(&v_full[jt & 1], (jt >> 1) & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + L::KV + (jt & 1) * 2 * Tile<D>::BYTES + Tile<D>::BYTES);
        const uint32_t tP = tmem + 128 * g, tO = tmem + 256 + 128 * g;
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts(tO, tP + kk * 8, mnmajor_desc(sv, kk), id_o, (jt > 0 || kk > 0));
        pending[g] = false;
      };
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&k_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + L::KV + (j & 1) * 2 * Tile<D>::BYTES);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (pending[g]) issue_pv(g, j - 1);
          if (j <= last[g]) {
            const uint32_t tS = tmem + 128 * g;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              umma_f16_ss(tS, kmajor_desc(sq[g], kk), kmajor_desc(sk, kk), id_s, kk > 0);
            umma_commit(&s_full[g]);
            pending[g] = true;
          }
        }
        if (j > 0) umma_commit(&kv_empty[(j - 1) & 1]);
      }
      for (int g = 0; g < 2; ++g)
        if (pending[g]) issue_pv(g, last[g]);
      umma_commit(&o_full[0]);
      umma_commit(&o_full[1]);
    }
  } else {
    // ---------------- softmax warpgroups: thread = query row of tile g
    const int g = warp >> 2;
    const int quad = warp & 3;
    if (g == 0 || has_b) {
      const int r = quad * 32 + lane;
      const int qt = qtile[g];
      const int qrow = qt * AT_TILE + r;
      const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
      const uint32_t tS = tmem + 128 * g + lane_off, tO = tmem + 256 + 128 * g + lane_off;
      const float c = p.scale_log2;
      float m_used = -INFINITY, l_run = 0.f;
      for (int j = 0; j <= qt; ++j) {
        mbar_wait(&s_full[g], j & 1);
        tc_fence_after();
        uint32_t raw[AT_TILE];
#pragma unroll
        for (int ch = 0; ch < AT_TILE / 32; ++ch)
          tmem_ld32(tS + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(raw + ch * 32));
        tmem_wait_ld();
        float mx = -INFINITY;
        if (j == qt) {
#pragma unroll
          for (int i = 0; i < AT_TILE; ++i) {
            if (i > r) raw[i] = __float_as_uint(-INFINITY);
            mx = fmaxf(mx, __uint_as_float(raw[i]));
          }
        } else {
#pragma unroll
          for (int i = 0; i < AT_TILE; ++i) mx = fmaxf(mx, __uint_as_float(raw[i]));
        }
        mx *= c;
        const float m_new = (mx > m_used + 8.0f) ? mx : m_used;
        const float alpha = fast_exp2(m_used - m_new);
        if (j > 0 && __any_sync(0xffffffffu, m_new != m_used)) {
#pragma unroll
          for (int ch = 0; ch < D / 16; ++ch) {
            uint32_t o16[16];
            tmem_ld16(tO + ch * 16, o16);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o16[i] = __float_as_uint(__uint_as_float(o16[i]) * alpha);
            tmem_st16(tO + ch * 16, o16);
          }
        }
        m_used = m_new;
        const float neg_m = -m_new;
        float rs = 0.f;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float e0 = fast_exp2(fmaf(__uint_as_float(raw[half * 64 + 2 * i]), c, neg_m));
            const float e1 = fast_exp2(fmaf(__uint_as_float(raw[half * 64 + 2 * i + 1]), c, neg_m));
            rs += e0 + e1;
            pk[i] = pack_bf16(e0, e1);
          }
          tmem_st32(tS + half * 32, pk);  // P over the first 64 columns of S
        }
        tmem_wait_st();
        l_run = l_run * alpha + rs;
        tc_fence_before();
        mbar_arrive(&p_full[g]);
      }
      mbar_wait(&o_full[g], 0);
      tc_fence_after();
      const float inv_l = 1.f / l_run;
      __nv_bfloat16* orow = p.o + (static_cast<int64_t>(qrow) * p.b + bi) * p.ld_o + head * D;
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch) {
        uint32_t o32[32];
        tmem_ld32(tO + ch * 32, o32);
        tmem_wait_ld();
        if (qrow < p.s) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            float f[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(o32[v * 8 + i]) * inv_l;
            *reinterpret_cast<uint4*>(orow + ch * 32 + v * 8) =
                make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]),
                           pack_bf16(f[6], f[7]));
          }
        }
      }
      if (qrow < p.s) p.lse[static_cast<int64_t>(bh) * p.s + qrow] = (m_used + log2f(l_run)) * LN2;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
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

// =====================================================================================
// backward v2
// =====================================================================================
//
// CTA = one 128-row key tile of one (batch, head), walking query tiles diag..end.
//   warps 0-7   compute: warpgroup g handles query columns [64g, 64g+64) of the
//               transposed tiles; thread = key row.  P^T goes back into TMEM
//               (A operand of dV += P^T dO), dS^T into a swizzled smem tile
//               (A operand of dK += dS^T Q, and - read MN-major - of dQ = dS K).
//   warps 8-11  dQ reduction: TMEM -> registers -> fp32 vector atomics, so the
//               global reduction overlaps the next tile's MMAs and softmax.
//   warp 12     TMA (K, V once; Q, dO double-buffered).
//   warp 13     MMA issuer + TMEM owner.
// TMEM: dK 0-127 | dV 128-255 | S^T (P^T in 256-287 / 320-351) 256-383 | dP^T = dQ 384-511.
// MMA order per query tile i:  S^T(i), [dQ(i-1) read out] dP^T(i), [P^T(i)] dV,
// [dS^T(i)] dK, dQ(i)  - so S^T(i+1) runs while the reducers drain dQ(i).

constexpr int BWD2_THREADS = 448;

template <int D>
struct Bwd2Smem {
  static constexpr int K = 0;
  static constexpr int V = K + Tile<D>::BYTES;
  static constexpr int Q = V + Tile<D>::BYTES;        // 2 stages
  static constexpr int DO = Q + 2 * Tile<D>::BYTES;   // 2 stages
  static constexpr int DST = DO + 2 * Tile<D>::BYTES;  // dS^T [kv x q], 2 atoms
  static constexpr int STAT = DST + AT_TILE * AT_TILE * 2;  // [2 slots][lse2 | delta][128]
  static constexpr int BAR = STAT + 2 * 2 * AT_TILE * 4;
  static constexpr int TOTAL = BAR + 256;  // requires a 1024-aligned dynamic smem base
};

HX_DEVICE void named_barrier_sync(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int D>
__global__ void __launch_bounds__(BWD2_THREADS, 1)
    attn_bwd2_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                     const AttnParams p) {
  using L = Bwd2Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* kv_full = bars;         // 1
  uint64_t* qdo_full = bars + 1;    // 2
  uint64_t* qdo_empty = bars + 3;   // 2
  uint64_t* s_full = bars + 5;
  uint64_t* dp_full = bars + 6;
  uint64_t* p_full = bars + 7;      // 256 arrivals
  uint64_t* ds_full = bars + 8;     // 256 arrivals
  uint64_t* dq_full = bars + 9;
  uint64_t* dq_free = bars + 10;    // 128 arrivals
  uint64_t* acc_full = bars + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  float* stat = reinterpret_cast<float*>(smem + L::STAT);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int kt = static_cast<int>(blockIdx.x);
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;
  const int n_it = nq - kt;

  if (warp == 12 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    for (int i = 0; i < 12; ++i)
      mbar_init(&bars[i], (i == 7 || i == 8) ? 256 : (i == 10 ? 128 : 1));
    fence_barrier_init();
  }
  if (warp == 13) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDK = tmem, tDV = tmem + 128, tS = tmem + 256, tDP = tmem + 384;

  if (warp == 12) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_arrive_expect_tx(kv_full, 2 * Tile<D>::BYTES);
      tma_tile<D>(smem + L::K, &tm_qkv, kv_full, kcol, bi, kt * AT_TILE);
      tma_tile<D>(smem + L::V, &tm_qkv, kv_full, vcol, bi, kt * AT_TILE);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1, q0 = (kt + it) * AT_TILE;
        mbar_wait(&qdo_empty[st], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qdo_full[st], 2 * Tile<D>::BYTES);
        tma_tile<D>(smem + L::Q + st * Tile<D>::BYTES, &tm_qkv, &qdo_full[st], qcol, bi, q0);
        tma_tile<D>(smem + L::DO + st * Tile<D>::BYTES, &tm_do, &qdo_full[st], head * D, bi, q0);
      }
    }
  } else if (warp == 13) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t id_sp = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_kv = idesc_bf16(128, D, false, true);
      constexpr uint32_t id_q = idesc_bf16(128, D, true, true);
      const uint32_t sk = smem_u32(smem + L::K), sv = smem_u32(smem + L::V);
      const uint32_t sdst = smem_u32(smem + L::DST);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1;
        const uint32_t sq = smem_u32(smem + L::Q + st * Tile<D>::BYTES);
        const uint32_t sdo = smem_u32(smem + L::DO + st * Tile<D>::BYTES);
        mbar_wait(&qdo_full[st], (it >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tS, kmajor_desc(sk, kk), kmajor_desc(sq, kk), id_sp, kk > 0);
        umma_commit(s_full);
        if (it > 0) {
          mbar_wait(dq_free, (it - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tDP, kmajor_desc(sv, kk), kmajor_desc(sdo, kk), id_sp, kk > 0);
        umma_commit(dp_full);
        mbar_wait(p_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)  // P^T of warpgroup kk/4 at 256 + 64*(kk/4)
          umma_f16_ts(tDV, tS + (kk >> 2) * 64 + (kk & 3) * 8, mnmajor_desc(sdo, kk), id_kv,
                      it > 0 || kk > 0);
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ss(tDK, kmajor_desc(sdst, kk), mnmajor_desc(sq, kk), id_kv, it > 0 || kk > 0);
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ss(tDP, mnmajor_desc(sdst, kk), mnmajor_desc(sk, kk), id_q, kk > 0);
        umma_commit(dq_full);
        umma_commit(&qdo_empty[st]);
      }
      umma_commit(acc_full);
    }
  } else if (warp < 8) {
    // ---------------- compute: thread = key row c, query columns [qoff, qoff+64)
    const int g = warp >> 2, quad = warp & 3;
    const int c = quad * 32 + lane;
    const int qoff = 64 * g;
    const int ct = threadIdx.x;  // 0..255
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row_base = static_cast<int64_t>(bh) * p.s;
    uint8_t* dst = smem + L::DST;
    for (int it = 0; it < n_it; ++it) {
      const int qtile = kt + it, q0 = qtile * AT_TILE;
      float* s_lse = stat + (it & 1) * 2 * AT_TILE;
      float* s_del = s_lse + AT_TILE;
      {
        const int qi = ct & (AT_TILE - 1);
        const int q = q0 + qi;
        if (ct < AT_TILE) s_lse[qi] = q < p.s ? p.lse[row_base + q] * LOG2E : 0.f;
        else s_del[qi] = q < p.s ? p.delta[row_base + q] : 0.f;
      }
      named_barrier_sync(1, 256);
      const bool diag = (qtile == kt);
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      uint32_t raw[64];
      tmem_ld32(tS + lane_off + qoff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tS + lane_off + qoff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      float pv[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int qi = qoff + j;
        float pr = fast_exp2(fmaf(__uint_as_float(raw[j]), p.scale_log2, -s_lse[qi]));
        if ((diag && qi < c) || q0 + qi >= p.s) pr = 0.f;
        pv[j] = pr;
      }
      {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) pk[j] = pack_bf16(pv[2 * j], pv[2 * j + 1]);
        tmem_st32(tS + lane_off + qoff, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
      mbar_wait(dp_full, it & 1);
      tc_fence_after();
      tmem_ld32(tDP + lane_off + qoff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tDP + lane_off + qoff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        float ds[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int j = v * 8 + i;
          ds[i] = pv[j] * (__uint_as_float(raw[j]) - s_del[qoff + j]);
        }
        *reinterpret_cast<uint4*>(dst + swz_off(c, qoff + v * 8)) =
            make_uint4(pack_bf16(ds[0], ds[1]), pack_bf16(ds[2], ds[3]), pack_bf16(ds[4], ds[5]),
                       pack_bf16(ds[6], ds[7]));
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    // dK, dV epilogue (rows c, columns [64g, 64g+64))
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int krow = kt * AT_TILE + c;
    const int64_t tok = static_cast<int64_t>(krow) * p.b + bi;
    __nv_bfloat16* dk = p.dqkv + tok * p.ld_dqkv + p.h + head * D;
    __nv_bfloat16* dv = p.dqkv + tok * p.ld_dqkv + 2 * p.h + head * D;
#pragma unroll
    for (int ch = 0; ch < D / 64; ++ch) {
      const int col = g * (D / 2) + ch * 32;
      if (col >= (g + 1) * (D / 2)) break;
      uint32_t rk[32], rv[32];
      tmem_ld32(tDK + lane_off + col, rk);
      tmem_ld32(tDV + lane_off + col, rv);
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
          *reinterpret_cast<uint4*>(dk + col + v * 8) =
              make_uint4(pack_bf16(fk[0], fk[1]), pack_bf16(fk[2], fk[3]), pack_bf16(fk[4], fk[5]), pack_bf16(fk[6], fk[7]));
          *reinterpret_cast<uint4*>(dv + col + v * 8) =
              make_uint4(pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
        }
      }
    }
  } else {
    // ---------------- dQ reducers (warps 8-11): thread = query row
    const int quad = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row_base = static_cast<int64_t>(bh) * p.s;
    for (int it = 0; it < n_it; ++it) {
      const int q = (kt + it) * AT_TILE + quad * 32 + lane;
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      float* dq = p.dq_acc + (row_base + q) * D;
#pragma unroll
      for (int half = 0; half < D / 64; ++half) {
        uint32_t r0[32], r1[32];
        tmem_ld32(tDP + lane_off + half * 64, r0);
        tmem_ld32(tDP + lane_off + half * 64 + 32, r1);
        tmem_wait_ld();
        if (half == D / 64 - 1) {
          tc_fence_before();
          mbar_arrive(dq_free);
        }
        if (q < p.s) {
#pragma unroll
          for (int v = 0; v < 8; ++v)
            atomicAdd(reinterpret_cast<float4*>(dq + half * 64 + 4 * v),
                      make_float4(__uint_as_float(r0[4 * v]) * p.scale, __uint_as_float(r0[4 * v + 1]) * p.scale,
                                  __uint_as_float(r0[4 * v + 2]) * p.scale, __uint_as_float(r0[4 * v + 3]) * p.scale));
#pragma unroll
          for (int v = 0; v < 8; ++v)
            atomicAdd(reinterpret_cast<float4*>(dq + half * 64 + 32 + 4 * v),
                      make_float4(__uint_as_float(r1[4 * v]) * p.scale, __uint_as_float(r1[4 * v + 1]) * p.scale,
                                  __uint_as_float(r1[4 * v + 2]) * p.scale, __uint_as_float(r1[4 * v + 3]) * p.scale));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// =====================================================================================
// backward v3: atomic-free split into a dK/dV kernel and a dQ kernel
// =====================================================================================
//
// dK/dV kernel: CTA = one 128-row key tile, walks query tiles diag..end.
//   MMA order per query tile i: S^T(i), dP^T(i), [P^T(i) in TMEM] dV += P^T dO,
//   [dS^T(i) in smem] dK += dS^T Q; S^T(i+1) follows immediately (P^T(i) was
//   consumed by dV(i) earlier in the same in-order MMA stream).
//   TMEM: dK 0-127 | dV 128-255 | S^T (P^T at 256+64g) 256-383 | dP^T 384-511.
// dQ kernel: CTA = one 128-row query tile, walks key tiles 0..diag.
//   S(j) double-buffered in TMEM so S(j+1) overlaps the softmax of tile j;
//   dQ accumulates in TMEM across all key tiles and is written once as bf16.
//   TMEM: S0 0-127 | S1 128-255 | dP 256-383 | dQ 384-511.
// Both: warps 0-7 compute (warpgroup g owns columns [64g, 64g+64) of the
// 128-wide score tiles, thread = TMEM lane = row), warp 8 TMA, warp 9 MMA.

constexpr int BWD3_THREADS = 320;

template <int D>
struct KVSmem {
  static constexpr int K = 0;
  static constexpr int V = K + Tile<D>::BYTES;
  static constexpr int Q = V + Tile<D>::BYTES;        // 2 stages
  static constexpr int DO = Q + 2 * Tile<D>::BYTES;   // 2 stages
  static constexpr int DST = DO + 2 * Tile<D>::BYTES;  // dS^T [kv x q]
  static constexpr int STAT = DST + AT_TILE * AT_TILE * 2;  // [2 slots][lse2 | delta][128]
  static constexpr int BAR = STAT + 2 * 2 * AT_TILE * 4;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(BWD3_THREADS, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                         const AttnParams p) {
  using L = KVSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* kv_full = bars;        // 1
  uint64_t* qdo_full = bars + 1;   // 2
  uint64_t* qdo_empty = bars + 3;  // 2
  uint64_t* s_full = bars + 5;
  uint64_t* dp_full = bars + 6;
  uint64_t* p_full = bars + 7;     // 256 arrivals
  uint64_t* ds_full = bars + 8;    // 256 arrivals
  uint64_t* acc_full = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  float* stat = reinterpret_cast<float*>(smem + L::STAT);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int kt = static_cast<int>(blockIdx.x);
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;
  const int n_it = nq - kt;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    for (int i = 0; i < 10; ++i) mbar_init(&bars[i], (i == 7 || i == 8) ? 256 : 1);
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
      tma_tile<D>(smem + L::K, &tm_qkv, kv_full, kcol, bi, kt * AT_TILE);
      tma_tile<D>(smem + L::V, &tm_qkv, kv_full, vcol, bi, kt * AT_TILE);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1, q0 = (kt + it) * AT_TILE;
        mbar_wait(&qdo_empty[st], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qdo_full[st], 2 * Tile<D>::BYTES);
        tma_tile<D>(smem + L::Q + st * Tile<D>::BYTES, &tm_qkv, &qdo_full[st], qcol, bi, q0);
        tma_tile<D>(smem + L::DO + st * Tile<D>::BYTES, &tm_do, &qdo_full[st], head * D, bi, q0);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_sp = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_kv = idesc_bf16(128, D, false, true);
      const uint32_t sk = smem_u32(smem + L::K), sv = smem_u32(smem + L::V);
      const uint32_t sdst = smem_u32(smem + L::DST);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1;
        const uint32_t sq = smem_u32(smem + L::Q + st * Tile<D>::BYTES);
        const uint32_t sdo = smem_u32(smem + L::DO + st * Tile<D>::BYTES);
        mbar_wait(&qdo_full[st], (it >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tS, kmajor_desc(sk, kk), kmajor_desc(sq, kk), id_sp, kk > 0);
        umma_commit(s_full);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tDP, kmajor_desc(sv, kk), kmajor_desc(sdo, kk), id_sp, kk > 0);
        umma_commit(dp_full);
        mbar_wait(p_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts(tDV, tS + (kk >> 2) * 64 + (kk & 3) * 8, mnmajor_desc(sdo, kk), id_kv,
                      it > 0 || kk > 0);
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ss(tDK, kmajor_desc(sdst, kk), mnmajor_desc(sq, kk), id_kv, it > 0 || kk > 0);
        umma_commit(&qdo_empty[st]);
      }
      umma_commit(acc_full);
    }
  } else {
    const int g = warp >> 2, quad = warp & 3;
    const int c = quad * 32 + lane;
    const int qoff = 64 * g;
    const int ct = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row_base = static_cast<int64_t>(bh) * p.s;
    uint8_t* dst = smem + L::DST;
    for (int it = 0; it < n_it; ++it) {
      const int qtile = kt + it, q0 = qtile * AT_TILE;
      float* s_lse = stat + (it & 1) * 2 * AT_TILE;
      float* s_del = s_lse + AT_TILE;
      {
        const int qi = ct & (AT_TILE - 1);
        const int q = q0 + qi;
        if (ct < AT_TILE) s_lse[qi] = q < p.s ? p.lse[row_base + q] * LOG2E : 0.f;
        else s_del[qi] = q < p.s ? p.delta[row_base + q] : 0.f;
      }
      named_barrier_sync(1, 256);
      const bool diag = (qtile == kt);
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      uint32_t raw[64];
      tmem_ld32(tS + lane_off + qoff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tS + lane_off + qoff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int qi = qoff + 2 * j;
        float p0 = fast_exp2(fmaf(__uint_as_float(raw[2 * j]), p.scale_log2, -s_lse[qi]));
        float p1 = fast_exp2(fmaf(__uint_as_float(raw[2 * j + 1]), p.scale_log2, -s_lse[qi + 1]));
        if ((diag && qi < c) || q0 + qi >= p.s) p0 = 0.f;
        if ((diag && qi + 1 < c) || q0 + qi + 1 >= p.s) p1 = 0.f;
        pk[j] = pack_bf16(p0, p1);
      }
      tmem_st32(tS + lane_off + qoff, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
      mbar_wait(dp_full, it & 1);
      tc_fence_after();
      tmem_ld32(tDP + lane_off + qoff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tDP + lane_off + qoff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = v * 4 + i;  // packed pair index
          const float2 pp = unpack_bf16(pk[j]);
          const int qi = qoff + 2 * j;
          w[i] = pack_bf16(pp.x * (__uint_as_float(raw[2 * j]) - s_del[qi]),
                           pp.y * (__uint_as_float(raw[2 * j + 1]) - s_del[qi + 1]));
        }
        *reinterpret_cast<uint4*>(dst + swz_off(c, qoff + v * 8)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int krow = kt * AT_TILE + c;
    const int64_t tok = static_cast<int64_t>(krow) * p.b + bi;
    __nv_bfloat16* dk = p.dqkv + tok * p.ld_dqkv + p.h + head * D;
    __nv_bfloat16* dv = p.dqkv + tok * p.ld_dqkv + 2 * p.h + head * D;
#pragma unroll
    for (int ch = 0; ch < D / 64; ++ch) {
      const int col = g * (D / 2) + ch * 32;
      uint32_t rk[32], rv[32];
      tmem_ld32(tDK + lane_off + col, rk);
      tmem_ld32(tDV + lane_off + col, rv);
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
          *reinterpret_cast<uint4*>(dk + col + v * 8) =
              make_uint4(pack_bf16(fk[0], fk[1]), pack_bf16(fk[2], fk[3]), pack_bf16(fk[4], fk[5]), pack_bf16(fk[6], fk[7]));
          *reinterpret_cast<uint4*>(dv + col + v * 8) =
              make_uint4(pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
struct QSmem {
  static constexpr int Q = 0;
  static constexpr int DO = Q + Tile<D>::BYTES;
  static constexpr int KV = DO + Tile<D>::BYTES;          // 2 stages x (K, V)
  static constexpr int DS = KV + 4 * Tile<D>::BYTES;       // dS [q x kv]
  static constexpr int BAR = DS + AT_TILE * AT_TILE * 2;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(BWD3_THREADS, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                       const AttnParams p) {
  using L = QSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;          // 1
  uint64_t* kv_full = bars + 1;     // 2
  uint64_t* kv_empty = bars + 3;    // 2
  uint64_t* s_full = bars + 5;      // 2
  uint64_t* s_free = bars + 7;      // 2, 256 arrivals
  uint64_t* dp_full = bars + 9;
  uint64_t* ds_full = bars + 10;    // 256 arrivals
  uint64_t* dq_done = bars + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int qt = nq - 1 - static_cast<int>(blockIdx.x);
  const int nkv = qt + 1;
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    for (int i = 0; i < 12; ++i)
      mbar_init(&bars[i], (i == 7 || i == 8 || i == 10) ? 256 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDP = tmem + 256, tDQ = tmem + 384;

  if (warp == 8) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * Tile<D>::BYTES);
      tma_tile<D>(smem + L::Q, &tm_qkv, q_full, qcol, bi, qt * AT_TILE);
      tma_tile<D>(smem + L::DO, &tm_do, q_full, head * D, bi, qt * AT_TILE);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* kb = smem + L::KV + st * 2 * Tile<D>::BYTES;
        mbar_arrive_expect_tx(&kv_full[st], 2 * Tile<D>::BYTES);
        tma_tile<D>(kb, &tm_qkv, &kv_full[st], kcol, bi, j * AT_TILE);
        tma_tile<D>(kb + Tile<D>::BYTES, &tm_qkv, &kv_full[st], vcol, bi, j * AT_TILE);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_sp = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_q = idesc_bf16(128, D, false, true);
      const uint32_t sq = smem_u32(smem + L::Q), sdo = smem_u32(smem + L::DO);
      const uint32_t sds = smem_u32(smem + L::DS);
      auto sk = [&](int j) { return smem_u32(smem + L::KV + (j & 1) * 2 * Tile<D>::BYTES); };
      auto issue_s = [&](int j) {
        mbar_wait(&kv_full[j & 1], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&s_free[j & 1], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t ts = tmem + (j & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(ts, kmajor_desc(sq, kk), kmajor_desc(sk(j), kk), id_sp, kk > 0);
        umma_commit(&s_full[j & 1]);
      };
      auto issue_dp = [&](int j) {
        const uint32_t sv = sk(j) + Tile<D>::BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tDP, kmajor_desc(sdo, kk), kmajor_desc(sv, kk), id_sp, kk > 0);
        umma_commit(dp_full);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      issue_dp(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ss(tDQ, kmajor_desc(sds, kk), mnmajor_desc(sk(j), kk), id_q, j > 0 || kk > 0);
        umma_commit(&kv_empty[j & 1]);
        if (j + 1 < nkv) issue_dp(j + 1);
      }
      umma_commit(dq_done);
    }
  } else {
    // compute: thread = query row r; warpgroup g owns key columns [64g, 64g+64)
    const int g = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const int koff = 64 * g;
    const int q = qt * AT_TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row = static_cast<int64_t>(bh) * p.s + q;
    const float lse2 = q < p.s ? p.lse[row] * LOG2E : 0.f;
    const float dlt = q < p.s ? p.delta[row] : 0.f;
    uint8_t* ds_s = smem + L::DS;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t raw[64];
      const uint32_t ts = tmem + (j & 1) * 128 + lane_off + koff;
      tmem_ld32(ts, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(ts + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_free[j & 1]);
      const bool diag = (j == qt);
      float pv[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        float pr = fast_exp2(fmaf(__uint_as_float(raw[i]), p.scale_log2, -lse2));
        if (diag && koff + i > r) pr = 0.f;
        pv[i] = pr;
      }
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
      tmem_ld32(tDP + lane_off + koff, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tDP + lane_off + koff + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        float ds[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) ds[i] = pv[v * 8 + i] * (__uint_as_float(raw[v * 8 + i]) - dlt);
        *reinterpret_cast<uint4*>(ds_s + swz_off(r, koff + v * 8)) =
            make_uint4(pack_bf16(ds[0], ds[1]), pack_bf16(ds[2], ds[3]), pack_bf16(ds[4], ds[5]),
                       pack_bf16(ds[6], ds[7]));
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    __nv_bfloat16* dqp = p.dqkv + (static_cast<int64_t>(q) * p.b + bi) * p.ld_dqkv + head * D;
#pragma unroll
    for (int ch = 0; ch < D / 64; ++ch) {
      const int col = g * (D / 2) + ch * 32;
      uint32_t rq[32];
      tmem_ld32(tDQ + lane_off + col, rq);
      tmem_wait_ld();
      if (q < p.s) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(rq[v * 8 + i]) * p.scale;
          *reinterpret_cast<uint4*>(dqp + col + v * 8) =
              make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// =====================================================================================
// backward v4: split kernels with a 64-wide streamed tile, double-buffered S/dP
// =====================================================================================
//
// Halving the streamed tile (query tile in dK/dV, key tile in dQ) to 64 lets both
// score tiles (S and dP) be double-buffered in TMEM next to the two 128-column
// accumulators, so the tensor core computes S/dP of tile i+1 while the compute
// warps turn tile i into P and dS.  N=64 MMAs keep the per-FLOP rate of N=128.
//
// dK/dV: TMEM dK 0-127 | dV 128-255 | S^T[b] 256+64b (P^T in its first 32 cols,
//        16 per warpgroup) | dP^T[b] 384+64b.   smem: K, V (128 rows), Q / dO
//        (64 rows, 3 stages), dS^T [128 x 64] x 2.
// dQ:    TMEM S[b] 64b | dP[b] 128+64b | dQ 256-383.   smem: Q, dO (128 rows),
//        K / V (64 rows, 3 stages), dS [128 x 64] x 2.
constexpr int BT = 64;        // streamed tile
constexpr int BT_STAGES = 3;

template <int D>
struct Half {  // [64 rows x D] tile
  static constexpr int BYTES = BT * D * 2;
};

// K-major / MN-major descriptors for tiles with `rows` rows (atom = rows*128 bytes).
HX_DEVICE uint64_t kdesc(uint32_t base, int kk, int rows) {
  return sw128_desc(base + (kk >> 2) * rows * 128 + (kk & 3) * 32, 16, 1024);
}
HX_DEVICE uint64_t mndesc(uint32_t base, int kk, int rows) {
  return sw128_desc(base + kk * 2048, rows * 128, 1024);
}
template <int D>
HX_DEVICE void tma_tile_rows(void* dst, const CUtensorMap* map, uint64_t* bar, int col0, int bi, int s0, int rows) {
#pragma unroll
  for (int a = 0; a < D / 64; ++a)
    tma_load_3d(static_cast<uint8_t*>(dst) + a * rows * 128, map, bar, col0 + 64 * a, bi, s0);
}
// 64-row swizzled tile: byte offset of 16-byte chunk (row, col), col < 64.
HX_DEVICE uint32_t swz64(int row, int col) { return row * 128 + ((((col >> 3) & 7) ^ (row & 7)) << 4); }

constexpr int BWD4_THREADS = 320;

template <int D>
struct KV4Smem {
  static constexpr int K = 0;
  static constexpr int V = K + Tile<D>::BYTES;
  static constexpr int Q = V + Tile<D>::BYTES;              // BT_STAGES x [64 x D]
  static constexpr int DO = Q + BT_STAGES * Half<D>::BYTES;  // BT_STAGES x [64 x D]
  static constexpr int DST = DO + BT_STAGES * Half<D>::BYTES;  // 2 x [128 x 64]
  static constexpr int STAT = DST + 2 * AT_TILE * BT * 2;     // [2][lse2 | delta][64]
  static constexpr int BAR = STAT + 2 * 2 * BT * 4;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(BWD4_THREADS, 1)
    attn_bwd_dkdv4_kernel(const __grid_constant__ CUtensorMap tm_qkv128, const __grid_constant__ CUtensorMap tm_qkv64,
                          const __grid_constant__ CUtensorMap tm_do64, const AttnParams p) {
  using L = KV4Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* kv_full = bars;                  // 1
  uint64_t* qdo_full = bars + 1;             // BT_STAGES
  uint64_t* qdo_empty = bars + 4;            // BT_STAGES
  uint64_t* sdp_full = bars + 7;             // 2
  uint64_t* p_full = bars + 9;               // 256 arrivals
  uint64_t* ds_full = bars + 10;             // 256 arrivals
  uint64_t* acc_full = bars + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  float* stat = reinterpret_cast<float*>(smem + L::STAT);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + BT - 1) / BT;           // 64-row query tiles
  const int kt = static_cast<int>(blockIdx.x);  // 128-row key tile
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;
  const int q_first = 2 * kt;                   // first query tile touching the diagonal
  const int n_it = nq - q_first;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv128);
    tma_prefetch(&tm_qkv64);
    tma_prefetch(&tm_do64);
    for (int i = 0; i < 12; ++i) mbar_init(&bars[i], (i == 9 || i == 10) ? 256 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDK = tmem, tDV = tmem + 128, tS0 = tmem + 256, tDP0 = tmem + 384;

  if (warp == 8) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * Tile<D>::BYTES);
      tma_tile_rows<D>(smem + L::K, &tm_qkv128, kv_full, kcol, bi, kt * AT_TILE, AT_TILE);
      tma_tile_rows<D>(smem + L::V, &tm_qkv128, kv_full, vcol, bi, kt * AT_TILE, AT_TILE);
      for (int it = 0; it < n_it; ++it) {
        const int st = it % BT_STAGES, q0 = (q_first + it) * BT;
        mbar_wait(&qdo_empty[st], ((it / BT_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&qdo_full[st], 2 * Half<D>::BYTES);
        tma_tile_rows<D>(smem + L::Q + st * Half<D>::BYTES, &tm_qkv64, &qdo_full[st], qcol, bi, q0, BT);
        tma_tile_rows<D>(smem + L::DO + st * Half<D>::BYTES, &tm_do64, &qdo_full[st], head * D, bi, q0, BT);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_sp = idesc_bf16(128, BT, false, false);  // S^T, dP^T: M=128 kv, N=64 q
      constexpr uint32_t id_kv = idesc_bf16(128, D, false, true);    // dV, dK
      const uint32_t sk = smem_u32(smem + L::K), sv = smem_u32(smem + L::V);
      auto issue_sdp = [&](int it) {
        const int st = it % BT_STAGES, b = it & 1;
        mbar_wait(&qdo_full[st], (it / BT_STAGES) & 1);
        tc_fence_after();
        const uint32_t sq = smem_u32(smem + L::Q + st * Half<D>::BYTES);
        const uint32_t sdo = smem_u32(smem + L::DO + st * Half<D>::BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tS0 + 64 * b, kdesc(sk, kk, AT_TILE), kdesc(sq, kk, BT), id_sp, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tDP0 + 64 * b, kdesc(sv, kk, AT_TILE), kdesc(sdo, kk, BT), id_sp, kk > 0);
        umma_commit(&sdp_full[b]);
      };
      mbar_wait(kv_full, 0);
      issue_sdp(0);
      for (int it = 0; it < n_it; ++it) {
        const int st = it % BT_STAGES, b = it & 1;
        if (it + 1 < n_it) issue_sdp(it + 1);
        const uint32_t sq = smem_u32(smem + L::Q + st * Half<D>::BYTES);
        const uint32_t sdo = smem_u32(smem + L::DO + st * Half<D>::BYTES);
        const uint32_t sdst = smem_u32(smem + L::DST + b * AT_TILE * BT * 2);
        mbar_wait(p_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk)  // P^T of warpgroup kk/2 at S^T[b] + 32*(kk/2)
          umma_f16_ts(tDV, tS0 + 64 * b + (kk >> 1) * 32 + (kk & 1) * 8, mndesc(sdo, kk, BT), id_kv,
                      it > 0 || kk > 0);
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk)
          umma_f16_ss(tDK, kdesc(sdst, kk, AT_TILE), mndesc(sq, kk, BT), id_kv, it > 0 || kk > 0);
        umma_commit(&qdo_empty[st]);
      }
      umma_commit(acc_full);
    }
  } else {
    // compute: thread = key row c; warpgroup g owns query columns [32g, 32g+32) of each tile
    const int g = warp >> 2, quad = warp & 3;
    const int c = quad * 32 + lane;
    const int qoff = 32 * g;
    const int ct = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row_base = static_cast<int64_t>(bh) * p.s;
    const int kv_row = kt * AT_TILE + c;
    for (int it = 0; it < n_it; ++it) {
      const int b = it & 1;
      const int q0 = (q_first + it) * BT;
      float* s_lse = stat + b * 2 * BT;
      float* s_del = s_lse + BT;
      if (ct < 2 * BT) {
        const int qi = ct & (BT - 1);
        const int q = q0 + qi;
        if (ct < BT) s_lse[qi] = q < p.s ? p.lse[row_base + q] * LOG2E : 0.f;
        else s_del[qi] = q < p.s ? p.delta[row_base + q] : 0.f;
      }
      named_barrier_sync(1, 256);
      mbar_wait(&sdp_full[b], (it >> 1) & 1);
      tc_fence_after();
      uint32_t rs[32], rd[32];
      tmem_ld32(tS0 + 64 * b + lane_off + qoff, rs);
      tmem_ld32(tDP0 + 64 * b + lane_off + qoff, rd);
      tmem_wait_ld();
      const bool need_mask = q0 < (kt + 1) * AT_TILE || q0 + BT > p.s;  // tile touches the diagonal / tail
      uint32_t pk[16];
      float ds[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int qi = qoff + j;
        float pr = fast_exp2(fmaf(__uint_as_float(rs[j]), p.scale_log2, -s_lse[qi]));
        if (need_mask && (q0 + qi < kv_row || q0 + qi >= p.s)) pr = 0.f;
        ds[j] = pr * (__uint_as_float(rd[j]) - s_del[qi]);
        rs[j] = __float_as_uint(pr);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(__uint_as_float(rs[2 * j]), __uint_as_float(rs[2 * j + 1]));
      tmem_st16(tS0 + 64 * b + lane_off + qoff, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
      uint8_t* dst = smem + L::DST + b * AT_TILE * BT * 2;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        *reinterpret_cast<uint4*>(dst + swz64(c, qoff + v * 8)) =
            make_uint4(pack_bf16(ds[v * 8], ds[v * 8 + 1]), pack_bf16(ds[v * 8 + 2], ds[v * 8 + 3]),
                       pack_bf16(ds[v * 8 + 4], ds[v * 8 + 5]), pack_bf16(ds[v * 8 + 6], ds[v * 8 + 7]));
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int64_t tok = static_cast<int64_t>(kv_row) * p.b + bi;
    __nv_bfloat16* dk = p.dqkv + tok * p.ld_dqkv + p.h + head * D;
    __nv_bfloat16* dv = p.dqkv + tok * p.ld_dqkv + 2 * p.h + head * D;
#pragma unroll
    for (int ch = 0; ch < D / 64; ++ch) {
      const int col = g * (D / 2) + ch * 32;
      uint32_t rk[32], rv[32];
      tmem_ld32(tDK + lane_off + col, rk);
      tmem_ld32(tDV + lane_off + col, rv);
      tmem_wait_ld();
      if (kv_row < p.s) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float fk[8], fv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            fk[i] = __uint_as_float(rk[v * 8 + i]) * p.scale;
            fv[i] = __uint_as_float(rv[v * 8 + i]);
          }
          *reinterpret_cast<uint4*>(dk + col + v * 8) =
              make_uint4(pack_bf16(fk[0], fk[1]), pack_bf16(fk[2], fk[3]), pack_bf16(fk[4], fk[5]), pack_bf16(fk[6], fk[7]));
          *reinterpret_cast<uint4*>(dv + col + v * 8) =
              make_uint4(pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
struct Q4Smem {
  static constexpr int Q = 0;
  static constexpr int DO = Q + Tile<D>::BYTES;
  static constexpr int KV = DO + Tile<D>::BYTES;             // BT_STAGES x (K, V) [64 x D]
  static constexpr int DS = KV + BT_STAGES * 2 * Half<D>::BYTES;  // 2 x [128 x 64]
  static constexpr int BAR = DS + 2 * AT_TILE * BT * 2;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(BWD4_THREADS, 1)
    attn_bwd_dq4_kernel(const __grid_constant__ CUtensorMap tm_qkv128, const __grid_constant__ CUtensorMap tm_qkv64,
                        const __grid_constant__ CUtensorMap tm_do128, const AttnParams p) {
  using L = Q4Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;               // 1
  uint64_t* kv_full = bars + 1;          // BT_STAGES
  uint64_t* kv_empty = bars + 4;         // BT_STAGES
  uint64_t* sdp_full = bars + 7;         // 2
  uint64_t* ds_full = bars + 9;          // 256 arrivals
  uint64_t* dq_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int qt = nq - 1 - static_cast<int>(blockIdx.x);
  const int q_last = min(p.s, (qt + 1) * AT_TILE) - 1;
  const int nkv = q_last / BT + 1;  // 64-row key tiles 0 .. diag
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv128);
    tma_prefetch(&tm_qkv64);
    tma_prefetch(&tm_do128);
    for (int i = 0; i < 11; ++i) mbar_init(&bars[i], i == 9 ? 256 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS0 = tmem, tDP0 = tmem + 128, tDQ = tmem + 256;

  if (warp == 8) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * Tile<D>::BYTES);
      tma_tile_rows<D>(smem + L::Q, &tm_qkv128, q_full, qcol, bi, qt * AT_TILE, AT_TILE);
      tma_tile_rows<D>(smem + L::DO, &tm_do128, q_full, head * D, bi, qt * AT_TILE, AT_TILE);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % BT_STAGES;
        mbar_wait(&kv_empty[st], ((j / BT_STAGES) & 1) ^ 1);
        uint8_t* kb = smem + L::KV + st * 2 * Half<D>::BYTES;
        mbar_arrive_expect_tx(&kv_full[st], 2 * Half<D>::BYTES);
        tma_tile_rows<D>(kb, &tm_qkv64, &kv_full[st], kcol, bi, j * BT, BT);
        tma_tile_rows<D>(kb + Half<D>::BYTES, &tm_qkv64, &kv_full[st], vcol, bi, j * BT, BT);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_sp = idesc_bf16(128, BT, false, false);  // S, dP: M=128 q, N=64 kv
      constexpr uint32_t id_q = idesc_bf16(128, D, false, true);     // dQ += dS K
      const uint32_t sq = smem_u32(smem + L::Q), sdo = smem_u32(smem + L::DO);
      auto skv = [&](int j) { return smem_u32(smem + L::KV + (j % BT_STAGES) * 2 * Half<D>::BYTES); };
      auto issue_sdp = [&](int j) {
        const int st = j % BT_STAGES, b = j & 1;
        mbar_wait(&kv_full[st], (j / BT_STAGES) & 1);
        tc_fence_after();
        const uint32_t sk = skv(j), sv = sk + Half<D>::BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tS0 + 64 * b, kdesc(sq, kk, AT_TILE), kdesc(sk, kk, BT), id_sp, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ss(tDP0 + 64 * b, kdesc(sdo, kk, AT_TILE), kdesc(sv, kk, BT), id_sp, kk > 0);
        umma_commit(&sdp_full[b]);
      };
      mbar_wait(q_full, 0);
      issue_sdp(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_sdp(j + 1);
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
        const uint32_t sds = smem_u32(smem + L::DS + (j & 1) * AT_TILE * BT * 2);
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk)
          umma_f16_ss(tDQ, kdesc(sds, kk, AT_TILE), mndesc(skv(j), kk, BT), id_q, j > 0 || kk > 0);
        umma_commit(&kv_empty[j % BT_STAGES]);
      }
      umma_commit(dq_done);
    }
  } else {
    // compute: thread = query row r; warpgroup g owns key columns [32g, 32g+32)
    const int g = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const int koff = 32 * g;
    const int q = qt * AT_TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const int64_t row = static_cast<int64_t>(bh) * p.s + q;
    const float lse2 = q < p.s ? p.lse[row] * LOG2E : 0.f;
    const float dlt = q < p.s ? p.delta[row] : 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      mbar_wait(&sdp_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t rs[32], rd[32];
      tmem_ld32(tS0 + 64 * b + lane_off + koff, rs);
      tmem_ld32(tDP0 + 64 * b + lane_off + koff, rd);
      tmem_wait_ld();
      const int k0 = j * BT + koff;
      const bool need_mask = k0 + 31 > qt * AT_TILE;  // some key index may exceed some query index
      float ds[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float pr = fast_exp2(fmaf(__uint_as_float(rs[i]), p.scale_log2, -lse2));
        if (need_mask && k0 + i > q) pr = 0.f;
        ds[i] = pr * (__uint_as_float(rd[i]) - dlt);
      }
      uint8_t* dss = smem + L::DS + b * AT_TILE * BT * 2;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        *reinterpret_cast<uint4*>(dss + swz64(r, koff + v * 8)) =
            make_uint4(pack_bf16(ds[v * 8], ds[v * 8 + 1]), pack_bf16(ds[v * 8 + 2], ds[v * 8 + 3]),
                       pack_bf16(ds[v * 8 + 4], ds[v * 8 + 5]), pack_bf16(ds[v * 8 + 6], ds[v * 8 + 7]));
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    __nv_bfloat16* dqp = p.dqkv + (static_cast<int64_t>(q) * p.b + bi) * p.ld_dqkv + head * D;
#pragma unroll
    for (int ch = 0; ch < D / 64; ++ch) {
      const int col = g * (D / 2) + ch * 32;
      uint32_t rq[32];
      tmem_ld32(tDQ + lane_off + col, rq);
      tmem_wait_ld();
      if (q < p.s) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(rq[v * 8 + i]) * p.scale;
          *reinterpret_cast<uint4*>(dqp + col + v * 8) =
              make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// =====================================================================================
// dQ kernel v5: every A operand in TMEM (smem traffic = one 64-row B tile per MMA)
// =====================================================================================
//
// Q and dO are constant for the CTA: the compute warps copy them once into TMEM
// in the packed A-operand layout (lane = query row, column c = K pair 2c,2c+1).
// dS(j) goes from registers straight into TMEM over its own S columns.  All
// three MMAs per 64-row key tile are then TS-form, reading only K_j / V_j from
// shared memory: S = Q K_j^T, dP = dO V_j^T, dQ += dS K_j.
// TMEM: S[b] 64b (dS at S[b] + 32g) | dP[b] 128+64b | dQ 256 | Q 384 | dO 384+D/2.

template <int D>
struct Q5Smem {
  static constexpr int STAGES = 4;
  static constexpr int KV = 0;  // STAGES x (K, V) [64 x D]
  static constexpr int BAR = KV + STAGES * 2 * Half<D>::BYTES;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(BWD4_THREADS, 1)
    attn_bwd_dq5_kernel(const __grid_constant__ CUtensorMap tm_qkv64, const __nv_bfloat16* __restrict__ qkv,
                        int ld_qkv, const __nv_bfloat16* __restrict__ d_o, int ld_o, const AttnParams p) {
  using L = Q5Smem<D>;
  constexpr int ST = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* kv_full = bars;             // ST
  uint64_t* kv_empty = bars + ST;       // ST
  uint64_t* sdp_full = bars + 2 * ST;   // 2
  uint64_t* ds_full = bars + 2 * ST + 2;  // 256 arrivals
  uint64_t* qdo_ready = bars + 2 * ST + 3;  // 256 arrivals
  uint64_t* dq_done = bars + 2 * ST + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 5);
  constexpr int NBARS = 2 * ST + 5;

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int qt = nq - 1 - static_cast<int>(blockIdx.x);
  const int q_last = min(p.s, (qt + 1) * AT_TILE) - 1;
  const int nkv = q_last / BT + 1;
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv64);
    for (int i = 0; i < NBARS; ++i)
      mbar_init(&bars[i], (i == 2 * ST + 2 || i == 2 * ST + 3) ? 256 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS0 = tmem, tDP0 = tmem + 128, tDQ = tmem + 256, tQ = tmem + 384, tDO = tmem + 384 + D / 2;

  if (warp == 8) {
    if (lane == 0) {
      for (int j = 0; j < nkv; ++j) {
        const int st = j % ST;
        mbar_wait(&kv_empty[st], ((j / ST) & 1) ^ 1);
        uint8_t* kb = smem + L::KV + st * 2 * Half<D>::BYTES;
        mbar_arrive_expect_tx(&kv_full[st], 2 * Half<D>::BYTES);
        tma_tile_rows<D>(kb, &tm_qkv64, &kv_full[st], kcol, bi, j * BT, BT);
        tma_tile_rows<D>(kb + Half<D>::BYTES, &tm_qkv64, &kv_full[st], vcol, bi, j * BT, BT);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t id_sp = idesc_bf16(128, BT, false, false);
      constexpr uint32_t id_q = idesc_bf16(128, D, false, true);
      auto skv = [&](int j) { return smem_u32(smem + L::KV + (j % ST) * 2 * Half<D>::BYTES); };
      auto issue_sdp = [&](int j) {
        const int b = j & 1;
        mbar_wait(&kv_full[j % ST], (j / ST) & 1);
        tc_fence_after();
        const uint32_t sk = skv(j), sv = sk + Half<D>::BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ts(tS0 + 64 * b, tQ + kk * 8, kdesc(sk, kk, BT), id_sp, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ts(tDP0 + 64 * b, tDO + kk * 8, kdesc(sv, kk, BT), id_sp, kk > 0);
        umma_commit(&sdp_full[b]);
      };
      mbar_wait(qdo_ready, 0);
      tc_fence_after();
      issue_sdp(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_sdp(j + 1);
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
        const uint32_t tds = tS0 + 64 * (j & 1);
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk)
          umma_f16_ts(tDQ, tds + (kk >> 1) * 32 + (kk & 1) * 8, mndesc(skv(j), kk, BT), id_q, j > 0 || kk > 0);
        umma_commit(&kv_empty[j % ST]);
      }
      umma_commit(dq_done);
    }
  } else {
    const int g = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const int koff = 32 * g;
    const int q = qt * AT_TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    {  // Q and dO rows -> TMEM (this warpgroup's half of the head dimension)
      const int64_t tok = static_cast<int64_t>(q) * p.b + bi;
      const uint4* qsrc = reinterpret_cast<const uint4*>(qkv + tok * ld_qkv + head * D + g * (D / 2));
      const uint4* osrc = reinterpret_cast<const uint4*>(d_o + tok * ld_o + head * D + g * (D / 2));
      // D/2 bf16 per warpgroup = D/16 uint4 = D/4 packed TMEM columns
      if constexpr (D == 128) {
        uint32_t wq[32], wo[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 a = q < p.s ? qsrc[v] : make_uint4(0, 0, 0, 0);
          const uint4 o = q < p.s ? osrc[v] : make_uint4(0, 0, 0, 0);
          wq[4 * v] = a.x; wq[4 * v + 1] = a.y; wq[4 * v + 2] = a.z; wq[4 * v + 3] = a.w;
          wo[4 * v] = o.x; wo[4 * v + 1] = o.y; wo[4 * v + 2] = o.z; wo[4 * v + 3] = o.w;
        }
        tmem_st32(tQ + lane_off + g * 32, wq);
        tmem_st32(tDO + lane_off + g * 32, wo);
      } else {
        uint32_t wq[16], wo[16];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint4 a = q < p.s ? qsrc[v] : make_uint4(0, 0, 0, 0);
          const uint4 o = q < p.s ? osrc[v] : make_uint4(0, 0, 0, 0);
          wq[4 * v] = a.x; wq[4 * v + 1] = a.y; wq[4 * v + 2] = a.z; wq[4 * v + 3] = a.w;
          wo[4 * v] = o.x; wo[4 * v + 1] = o.y; wo[4 * v + 2] = o.z; wo[4 * v + 3] = o.w;
        }
        tmem_st16(tQ + lane_off + g * 16, wq);
        tmem_st16(tDO + lane_off + g * 16, wo);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(qdo_ready);
    }
    const int64_t row = static_cast<int64_t>(bh) * p.s + q;
    const float lse2 = q < p.s ? p.lse[row] * LOG2E : 0.f;
    const float dlt = q < p.s ? p.delta[row] : 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      mbar_wait(&sdp_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t rs[32], rd[32];
      tmem_ld32(tS0 + 64 * b + lane_off + koff, rs);
      tmem_ld32(tDP0 + 64 * b + lane_off + koff, rd);
      tmem_wait_ld();
      const int k0 = j * BT + koff;
      const bool need_mask = k0 + 31 > qt * AT_TILE;
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float p0 = fast_exp2(fmaf(__uint_as_float(rs[2 * i]), p.scale_log2, -lse2));
        float p1 = fast_exp2(fmaf(__uint_as_float(rs[2 * i + 1]), p.scale_log2, -lse2));
        if (need_mask && k0 + 2 * i > q) p0 = 0.f;
        if (need_mask && k0 + 2 * i + 1 > q) p1 = 0.f;
        pk[i] = pack_bf16(p0 * (__uint_as_float(rd[2 * i]) - dlt), p1 * (__uint_as_float(rd[2 * i + 1]) - dlt));
      }
      tmem_st16(tS0 + 64 * b + lane_off + koff, pk);  // dS over this warpgroup's own S columns
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    __nv_bfloat16* dqp = p.dqkv + (static_cast<int64_t>(q) * p.b + bi) * p.ld_dqkv + head * D;
#pragma unroll
    for (int ch = 0; ch < D / 64; ++ch) {
      const int col = g * (D / 2) + ch * 32;
      uint32_t rq[32];
      tmem_ld32(tDQ + lane_off + col, rq);
      tmem_wait_ld();
      if (q < p.s) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(rq[v * 8 + i]) * p.scale;
          *reinterpret_cast<uint4*>(dqp + col + v * 8) =
              make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
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
      if (dq_acc) {
        reinterpret_cast<uint4*>(dq_acc + row * D)[sub * 2] = make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4*>(dq_acc + row * D)[sub * 2 + 1] = make_uint4(0, 0, 0, 0);
      }
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
  static const bool v1 = getenv("HX_ATTN_FWD_V1") != nullptr;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FwdSmem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_fwd2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Fwd2Smem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  if (v1) {
    attn_fwd_kernel<D><<<dim3(nq, p.b * p.heads), AT_THREADS, FwdSmem<D>::TOTAL, st>>>(tm, p);
  } else {
    attn_fwd2_kernel<D><<<dim3((nq + 1) / 2, p.b * p.heads), FWD2_THREADS, Fwd2Smem<D>::TOTAL, st>>>(tm, p);
  }
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
  // HX_ATTN_BWD=1 / 2: the earlier single-kernel variants with dQ atomics (kept for A/B runs)
  static const int variant = getenv("HX_ATTN_BWD") ? atoi(getenv("HX_ATTN_BWD")) : 4;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdSmem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Bwd2Smem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, KVSmem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, QSmem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dkdv4_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, KV4Smem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq4_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q4Smem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq5_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q5Smem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const bool atomics = variant < 3;
  attn_bwd_pre_kernel<D><<<(tokens + 7) / 8, 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(d_o), ld_o,
      const_cast<float*>(p.delta), atomics ? p.dq_acc : nullptr, p.s, p.b, p.heads);
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  dim3 grid(nq, p.b * p.heads);
  if (variant == 4) {
    CUtensorMap tq64, tdo64;
    e = make_tma_3d_rows(&tq64, qkv, 3 * p.h, p.b, p.s, ld_qkv, 64, BT);
    if (e == cudaSuccess) e = make_tma_3d_rows(&tdo64, d_o, p.h, p.b, p.s, ld_o, 64, BT);
    if (e != cudaSuccess) return e;
    attn_bwd_dkdv4_kernel<D><<<grid, BWD4_THREADS, KV4Smem<D>::TOTAL, st>>>(tq, tq64, tdo64, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static const bool dq4 = getenv("HX_ATTN_DQ4") != nullptr;
    if (dq4)
      attn_bwd_dq4_kernel<D><<<grid, BWD4_THREADS, Q4Smem<D>::TOTAL, st>>>(tq, tq64, tdo, p);
    else
      attn_bwd_dq5_kernel<D><<<grid, BWD4_THREADS, Q5Smem<D>::TOTAL, st>>>(
          tq64, static_cast<const __nv_bfloat16*>(qkv), ld_qkv, static_cast<const __nv_bfloat16*>(d_o), ld_o, p);
    return cudaGetLastError();
  }
  if (!atomics) {
    attn_bwd_dkdv_kernel<D><<<grid, BWD3_THREADS, KVSmem<D>::TOTAL, st>>>(tq, tdo, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    attn_bwd_dq_kernel<D><<<grid, BWD3_THREADS, QSmem<D>::TOTAL, st>>>(tq, tdo, p);
    return cudaGetLastError();
  }
  if (variant == 1)
    attn_bwd_kernel<D><<<grid, AT_THREADS, BwdSmem<D>::TOTAL, st>>>(tq, tdo, p);
  else
    attn_bwd2_kernel<D><<<grid, BWD2_THREADS, Bwd2Smem<D>::TOTAL, st>>>(tq, tdo, p);
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
