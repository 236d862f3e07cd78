// Causal flash attention forward on tcgen05 / TMEM / TMA (sm_100a).
// Replaces the reference's whole-matrix fp64 attention (P/runtime/mathops.py:83-100):
//   O = softmax(Q K^T / sqrt(d) + causal mask) V, plus the natural-log LSE per row.
//
// CTA = query tiles (2t, 2t+1) of one (batch, head); heaviest pairs first.
// Two softmax warpgroups (warps 0-3 -> tile A, 4-7 -> tile B) alternate with the
// tensor core: while group A exponentiates S_A(j), the tensor core runs
// O_B += P_B(j-1) V(j-1) and S_B(j) = Q_B K(j)^T, and vice versa.
//   S = Q K^T    SS-MMA (Q, K from smem)           -> TMEM S_g (fp32, 128 cols)
//   P            bf16, written back over the first 64 columns of S_g
//   O += P V     TS-MMA (A = P from TMEM, B = V MN-major from smem) -> TMEM O_g
// O is rescaled only when a row's running max grows by more than 2^8 (exponents
// stay <= 256, exact in fp32), so rescales are rare after the first tiles.
// Warp 8 issues TMA (Q once, K/V double-buffered), warp 9 issues MMAs and owns TMEM.
// TMEM (512 columns): S_A 0-127 | S_B 128-255 | O_A 256-383 | O_B 384-511.
#include "attention_common.cuh"

namespace hx {

constexpr int FWD_THREADS = 320;

template <int D>
struct FwdSmem {
  static constexpr int QA = 0;
  static constexpr int QB = QA + Tile<D>::BYTES;
  static constexpr int KV = QB + Tile<D>::BYTES;  // 2 stages x (K, V)
  static constexpr int BAR = KV + 4 * Tile<D>::BYTES;
  static constexpr int TOTAL = BAR + 256;
};

template <int D>
__global__ void __launch_bounds__(FWD_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnParams p) {
  using L = FwdSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;          // 1
  uint64_t* k_full = bars + 1;      // 2
  uint64_t* v_full = bars + 3;      // 2
  uint64_t* kv_empty = bars + 5;    // 2
  uint64_t* s_full = bars + 7;      // 2 (per group)
  uint64_t* p_full = bars + 9;      // 2, 128 arrivals each
  uint64_t* o_full = bars + 11;     // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int npairs = (nq + 1) / 2;
  const int t = npairs - 1 - static_cast<int>(blockIdx.x);
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
      tma_tile_rows<D>(smem + L::QA, &tm_qkv, q_full, qcol, bi, qtile[0] * AT_TILE, AT_TILE);
      if (has_b) tma_tile_rows<D>(smem + L::QB, &tm_qkv, q_full, qcol, bi, qtile[1] * AT_TILE, AT_TILE);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* kb = smem + L::KV + st * 2 * Tile<D>::BYTES;
        mbar_arrive_expect_tx(&k_full[st], Tile<D>::BYTES);
        tma_tile_rows<D>(kb, &tm_qkv, &k_full[st], kcol, bi, j * AT_TILE, AT_TILE);
        mbar_arrive_expect_tx(&v_full[st], Tile<D>::BYTES);
        tma_tile_rows<D>(kb + Tile<D>::BYTES, &tm_qkv, &v_full[st], vcol, bi, j * AT_TILE, AT_TILE);
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
      auto issue_pv = [&](int g, int jt) {  // O_g += P_g(jt) V(jt)
        mbar_wait(&p_full[g], pcount[g] & 1);
        ++pcount[g];
        mbar_wait(&v_full[jt & 1], (jt >> 1) & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + L::KV + (jt & 1) * 2 * Tile<D>::BYTES + Tile<D>::BYTES);
        const uint32_t tP = tmem + 128 * g, tO = tmem + 256 + 128 * g;
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts(tO, tP + kk * 8, mndesc(sv, kk, AT_TILE), id_o, (jt > 0 || kk > 0));
        pending[g] = false;
      };
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&k_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + L::KV + (j & 1) * 2 * Tile<D>::BYTES);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (pending[g]) issue_pv(g, j - 1);
          if (j <= last[g]) {  // S_g(j) = Q_g K(j)^T
            const uint32_t tS = tmem + 128 * g;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              umma_f16_ss(tS, kdesc(sq[g], kk, AT_TILE), kdesc(sk, kk, AT_TILE), id_s, kk > 0);
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
        if (j == qt) {  // diagonal tile: key index > query index is masked
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
          // O_g holds PV(j-1): complete, since S_g(j) was issued after it
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
            const float e0 = exp2_mixed(fmaf(__uint_as_float(raw[half * 64 + 2 * i]), c, neg_m), 2 * i);
            const float e1 = exp2_mixed(fmaf(__uint_as_float(raw[half * 64 + 2 * i + 1]), c, neg_m), 2 * i + 1);
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
      __nv_bfloat16* orow = p.o + (static_cast<int64_t>(qrow) * p.b + bi) * p.ld_o + head * D;
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch)
        tmem_row_to_global<32>(tO + ch * 32, orow + ch * 32, 1.f / l_run, qrow < p.s);
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

template <int D>
static cudaError_t fwd_launch(const void* qkv, int ld_qkv, const AttnParams& p, cudaStream_t st) {
  CUtensorMap tm;
  cudaError_t e = make_tma_3d_rows(&tm, qkv, 3 * p.h, p.b, p.s, ld_qkv, 64, AT_TILE);
  if (e != cudaSuccess) return e;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  attn_fwd_kernel<D><<<dim3((nq + 1) / 2, p.b * p.heads), FWD_THREADS, FwdSmem<D>::TOTAL, st>>>(tm, p);
  return cudaGetLastError();
}

cudaError_t attn_fwd_launch(const void* qkv, int ld_qkv, void* o, int ld_o, float* lse, int s, int b,
                            int heads, int d, cudaStream_t st) {
  AttnParams p{};
  p.s = s;
  p.b = b;
  p.heads = heads;
  p.h = heads * d;
  p.scale = 1.0f / sqrtf(static_cast<float>(d));
  p.scale_log2 = p.scale * LOG2E;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.ld_o = ld_o;
  p.lse = lse;
  if (d == 128) return fwd_launch<128>(qkv, ld_qkv, p, st);
  if (d == 64) return fwd_launch<64>(qkv, ld_qkv, p, st);
  return cudaErrorNotSupported;
}

}  // namespace hx
