// Causal flash attention forward, one 128-row query tile per CTA with the score
// tile double-buffered in TMEM (round 2; HX_ATTN_FWD=2 selects it).
//
// The two-tile kernel (attention_fwd.cu) keeps one S buffer per query tile, so
// S(j+1) of a tile can only be issued after PV(j) has read P(j) out of the same
// columns: per tile the chain S -> softmax -> PV -> S is serial, and the
// softmax of one warp per SMSP runs the MUFU at ~72% of its rate.  Here:
//   * one query tile per CTA: O (D cols) + S0 + S1 (128 cols each) fit TMEM, so
//     S(j+1) runs on the tensor core while the softmax works on S(j), and the
//     MMA warp issues PV(j), S(j+2) as soon as P(j) is stored;
//   * both softmax warpgroups work on the same rows: warpgroup h owns keys
//     64h..64h+63 of every row (two warps per SMSP on the exponentials); the
//     half-row maxima are exchanged through shared memory once per step (the
//     speculative-exponential scheme of attention_fwd.cu needs the row max only
//     to decide a redo), and the half row sums once at the end;
//   * P(j) is written over the first 32 columns of each half's own 64, so a
//     redo never needs scores another warp overwrote (they stay in registers).
// TMEM: O 0..D-1 | S0 D..D+127 | S1 D+128..D+255.  Warps 0-3: keys 0-63,
// 4-7: keys 64-127 (thread = query row), 8 TMA, 9 MMA, 10-11 idle.
#include "attention_common.cuh"

namespace hx {

constexpr int F1_THREADS = 384;
constexpr int F1_REGS_SOFTMAX = 208;  // 2 x 128 x 208 + 128 x 80 = 63.5 K of the launch 64.5 K
constexpr int F1_REGS_ISSUE = 80;

template <int D>
struct Fwd1Smem {
  static constexpr int NSLOT_FIT = (227 * 1024 - Tile<D>::BYTES - 4096 - 512) / Tile<D>::BYTES;
  static constexpr int NSLOT = NSLOT_FIT > 8 ? 8 : NSLOT_FIT;
  static constexpr int Q = 0;
  static constexpr int KV = Q + Tile<D>::BYTES;
  static constexpr int XCH = KV + NSLOT * Tile<D>::BYTES;  // [2 step parity][2 halves][128] f32 maxima, then sums
  static constexpr int BAR = XCH + 4 * 2 * 128 * 4;
  static constexpr int TOTAL = BAR + 512;
};

template <int D>
__global__ void __launch_bounds__(F1_THREADS, 1)
    attn_fwd1_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnParams p) {
  using L = Fwd1Smem<D>;
  constexpr int NS = L::NSLOT;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
#ifdef HX_WAIT_DEBUG
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("fwd1: smem base 0x%x bars at 0x%x (q_full, s_full x2, p_full x2, pv_done x2, o_full, kv_full x%d, kv_empty)\n",
           smem_u32(smem), smem_u32(bars), L::NSLOT);
#endif
  uint64_t* q_full = bars;          // 1
  uint64_t* s_full = bars + 1;      // 2 (per S buffer)
  uint64_t* p_full = bars + 3;      // 2, 256 arrivals each
  uint64_t* pv_done = bars + 5;     // 2 (PV of the step that used that buffer)
  uint64_t* o_full = bars + 7;      // 1
  uint64_t* kv_full = bars + 8;     // NS
  uint64_t* kv_empty = bars + 8 + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * NS);
  float* xch = reinterpret_cast<float*>(smem + L::XCH);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  int bh, t;
  band_order(static_cast<int>(blockIdx.x), nq, p.b * p.heads, p.band, bh, t);
  const int qt = nq - 1 - t;  // heaviest query tiles first
  const int nkv = qt + 1;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    for (int i = 0; i < 8 + 2 * NS; ++i) mbar_init(&bars[i], (i == 3 || i == 4) ? 256 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto slot_addr = [&](int n) { return smem + L::KV + (n % NS) * Tile<D>::BYTES; };
  auto finish = [&]() {
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
      tc_fence_after();
      tmem_dealloc(tmem, 512);
    }
  };

  if (warp >= 8) {
    regs_dec<F1_REGS_ISSUE>();
    if (warp == 8 && lane == 0) {  // ---------------- TMA: Q once, K(0) V(0) K(1) V(1) ... through the ring
      mbar_arrive_expect_tx(q_full, Tile<D>::BYTES);
      tma_tile_rows<D>(smem + L::Q, &tm_qkv, q_full, qcol, bi, qt * AT_TILE, AT_TILE);
      for (int n = 0; n < 2 * nkv; ++n) {
        const int sl = n % NS;
        mbar_wait_nohint(&kv_empty[sl], ((n / NS) & 1) ^ 1);
#ifdef HX_FWD_NOKV  // debug-only probe: no K/V traffic after the ring's first fill (wrong results)
        if (n >= NS) {
          mbar_arrive(&kv_full[sl]);
          continue;
        }
#endif
        mbar_arrive_expect_tx(&kv_full[sl], Tile<D>::BYTES);
        tma_tile_rows<D>(slot_addr(n), &tm_qkv, &kv_full[sl], (n & 1) ? vcol : kcol, bi, (n >> 1) * AT_TILE,
                         AT_TILE);
      }
    } else if (warp == 9 && lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t id_s = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_o = idesc_bf16(128, D, false, true);
      const uint32_t sq = smem_u32(smem + L::Q);
      auto wait_slot = [&](int n) {
        mbar_wait_nohint(&kv_full[n % NS], (n / NS) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int j) {  // S_b(j) = Q K(j)^T, b = j & 1
        wait_slot(2 * j);
        const uint32_t sk = smem_u32(slot_addr(2 * j));
        const uint32_t tS = tmem + D + 128 * (j & 1);
        const uint64_t dq = sw128_desc(sq, 16, 1024), dk = sw128_desc(sk, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * AT_TILE * 128 + (kk & 3) * 32) >> 4;
          umma_f16_ss(tS, dq + off, dk + off, id_s, kk > 0);
        }
        umma_commit(&s_full[j & 1]);
        umma_commit(&kv_empty[(2 * j) % NS]);  // K(j) read once S(j) completes
      };
      mbar_wait_nohint(q_full, 0);
      tc_fence_after();
      issue_s(0);
      if (nkv > 1) issue_s(1);
      for (int j = 0; j < nkv; ++j) {
        const int b = j & 1;
        mbar_wait_nohint(&p_full[b], (j >> 1) & 1);
        wait_slot(2 * j + 1);
        const uint32_t sv = smem_u32(slot_addr(2 * j + 1));
        const uint32_t tP = tmem + D + 128 * b, tO = tmem;
        const uint64_t dv = sw128_desc(sv, AT_TILE * 128, 1024);  // MN-major V, +2048 B per K-step
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)  // P keys 0-63 at cols 0-31, keys 64-127 at 64-95
          umma_f16_ts(tO, tP + (kk < 4 ? 8 * kk : 64 + 8 * (kk - 4)), dv + 128 * kk, id_o, (j > 0 || kk > 0));
        umma_commit(&kv_empty[(2 * j + 1) % NS]);
        umma_commit(&pv_done[b]);
        if (j + 2 < nkv) issue_s(j + 2);  // into the buffer PV(j) just read (in-order tensor pipe)
      }
      umma_commit(o_full);
    }
    finish();
    return;
  }

  regs_inc<F1_REGS_SOFTMAX>();
  {
    // ---------------- softmax: thread = query row r, warpgroup hf = key half
    const int hf = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const int qrow = qt * AT_TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const float c = p.scale_log2;
    float m_used = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      const uint32_t tS = tmem + D + 128 * b + 64 * hf + lane_off;
      mbar_wait_nohint(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t raw[64];
      tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(raw));
      tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
      tmem_wait_ld();
      if (j == qt) {  // diagonal tile: key index > query index is masked
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (64 * hf + i > r) raw[i] = __float_as_uint(-INFINITY);
      }
      // P = 2^(s*c - m) for this half's 64 keys as bf16 over its first 32 columns
      auto write_p = [&](float m) {
        const uint64_t c2 = f2pack(c, c), nm2 = f2pack(-m, -m);
        uint64_t rs2[2] = {f2pack(0.f, 0.f), f2pack(0.f, 0.f)};
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const uint64_t x2 =
              ffma2(f2pack(__uint_as_float(raw[2 * i]), __uint_as_float(raw[2 * i + 1])), c2, nm2);
          float e0, e1;
          pk[i] = exp2_pack_mixed(x2, i, e0, e1);
          rs2[i & 1] = fadd2(rs2[i & 1], f2pack(e0, e1));
        }
        tmem_st32(tS, pk);
        const float2 ra = f2unpack(rs2[0]), rb = f2unpack(rs2[1]);
        return (ra.x + ra.y) + (rb.x + rb.y);
      };
      auto half_max = [&]() {
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 64; i += 8)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            m4[k] = fmax3(m4[k], __uint_as_float(raw[i + 2 * k]), __uint_as_float(raw[i + 2 * k + 1]));
        return fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3])) * c;
      };
      float rowsum = 0.f;
      if (j > 0) rowsum = write_p(m_used);  // speculative: against the running max
      // the row max over both halves (the partner warp owns the same rows)
      float* xb = xch + (j & 1) * 256;
      xb[hf * 128 + r] = half_max();
      named_barrier_sync(1 + quad, 64);
      const float mx = fmaxf(xb[r], xb[128 + r]);
      const bool redo = j == 0 || __any_sync(0xffffffffu, mx > m_used + 8.0f);
      float alpha = 1.f;
      if (redo) {
        const float m_new = (mx > m_used + 8.0f) ? mx : m_used;
        alpha = fast_exp2(m_used - m_new);
        if (j > 0) {
          tmem_wait_st();
          // O holds PV(j-1) once it completes; rescale this half's D/2 columns
          mbar_wait_nohint(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
          const uint32_t tO = tmem + (D / 2) * hf + lane_off;
#pragma unroll
          for (int ch = 0; ch < D / 32; ++ch) {
            uint32_t o16[16];
            tmem_ld16(tO + ch * 16, o16);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o16[i] = __float_as_uint(__uint_as_float(o16[i]) * alpha);
            tmem_st16(tO + ch * 16, o16);
          }
        }
        m_used = m_new;
        rowsum = write_p(m_used);
      }
      tmem_wait_st();
      l_run = l_run * alpha + rowsum;
      tc_fence_before();
      mbar_arrive(&p_full[b]);
    }
    // full row sum = both halves' partial sums
    float* lx = xch + 512;
    lx[hf * 128 + r] = l_run;
    named_barrier_sync(1 + quad, 64);
    const float l_all = lx[r] + lx[128 + r];
    mbar_wait_nohint(o_full, 0);
    tc_fence_after();
    __nv_bfloat16* orow = p.o + (static_cast<int64_t>(qrow) * p.b + bi) * p.ld_o + head * D + (D / 2) * hf;
#pragma unroll
    for (int ch = 0; ch < D / 64; ++ch)
      tmem_row_to_global<32>(tmem + (D / 2) * hf + lane_off + ch * 32, orow + ch * 32, 1.f / l_all, qrow < p.s);
    if (hf == 0 && qrow < p.s) p.lse[static_cast<int64_t>(bh) * p.s + qrow] = (m_used + log2f(l_all)) * LN2;
  }
  finish();
}

template <int D>
static cudaError_t fwd1_launch_t(const void* qkv, int ld_qkv, const AttnParams& p, cudaStream_t st) {
  CUtensorMap tm;
  cudaError_t e = make_tma_3d_rows(&tm, qkv, 3 * p.h, p.b, p.s, ld_qkv, 64, AT_TILE);
  if (e != cudaSuccess) return e;
  static bool cfg = false;
  if (!cfg) {
    e = cudaFuncSetAttribute(attn_fwd1_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd1Smem<D>::TOTAL);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  attn_fwd1_kernel<D><<<nq * p.b * p.heads, F1_THREADS, Fwd1Smem<D>::TOTAL, st>>>(tm, p);
  return cudaGetLastError();
}

cudaError_t attn_fwd1_launch(const void* qkv, int ld_qkv, const AttnParams& p, int d, cudaStream_t st) {
  if (d == 128) return fwd1_launch_t<128>(qkv, ld_qkv, p, st);
  if (d == 64) return fwd1_launch_t<64>(qkv, ld_qkv, p, st);
  return cudaErrorNotSupported;
}

}  // namespace hx
