// Causal flash attention forward on tcgen05 / TMEM / TMA (sm_100a).
// Replaces the reference's whole-matrix fp64 attention (P/runtime/mathops.py:83-100):
//   O = softmax(Q K^T / sqrt(d) + causal mask) V, plus the natural-log LSE per row.
//
// CTA = query tiles (2t, 2t+1) of one (batch, head); heaviest pairs of all heads first.
// Two softmax warpgroups (warps 0-3 -> tile A, 4-7 -> tile B) alternate with the
// tensor core: while group A exponentiates S_A(j), the tensor core runs
// O_B += P_B(j-1) V(j-1) and S_B(j) = Q_B K(j)^T, and vice versa.
//   S = Q K^T    SS-MMA (Q, K from smem)           -> TMEM S_g (fp32, 128 cols)
//   P            bf16, written back over the first 64 columns of S_g
//   O += P V     TS-MMA (A = P from TMEM, B = V MN-major from smem) -> TMEM O_g
// O is rescaled only when a row's running max grows by more than 2^8 (exponents
// stay <= 256, exact in fp32), so rescales are rare after the first tiles.
// Warp 8 issues TMA (Q once, K/V through a 5-slot ring), warp 9 issues MMAs and owns TMEM;
// warps 10-11 idle (they complete warpgroup 2 for setmaxnreg).
// TMEM (512 columns): S_A 0-127 | S_B 128-255 | O_A 256-383 | O_B 384-511.
#include "attention_common.cuh"

namespace hx {

// 12 warps = 3 warpgroups: softmax WG0 / WG1, and WG2 = TMA (warp 8), MMA (warp
// 9), two idle warps (10, 11) so that setmaxnreg can move registers from WG2 to
// the softmax warpgroups (the instruction acts on whole warpgroups).
constexpr int FWD_THREADS = 384;

// Debug build only (-DHX_FWD_TRACE): clock64 stamps of CTA (0,0)'s pipeline
// events, read back with hx_debug_fwd_trace (tools/fwd_trace.py).
#ifdef HX_FWD_TRACE
__device__ long long g_fwd_trace[8][1024];
#define HX_TR(slot, idx) \
  if (blockIdx.x == 0 && (idx) < 1024) g_fwd_trace[slot][idx] = clock64()
#else
#define HX_TR(slot, idx)
#endif

// setmaxnreg budgets: 2 x 128 x 216 + 128 x 72 = 64 K registers.  The launch
// budget is 168 (65536 / 384, rounded down to 8).
constexpr int FWD_REGS_SOFTMAX = 216;
constexpr int FWD_REGS_ISSUE = 72;

// Barrier waits of the forward: mbarrier.try_wait without the 1 ms suspend hint
// the other kernels use (forward alone: 3.71 vs 3.85 ms at 1.3B/32k; the same
// change made the backward 1% slower, so it stays local).  HX_FWD_SPIN=1 makes
// the MMA issuer busy-poll instead (A/B only).
#ifndef HX_FWD_SPIN
#define HX_FWD_SPIN 0
#endif
HX_DEVICE void fwd_wait(uint64_t* bar, uint32_t parity) { mbar_wait_nohint(bar, parity); }
HX_DEVICE void fwd_wait_mma(uint64_t* bar, uint32_t parity) {
  if (HX_FWD_SPIN & 1) mbar_wait_spin(bar, parity);
  else mbar_wait_nohint(bar, parity);
}
HX_DEVICE void fwd_wait_softmax(uint64_t* bar, uint32_t parity) { mbar_wait_nohint(bar, parity); }

template <int D>
struct FwdSmem {
  // K and V tiles share one ring, in load order K(0) V(0) K(1) V(1) ...; as many
  // slots as fit next to the two Q tiles (5 at d=128), so the TMA loads of
  // K/V(j+1) are in flight during the whole of step j.
  static constexpr int NSLOT_FIT = (227 * 1024 - 2 * Tile<D>::BYTES - 512) / Tile<D>::BYTES;
  static constexpr int NSLOT = NSLOT_FIT > 8 ? 8 : NSLOT_FIT;
  static constexpr int QA = 0;
  static constexpr int QB = QA + Tile<D>::BYTES;
  static constexpr int KV = QB + Tile<D>::BYTES;
  static constexpr int BAR = KV + NSLOT * Tile<D>::BYTES;
  static constexpr int TOTAL = BAR + 512;
};

template <int D>
__global__ void __launch_bounds__(FWD_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnParams p) {
  using L = FwdSmem<D>;
  constexpr int NS = L::NSLOT;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;               // 1
  uint64_t* s_full = bars + 1;           // 2 (per group)
  uint64_t* p_full = bars + 3;           // 2, 128 arrivals each
  uint64_t* o_full = bars + 5;           // 2
  uint64_t* kv_full = bars + 7;          // NS
  uint64_t* kv_empty = bars + 7 + NS;    // NS
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7 + 2 * NS);

  const int warp = warp_id(), lane = lane_id();
  const int nq = (p.s + AT_TILE - 1) / AT_TILE;
  const int npairs = (nq + 1) / 2;
  // 1-D grid in bands of p.band (batch, head)s; inside a band, pair-major: each
  // head's heaviest pair launches before any lighter one (longest-processing-time
  // first), while the band keeps the concurrently streamed K/V in L2
  int bh, t;
  band_order(static_cast<int>(blockIdx.x), npairs, p.b * p.heads, p.band, bh, t);
  t = npairs - 1 - t;
  const int qtile[2] = {2 * t, 2 * t + 1};
  const bool has_b = qtile[1] < nq;
  const int last[2] = {qtile[0], has_b ? qtile[1] : -1};
  const int nkv = has_b ? qtile[1] + 1 : qtile[0] + 1;
  const int bi = bh / p.heads, head = bh % p.heads;
  const int qcol = head * D, kcol = p.h + head * D, vcol = 2 * p.h + head * D;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tm_qkv);
    for (int i = 0; i < 7 + 2 * NS; ++i) mbar_init(&bars[i], (i == 3 || i == 4) ? 128 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // ring slot n: K(n/2) for even n, V(n/2) for odd n
  auto slot_addr = [&](int n) { return smem + L::KV + (n % NS) * Tile<D>::BYTES; };

  // Each role ends the kernel itself (no code shared after the role branches,
  // so ptxas allocates each under its own setmaxnreg budget).
  auto finish = [&]() {
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
      tc_fence_after();
      tmem_dealloc(tmem, 512);
    }
  };
  if (warp >= 8) {
  regs_dec<FWD_REGS_ISSUE>();
  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_arrive_expect_tx(q_full, (has_b ? 2 : 1) * Tile<D>::BYTES);
      tma_tile_rows<D>(smem + L::QA, &tm_qkv, q_full, qcol, bi, qtile[0] * AT_TILE, AT_TILE);
      if (has_b) tma_tile_rows<D>(smem + L::QB, &tm_qkv, q_full, qcol, bi, qtile[1] * AT_TILE, AT_TILE);
      for (int n = 0; n < 2 * nkv; ++n) {
        const int sl = n % NS;
        fwd_wait(&kv_empty[sl], ((n / NS) & 1) ^ 1);
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
    }
  } else if (warp == 9) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t id_s = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_o = idesc_bf16(128, D, false, true);
      const uint32_t sq[2] = {smem_u32(smem + L::QA), smem_u32(smem + L::QB)};
      bool pending[2] = {false, false};
      int pcount[2] = {0, 0};
      auto wait_slot = [&](int n) {
        fwd_wait_mma(&kv_full[n % NS], (n / NS) & 1);
        tc_fence_after();
      };
      fwd_wait(q_full, 0);
      auto issue_pv = [&](int g, int jt) {  // O_g += P_g(jt) V(jt)
        wait_slot(2 * jt + 1);
        fwd_wait_mma(&p_full[g], pcount[g] & 1);
        ++pcount[g];
        tc_fence_after();
        const uint32_t sv = smem_u32(slot_addr(2 * jt + 1));
        const uint32_t tP = tmem + 128 * g, tO = tmem + 256 + 128 * g;
        HX_TR(2, 2 * jt + g);
        const uint64_t dv = sw128_desc(sv, AT_TILE * 128, 1024);  // MN-major V, +2048 B per K-step
#pragma unroll
        for (int kk = 0; kk < AT_TILE / 16; ++kk)
          umma_f16_ts(tO, tP + kk * 8, dv + 128 * kk, id_o, (jt > 0 || kk > 0));
        pending[g] = false;
      };
      for (int j = 0; j < nkv; ++j) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          // PV_g(j-1) only needs V(j-1): issue it before waiting for K(j)
          if (pending[g]) {
            issue_pv(g, j - 1);
            if (g == 1 || !pending[1]) umma_commit(&kv_empty[(2 * j - 1) % NS]);  // V(j-1) free
          }
          if (j <= last[g]) {  // S_g(j) = Q_g K(j)^T
            wait_slot(2 * j);
            const uint32_t sk = smem_u32(slot_addr(2 * j));
            const uint32_t tS = tmem + 128 * g;
            // descriptors as one base + compile-time offsets (64-col atoms, +32 B per step)
            const uint64_t dq = sw128_desc(sq[g], 16, 1024), dk = sw128_desc(sk, 16, 1024);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = ((kk >> 2) * AT_TILE * 128 + (kk & 3) * 32) >> 4;
              umma_f16_ss(tS, dq + off, dk + off, id_s, kk > 0);
            }
            umma_commit(&s_full[g]);
            HX_TR(3, 2 * j + g);
            pending[g] = true;
          }
        }
        umma_commit(&kv_empty[(2 * j) % NS]);  // K(j) free
      }
      for (int g = 0; g < 2; ++g)
        if (pending[g]) issue_pv(g, last[g]);
      umma_commit(&o_full[0]);
      umma_commit(&o_full[1]);
    }
  }
  finish();
  return;
  }
  regs_inc<FWD_REGS_SOFTMAX>();
  {
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
        fwd_wait_softmax(&s_full[g], j & 1);
        if (quad == 0 && lane == 0) HX_TR(g, 2 * j);
        tc_fence_after();
        uint32_t raw[AT_TILE];
#pragma unroll
        for (int ch = 0; ch < AT_TILE / 32; ++ch)
          tmem_ld32(tS + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(raw + ch * 32));
        tmem_wait_ld();
        if (quad == 0 && lane == 0) HX_TR(4 + g, j);
        if (j == qt) {  // diagonal tile: key index > query index is masked
#pragma unroll
          for (int i = 0; i < AT_TILE; ++i)
            if (i > r) raw[i] = __float_as_uint(-INFINITY);
        }
        // P = 2^(s*c - m) as bf16 over the first 64 columns of S; returns the row sum.
        // Packed pairs (FFMA2), row sum on packed pairs (FADD2).
        auto write_p = [&](float m) {
          const uint64_t c2 = f2pack(c, c), nm2 = f2pack(-m, -m);
          uint64_t rs2[2] = {f2pack(0.f, 0.f), f2pack(0.f, 0.f)};
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t pk[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const uint64_t x2 = ffma2(f2pack(__uint_as_float(raw[half * 64 + 2 * i]),
                                               __uint_as_float(raw[half * 64 + 2 * i + 1])), c2, nm2);
              float e0, e1;
              pk[i] = exp2_pack_mixed(x2, i, e0, e1);
              rs2[i & 1] = fadd2(rs2[i & 1], f2pack(e0, e1));
            }
            tmem_st32(tS + half * 32, pk);
          }
          const float2 ra = f2unpack(rs2[0]), rb = f2unpack(rs2[1]);
          return (ra.x + ra.y) + (rb.x + rb.y);
        };
        // row max: four independent 3-input-max chains
        auto row_max = [&]() {
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < AT_TILE; i += 8)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              m4[k] = fmax3(m4[k], __uint_as_float(raw[i + 2 * k]), __uint_as_float(raw[i + 2 * k + 1]));
          return fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3])) * c;
        };
        // Speculative exponentials (j > 0): P is computed against the running max
        // m_used while the tile's max is reduced alongside (independent
        // instructions, free issue slots next to the MUFU-bound exps), so the max
        // reduction leaves the softmax -> PV -> S chain.  Only when some row's max
        // grew by more than 2^8 does the warp redo the tile: rescale O, recompute P.
        float rowsum = 0.f;
        float mx = -INFINITY;
        bool redo = true;
        if (j > 0) {
          rowsum = write_p(m_used);
          mx = row_max();
          redo = __any_sync(0xffffffffu, mx > m_used + 8.0f);
        } else {
          mx = row_max();
        }
        float alpha = 1.f;
        if (redo) {
          const float m_new = (mx > m_used + 8.0f) ? mx : m_used;
          alpha = fast_exp2(m_used - m_new);
          if (j > 0) {
            tmem_wait_st();  // the speculative P stores land before being overwritten
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
          if (j > 0) {
            // The speculative P (keys 0-127 packed into columns 0-63) overwrote
            // the scores of keys 0-63 only: reload keys 64-127 from TMEM, so only
            // raw[0..63] had to stay live in registers across the speculative pass.
            tmem_ld32(tS + 64, *reinterpret_cast<uint32_t(*)[32]>(raw + 64));
            tmem_ld32(tS + 96, *reinterpret_cast<uint32_t(*)[32]>(raw + 96));
            tmem_wait_ld();
            if (j == qt) {
#pragma unroll
              for (int i = 64; i < AT_TILE; ++i)
                if (i > r) raw[i] = __float_as_uint(-INFINITY);
            }
          }
          rowsum = write_p(m_used);
        }
        if (quad == 0 && lane == 0) HX_TR(6 + g, j);
        tmem_wait_st();
        l_run = l_run * alpha + rowsum;
        tc_fence_before();
        mbar_arrive(&p_full[g]);
        if (quad == 0 && lane == 0) HX_TR(g, 2 * j + 1);
      }
      fwd_wait(&o_full[g], 0);
      tc_fence_after();
      __nv_bfloat16* orow = p.o + (static_cast<int64_t>(qrow) * p.b + bi) * p.ld_o + head * D;
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch)
        tmem_row_to_global<32>(tO + ch * 32, orow + ch * 32, 1.f / l_run, qrow < p.s);
      if (qrow < p.s) p.lse[static_cast<int64_t>(bh) * p.s + qrow] = (m_used + log2f(l_run)) * LN2;
    }
  }
  finish();
}

#ifdef HX_FWD_TRACE
extern "C" HX_API int hx_debug_fwd_trace(long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_fwd_trace, sizeof(g_fwd_trace)));
}
#endif

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
  attn_fwd_kernel<D><<<((nq + 1) / 2) * p.b * p.heads, FWD_THREADS, FwdSmem<D>::TOTAL, st>>>(tm, p);
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
  // Forward band: as many heads as keep their K/V (2 * s * d bf16 each) within
  // ~64 MB of L2.  In the GPT-1.3B/32k bench step (1.3B: 16 MB per head) bands of
  // 4 heads ran the forward in 4.31-4.34 ms against 4.38-4.40 (1 head) and
  // 4.40-4.47 (all 16 heads, 5x the DRAM reads; lower clocks under the power cap).
  {
    const int64_t per_head = 2LL * s * d * 2;
    int band = static_cast<int>((64LL << 20) / (per_head > 0 ? per_head : 1));
    static const int forced = getenv("HX_ATTN_FWD_BAND") ? atoi(getenv("HX_ATTN_FWD_BAND")) : 0;
    if (forced > 0) band = forced;
    p.band = band < 1 ? 1 : band;
  }
  p.o = static_cast<__nv_bfloat16*>(o);
  p.ld_o = ld_o;
  p.lse = lse;
  // HX_ATTN_FWD=2: one query tile per CTA with double-buffered S (attention_fwd1.cu)
  static const int variant = getenv("HX_ATTN_FWD") ? atoi(getenv("HX_ATTN_FWD")) : 1;
  if (variant == 2) return attn_fwd1_launch(qkv, ld_qkv, p, d, st);
  if (d == 128) return fwd_launch<128>(qkv, ld_qkv, p, st);
  if (d == 64) return fwd_launch<64>(qkv, ld_qkv, p, st);
  return cudaErrorNotSupported;
}

}  // namespace hx
