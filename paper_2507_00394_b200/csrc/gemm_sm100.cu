// Persistent tcgen05 GEMM for the helix components (SURVEY.md §2.2 K2, K4, K6,
// K7, K9, K11, K13, K14):
//
//   C[M,N] (epilogue)= op(A)[M,K] * op(B)[K,N],  bf16 operands, f32 accumulate
//
// Operand storage (row-major in HBM, "ld" = row stride in elements):
//   a_mn = 0 : A stored [M, K] (K contiguous)   -> UMMA K-major
//   a_mn = 1 : A stored [K, M] (M contiguous)   -> UMMA MN-major (weight grads, X^T * dY)
//   b_mn = 0 : B stored [N, K] (K contiguous)   -> UMMA K-major  (input grads, dY * W^T)
//   b_mn = 1 : B stored [K, N] (N contiguous)   -> UMMA MN-major (forward, X * W)
//
// Default for large GEMMs: gemm_2sm_kernel, CTA pairs (cta_group::2) computing
// 256 x 256 tiles with 256x256x16 MMAs (see its comment).  The single-CTA kernel
// below serves GEMMs too small to pair.
//
// Structure (one CTA per SM, 256 threads):
//   warp 0 lane 0 : TMA producer, STAGES-deep smem ring (128B-swizzled tiles)
//   warp 1 lane 0 : UMMA issuer, 128 x BN x 16 tcgen05.mma, accumulator in TMEM,
//                   two accumulator buffers so the epilogue of tile i overlaps
//                   the MMAs of tile i+1
//   warp 2        : TMEM allocator
//   warps 4..7    : epilogue: tcgen05.ld 32 columns at a time, fused op, store
// Tiles are visited in M-grouped raster order (16 M-blocks per group) so the
// concurrently resident A and B panels stay in the 126 MB L2.
#include "hx_common.cuh"
#include "hx_gemm.h"

namespace hx {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;
constexpr int GEMM_GROUP_M = 16;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
  static constexpr int SMEM_BYTES = BAR_OFFSET + 256 + 1024;  // barriers + align slack
  static constexpr int TMEM_COLS = 2 * BN;
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb,
                                            int group_m = GEMM_GROUP_M) {
  const int per_group = group_m * num_n;
  const int group = t / per_group;
  const int first_m = group * group_m;
  const int gm = min(num_m - first_m, group_m);
  const int r = t - group * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

// The bf16 aux operand (residual or GeLU pre-activation) of 32 columns of one
// row, loaded ahead of its accumulator so the load latency overlaps the MMAs.
__device__ __forceinline__ void epilogue_aux_load(const GemmParams& p, int row, int col, uint4 (&a)[4]) {
  if ((p.epi != HX_EPI_RESID_BF16 && p.epi != HX_EPI_DGELU) || row >= p.M) return;
  const __nv_bfloat16* aux = reinterpret_cast<const __nv_bfloat16*>(p.aux) + static_cast<int64_t>(row) * p.ld_aux + col;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (col + 8 * j + 8 <= p.N) a[j] = __ldg(reinterpret_cast<const uint4*>(aux + 8 * j));
}

// Fused epilogue for 32 consecutive accumulator columns of one row (aux, when
// the epilogue has one, preloaded by epilogue_aux_load).
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int row, int col,
                                               const uint32_t (&acc)[32], const uint4 (&pre)[4]) {
  if (row >= p.M) return;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(acc[i]);
  const int epi = p.epi;
  if (epi == HX_EPI_STORE_F32 || epi == HX_EPI_ACC_F32) {
    float* out = reinterpret_cast<float*>(p.out) + static_cast<int64_t>(row) * p.ldo + col;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (col + 4 * j + 4 > p.N) break;
      float4 w = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      if (epi == HX_EPI_ACC_F32 && p.ksplit > 1) {  // K slices of one tile race: add in L2
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out + 4 * j), "f"(w.x), "f"(w.y),
                     "f"(w.z), "f"(w.w)
                     : "memory");
        continue;
      }
      if (epi == HX_EPI_ACC_F32) {
        float4 o = *reinterpret_cast<float4*>(out + 4 * j);
        w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
      }
      *reinterpret_cast<float4*>(out + 4 * j) = w;
    }
    return;
  }
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + static_cast<int64_t>(row) * p.ldo + col;
  __nv_bfloat16* out2 =
      p.out2 ? reinterpret_cast<__nv_bfloat16*>(p.out2) + static_cast<int64_t>(row) * p.ldo2 + col
             : nullptr;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (col + 8 * j + 8 > p.N) break;
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = v[8 * j + i];
    if (epi == HX_EPI_RESID_BF16 || epi == HX_EPI_DGELU) {
      const uint4 a = pre[j];
      const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = unpack_bf16(aw[i]);
        if (epi == HX_EPI_RESID_BF16) {
          x[2 * i] += f.x;
          x[2 * i + 1] += f.y;
        } else {
          const float2 d = gelu_erf_grad_pair(f.x, f.y);
          x[2 * i] *= d.x;
          x[2 * i + 1] *= d.y;
        }
      }
    }
    uint4 o;
    o.x = pack_bf16(x[0], x[1]);
    o.y = pack_bf16(x[2], x[3]);
    o.z = pack_bf16(x[4], x[5]);
    o.w = pack_bf16(x[6], x[7]);
    *reinterpret_cast<uint4*>(out + 8 * j) = o;
    if (epi == HX_EPI_GELU) {
      uint32_t gw[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 t = gelu_erf_pair(x[2 * i], x[2 * i + 1]);
        gw[i] = pack_bf16(t.x, t.y);
      }
      *reinterpret_cast<uint4*>(out2 + 8 * j) = make_uint4(gw[0], gw[1], gw[2], gw[3]);
    }
  }
}

// bf16 epilogues (STORE / RESID / GELU / DGELU) of 32 accumulator columns of
// one row, packed to bf16 pairs: o = the output, o2 = GeLU(output) for GELU.
__device__ __forceinline__ void epilogue_values(int epi, const uint32_t (&acc)[32], const uint4 (&pre)[4],
                                                uint32_t (&o)[16], uint32_t (&o2)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __uint_as_float(acc[8 * j + i]);
    if (epi == HX_EPI_RESID_BF16 || epi == HX_EPI_DGELU) {
      const uint32_t aw[4] = {pre[j].x, pre[j].y, pre[j].z, pre[j].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = unpack_bf16(aw[i]);
        if (epi == HX_EPI_RESID_BF16) {
          x[2 * i] += f.x;
          x[2 * i + 1] += f.y;
        } else {
          const float2 d = gelu_erf_grad_pair(f.x, f.y);
          x[2 * i] *= d.x;
          x[2 * i + 1] *= d.y;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) o[4 * j + i] = pack_bf16(x[2 * i], x[2 * i + 1]);
    if (epi == HX_EPI_GELU) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 t = gelu_erf_pair(x[2 * i], x[2 * i + 1]);
        o2[4 * j + i] = pack_bf16(t.x, t.y);
      }
    }
  }
}

// CL = true: clusters of 2 CTAs on vertically adjacent M-blocks that share the
// B panel.  Each CTA TMA-loads its own A tile and HALF of the B tile, multicast
// to both CTAs, so L2->SM traffic per MMA drops from (A + B) to (A + B/2): 48 ->
// 32 KB per 64-deep stage at BN = 256.  A stage is refilled only after both
// CTAs' MMAs released it (multicast commits on a count-2 empty barrier).
template <int BN, bool A_MN, bool B_MN, bool CL>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tm_a,
                      const __grid_constant__ CUtensorMap tm_b, const GemmParams p) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFFSET);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_m = (p.M + GEMM_BM - 1) / GEMM_BM;
  const int num_n = (p.N + BN - 1) / BN;
  const int num_k = (p.K + GEMM_BK - 1) / GEMM_BK;
  // persistent walk over (cluster) tiles: with CL a tile is an M-block pair
  const int rank = CL ? static_cast<int>(cluster_ctarank()) : 0;
  const int num_m_w = CL ? num_m / 2 : num_m;
  const int num_tiles = num_m_w * num_n;
  const int first = CL ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int stride = CL ? static_cast<int>(nclusters_x()) : static_cast<int>(gridDim.x);
  auto coords = [&](int t, int& mb, int& nb) {
    tile_coords(t, num_m_w, num_n, mb, nb);
    if (CL) mb = 2 * mb + rank;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_a);
    tma_prefetch(&tm_b);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  if (CL) cluster_sync();  // peers' barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = first; t < num_tiles; t += stride) {
        int mb, nb;
        coords(t, mb, nb);
        const int m0 = mb * GEMM_BM, n0 = nb * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          const int k0 = kb * GEMM_BK;
          if (A_MN) {
            tma_load_2d(sa, &tm_a, &full[stage], m0, k0);
            tma_load_2d(sa + 8192, &tm_a, &full[stage], m0 + 64, k0);
          } else {
            tma_load_2d(sa, &tm_a, &full[stage], k0, m0);
          }
          if (CL) {  // this CTA's half of B, multicast to both CTAs of the pair
            if (B_MN) {
#pragma unroll
              for (int j = rank * (BN / 128); j < (rank + 1) * (BN / 128); ++j)
                tma_load_2d_mc(sb + j * 8192, &tm_b, &full[stage], n0 + 64 * j, k0, 0x3);
            } else {
              tma_load_2d_mc(sb + rank * (BN / 2) * 128, &tm_b, &full[stage], k0, n0 + rank * (BN / 2), 0x3);
            }
          } else if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * 8192, &tm_b, &full[stage], n0 + 64 * j, k0);
          } else {
            tma_load_2d(sb, &tm_b, &full[stage], k0, n0);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- UMMA issuer
      constexpr uint32_t idesc = idesc_bf16(GEMM_BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = first; t < num_tiles; t += stride, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
            const uint64_t da = A_MN ? sw128_desc(sa + kk * 2048, 8192, 1024)
                                     : sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? sw128_desc(sb + kk * 2048, 8192, 1024)
                                     : sw128_desc(sb + kk * 32, 16, 1024);
            umma_f16_ss(d_tmem, da, db, idesc, (kb | kk) != 0);
          }
          if (CL)
            umma_commit_mc(&empty[stage], 0x3);  // the stage holds both CTAs' B halves
          else
            umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue
    const int sub = warp & 3;  // TMEM lane quadrant this warp may access
    int it = 0;
    for (int t = first; t < num_tiles; t += stride, ++it) {
      int mb, nb;
      coords(t, mb, nb);
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = mb * GEMM_BM + sub * 32 + lane;
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(sub * 32) << 16);
      uint4 aux_c[4], aux_n[4];
      epilogue_aux_load(p, row, nb * BN, aux_c);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int col = nb * BN + c * 32;
        if (col >= p.N) break;  // warp-uniform
        if (c + 1 < BN / 32 && col + 32 < p.N) epilogue_aux_load(p, row, col + 32, aux_n);
        uint32_t r[32];
        tmem_ld32(taddr + c * 32, r);
        tmem_wait_ld();
        epilogue_chunk(p, row, col, r, aux_c);
#pragma unroll
        for (int j = 0; j < 4; ++j) aux_c[j] = aux_n[j];
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (CL) cluster_sync();  // no CTA leaves while its peer may still multicast into it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}


// ------------------------------------------------------------------ 2-CTA (cta_group::2)
// One 256 x 256 output tile per CTA pair: the leader issues 256x256x16 MMAs whose
// A rows and B columns come half from each CTA's smem, so each SM stages only
// its own 128 A rows and 128 B columns per k-block (32 KB instead of 48 KB):
// 6 stages in flight instead of 4, and half the L2->SM traffic for B.
// Both CTAs' TMA loads complete on the leader's full barrier; the leader's
// commits release both CTAs' stages (empty) and accumulators (tfull); both
// CTAs' epilogue threads return accumulators on the leader's tempty barrier.
constexpr int G2_STAGES = 6;
constexpr int G2_A_BYTES = GEMM_BM * GEMM_BK * 2;   // 16 KB: this CTA's 128 rows
constexpr int G2_B_BYTES = 128 * GEMM_BK * 2;       // 16 KB: this CTA's 128 of 256 columns
constexpr int G2_STAGE_BYTES = G2_A_BYTES + G2_B_BYTES;
// bf16 epilogues stage each warp's 32 x 32 output chunk (SWIZZLE_64B) here and
// TMA-store it: per warp 2 buffers x (1 or 2 outputs) x 2 KB, 32 KB in all
constexpr int G2_STG_OFFSET = G2_STAGES * G2_STAGE_BYTES;
constexpr int G2_STG_BYTES = 32768;
constexpr int G2_BAR_OFFSET = G2_STG_OFFSET + G2_STG_BYTES;
constexpr int G2_SMEM_BYTES = G2_BAR_OFFSET + 256 + 1024;

// EW epilogue warps (4 or 8): with 8, warps 4..7 drain accumulator columns
// 0..127 and warps 8..11 columns 128..255 of their TMEM lane quadrant (warp & 3),
// so the fused epilogues (GeLU, GeLU', residual) keep up with the MMAs.
template <bool A_MN, bool B_MN, int EW>
__global__ void __launch_bounds__(128 + 32 * EW, 1)
    gemm_2sm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                    const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_c2,
                    const GemmParams p) {
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G2_BAR_OFFSET);
  uint64_t* empty = full + G2_STAGES;
  uint64_t* tfull = empty + G2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int rank = static_cast<int>(cluster_ctarank());
  const bool leader = rank == 0;
  const int num_m = (p.M + GEMM_BM - 1) / GEMM_BM;
  const int num_n = (p.N + BN - 1) / BN;
  const int num_k = (p.K + GEMM_BK - 1) / GEMM_BK;
  const int num_tiles = (num_m / 2) * num_n;
  // work unit u = (tile u / S, K slice u % S): slices of one tile run on different pairs
  const int S = p.ksplit;
  const int num_units = num_tiles * S;
  auto kslice = [&](int u, int& kb0, int& kb1) {
    const int ks = u % S;
    kb0 = ks * num_k / S;
    kb1 = (ks + 1) * num_k / S;
  };
  const int first = static_cast<int>(cluster_id_x());
  const int stride = static_cast<int>(nclusters_x());

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_a);
    tma_prefetch(&tm_b);
    for (int s = 0; s < G2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EW);  // one arrival per epilogue warp of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs): own A rows + own half of B
      int stage = 0;
      uint32_t phase = 0;
      for (int u = first; u < num_units; u += stride) {
        int mp, nb, kb0, kb1;
        tile_coords(u / S, num_m / 2, num_n, mp, nb, p.group_m);
        kslice(u, kb0, kb1);
        const int m0 = (2 * mp + rank) * GEMM_BM, n0 = nb * BN + rank * 128;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t bar = mapa_shared(&full[stage], 0);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * G2_STAGE_BYTES);
          uint8_t* sa = smem + stage * G2_STAGE_BYTES;
          uint8_t* sb = sa + G2_A_BYTES;
          const int k0 = kb * GEMM_BK;
          if (A_MN) {
            tma_load_2d_2sm(sa, &tm_a, bar, m0, k0);
            tma_load_2d_2sm(sa + 8192, &tm_a, bar, m0 + 64, k0);
          } else {
            tma_load_2d_2sm(sa, &tm_a, bar, k0, m0);
          }
          if (B_MN) {
            tma_load_2d_2sm(sb, &tm_b, bar, n0, k0);
            tma_load_2d_2sm(sb + 8192, &tm_b, bar, n0 + 64, k0);
          } else {
            tma_load_2d_2sm(sb, &tm_b, bar, k0, n0);
          }
          if (++stage == G2_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- UMMA issuer (pair leader): 256 x 256 x 16 per instruction
      constexpr uint32_t idesc = idesc_bf16(2 * GEMM_BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = first; u < num_units; u += stride, ++it) {
        const int acc = it & 1;
        int kb0, kb1;
        kslice(u, kb0, kb1);
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * G2_STAGE_BYTES);
          const uint32_t sb = sa + G2_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
            const uint64_t da = A_MN ? sw128_desc(sa + kk * 2048, 8192, 1024)
                                     : sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? sw128_desc(sb + kk * 2048, 8192, 1024)
                                     : sw128_desc(sb + kk * 32, 16, 1024);
            umma_f16_ss_2sm(d_tmem, da, db, idesc, (kb != kb0) || kk != 0);
          }
          umma_commit_2sm_mc(&empty[stage], 0x3);
          if (++stage == G2_STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc(&tfull[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): this CTA's 128 rows of the 256 x 256 tile
    const int sub = warp & 3;
    constexpr int CPW = (BN / 32) * 4 / EW;     // 32-column chunks per warp
    const int c0 = ((warp - 4) / 4) * CPW;      // this warp's first chunk
    const uint32_t tempty_leader0 = mapa_shared(&tempty[0], 0);
    // bf16 outputs leave through smem + TMA stores (coalesced, async); fp32 ones
    // (weight-gradient accumulation) keep the per-row path
    const int nout = p.epi == HX_EPI_GELU ? 2 : 1;
    // staging buffers per warp: 2 (double-buffered) if they fit, else 1
    const int nbuf = nout * 2 * 2048 * EW <= G2_STG_BYTES ? 2 : 1;
    const bool tma_out = p.tma_store && p.epi != HX_EPI_ACC_F32 && p.epi != HX_EPI_STORE_F32 &&
                         nout * nbuf * 2048 * EW <= G2_STG_BYTES;
    uint8_t* stg = smem + G2_STG_OFFSET + (warp - 4) * (G2_STG_BYTES / EW);
    int kbuf = 0;
    int it = 0;
    for (int u = first; u < num_units; u += stride, ++it) {
      int mp, nb;
      tile_coords(u / S, num_m / 2, num_n, mp, nb, p.group_m);
      const int acc = it & 1;
      const int row0 = (2 * mp + rank) * GEMM_BM + sub * 32;
      const int row = row0 + lane;
      // aux (residual / GeLU pre-activation) two chunks ahead: the first two chunks'
      // are loaded before the accumulator is ready, chunk c + 2's while chunk c is
      // processed (one chunk ahead left the GeLU' epilogue waiting on DRAM at every
      // chunk's first aux use: 10% of its stall samples).  The chunk loop is
      // unrolled so the three aux slots stay in registers.
      uint4 aux[3][4];
      epilogue_aux_load(p, row, nb * BN + c0 * 32, aux[0]);
      if (CPW > 1) epilogue_aux_load(p, row, nb * BN + (c0 + 1) * 32, aux[1]);
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(sub * 32) << 16);
#pragma unroll
      for (int ci = 0; ci < CPW; ++ci) {
        const int c = c0 + ci;
        const int col = nb * BN + c * 32;
        if (col >= p.N) break;  // warp-uniform
        if (ci + 2 < CPW && col + 64 < p.N) epilogue_aux_load(p, row, col + 64, aux[(ci + 2) % 3]);
        uint32_t r[32];
        tmem_ld32(taddr + c * 32, r);
        tmem_wait_ld();
        if (tma_out) {
          uint32_t o[16], o2[16];
          epilogue_values(p.epi, r, aux[ci % 3], o, o2);
          uint8_t* buf = stg + (nbuf == 2 ? (kbuf & 1) * (nout * 2048) : 0);
          if (lane == 0) {  // the store that last read this buffer is done
            if (nbuf == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          // row `lane` of the 32 x 64-byte box, SWIZZLE_64B: 16-byte chunk j at j ^ ((row >> 1) & 3)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int off = lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
            *reinterpret_cast<uint4*>(buf + off) = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
            if (nout == 2)
              *reinterpret_cast<uint4*>(buf + 2048 + off) =
                  make_uint4(o2[4 * j], o2[4 * j + 1], o2[4 * j + 2], o2[4 * j + 3]);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_c, buf, col, row0);
            if (nout == 2) tma_store_2d(&tm_c2, buf + 2048, col, row0);
            bulk_commit();
          }
          ++kbuf;
        } else {
          epilogue_chunk(p, row, col, r, aux[ci % 3]);
        }
      }
      // every lane's tcgen05.ld has completed (wait::ld above); one arrival per warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
    }
  }
  if (warp >= 4 && lane == 0) bulk_wait_all();  // epilogue TMA stores have left smem
  __syncthreads();
  cluster_sync();  // the peer's smem / barriers stay valid until both CTAs are done
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 2 * BN);
  }
}

template <bool A_MN, bool B_MN, int EW>
static cudaError_t launch_gemm_2sm_ew(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                                      int num_sms, cudaStream_t stream) {
  // output tensor maps of the TMA-store epilogue (bf16 [M, N], 32 x 32 boxes)
  CUtensorMap tc = ta, tc2 = ta;
  if (p.epi != HX_EPI_ACC_F32 && p.epi != HX_EPI_STORE_F32) {
    cudaError_t e = make_tma_2d_sw64(&tc, p.out, p.M, p.N, p.ldo, 32, 32);
    if (e == cudaSuccess && p.epi == HX_EPI_GELU) e = make_tma_2d_sw64(&tc2, p.out2, p.M, p.N, p.ldo2, 32, 32);
    if (e != cudaSuccess) return e;
  }
  auto kern = gemm_2sm_kernel<A_MN, B_MN, EW>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G2_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int pairs = ((p.M + GEMM_BM - 1) / GEMM_BM / 2) * ((p.N + 255) / 256) * p.ksplit;
  int grid = 2 * (pairs < num_sms / 2 ? pairs : num_sms / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128 + 32 * EW);
  cfg.dynamicSmemBytes = G2_SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tc2, p);
}

// Epilogue warps (HX_GEMM_EPI_WARPS=4/8 forces one for A/B runs; 8 by default).
// Measured in the GPT-1.3B/32k bench step: W2^T * GeLU' (reads m1) 0.72 -> 1.00
// PFLOP/s with 8 warps.  W1 + GeLU (writes m1 and g) was slower with 8 warps on
// the per-row store path (1.03 -> 0.90); with the TMA-store epilogue (8 warps,
// single-buffered staging for its two outputs) it is faster than with 4
// (HX_GEMM_GELU_WARPS A/B: 375 vs 402 ms of GEMM per step, +1.3% tokens/s).
template <bool A_MN, bool B_MN>
static cudaError_t launch_gemm_2sm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                                   int num_sms, cudaStream_t stream) {
  static const int forced = getenv("HX_GEMM_EPI_WARPS") ? atoi(getenv("HX_GEMM_EPI_WARPS")) : 0;
  static const int gelu_ew = getenv("HX_GEMM_GELU_WARPS") ? atoi(getenv("HX_GEMM_GELU_WARPS")) : 8;
  const int ew = forced ? forced : (p.epi == HX_EPI_GELU ? gelu_ew : 8);
  if (ew == 4) return launch_gemm_2sm_ew<A_MN, B_MN, 4>(ta, tb, p, num_sms, stream);
  return launch_gemm_2sm_ew<A_MN, B_MN, 8>(ta, tb, p, num_sms, stream);
}

// ------------------------------------------------------------------ host side

template <int BN, bool A_MN, bool B_MN, bool CL>
static cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                               int num_sms, cudaStream_t stream) {
  using C = GemmCfg<BN>;
  auto kern = gemm_sm100_kernel<BN, A_MN, B_MN, CL>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e == cudaSuccess && CL) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = ((p.M + GEMM_BM - 1) / GEMM_BM) * ((p.N + BN - 1) / BN);
  int grid = tiles < num_sms ? tiles : num_sms;
  if (!CL) {
    kern<<<grid, GEMM_THREADS, C::SMEM_BYTES, stream>>>(ta, tb, p);
    return cudaGetLastError();
  }
  grid &= ~1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
}

static int pick_bn(int M, int N, int num_sms) {
  if (N <= 128) return 128;
  const long mb = (M + GEMM_BM - 1) / GEMM_BM;
  const long t256 = mb * ((N + 255) / 256), t128 = mb * ((N + 127) / 128);
  auto eff = [&](long tiles, double work_per_tile) {
    const long waves = (tiles + num_sms - 1) / num_sms;
    return (tiles * work_per_tile) / (waves * num_sms * work_per_tile);
  };
  // 256-wide tiles halve A re-reads and smem traffic per FLOP; only give them up
  // for a clearly better wave quantisation.
  // Measured on B200: 128-wide tiles run ~20% slower per FLOP (they need 96 B/clk
  // of smem operand bandwidth vs 64 for 256-wide), so only a large wave-
  // quantisation gain justifies them.
  return eff(t128, 1.0) > eff(t256, 1.0) + 0.25 ? 128 : 256;
}

// K slices per 256 x 256 tile for the pair kernel.  Only fp32-accumulating GEMMs
// (weight gradients: few tiles, long K) split, and only when the slices fill the
// pair slots clearly better than whole tiles do; each slice keeps >= 2048 of K.
// At most 2 slices: measured at GPT-1.3B/32k, 2 slices take the MLP weight
// gradients (256 tiles on 74 pairs) from 0.81-0.88 to 0.74-0.78 ms, while 3
// slices (qkv, 192 tiles) were 4% and 8 slices (o, 64 tiles) 26% slower than
// none: the red.global traffic then outweighs the better wave fill.
// HX_GEMM_KSPLIT=n forces n (1 disables), for A/B runs.
static int pick_ksplit(const GemmParams& p, int tiles, int slots) {
  static const int forced = getenv("HX_GEMM_KSPLIT") ? atoi(getenv("HX_GEMM_KSPLIT")) : 0;
  if (p.epi != HX_EPI_ACC_F32) return 1;
  if (forced > 0) return forced;
  auto eff = [&](int s) {
    const long units = static_cast<long>(tiles) * s;
    const long waves = (units + slots - 1) / slots;
    return static_cast<double>(units) / static_cast<double>(waves * slots);
  };
  int best = 1;
  for (int s = 2; s <= 2 && p.K / s >= 2048; ++s)
    if (eff(s) > eff(best) + 0.05) best = s;
  return best;
}

// Tile raster of the pair kernel: pair-rows per M-group (M fastest inside a
// group, groups in order).  Picked to minimise the modelled DRAM bytes of the
// operand panels: a wave of `conc` concurrent tiles re-reads A panels once per
// n-column wave unless the group's A panels stay in L2, and B panels once per
// group unless all of B stays in L2.  Narrow-N GEMMs (N = 2048: 8 tile columns)
// then run whole tile rows per wave (A read once) instead of 16-row groups that
// read A 1.7x; wide-N weight gradients keep the tall groups.
// HX_GEMM_GROUP=n forces n, for A/B runs.
static int pick_group(const GemmParams& p, int num_mp, int num_n, int conc) {
  static const int forced = getenv("HX_GEMM_GROUP") ? atoi(getenv("HX_GEMM_GROUP")) : 0;
  if (forced > 0) return forced;
  const double budget = 16.0 * (1 << 20);  // L2 bytes a group's panels may hold across waves
  const double a_panel = 256.0 * p.K * 2, b_panel = 256.0 * p.K * 2;
  const double a_total = a_panel * num_mp, b_total = b_panel * num_n;
  double best_bytes = 0;
  int best = GEMM_GROUP_M;
  for (int g : {GEMM_GROUP_M, 8, 4, 2, 1}) {
    double a_rd, b_rd;
    if (conc >= g * num_n) {  // a wave covers whole tile rows
      const double m_conc = static_cast<double>(conc) / num_n;
      a_rd = a_total;
      b_rd = b_total <= budget ? b_total : b_total * num_mp / m_conc;
    } else {
      const int m_conc = g < num_mp ? g : num_mp;
      const double n_conc = static_cast<double>(conc) / m_conc;
      a_rd = m_conc * a_panel <= budget ? a_total : a_total * num_n / n_conc;
      b_rd = b_total <= budget ? b_total : b_total * ((num_mp + g - 1) / g);
    }
    if (g == GEMM_GROUP_M || a_rd + b_rd < 0.95 * best_bytes) {
      best_bytes = a_rd + b_rd;
      best = g;
    }
  }
  return best;
}

cudaError_t gemm_launch(const GemmOperand& a, const GemmOperand& b, const GemmParams& p,
                        cudaStream_t stream) {
  const int num_sms = hx::num_sms();  // persistent grid size (honours HX_SM_RESERVE)
  const int bn = pick_bn(p.M, p.N, num_sms);
  CUtensorMap ta, tb;
  // A: K-major [M,K] box {64,128}; MN-major [K,M] box {64,64}
  cudaError_t e = a.mn ? make_tma_2d(&ta, a.ptr, p.K, p.M, a.ld, 64, 64)
                       : make_tma_2d(&ta, a.ptr, p.M, p.K, a.ld, 64, GEMM_BM);
  if (e != cudaSuccess) return e;
  // 2-CTA clusters with B multicast when the M-blocks pair up evenly and there are
  // enough tile pairs to fill the machine (HX_GEMM_CLUSTER=0 disables, for A/B runs)
  // HX_GEMM_CLUSTER: 2 (default) cta_group::2 pairs, 1 B-multicast pairs, 0 single CTAs
  static const int cl_mode = getenv("HX_GEMM_CLUSTER") ? atoi(getenv("HX_GEMM_CLUSTER")) : 2;
  const int num_m = (p.M + GEMM_BM - 1) / GEMM_BM;
  const int pairs = (num_m / 2) * ((p.N + 255) / 256);
  const bool pairable = bn == 256 && num_m % 2 == 0 && pairs >= num_sms / 2;
  const bool cl = cl_mode != 0 && pairable;
  // cta_group::2 also wins with fewer tiles than pairs of SMs (e.g. the 2048 x 2048
  // weight gradient: 64 pairs); only tiny GEMMs stay on single CTAs
  if (cl_mode == 2 && num_m % 2 == 0 && p.N > 128 && pairs >= 32) {
    GemmParams q = p;
    static const int tma_store = getenv("HX_GEMM_TMA_STORE") ? atoi(getenv("HX_GEMM_TMA_STORE")) : 1;
    q.tma_store = tma_store;
    q.ksplit = pick_ksplit(p, pairs, num_sms / 2);
    q.group_m = pick_group(p, num_m / 2, (p.N + 255) / 256, (num_sms / 2) / q.ksplit);
    e = b.mn ? make_tma_2d(&tb, b.ptr, p.K, p.N, b.ld, 64, 64) : make_tma_2d(&tb, b.ptr, p.N, p.K, b.ld, 64, 128);
    if (e != cudaSuccess) return e;
    if (a.mn && b.mn) return launch_gemm_2sm<true, true>(ta, tb, q, num_sms, stream);
    if (!a.mn && b.mn) return launch_gemm_2sm<false, true>(ta, tb, q, num_sms, stream);
    if (!a.mn && !b.mn) return launch_gemm_2sm<false, false>(ta, tb, q, num_sms, stream);
    return cudaErrorNotSupported;
  }
  e = b.mn ? make_tma_2d(&tb, b.ptr, p.K, p.N, b.ld, 64, 64)
           : make_tma_2d(&tb, b.ptr, p.N, p.K, b.ld, 64, cl ? bn / 2 : bn);
  if (e != cudaSuccess) return e;
#define HX_GEMM_CASE(BN_, AM_, BM_)                                                   \
  if (bn == BN_ && a.mn == AM_ && b.mn == BM_)                                          \
    return cl ? launch_gemm<BN_, AM_, BM_, true>(ta, tb, p, num_sms, stream)             \
              : launch_gemm<BN_, AM_, BM_, false>(ta, tb, p, num_sms, stream);
  HX_GEMM_CASE(256, false, true)
  HX_GEMM_CASE(256, false, false)
  HX_GEMM_CASE(256, true, true)
  HX_GEMM_CASE(128, false, true)
  HX_GEMM_CASE(128, false, false)
  HX_GEMM_CASE(128, true, true)
#undef HX_GEMM_CASE
  return cudaErrorNotSupported;
}

}  // namespace hx
