// Paper §4.6 extras (no reference code): word +
// position embeddings in front of layer 0 and the tied-weight next-token
// prediction whose logits and cross-entropy are computed in the backward pass,
// chunk by chunk, so the [s, b, V] logits are never stashed.  The three GEMMs
// of the head (logits, dz, dW_emb) run on the tcgen05 GEMM; the kernels here are
// the HBM-bound pieces:
//
//   embed_fwd   x[t] = W_emb[tok[t]] + W_pos[t / b]          reads 2*T*h*2, writes T*h*2 bytes
//   embed_bwd   dW_emb[tok[t]] += dx[t] (fp32 vector atomics), dW_pos[si] += sum_b dx[si*b + bi]
//   ce_loss     per logits row: lse over the V real columns, loss += lse - z[label],
//               dlogits = (softmax - onehot) * scale in place (padded columns -> 0)
//                                                             reads 2*V*2, writes V*2 bytes per row
#include "hx_common.cuh"
#include "hx_gemm.h"

namespace hx {

HX_DEVICE void unpack8_lm(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = unpack_bf16(w[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}

// One warp per token row; 16-byte vectors.
__global__ void __launch_bounds__(256) embed_fwd_kernel(const int* __restrict__ tok,
                                                         const __nv_bfloat16* __restrict__ w_emb,
                                                         const __nv_bfloat16* __restrict__ w_pos,
                                                         __nv_bfloat16* __restrict__ x, int T, int b, int h) {
  const int lane = lane_id();
  const int nvec = h / 8;
  for (int t = blockIdx.x * 8 + warp_id(); t < T; t += gridDim.x * 8) {
    const int id = tok[t];
    const uint4* we = reinterpret_cast<const uint4*>(w_emb + static_cast<int64_t>(id) * h);
    const uint4* wp = reinterpret_cast<const uint4*>(w_pos + static_cast<int64_t>(t / b) * h);
    uint4* xr = reinterpret_cast<uint4*>(x + static_cast<int64_t>(t) * h);
    for (int c = lane; c < nvec; c += 32) {
      float a[8], p[8];
      unpack8_lm(__ldg(we + c), a);
      unpack8_lm(__ldg(wp + c), p);
      xr[c] = make_uint4(pack_bf16(a[0] + p[0], a[1] + p[1]), pack_bf16(a[2] + p[2], a[3] + p[3]),
                         pack_bf16(a[4] + p[4], a[5] + p[5]), pack_bf16(a[6] + p[6], a[7] + p[7]));
    }
  }
}

// Word-embedding gradient: one warp per token, fp32 vector atomics (tokens repeat).
// Position-embedding gradient: one warp per sequence position, summed over the
// batch in registers (each (position, column) is owned by one lane: no atomics).
__global__ void __launch_bounds__(256) embed_bwd_kernel(const int* __restrict__ tok,
                                                         const __nv_bfloat16* __restrict__ dx,
                                                         float* __restrict__ dw_emb, float* __restrict__ dw_pos,
                                                         int s, int b, int h) {
  const int lane = lane_id();
  const int nvec = h / 8;
  const int T = s * b;
  const int warps = gridDim.x * 8;
  for (int w = blockIdx.x * 8 + warp_id(); w < T + s; w += warps) {
    if (w < T) {
      const uint4* dr = reinterpret_cast<const uint4*>(dx + static_cast<int64_t>(w) * h);
      float* dst = dw_emb + static_cast<int64_t>(tok[w]) * h;
      for (int c = lane; c < nvec; c += 32) {
        float f[8];
        unpack8_lm(dr[c], f);
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 8 * c), "f"(f[0]), "f"(f[1]),
                     "f"(f[2]), "f"(f[3])
                     : "memory");
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 8 * c + 4), "f"(f[4]),
                     "f"(f[5]), "f"(f[6]), "f"(f[7])
                     : "memory");
      }
    } else {
      const int si = w - T;
      float* dst = dw_pos + static_cast<int64_t>(si) * h;
      for (int c = lane; c < nvec; c += 32) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int bi = 0; bi < b; ++bi) {
          float f[8];
          unpack8_lm(reinterpret_cast<const uint4*>(dx + (static_cast<int64_t>(si) * b + bi) * h)[c], f);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] += f[k];
        }
        float4* d4 = reinterpret_cast<float4*>(dst + 8 * c);
        float4 u = d4[0], v = d4[1];
        u.x += acc[0]; u.y += acc[1]; u.z += acc[2]; u.w += acc[3];
        v.x += acc[4]; v.y += acc[5]; v.z += acc[6]; v.w += acc[7];
        d4[0] = u;
        d4[1] = v;
      }
    }
  }
}

HX_DEVICE float block_reduce_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < static_cast<int>(blockDim.x / 32); ++i) r = fmaxf(r, red[i]);
  return r;
}
HX_DEVICE float block_reduce_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x / 32); ++i) r += red[i];
  return r;
}

// One CTA per logits row.  Pass 1: online max / sum of exp over the V real
// columns; pass 2 (an L2 re-read): dlogits in place, padded columns zeroed.
__global__ void __launch_bounds__(512) ce_loss_kernel(__nv_bfloat16* __restrict__ logits, int ld,
                                                       const int* __restrict__ labels, int vocab, int vpad,
                                                       float scale, double* __restrict__ loss_acc,
                                                       int* __restrict__ count_acc) {
  __shared__ float red[16];
  const int row = blockIdx.x;
  __nv_bfloat16* z = logits + static_cast<int64_t>(row) * ld;
  const int label = labels[row];
  const int nvec = vpad / 8;
  const uint4* zr = reinterpret_cast<const uint4*>(z);
  float m = -INFINITY, ssum = 0.f;
  for (int c = threadIdx.x; c < nvec; c += blockDim.x) {
    float f[8];
    unpack8_lm(zr[c], f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (8 * c + k < vocab) {
        const float v = f[k];
        if (v > m) {
          ssum = ssum * __expf(m - v) + 1.f;
          m = v;
        } else {
          ssum += __expf(v - m);
        }
      }
    }
  }
  const float gm = block_reduce_max(m, red);
  const float gs = block_reduce_sum(m == -INFINITY ? 0.f : ssum * __expf(m - gm), red);
  const float lse = gm + __logf(gs);
  if (threadIdx.x == 0 && label >= 0) {
    atomicAdd(loss_acc, static_cast<double>(lse - __bfloat162float(z[label])));
    atomicAdd(count_acc, 1);
  }
  __syncthreads();  // the label's logit is read before dlogits overwrite it
  uint4* wr = reinterpret_cast<uint4*>(z);
  for (int c = threadIdx.x; c < nvec; c += blockDim.x) {
    float f[8], o[8];
    unpack8_lm(zr[c], f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int col = 8 * c + k;
      o[k] = (col < vocab && label >= 0) ? (__expf(f[k] - lse) - (col == label ? 1.f : 0.f)) * scale : 0.f;
    }
    wr[c] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
  }
}

cudaError_t embed_fwd_launch(const int* tok, const void* w_emb, const void* w_pos, void* x, int s, int b, int h,
                             cudaStream_t st) {
  const int T = s * b;
  int grid = (T + 7) / 8;
  if (grid > num_sms() * 8) grid = num_sms() * 8;
  embed_fwd_kernel<<<grid, 256, 0, st>>>(tok, static_cast<const __nv_bfloat16*>(w_emb),
                                         static_cast<const __nv_bfloat16*>(w_pos), static_cast<__nv_bfloat16*>(x),
                                         T, b, h);
  return cudaGetLastError();
}

cudaError_t embed_bwd_launch(const int* tok, const void* dx, float* dw_emb, float* dw_pos, int s, int b, int h,
                             cudaStream_t st) {
  int grid = (s * b + s + 7) / 8;
  if (grid > num_sms() * 8) grid = num_sms() * 8;
  embed_bwd_kernel<<<grid, 256, 0, st>>>(tok, static_cast<const __nv_bfloat16*>(dx), dw_emb, dw_pos, s, b, h);
  return cudaGetLastError();
}

cudaError_t ce_loss_launch(void* logits, int ld, const int* labels, int rows, int vocab, int vpad, float scale,
                           double* loss_acc, int* count_acc, cudaStream_t st) {
  ce_loss_kernel<<<rows, 512, 0, st>>>(static_cast<__nv_bfloat16*>(logits), ld, labels, vocab, vpad, scale,
                                       loss_acc, count_acc);
  return cudaGetLastError();
}

}  // namespace hx
