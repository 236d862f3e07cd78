// Internal host/device interfaces shared by the libhx translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hx.h"

namespace hx {

struct GemmOperand {
  const void* ptr;
  int ld;    // row stride in elements of the stored matrix
  bool mn;   // false: K contiguous; true: M (for A) / N (for B) contiguous
};

struct GemmParams {
  int M, N, K;
  int epi;               // HX_EPI_*
  void* out;             // bf16 or f32 [M, N] with row stride ldo
  int ldo;
  const void* aux;       // bf16 [M, N]: residual (RESID) or GeLU pre-activation (DGELU)
  int ld_aux;
  void* out2;            // bf16 [M, N]: GeLU output (GELU)
  int ldo2;
  int ksplit;            // K slices per tile (pair kernel, ACC_F32 only; set by gemm_launch)
  int group_m;           // tile-raster M-group in pair-rows (pair kernel; set by gemm_launch)
  int tma_store;         // bf16 outputs via smem + TMA store (pair kernel; HX_GEMM_TMA_STORE=0 disables)
};

// 2-D bf16 tensor map over a row-major [rows, cols] matrix with row stride ld,
// SWIZZLE_128B, box {box_cols, box_rows}.  OOB reads are zero-filled.
cudaError_t make_tma_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
                        uint32_t box_cols, uint32_t box_rows);

// 2-D bf16 tensor map as make_tma_2d but SWIZZLE_64B (box_cols * 2 bytes = 64):
// the GEMM epilogue's TMA stores of 32-column row chunks.
cudaError_t make_tma_2d_sw64(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
                             uint32_t box_cols, uint32_t box_rows);

// 3-D bf16 tensor map over activations stored token-major [s][b][ld]: dims
// {cols, b, s}, box {box_cols, 1, box_rows} (one batch column, box_rows tokens).
cudaError_t make_tma_3d_rows(CUtensorMap* map, const void* ptr, uint64_t cols, uint64_t b, uint64_t s,
                             uint64_t ld, uint32_t box_cols, uint32_t box_rows);

// 3-D fp32 tensor map over a dense [d2][d1][d0] array, SWIZZLE_128B, box
// {box0, box1, 1} (box0 * 4 bytes must be 128).  Used for TMA reduce-adds.
cudaError_t make_tma_f32_3d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                            uint32_t box0, uint32_t box1);

cudaError_t ln_fwd_launch(const void* x, const float* g, const float* b, void* y, int rows, int h,
                          cudaStream_t st);
cudaError_t ln_bwd_launch(const void* dy, const void* x, const float* g, const void* dres, void* dx,
                          float* dg, float* db, float* stats, int rows, int h, cudaStream_t st);
cudaError_t mse_loss_launch(const void* z, int64_t n, void* dz, double* sumsq, cudaStream_t st);
cudaError_t axpy_f32_launch(float* y, const float* x, int64_t n, cudaStream_t st);
cudaError_t attn_fwd_launch(const void* qkv, int ld_qkv, void* o, int ld_o, float* lse, int s, int b,
                            int heads, int d, cudaStream_t st);
struct AttnParams;
cudaError_t attn_fwd1_launch(const void* qkv, int ld_qkv, const AttnParams& p, int d, cudaStream_t st);
cudaError_t attn_bwd_delta_launch(const void* o, const void* d_o, int ld_o, float* delta, int s, int b, int heads,
                                  int d, cudaStream_t st);
cudaError_t attn_bwd_launch(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o,
                            const float* lse, float* delta, float* dq_acc, void* dqkv, int ld_dqkv,
                            int s, int b, int heads, int d, cudaStream_t st);

cudaError_t embed_fwd_launch(const int* tok, const void* w_emb, const void* w_pos, void* x, int s, int b, int h,
                             cudaStream_t st);
cudaError_t embed_bwd_launch(const int* tok, const void* dx, float* dw_emb, float* dw_pos, int s, int b, int h,
                             cudaStream_t st);
cudaError_t ce_loss_launch(void* logits, int ld, const int* labels, int rows, int vocab, int vpad, float scale,
                           double* loss_acc, int* count_acc, cudaStream_t st);

cudaError_t gemm_launch(const GemmOperand& a, const GemmOperand& b, const GemmParams& p,
                        cudaStream_t stream);

int num_sms();

}  // namespace hx
