// extern "C" boundary of libhx (declared in include/hx.h): argument checks,
// TMA tensor-map encoding, kernel dispatch, launch accounting.
#include <atomic>
#include <cstdio>

#include "hx_common.cuh"
#include "hx_gemm.h"

namespace hx {

static std::atomic<long long> g_launches{0};
// -1: not set through hx_set_sm_reserve, fall back to the HX_SM_RESERVE env var
static std::atomic<int> g_sm_reserve{-1};

// SMs available to persistent kernels.  The reserve leaves SMs free for
// concurrently running NCCL point-to-point kernels in multi-stage runs, so a
// statically scheduled persistent GEMM never waits for a CTA slot.
int num_sms() {
  static int total = 0;
  static int env_reserve = 0;
  if (total == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&total, cudaDevAttrMultiProcessorCount, dev);
    if (total <= 0) total = 148;
    const char* r = getenv("HX_SM_RESERVE");
    env_reserve = r ? atoi(r) : 0;
  }
  int reserve = g_sm_reserve.load();
  if (reserve < 0) reserve = env_reserve;
  return (reserve > 0 && reserve < total) ? total - reserve : total;
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

static cudaError_t encode(CUtensorMap* map, const void* ptr, cuuint32_t rank, const cuuint64_t* dims,
                          const cuuint64_t* strides, const cuuint32_t* box,
                          CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiled fn = encode_fn();
  if (!fn) return cudaErrorInitializationError;
  cuuint32_t elem_strides[3] = {1, 1, 1};
  CUresult r = fn(map, dtype, rank, const_cast<void*>(ptr), dims, strides, box,
                  elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_tma_2d_sw64(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
                             uint32_t box_cols, uint32_t box_rows) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  return encode(map, ptr, 2, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_64B);
}

cudaError_t make_tma_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
                        uint32_t box_cols, uint32_t box_rows) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  return encode(map, ptr, 2, dims, strides, box);
}

cudaError_t make_tma_3d_rows(CUtensorMap* map, const void* ptr, uint64_t cols, uint64_t b, uint64_t s,
                             uint64_t ld, uint32_t box_cols, uint32_t box_rows) {
  const cuuint64_t dims[3] = {cols, b, s};
  const cuuint64_t strides[2] = {ld * 2, ld * b * 2};
  const cuuint32_t box[3] = {box_cols, 1, box_rows};
  return encode(map, ptr, 3, dims, strides, box);
}

cudaError_t make_tma_f32_3d(CUtensorMap* map, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                            uint32_t box0, uint32_t box1) {
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {d0 * 4, d0 * d1 * 4};
  const cuuint32_t box[3] = {box0, box1, 1};
  return encode(map, ptr, 3, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

}  // namespace hx

using namespace hx;

static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
static inline int ret(cudaError_t e, int kernels) {
  if (e == cudaSuccess) {
    g_launches += kernels;
    return HX_OK;
  }
  return static_cast<int>(e);
}

extern "C" {

int hx_version(void) { return 100; }

long long hx_launch_count(void) { return g_launches.load(); }

int hx_set_sm_reserve(int sms) {
  if (sms < 0 || sms > 64) return HX_E_SHAPE;
  g_sm_reserve.store(sms);
  return HX_OK;
}

int hx_gemm(const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C, int ldc, int M,
            int N, int K, int epi, const void* aux, int ld_aux, void* out2, int ld_out2, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0) return HX_E_SHAPE;
  // K (the reduction extent) needs 16-byte granularity only for a K-major
  // operand; an MN-major one (the weight-gradient form X^T dY over a ragged MLP
  // row slab) reads its K tail through TMA out-of-bounds zero fill
  if (((!a_mn || !b_mn) && K % 8) || N % 8 || lda % 8 || ldb % 8 || ldc % 4) return HX_E_SHAPE;
  if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return HX_E_ALIGN;
  if (epi < HX_EPI_STORE_BF16 || epi > HX_EPI_STORE_F32) return HX_E_UNSUPPORTED;
  if (epi == HX_EPI_ACC_F32 || epi == HX_EPI_STORE_F32) {
    if (ldc % 4) return HX_E_SHAPE;
  } else if (ldc % 8) {
    return HX_E_SHAPE;
  }
  if ((epi == HX_EPI_RESID_BF16 || epi == HX_EPI_DGELU) && (!aux || !aligned16(aux) || ld_aux % 8))
    return HX_E_ALIGN;
  if (epi == HX_EPI_GELU && (!out2 || !aligned16(out2) || ld_out2 % 8)) return HX_E_ALIGN;
  if (!a_mn && lda < K) return HX_E_SHAPE;
  if (a_mn && lda < M) return HX_E_SHAPE;
  if (!b_mn && ldb < K) return HX_E_SHAPE;
  if (b_mn && ldb < N) return HX_E_SHAPE;
  GemmOperand a{A, lda, a_mn != 0}, b{B, ldb, b_mn != 0};
  GemmParams p{M, N, K, epi, C, ldc, aux, ld_aux, out2, ld_out2, 1, 16};
  return ret(gemm_launch(a, b, p, as_stream(stream)), 1);
}

int hx_ln_fwd(const void* x, const float* gain, const float* bias, void* y, int rows, int h, void* stream) {
  if (rows <= 0 || h <= 0 || h % 8 || h > 8192) return HX_E_SHAPE;
  if (!aligned16(x) || !aligned16(y) || !aligned16(gain) || !aligned16(bias)) return HX_E_ALIGN;
  return ret(ln_fwd_launch(x, gain, bias, y, rows, h, as_stream(stream)), 1);
}

int hx_ln_bwd(const void* dy, const void* x, const float* gain, const void* dres, void* dx, float* dgain_acc,
              float* dbias_acc, float* stats_ws, int rows, int h, void* stream) {
  if (rows <= 0 || h <= 0 || h % 8 || h > 8192) return HX_E_SHAPE;
  if (!aligned16(dy) || !aligned16(x) || !aligned16(dx) || !aligned16(gain) || (dres && !aligned16(dres)) ||
      !aligned16(stats_ws))
    return HX_E_ALIGN;
  return ret(ln_bwd_launch(dy, x, gain, dres, dx, dgain_acc, dbias_acc, stats_ws, rows, h, as_stream(stream)), 2);
}

int hx_attn_fwd(const void* qkv, int ld_qkv, void* o, int ld_o, float* lse, int s, int b, int heads, int d,
                void* stream) {
  if (d != 64 && d != 128) return HX_E_UNSUPPORTED;
  if (s <= 0 || b <= 0 || heads <= 0 || ld_qkv < 3 * heads * d || ld_o < heads * d) return HX_E_SHAPE;
  if (ld_qkv % 8 || ld_o % 8) return HX_E_SHAPE;
  if (!aligned16(qkv) || !aligned16(o) || !aligned16(lse)) return HX_E_ALIGN;
  return ret(attn_fwd_launch(qkv, ld_qkv, o, ld_o, lse, s, b, heads, d, as_stream(stream)), 1);
}

int hx_attn_bwd(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o, const float* lse,
                float* delta_ws, float* dq_ws, void* dqkv, int ld_dqkv, int s, int b, int heads, int d,
                void* stream) {
  if (d != 64 && d != 128) return HX_E_UNSUPPORTED;
  if (s <= 0 || b <= 0 || heads <= 0 || ld_qkv < 3 * heads * d || ld_o < heads * d ||
      ld_dqkv < 3 * heads * d)
    return HX_E_SHAPE;
  if (ld_qkv % 8 || ld_o % 8 || ld_dqkv % 8) return HX_E_SHAPE;
  if (!aligned16(qkv) || !aligned16(o) || !aligned16(d_o) || !aligned16(lse) || !aligned16(delta_ws) ||
      !aligned16(dq_ws) || !aligned16(dqkv))
    return HX_E_ALIGN;
  return ret(attn_bwd_launch(qkv, ld_qkv, o, d_o, ld_o, lse, delta_ws, dq_ws, dqkv, ld_dqkv, s, b, heads, d,
                             as_stream(stream)),
             o != nullptr ? 3 : 2);
}

long long hx_attn_bwd_ws_bytes(int s, int b, int heads, int d) {
  if (s <= 0 || b <= 0 || heads <= 0 || d <= 0) return 0;
  return static_cast<long long>(s) * b * heads * d * 4;  // the fp32 dQ accumulator
}

int hx_attn_bwd_delta(const void* o, const void* d_o, int ld_o, float* delta, int s, int b, int heads, int d,
                      void* stream) {
  if (d != 64 && d != 128) return HX_E_UNSUPPORTED;
  if (s <= 0 || b <= 0 || heads <= 0 || ld_o < heads * d || ld_o % 8) return HX_E_SHAPE;
  if (!aligned16(o) || !aligned16(d_o) || !aligned16(delta)) return HX_E_ALIGN;
  return ret(attn_bwd_delta_launch(o, d_o, ld_o, delta, s, b, heads, d, as_stream(stream)), 1);
}

int hx_embed_fwd(const int* tokens, const void* w_emb, const void* w_pos, void* x, int s, int b, int h,
                 void* stream) {
  if (s <= 0 || b <= 0 || h <= 0 || h % 8) return HX_E_SHAPE;
  if (!aligned16(w_emb) || !aligned16(w_pos) || !aligned16(x)) return HX_E_ALIGN;
  return ret(embed_fwd_launch(tokens, w_emb, w_pos, x, s, b, h, as_stream(stream)), 1);
}

int hx_embed_bwd(const int* tokens, const void* dx, float* dw_emb, float* dw_pos, int s, int b, int h,
                 void* stream) {
  if (s <= 0 || b <= 0 || h <= 0 || h % 8) return HX_E_SHAPE;
  if (!aligned16(dx) || !aligned16(dw_emb) || !aligned16(dw_pos)) return HX_E_ALIGN;
  return ret(embed_bwd_launch(tokens, dx, dw_emb, dw_pos, s, b, h, as_stream(stream)), 1);
}

int hx_ce_loss(void* logits, int ld, const int* labels, int rows, int vocab, int vpad, float scale,
               double* loss_acc, int* count_acc, void* stream) {
  if (rows <= 0 || vocab <= 0 || vpad < vocab || vpad % 8 || ld < vpad || ld % 8) return HX_E_SHAPE;
  if (!aligned16(logits)) return HX_E_ALIGN;
  return ret(ce_loss_launch(logits, ld, labels, rows, vocab, vpad, scale, loss_acc, count_acc, as_stream(stream)),
             1);
}

int hx_mse_loss(const void* z, long long n, void* dz, double* sumsq_acc, void* stream) {
  if (n <= 0 || n % 8) return HX_E_SHAPE;
  if (!aligned16(z) || !aligned16(dz)) return HX_E_ALIGN;
  return ret(mse_loss_launch(z, n, dz, sumsq_acc, as_stream(stream)), 1);
}

int hx_axpy_f32(float* y, const float* x, long long n, void* stream) {
  if (n <= 0) return HX_E_SHAPE;
  if (!aligned16(y) || !aligned16(x)) return HX_E_ALIGN;
  return ret(axpy_f32_launch(y, x, n, as_stream(stream)), 1);
}

int hx_zero(void* ptr, long long bytes, void* stream) {
  if (bytes < 0) return HX_E_SHAPE;
  if (bytes == 0) return HX_OK;
  return ret(cudaMemsetAsync(ptr, 0, static_cast<size_t>(bytes), as_stream(stream)), 0);
}

}  // extern "C"
