/*
 * libhx — C-ABI of the B200 (sm_100a) HelixPipe stage-execution kernels.
 *
 * The reference (pipelab, pure Python/NumPy) has no FFI: its stage-execution
 * boundary is the per-component function layer called by the executor.  Each
 * entry point below replaces one of those reference functions (file:line under
 * /root/reference/pkg/src/pipelab) and is what a maintainer would bind with
 * ctypes from the executor.
 *
 * Conventions
 *   - all pointers are device pointers; activations are bf16 row-major
 *     [s*b, width] (token-major, the reference's [s, b, h] layout flattened);
 *     LayerNorm gains/biases and gradient accumulators are fp32;
 *   - `stream` is a cudaStream_t passed as void*; calls are stream-ordered,
 *     never synchronise the host and never allocate (caller-provided memory);
 *   - return 0 on success, a cudaError_t value on a CUDA error, or an
 *     HX_E_* code when arguments violate the documented constraints.
 */
#ifndef HX_H_
#define HX_H_

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HX_API __attribute__((visibility("default")))
#else
#define HX_API
#endif

#define HX_OK 0
#define HX_E_SHAPE 1001       /* dimension not supported / inconsistent      */
#define HX_E_ALIGN 1002       /* pointer or stride not 16-byte aligned        */
#define HX_E_UNSUPPORTED 1003 /* e.g. head_dim outside {64, 128}              */

/* GEMM epilogues */
#define HX_EPI_STORE_BF16 0 /* C = acc (bf16)                                  */
#define HX_EPI_RESID_BF16 1 /* C = acc + aux (bf16 residual)                    */
#define HX_EPI_GELU 2       /* C = acc (pre-activation), out2 = gelu_erf(acc)  */
#define HX_EPI_DGELU 3      /* C = acc * gelu_erf'(aux)                         */
#define HX_EPI_ACC_F32 4    /* C(f32) += acc      (weight-gradient accumulate)  */
#define HX_EPI_STORE_F32 5  /* C(f32) = acc                                     */

/* Library version (major*10000 + minor*100 + patch). */
HX_API int hx_version(void);

/* Number of kernels this library launched since load (host-side counter). */
HX_API long long hx_launch_count(void);

/*
 * Leave `sms` SMs (0..64) free of persistent-kernel CTAs, for NCCL p2p kernels
 * running beside them when one stage runs per GPU (the reference's stage
 * threads, P/runtime/executor.py:334-382, become ranks).  Overrides the
 * HX_SM_RESERVE environment variable; applies to launches after the call.
 */
HX_API int hx_set_sm_reserve(int sms);

/*
 * C[M,N] (epi)= op(A)[M,K] * op(B)[K,N], bf16 in, fp32 accumulate (tcgen05/TMEM).
 *   a_mn=0: A stored [M,K] row-major (lda >= K);  a_mn=1: A stored [K,M] (lda >= M)
 *   b_mn=0: B stored [N,K] row-major (ldb >= K);  b_mn=1: B stored [K,N] (ldb >= N)
 * Replaces mathops.linear / linear_backward_x / linear_backward_w
 * (P/runtime/mathops.py:21-32) and the fused epilogues of
 * layers._post_trunk / mlp_forward / mlp_backward_b (layers.py:122-137,
 * mathops.py:122-157).  Constraints: K, N, lda, ldb, ldc multiples of 8.
 */
HX_API int hx_gemm(const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C, int ldc,
            int M, int N, int K, int epi, const void* aux, int ld_aux, void* out2, int ld_out2,
            void* stream);

/*
 * y = LayerNorm(x) * gain + bias over the last dim (biased variance, eps 1e-5).
 * Replaces mathops.layernorm (P/runtime/mathops.py:44-49).  h % 8 == 0, h <= 8192.
 */
HX_API int hx_ln_fwd(const void* x, const float* gain, const float* bias, void* y, int rows, int h,
              void* stream);

/*
 * dx = LN_B(dy, x, gain) (+ dres if non-null); dgain_acc += sum_rows dy*xhat;
 * dbias_acc += sum_rows dy.  Stats are recomputed from x as the reference does
 * and left in stats_ws (2*rows floats: mean, rstd per row).
 * Replaces mathops.layernorm_backward_b/_w (P/runtime/mathops.py:52-72) plus the
 * residual adds of layers.py:149 and :198.
 */
HX_API int hx_ln_bwd(const void* dy, const void* x, const float* gain, const void* dres, void* dx,
              float* dgain_acc, float* dbias_acc, float* stats_ws, int rows, int h, void* stream);

/*
 * Causal multi-head attention forward (flash, tcgen05).  qkv is [s*b, ld_qkv]
 * with q, k, v of head j at columns j*d, h + j*d, 2h + j*d (h = heads*d);
 * o is [s*b, ld_o] (head j at columns j*d); lse is [b, heads, s] (natural log
 * of the softmax denominator of the scaled scores, max folded in).
 * Replaces mathops.attention (P/runtime/mathops.py:83-100).  d in {64, 128}.
 */
HX_API int hx_attn_fwd(const void* qkv, int ld_qkv, void* o, int ld_o, float* lse, int s, int b,
                int heads, int d, void* stream);

/*
 * Causal attention backward.  Writes dq, dk, dv into dqkv ([s*b, ld_dqkv], same
 * column layout as qkv).  Workspaces: delta [b*heads*s] f32 (overwritten) and
 * dq_ws of hx_attn_bwd_ws_bytes(s, b, heads, d) bytes (the fp32 dQ
 * accumulator; overwritten, no state kept between calls).  With
 * o == NULL, delta is an input instead: D = rowsum(dO * O) from
 * hx_attn_bwd_delta (computed on the stage that holds O, so the attention
 * stage need not stash it).
 * Replaces mathops.attention_backward (P/runtime/mathops.py:103-116).
 */
HX_API int hx_attn_bwd(const void* qkv, int ld_qkv, const void* o, const void* d_o, int ld_o,
                const float* lse, float* delta_ws, float* dq_ws, void* dqkv, int ld_dqkv, int s,
                int b, int heads, int d, void* stream);

/* Bytes of hx_attn_bwd's dq_ws workspace (0 for invalid shapes). */
HX_API long long hx_attn_bwd_ws_bytes(int s, int b, int heads, int d);

/*
 * delta[b, heads, s] = rowsum(d_o * o) per head (f32), the flash backward's
 * D term (P/runtime/mathops.py:113: the rowsum(dP * P) of the reference,
 * which equals rowsum(dO * O)).  o, d_o: [s*b, ld_o] bf16.
 */
HX_API int hx_attn_bwd_delta(const void* o, const void* d_o, int ld_o, float* delta, int s, int b, int heads,
                             int d, void* stream);

/*
 * Paper §4.6 extras (the reference has no code for them,
 * SPEC.md:467).  Word + position embeddings in front of layer 0:
 * x[t] = w_emb[tokens[t]] + w_pos[t / b] (t = s_idx * b + b_idx; bf16 [*, h]).
 * tokens must lie in [0, rows of w_emb).
 */
HX_API int hx_embed_fwd(const int* tokens, const void* w_emb, const void* w_pos, void* x, int s, int b, int h,
                        void* stream);
/* dw_emb[tokens[t]] += dx[t] (fp32 atomics), dw_pos[s_idx] += sum_b dx[s_idx * b + b_idx]. */
HX_API int hx_embed_bwd(const int* tokens, const void* dx, float* dw_emb, float* dw_pos, int s, int b, int h,
                        void* stream);
/*
 * Next-token cross-entropy over a chunk of logits rows ([rows, ld] bf16, the
 * first vocab of vpad columns real): loss_acc[0] += sum over rows with
 * labels[r] >= 0 of lse(row) - row[labels[r]]; count_acc[0] += that row count;
 * the logits are overwritten by dlogits = (softmax - onehot) * scale (padded
 * columns and ignored rows: 0).  The loss-in-backward head of PAPER.md:443-444.
 */
HX_API int hx_ce_loss(void* logits, int ld, const int* labels, int rows, int vocab, int vpad, float scale,
                      double* loss_acc, int* count_acc, void* stream);

/*
 * sumsq_acc[0] += sum(z^2) (fp64); dz = z * 2/n.  loss = sumsq/n (host divides).
 * Replaces model.loss_and_grad (P/runtime/model.py:61-64).
 */
HX_API int hx_mse_loss(const void* z, long long n, void* dz, double* sumsq_acc, void* stream);

/* y[i] += x[i] (fp32): micro-batch gradient accumulation (executor.py:406-412). */
HX_API int hx_axpy_f32(float* y, const float* x, long long n, void* stream);

/* Zero `bytes` of device memory on `stream` (cudaMemsetAsync). */
HX_API int hx_zero(void* ptr, long long bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HX_H_ */
