/*
 * amdp_kernels.h — C-ABI of the sm_100a kernels under the AMDP stage executor.
 *
 * The reference (ppsim, /root/reference/proj/include/ppsim) has no kernels: a stage's
 * forward/backward is an opaque cost (`ClusterSpec::fwd_cost/bwd_cost`,
 * types.hpp:63-64) and the window update is a zero-duration Reduce/Broadcast event
 * (builder.hpp:272-304).  These entry points are the real work those events stand
 * for.  Conventions (all functions):
 *   - plain pointers to caller-owned device memory, sizes in elements;
 *   - stream-ordered on `stream` (a cudaStream_t), never synchronising;
 *   - return 0 on success, a positive cudaError_t value on a CUDA failure, or a
 *     negative AMDP_ERR_* code for invalid arguments; no exceptions cross the ABI.
 * bf16 tensors are `uint16_t` bit patterns in this header (no CUDA types needed).
 */
#ifndef AMDP_KERNELS_H_
#define AMDP_KERNELS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#pragma GCC visibility push(default)

typedef struct CUstream_st* amdp_stream_t;

#define AMDP_ERR_INVALID (-1)
#define AMDP_ERR_TMA (-2)
#define AMDP_ERR_CUDA (-3)
#define AMDP_ERR_UNSUPPORTED (-4)

/* ---------------------------------------------------------------- GEMM
 * C[m][n] = epilogue(alpha * sum_k A(m,k) * B(n,k)), bf16 operands, fp32 accumulate.
 *   A(m,k) = a_mn_major ? A[k*lda + m] : A[m*lda + k]
 *   B(n,k) = b_mn_major ? B[k*ldb + n] : B[n*ldb + k]
 * K must be a multiple of 64, N a multiple of 8; M, N otherwise arbitrary.
 * Used for every stage contraction: forward X.W^T (both K-major), activation
 * gradient dY.W (B MN-major) and weight gradient dY^T.X (both MN-major).          */
enum amdp_epilogue {
  AMDP_EPI_STORE_BF16 = 0, /* C bf16 = acc                                          */
  AMDP_EPI_GELU = 1,       /* C bf16 = gelu(acc); C2 bf16 = acc (pre-activation)    */
  AMDP_EPI_RESIDUAL = 2,   /* C bf16 = acc + aux (bf16 residual stream)             */
  AMDP_EPI_ACCUM_F32 = 3,  /* C f32 += acc (window gradient accumulation)           */
  AMDP_EPI_GELU_BWD = 4,   /* C bf16 = acc * gelu'(aux), aux = pre-activation       */
  AMDP_EPI_STORE_F32 = 5,  /* C f32 = acc                                           */
  AMDP_EPI_ROWDOT = 6      /* C bf16 = acc, and per row and rowdot_seg-column segment
                              rowdot[(m / rowdot_seq) * (N / rowdot_seg) + n / rowdot_seg]
                                    [m % rowdot_seq] = sum bf16(acc) * aux over the segment
                              (attention backward's delta = rowsum(dO * O) per head, fused
                              into the dO GEMM); A and B K-major, rowdot_seg a multiple of 64 */
};

typedef struct amdp_gemm_args {
  int M, N, K;
  const void* A;
  int lda;
  int a_mn_major;
  const void* B;
  int ldb;
  int b_mn_major;
  void* C;
  int ldc;
  const void* aux;
  int ld_aux;
  void* C2;
  int ldc2;
  int epilogue;
  float alpha;
  float* rowdot;     /* AMDP_EPI_ROWDOT only */
  int rowdot_seg;
  int rowdot_seq;
} amdp_gemm_args;

int amdp_gemm(const amdp_gemm_args* args, amdp_stream_t stream);

/* ---------------------------------------------------------------- attention
 * Causal (or full) multi-head attention over `batch` sequences of `seq` tokens.
 * qkv: [batch*seq][3*H*D] bf16 rows holding q | k | v (head-major inside each);
 * out: [batch*seq][H*D] bf16; lse: [batch][H][seq] fp32 log-sum-exp (saved for bwd).
 * D in {32, 64, 80, 128}.  key_len (bidirectional models only; NULL = none): device int32
 * [batch], the number of valid keys of each sequence — keys at positions >= key_len[b] are
 * padding and get no attention weight (BERT padding mask); padded query rows still get an
 * output (their loss is masked by the labels).                                       */
int amdp_attention_fwd(const uint16_t* qkv, uint16_t* out, float* lse, int batch, int seq,
                       int heads, int head_dim, int causal, const int32_t* key_len,
                       amdp_stream_t stream);
/* dout: [batch*seq][H*D]; writes dqkv [batch*seq][3*H*D] (dq | dk | dv).
 * workspace: at least amdp_attention_bwd_workspace() bytes (either causal value), or
 * amdp_attention_bwd_workspace_causal() for the causal value passed: delta[batch][H][seq]
 * (padded to 256 B), then the dS^T scratch of the tiled kernels
 * (amdp_attention_bwd_scratch_bytes: the dK/dV kernel stores dS^T there and dQ = dS K reads
 * it back instead of recomputing S, dP and the softmax).                             */
size_t amdp_attention_bwd_workspace(int batch, int seq, int heads, int head_dim);
size_t amdp_attention_bwd_workspace_causal(int batch, int seq, int heads, int head_dim, int causal);
size_t amdp_attention_bwd_scratch_bytes(int batch, int seq, int heads, int head_dim, int causal);
/* The same backward with delta[batch][H][seq] = rowsum(dout * out) per head supplied by the
 * caller (e.g. from the dO GEMM's AMDP_EPI_ROWDOT epilogue); tcgen05 path only
 * (amdp_attention_bwd_delta_supported), AMDP_ERR_UNSUPPORTED otherwise.             */
int amdp_attention_bwd_delta_supported(int seq, int head_dim);
/* Which implementation amdp_attention_fwd (backward = 0) / amdp_attention_bwd (1) dispatches
 * to for this shape: AMDP_ATTN_IMPL_TCGEN05 (tcgen05/TMEM/TMA: tiled kernels for head_dim
 * 64 / 80 / 128 with seq % 256 == 0 forward, seq % 128 == 0 backward; one-tile kernels for
 * seq <= 128 with head_dim 32 / 64), or -1 (unsupported: the calls return
 * AMDP_ERR_UNSUPPORTED).  AMDP_ATTN_IMPL_MMA_SYNC is no longer returned (kept for ABI
 * stability; round 1's warp-level fallback was removed).                                    */
enum { AMDP_ATTN_IMPL_MMA_SYNC = 0, AMDP_ATTN_IMPL_TCGEN05 = 1 };
int amdp_attention_impl(int seq, int head_dim, int backward);
int amdp_attention_bwd_delta(const uint16_t* qkv, const uint16_t* dout, const float* lse, const float* delta,
                             uint16_t* dqkv, int batch, int seq, int heads, int head_dim, int causal,
                             const int32_t* key_len, amdp_stream_t stream);
/* amdp_attention_bwd_delta with the dS^T scratch (amdp_attention_bwd_scratch_bytes for this
 * causal value; NULL = the dQ kernel that recomputes S / dP instead).                 */
int amdp_attention_bwd_delta_ws(const uint16_t* qkv, const uint16_t* dout, const float* lse, const float* delta,
                                uint16_t* dqkv, void* scratch, int batch, int seq, int heads, int head_dim,
                                int causal, const int32_t* key_len, amdp_stream_t stream);
int amdp_attention_bwd(const uint16_t* qkv, const uint16_t* out, const uint16_t* dout,
                       const float* lse, uint16_t* dqkv, void* workspace, int batch, int seq,
                       int heads, int head_dim, int causal, const int32_t* key_len,
                       amdp_stream_t stream);

/* ---------------------------------------------------------------- LayerNorm
 * y = (x - mean) * rstd * gamma + beta over rows of width `cols` (bf16 in/out,
 * fp32 gamma/beta/statistics).  mean/rstd: [rows] fp32, saved for backward.        */
/* f = gelu_tanh(u) elementwise, bf16 in / out (the GEMM GELU epilogue's formula). */
int amdp_gelu_fwd(const uint16_t* u, uint16_t* f, int64_t n, amdp_stream_t stream);
int amdp_layernorm_fwd(const uint16_t* x, const float* gamma, const float* beta, uint16_t* y,
                       float* mean, float* rstd, int rows, int cols, float eps,
                       amdp_stream_t stream);
/* dx = resid_grad + LN-backward(dy); dgamma/dbeta are ACCUMULATED (+=) in fp32.
 * resid_grad may be NULL (treated as zero) and may alias dx.
 * workspace: at least amdp_layernorm_bwd_workspace() bytes.                        */
size_t amdp_layernorm_bwd_workspace(int rows, int cols);
int amdp_layernorm_bwd(const uint16_t* dy, const uint16_t* x, const float* gamma,
                       const float* mean, const float* rstd, const uint16_t* resid_grad,
                       uint16_t* dx, float* dgamma, float* dbeta, void* workspace, int rows,
                       int cols, amdp_stream_t stream);
/* Deferred dgamma / dbeta (one column reduction per optimizer window instead of per call):
 * amdp_layernorm_bwd_rows writes dx like amdp_layernorm_bwd and ADDS its per-CTA column
 * partials into part[amdp_layernorm_bwd_parts(rows, cols)][2][cols] (zero-initialised by the
 * caller, then kept between calls of the same rows / cols on one stream); the flush adds the
 * column sums into dgamma / dbeta and zeroes part.  bwd_parts returns 0 (and bwd_rows
 * AMDP_ERR_UNSUPPORTED) for widths the row-group kernel does not take (cols % 256 != 0 or
 * cols > 4096): use amdp_layernorm_bwd there.                                          */
int amdp_layernorm_bwd_parts(int rows, int cols);
int amdp_layernorm_bwd_rows(const uint16_t* dy, const uint16_t* x, const float* gamma,
                            const float* mean, const float* rstd, const uint16_t* resid_grad,
                            uint16_t* dx, float* part, int rows, int cols, amdp_stream_t stream);
int amdp_layernorm_dgb_flush(float* part, int nparts, int cols, float* dgamma, float* dbeta,
                             amdp_stream_t stream);

/* ---------------------------------------------------------------- embedding
 * x[t] = wte[tokens[t]] + wpe[t % seq]   (bf16 tables, bf16 out)                    */
int amdp_embedding_fwd(const int32_t* tokens, const uint16_t* wte, const uint16_t* wpe,
                       uint16_t* x, int ntok, int seq, int hidden, amdp_stream_t stream);
/* dwte[tokens[t]] += dx[t]; dwpe[p] += sum over sequences of dx[b*seq+p]  (fp32).
 * Deterministic (no atomics): the (token, position) keys are sorted on the device and every
 * token's rows are summed in position order.  workspace: 4 * ntok bytes; ntok <= 16384,
 * vocab < 2^18.                                                                     */
int amdp_embedding_bwd(const int32_t* tokens, const uint16_t* dx, float* dwte, float* dwpe,
                       void* workspace, int ntok, int seq, int hidden, amdp_stream_t stream);

/* ---------------------------------------------------------------- cross-entropy
 * Fused softmax cross-entropy over bf16 logits [ntok][vocab] (row stride ld):
 * row_loss[t] = lse_t - logit[t][label_t] (scratch, ntok floats), then
 * loss_sum[0] += sum_t row_loss[t] in a fixed order (deterministic, no atomics);
 * logits are overwritten IN PLACE by d(loss * scale)/dlogits = scale*(softmax - onehot).
 * Labels < 0 are ignored (zero gradient, no loss).                                 */
int amdp_xent_fwd_bwd(uint16_t* logits, const int32_t* labels, float* loss_sum, float* row_loss,
                      int ntok, int vocab, int ld, float scale, amdp_stream_t stream);

/* ---------------------------------------------------------------- fp32 validation mode
 * The stage math in fp32 end to end on the CUDA cores (no bf16 storage, no tensor-core or SFU
 * approximations), deterministic: the engine's fp32 validation mode
 * (amdp_model_config.fp32_validation) runs these instead of the bf16 tcgen05 kernels so that
 * losses / weights can be checked against the fp64 CPU oracle at a tight tolerance.  Same
 * argument conventions as the bf16 kernels above with float tensors (GEMM: every epilogue
 * except AMDP_EPI_ROWDOT; C, C2, aux are fp32).                                       */
int amdp_f32_gemm(const amdp_gemm_args* args, amdp_stream_t stream);
int amdp_f32_layernorm_fwd(const float* x, const float* gamma, const float* beta, float* y,
                           float* mean, float* rstd, int rows, int cols, float eps,
                           amdp_stream_t stream);
int amdp_f32_layernorm_bwd(const float* dy, const float* x, const float* gamma,
                           const float* mean, const float* rstd, const float* resid_grad,
                           float* dx, float* dgamma, float* dbeta, int rows, int cols,
                           amdp_stream_t stream);
int amdp_f32_attention_fwd(const float* qkv, float* out, float* lse, int batch, int seq,
                           int heads, int head_dim, int causal, const int32_t* key_len,
                           amdp_stream_t stream);
size_t amdp_f32_attention_bwd_workspace(int batch, int seq, int heads);
int amdp_f32_attention_bwd(const float* qkv, const float* out, const float* dout,
                           const float* lse, float* dqkv, float* workspace, int batch, int seq,
                           int heads, int head_dim, int causal, const int32_t* key_len,
                           amdp_stream_t stream);
int amdp_f32_embedding_fwd(const int32_t* tokens, const float* wte, const float* wpe, float* x,
                           int ntok, int seq, int hidden, amdp_stream_t stream);
int amdp_f32_embedding_bwd(const int32_t* tokens, const float* dx, float* dwte, float* dwpe,
                           void* workspace, int ntok, int seq, int hidden, amdp_stream_t stream);
int amdp_f32_xent_fwd_bwd(float* logits, const int32_t* labels, float* loss_sum,
                          float* row_loss, int ntok, int vocab, int ld, float scale,
                          amdp_stream_t stream);

/* ---------------------------------------------------------------- optimizer
 * One fused pass per parameter: g = grad (fp32, then zeroed), state update, fp32
 * master update, bf16 copy refresh.  Modes:
 *   AMDP_OPT_REF_ADAMTYPE: the reference rule (optim.hpp:256-266): m = b1 m + (1-b1) g;
 *      v = b2 v + (1-b2) g^2; P = clamp(1/(sqrt(v)+eps), cmin, cmax); theta -= lr P m
 *   AMDP_OPT_ADAMW: bias-corrected Adam with decoupled weight decay (step >= 1).
 *   AMDP_OPT_SGD / AMDP_OPT_MOMENTUM: optim.hpp:243-255.
 * grad_scale multiplies g first (1/num_accumulated for a mean, or a clip factor). */
enum amdp_opt_kind {
  AMDP_OPT_SGD = 0,
  AMDP_OPT_MOMENTUM = 1,
  AMDP_OPT_REF_ADAMTYPE = 2,
  AMDP_OPT_ADAMW = 3
};
typedef struct amdp_opt_args {
  int kind;
  float lr, beta1, beta2, eps, weight_decay, clamp_min, clamp_max, grad_scale;
  int step; /* 1-based update count (AdamW bias correction) */
} amdp_opt_args;
int amdp_optimizer_step(const amdp_opt_args* args, float* master, float* m, float* v,
                        float* grad, uint16_t* weight_bf16, int64_t n, amdp_stream_t stream);
/* sum of squares of grad (fp32) accumulated into out[0] (for global-norm clipping) */
int amdp_sumsq(const float* x, int64_t n, float* out, amdp_stream_t stream);

/* ---------------------------------------------------------------- utilities      */
int amdp_fill_normal_bf16_f32(uint16_t* w_bf16, float* w_f32, int64_t n, uint64_t seed,
                              float stddev, amdp_stream_t stream);
int amdp_fill_const_f32(float* x, int64_t n, float value, amdp_stream_t stream);

/* Diagnostics: CTA 0 of the tensor-core attention forward records clock64() at each
 * pipeline hand-off into device_buf (>= 16*64 int64; NULL disables). */
int amdp_debug_attention_trace(long long* device_buf);
/* Every CTA of the attention forward writes (start ns, end ns, smid) at 3*blockIdx. */
int amdp_debug_attention_cta_times(long long* device_buf);
int amdp_debug_attention_bwd_trace(long long* device_buf); /* CTA 0 of the dQ kernel */

/* Library identification (for the loader's sanity check). */
const char* amdp_version(void);

#pragma GCC visibility pop
#ifdef __cplusplus
}
#endif

#endif /* AMDP_KERNELS_H_ */
