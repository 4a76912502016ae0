/*
 * dawnpiper.h -- C ABI of the B200 (sm_100a) pipeline-training extension.
 *
 * The reference (`dawnplan`, pure Python) has no native interface: its
 * pipeline run is the analytic `simulate(plan, g, cfg)` (simulate.py:130).
 * This ABI is what the B200 replacement of that run binds: the per-stage
 * executor's kernels (the fine-grained node vocabulary of synth.py:22-26,
 * 93-107), the swap engine's transfers for memopt `swap` actions
 * (memopt.py:208,282), and the boundary P2P copies of `_boundary_bytes`
 * (simulate.py:93-100).  See INTEGRATION.md for the ctypes binding.
 *
 * Conventions
 *   - every function returns 0 on success, 1 on a bad argument, 2 on a CUDA
 *     error; dpn_last_error() returns the calling thread's last message;
 *   - no C++ exception crosses the ABI; no torch type appears in it;
 *   - pointers are device pointers unless named host_*; the caller owns all
 *     memory and keeps it alive until work on `stream` completes;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream);
 *   - "bf16" buffers are IEEE bfloat16, "f32" buffers IEEE float.
 */
#ifndef DAWNPIPER_H_
#define DAWNPIPER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPN_ABI_VERSION 1

/* ---- runtime ------------------------------------------------------------ */
const char* dpn_last_error(void);
int dpn_version(void);
/* Bind the calling thread to `device`; fails unless it is an sm_100 part. */
int dpn_init(int device);
int dpn_host_alloc(int64_t bytes, void** out);   /* pinned, portable */
int dpn_host_free(void* host_ptr);
int dpn_memset_async(void* dst, int value, int64_t bytes, void* stream);

/* Per-stage device arenas (runtime/arena.py).  One cudaMalloc of cap_bytes per arena; torch's
 * caching allocator draws its segments from it through a MemPool whose pluggable allocator is
 * dpn_arena_malloc / dpn_arena_free, so the arena is the stage's device-memory cap and its
 * high-water mark the stage's measured peak.  The arena serving a malloc is the calling thread's
 * current one (dpn_arena_select; -1 = none, mallocs then fail). */
int dpn_arena_create(int device, int64_t cap_bytes, int* handle);
int dpn_arena_destroy(int handle);
int dpn_arena_select(int handle);
int dpn_arena_stats(int handle, int64_t* in_use, int64_t* peak, int64_t* cap);
int dpn_arena_reset_peak(int handle);
void* dpn_arena_malloc(size_t size, int device, void* stream);    /* torch pluggable (cudaStream_t) */
void dpn_arena_free(void* ptr, size_t size, int device, void* stream);
/* Free every arena the library created (device synchronize first). */
int dpn_destroy(void);

/* Swap engine (memopt swap actions).  The copy is issued on copy_stream after
 * it waits for ready_event (if non-NULL); done_event (if non-NULL) is recorded
 * after the copy.  Replaces the analytic swap window of memopt.py:137-143. */
int dpn_swap_out(void* host_dst, const void* dev_src, int64_t bytes, void* copy_stream,
                 void* ready_event, void* done_event);
int dpn_swap_in(void* dev_dst, const void* host_src, int64_t bytes, void* copy_stream,
                void* ready_event, void* done_event);

/* Boundary activation / gradient hand-off between stages (simulate.py:93-114):
 * device-to-device when co-located, cudaMemcpyPeerAsync over NVLink otherwise. */
int dpn_p2p_copy(void* dst, int dst_dev, const void* src, int src_dev, int64_t bytes, void* stream);
int dpn_enable_peer(int dev, int peer);

/* ---- dense contraction (tcgen05 / TMEM / TMA) ----------------------------
 * C[z] = epi(alpha * A[z] B[z]^T), A[z]: M x K, B[z]: N x K, z = z1 + batch1*z2.
 * A K-major: element (m,k) at A + z1*a_s1 + z2*a_s2 + m*lda + k;
 * A MN-major: element (m,k) at A + z1*a_s1 + z2*a_s2 + k*lda + m (same for B).
 * Epilogue: + bias[n] (bf16), + residual (bf16, C layout with ldr/r_s*) or
 * x gelu'(residual) (residual_mode 1),
 * optional tanh-GELU (aux, if set, receives the pre-GELU value), store as
 * bf16 or f32 (optionally accumulating into f32).  Operand bases 16-byte
 * aligned, lda/ldb/ldc and batch strides multiples of 8 elements. */
typedef struct {
  int64_t M, N, K;
  int64_t batch1, batch2;
  const void* A; int64_t lda, a_s1, a_s2; int32_t a_mn_major;
  const void* B; int64_t ldb, b_s1, b_s2; int32_t b_mn_major;
  void* C; int64_t ldc, c_s1, c_s2; int32_t c_dtype; /* 0 f32, 1 bf16 */ int32_t accumulate;
  const void* bias;
  const void* residual; int64_t ldr, r_s1, r_s2;
  int32_t residual_mode; /* 0: C += residual; 1: C *= gelu'(residual) (fused GELU backward) */
  void* aux;
  float alpha; int32_t gelu;
  int32_t block_n; /* 0 = heuristic, else 64 / 128 / 256 */
  int32_t split_k; /* f32 output without bias/residual/GELU only: 0 = heuristic, 1 = off, n = n splits */
  int32_t cta_group; /* 0 = heuristic, 1 = one CTA per tile, 2 = CTA pair (tcgen05 cta_group::2, 256-row tile), 4 = two pairs sharing A by TMA multicast (block_n 256) */
  int32_t epilogue; /* 0 = TMA-staged stores when unbatched (default), 1 = direct per-thread stores */
  float* colsum; /* optional (bf16 C, TMA-staged epilogue): colsum[n] += sum_m C[m, n] of the stored
                    values -- the bias gradient of the linear whose output gradient C is, fused
                    into the GEMM that produces it (replaces a dpn_colsum pass over C) */
} dpn_gemm_args;
int dpn_gemm(const dpn_gemm_args* args, void* stream);

/* ---- fused attention (tcgen05 flash-style; head_dim 64) ------------------
 * qkv: [batch*seq, 3*heads*64] bf16 (Q | K | V column blocks, head-major within
 * each), out: [batch*seq, heads*64] bf16, lse: [batch, heads, seq] f32 (natural
 * log-sum-exp of scale * QK^T per query, saved for the backward).  seq % 64 == 0. */
int dpn_attn_fwd(const void* qkv, void* out, float* lse, int64_t batch, int64_t seq, int64_t heads,
                 int64_t head_dim, float scale, int causal, void* stream);
/* Backward: writes all of dqkv (dQ | dK | dV) from qkv, out, dout (= dL/dout) and
 * the forward's lse.  workspace: >= batch*seq*heads*64 + batch*heads*seq floats. */
int dpn_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                 float* workspace, int64_t workspace_floats, int64_t batch, int64_t seq,
                 int64_t heads, int64_t head_dim, float scale, int causal, float* dbias, void* stream);
/* dbias (optional, 16-byte aligned f32 [3H]): += the column sums of dQ | dK | dV --
 * the fused QKV projection's bias gradient, accumulated by the dQ store and the
 * dK / dV drain (replaces a dpn_colsum pass over dqkv). */

/* Cross-attention (T5 decoder): q [batch*q_seq, heads*64], kv [batch*kv_seq,
 * 2*heads*64] (K | V column blocks), out [batch*q_seq, heads*64], lse [batch,
 * heads, q_seq]; no mask.  Backward writes dq (like q) and dkv (like kv);
 * workspace >= batch*q_seq*heads*64 + batch*heads*q_seq floats. */
int dpn_attn_fwd_cross(const void* q, const void* kv, void* out, float* lse, int64_t batch,
                       int64_t q_seq, int64_t kv_seq, int64_t heads, int64_t head_dim, float scale,
                       void* stream);
int dpn_attn_bwd_cross(const void* q, const void* kv, const void* out, const void* dout,
                       const float* lse, void* dq, void* dkv, float* workspace,
                       int64_t workspace_floats, int64_t batch, int64_t q_seq, int64_t kv_seq,
                       int64_t heads, int64_t head_dim, float scale, void* stream);

/* ---- node kernels (bf16 storage, fp32 math) ------------------------------ */
/* ln1 / ln2 / lnf: y = (x - mean) * rstd * gamma + beta; mean/rstd saved (f32 [rows]). */
int dpn_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean,
                      float* rstd, int64_t rows, int64_t cols, float eps, void* stream);
/* dx = LN'(dy) (+ dx_add if non-NULL, may alias dx); dgamma/dbeta += (f32), both
 * NULL to skip the parameter gradients.  workspace: unused since ABI 1.1 (pass
 * NULL / 0); kept so the signature is stable. */
int dpn_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean,
                      const float* rstd, void* dx, const void* dx_add, float* dgamma, float* dbeta,
                      int64_t rows, int64_t cols, float* workspace, int64_t workspace_floats,
                      void* stream);
/* LayerNorm backward in one pass: dx (+= dx_add when given), dgamma += sum dy * xhat,
 * dbeta += sum dy and, when dbias is given, dbias += column sums of the final dx (the
 * bias gradient of the linear node whose output gradient dx is).  Replaces the
 * ln_dx + column-reduction pair of dpn_layernorm_bwd for the fused executor path. */
int dpn_layernorm_bwd_fused(const void* dy, const void* x, const void* gamma, const float* mean,
                            const float* rstd, void* dx, const void* dx_add, float* dgamma,
                            float* dbeta, float* dbias, int64_t rows, int64_t cols, void* stream);
/* score: P = softmax(alpha * S) per row; causal masks key > (row % q_len). */
int dpn_softmax_fwd(const void* s, void* p, int64_t rows, int64_t cols, int64_t q_len, float alpha,
                    int causal, void* stream);
/* dS = alpha * P * (dP - rowsum(dP * P)) */
int dpn_softmax_bwd(const void* p, const void* dp, void* ds, int64_t rows, int64_t cols,
                    float alpha, void* stream);
int dpn_gelu_fwd(const void* x, void* y, int64_t n, void* stream);
int dpn_gelu_bwd(const void* dy, const void* x, void* dx, int64_t n, void* stream);
int dpn_add(const void* a, const void* b, void* out, int64_t n, void* stream);
int dpn_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream);
/* out[c] += sum_r x[r, c]   (bias gradients; single pass, vector atomics).
 * workspace: unused since ABI 1.1 (pass NULL / 0). */
int dpn_colsum(const void* x, int64_t rows, int64_t cols, int64_t ld, float* out, float* workspace,
               int64_t workspace_floats, void* stream);
/* head: *loss_sum += loss_scale * sum_r CE(logits[r, :vocab], labels[r]);
 * dlogits = (softmax - onehot) * grad_scale, pad columns [vocab, ld) zeroed.
 * dlogits may alias logits. */
int dpn_xent(const void* logits, int64_t ld, const int32_t* labels, int64_t rows, int64_t vocab,
             float grad_scale, float loss_scale, float* loss_sum, void* dlogits, void* stream);
/* embed: out[r] = tok[ids[r]] + pos[r % seq]; backward accumulates (f32). */
int dpn_embed_fwd(const int32_t* ids, const void* tok, const void* pos, void* out, int64_t rows,
                  int64_t seq, int64_t hidden, void* stream);
int dpn_embed_bwd(const int32_t* ids, const void* dout, float* dtok, float* dpos, int64_t rows,
                  int64_t seq, int64_t hidden, void* stream);
/* AdamW over a stage's flat f32 buffers; writes the new bf16 weight version. */
int dpn_adamw(float* w, float* m, float* v, const float* g, void* out_bf16, int64_t n, float lr,
              float beta1, float beta2, float eps, float weight_decay, int64_t step, void* stream);
/* AdamW with the step count in device memory (incremented, then used for the
 * bias corrections): replayable inside a CUDA graph. */
int dpn_adamw_dstep(float* w, float* m, float* v, const float* g, void* out_bf16, int64_t n,
                    float lr, float beta1, float beta2, float eps, float wd, int64_t* step_dev,
                    void* stream);

/* ---- CNN nodes (AmoebaNet-D; synth.py:123-135 conv / act / pool vocabulary) ----
 * Activations are NHWC bf16 viewed as [pixels, C], C % 8 == 0.  3x3 windows
 * use pad 1; output size (H-1)/stride+1.  Dense 1x1 convolutions are dpn_gemm. */
int dpn_relu_fwd(const void* x, void* y, int64_t n, void* stream);
int dpn_relu_bwd(const void* dy, const void* y, void* dx, int64_t n, void* stream);
/* depthwise 3x3, w: [C, 9] bf16; backward: dx (if non-NULL) and dw += (f32, if non-NULL) */
int dpn_dwconv3_fwd(const void* x, const void* w, void* y, int64_t b, int64_t H, int64_t W,
                    int64_t C, int64_t stride, void* stream);
int dpn_dwconv3_bwd(const void* x, const void* w, const void* dy, void* dx, float* dw, int64_t b,
                    int64_t H, int64_t W, int64_t C, int64_t stride, void* stream);
/* training-mode batch norm over P pixels; stats: [2, C] f32 (sum, sum of squares),
 * written by the forward and read by the backward.  Backward: dx, dgamma/dbeta +=
 * (f32); workspace >= 2*C floats. */
int dpn_bn_fwd(const void* x, const void* gamma, const void* beta, void* y, float* stats,
               int64_t P, int64_t C, float eps, void* stream);
int dpn_bn_bwd(const void* dy, const void* x, const float* stats, const void* gamma, void* dx,
               float* dgamma, float* dbeta, float* workspace, int64_t P, int64_t C, float eps,
               void* stream);
/* 3x3 pooling, mode 0 max (argmax: uint8 tap per output element), 1 average
 * (padding excluded from the count). */
int dpn_pool3_fwd(const void* x, void* y, void* argmax, int64_t b, int64_t H, int64_t W, int64_t C,
                  int64_t stride, int mode, void* stream);
int dpn_pool3_bwd(const void* dy, const void* argmax, void* dx, int64_t b, int64_t H, int64_t W,
                  int64_t C, int64_t stride, int mode, void* stream);
/* dst[r, :cols] (+)= src[r, :cols] with row strides lds / ldd (channel concat) */
int dpn_copy_cols(const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                  int accumulate, void* stream);
/* stem: cols[p, (r*3+s)*C + c] = x[n, ho*stride-1+r, wo*stride-1+s, c] (zero outside) */
int dpn_im2col3(const void* x, void* cols, int64_t b, int64_t H, int64_t W, int64_t C,
                int64_t stride, void* stream);
/* head: y[n, c] = mean over the HW pixels of sample n; backward spreads dy / HW */
int dpn_gap_fwd(const void* x, void* y, int64_t b, int64_t HW, int64_t C, void* stream);
int dpn_gap_bwd(const void* dy, void* dx, int64_t b, int64_t HW, int64_t C, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DAWNPIPER_H_ */
