/*
 * dsp_train.h — the training (backward) path of the DSP ST block.
 *
 * The paper's throughput numbers are training numbers (§4.2: "scale the number of GPUs
 * used for training"), and P:125 (§3.3) combines DSP with ZeRO, which shards the parameters and
 * therefore reduces their gradients over the ranks.  The backward of the DSP schedule reuses the
 * switch unchanged: a switch is a permutation of the activation's rows, so its adjoint is the
 * inverse switch (T->S backward = S->T; oracle/backward.py simulate_sharded_bwd pins it).
 *
 * Same conventions as dsp.h: device pointers, 16-B alignment, stream-ordered, dsp_status_t errors,
 * no allocation.  bf16 only; head dim 72 (C / num_heads, the paper's ST-DiT-XL width), sequence
 * lengths S and T each dividing or multiple of 128; raw (unprepared) weights; no cross stage,
 * Latte pair or positional embedding (the forward-only extras of dsp_block_weights_t must be NULL).
 *
 *   forward_train:  the forward of dsp_st_block_forward, additionally keeping the activations the
 *                   backward needs in `saved` (layout below).  COLLECTIVE.
 *   backward:       dx and the twelve weight gradients of the block for the upstream dy, from
 *                   `saved`.  Weight gradients are ACCUMULATED (+=) in fp32; at N > 1 they are
 *                   this rank's partial sums, reduced by dsp_grads_reduce.  COLLECTIVE.
 *
 * saved (per rank, tok = B*T*S/N tokens, elem = 2; offsets from dsp_train_saved_layout):
 *   h1 [tok, C]   LN1(x)             (T-sharded)      qkv_s [tok, 3C], o_s [tok, C], lse_s [tok, NH] f32
 *   y1s [tok, C]  y1 after the switch (S-sharded)     h2 = LN2(y1s), qkv_t, o_t, lse_t
 *   y2 [tok, C]   h3 = LN3(y2) [tok, C]               u = h3 W1^T, g = gelu_tanh(u) [tok, 4C]
 * lse rows are the log2-domain log-sum-exp of the scaled attention scores of each (token, head):
 * lse2 = log2 sum_j 2^(q.k_j log2(e) / sqrt(Dh)).
 */
#ifndef DSP_TRAIN_H_
#define DSP_TRAIN_H_

#include "dsp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* fp32 gradient accumulators of one block, same shapes as dsp_block_weights_t's twelve weights */
typedef struct {
  float *ln1_w, *ln1_b, *w_qkv_s, *w_o_s;
  float *ln2_w, *ln2_b, *w_qkv_t, *w_o_t;
  float *ln3_w, *ln3_b, *w_fc1, *w_fc2;
} dsp_block_grads_t;

/* byte offsets of the saved tensors (see above) and the total; host-only */
typedef struct {
  int64_t h1, qkv_s, o_s, lse_s, y1s, h2, qkv_t, o_t, lse_t, y2, h3, u, g, total;
} dsp_train_saved_layout_t;
dsp_status_t dsp_train_saved_layout(const dsp_shape_t* shape, int world, dsp_train_saved_layout_t* out);

/* context workspace (dsp_ctx_set_workspace) both calls need, host-only */
size_t dsp_train_workspace_bytes(const dsp_shape_t* shape, int world);

/* y_local = block(x_local) exactly as dsp_st_block_forward (raw weights), saving into `saved`
 * (>= dsp_train_saved_layout().total bytes, device, 256-B aligned).  x_local, y_local T-sharded
 * [B, T/N, S, C]; they must not overlap `saved` or the workspace.
 * Errors: NULL, SHAPE, DIVISIBILITY, ALIGNMENT, ALIAS, UNSUPPORTED (f32, Dh != 72, extras set,
 * sequence length neither dividing nor a multiple of 128, impl DSP_SWITCH_FUSED), WORKSPACE, CUDA, NCCL. */
dsp_status_t dsp_st_block_forward_train(dsp_ctx_t ctx, const dsp_shape_t* shape, const dsp_block_weights_t* w,
                                        const void* x_local, void* y_local, void* saved,
                                        dsp_switch_impl_t impl, void* stream);

/* Backward of the block at x_local (the forward_train input) for dy_local (both T-sharded
 * [B, T/N, S, C]): dx_local = d(block)/dx^T dy; grads += this rank's d(block)/dW^T dy (fp32).
 * Schedule: dy -> switch T->S (adjoint of the forward's S->T); MLP and temporal-stage backward on
 * S-shards; switch S->T (adjoint of T->S); spatial-stage backward on T-shards.  dx_local may
 * equal dy_local.  Errors: as dsp_st_block_forward_train. */
dsp_status_t dsp_st_block_backward(dsp_ctx_t ctx, const dsp_shape_t* shape, const dsp_block_weights_t* w,
                                   const void* saved, const void* x_local, const void* dy_local,
                                   void* dx_local, const dsp_block_grads_t* grads,
                                   dsp_switch_impl_t impl, void* stream);

/* Sum of every rank's fp32 gradients: zero_shard == 0: in-place all-reduce of buf[n]
 * (every rank gets the full sum); zero_shard == 1: ZeRO reduce-scatter, rank r receives elements
 * [r n/N, (r+1) n/N) of the sum in out[n/N] (n % N == 0).  NCCL on the context's communicator;
 * N == 1: no-op (zero_shard: copy).  COLLECTIVE.  Errors: NULL, SHAPE, NCCL, CUDA. */
dsp_status_t dsp_grads_reduce(dsp_ctx_t ctx, float* buf, int64_t n, int zero_shard, float* out, void* stream);

/* ---- building blocks (stage-level parity) ------------------------------------------------ */

/* dgrad of nn.Linear (R4): dX[M, K] = dY[M, N] W[N, K] (W in its forward [out, in] layout, read
 * as an MN-major tcgen05 operand: no transpose).  u != NULL: dX *= gelu_tanh'(u) elementwise
 * (u [M, K] bf16: the FC1 pre-activation; the GELU backward fused into the epilogue).
 * Requires K % 128 == 0, N % 8 == 0.  Errors: NULL, UNSUPPORTED, ALIGNMENT, ALIAS, CUDA. */
dsp_status_t dsp_linear_dgrad(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* dY, const void* W,
                              const void* u, void* dX, void* stream);

/* wgrad of nn.Linear: dW[N, K] (+)= dY[M, N]^T X[M, K] in fp32 (accumulate != 0: added to dW),
 * both activations token-major and read as MN-major operands; the token range is split over the
 * CTA pairs (fp32 partials in the workspace, summed in slice order: deterministic).  Requires
 * N % 64 == 0, K % 128 == 0; workspace >= dsp_wgrad_workspace_bytes(M, N, K).  */
size_t dsp_wgrad_workspace_bytes(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K);
dsp_status_t dsp_linear_wgrad(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* dY, const void* X,
                              float* dW, int accumulate, void* stream);

/* forward-train FC1: G = gelu_tanh(A W^T) and U = A W^T in one GEMM (both bf16 [M, N]) */
dsp_status_t dsp_linear_gelu_aux(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* A, const void* W,
                                 void* G, void* U, void* stream);

/* LayerNorm backward (R3) fused with the residual path: dx = dres + dLN(x)^T dh over
 * rows of C (dres may be NULL), and dgamma_dbeta[0:C] += sum_rows dh * xhat,
 * dgamma_dbeta[C:2C] += sum_rows dh (fp32).  bf16 x, gamma,
 * dh, dres, dx [rows, C]; C % 8 == 0, C <= 2048.  Workspace >= 8 rows + 2 C * 4 * ceil(rows / 64) bytes
 * (row statistics, then per-64-row column partials summed in chunk order). */
dsp_status_t dsp_layer_norm_bwd(dsp_ctx_t ctx, int64_t rows, int64_t C, const void* x, const void* gamma,
                                const void* dh, const void* dres, float eps, void* dx, float* dgamma_dbeta,
                                void* stream);

/* dsp_attention_core that also writes lse [tok, NH] (f32, log2 domain, see above) */
dsp_status_t dsp_attention_core_lse(dsp_ctx_t ctx, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C,
                                    int32_t num_heads, dsp_dim_t dim, const void* qkv, void* o, float* lse,
                                    void* stream);

/* Attention backward: from qkv [tok, 3C], o, dout [tok, C] and lse of the forward, the
 * gradient dqkv [tok, 3C] ([dq | dk | dv], same head layout as qkv).  tcgen05 kernel: per key tile
 * S^T = K Q^T, P^T = exp2(S^T scale - lse), dP^T = V dO^T, dS^T = P^T (dP^T - rowsum(dO o O)) / sqrt(Dh)
 * (P^T rounded to bf16 once, the same values in dV and dS), dV += P^T dO, dK += dS^T Q, dQ += dS K
 * (f32 TMA reduce-add across key tiles; one bf16 store when the sequence is one key tile).  Workspace >=
 * dsp_attention_bwd_workspace_bytes.  Errors: NULL, UNSUPPORTED (head dim != 72, C > 2048, sequence
 * length neither dividing nor a multiple of 128), ALIGNMENT, WORKSPACE, CUDA. */
size_t dsp_attention_bwd_workspace_bytes(int64_t tok, int64_t C, int32_t num_heads);
dsp_status_t dsp_attention_core_bwd(dsp_ctx_t ctx, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C,
                                    int32_t num_heads, dsp_dim_t dim, const void* qkv, const void* o,
                                    const void* dout, const float* lse, void* dqkv, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DSP_TRAIN_H_ */
