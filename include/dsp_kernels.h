/*
 * dsp_kernels.h — building-block entry points of the DSP hot path (same library,
 * same conventions as dsp.h: device pointers, 16-B alignment, stream-ordered,
 * dsp_status_t errors, no allocation).  dsp_st_block_forward is composed of exactly
 * these operations plus dsp_switch; they are exported so each stage can be checked
 * against the oracle on its own (stage-level parity, e.g. peaky softmax).
 */
#ifndef DSP_KERNELS_H_
#define DSP_KERNELS_H_

#include "dsp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Per-token LayerNorm over C ("Layer normalization is also applied before each
 * layer"; R3): y = (x - mean) / sqrt(var + eps) * gamma + beta, biased variance, fp32
 * math, output in `dtype`.  x, y: [rows, C] (may be equal); gamma, beta: [C].
 * Errors: NULL, SHAPE (rows < 0, C < 1), ALIGNMENT (C*elem % 16 for bf16). */
dsp_status_t dsp_layer_norm(dsp_ctx_t ctx, dsp_dtype_t dtype, int64_t rows, int64_t C,
                            const void* x, const void* gamma, const void* beta, float eps,
                            void* y, void* stream);

/* Linear layer epilogue kinds for dsp_linear. */
typedef enum {
  DSP_EPI_NONE = 0,      /* D = A W^T */
  DSP_EPI_RESIDUAL = 1,  /* D = R + A W^T        (R may equal D) */
  DSP_EPI_GELU = 2       /* D = gelu_tanh(A W^T) (R5) */
} dsp_epilogue_t;

/* D[M,N] = epi(A[M,K] * W[N,K]^T): nn.Linear without bias (R4).  All row-major.
 * bf16: persistent tcgen05 GEMM (TMA -> smem -> tcgen05.mma -> TMEM -> epilogue),
 * fp32 accumulation, requires K % 8 == 0 and N % 32 == 0 (else UNSUPPORTED).
 * f32 : SIMT check-path GEMM.  D must not overlap A or W. */
dsp_status_t dsp_linear(dsp_ctx_t ctx, dsp_dtype_t dtype, int64_t M, int64_t N, int64_t K,
                        const void* A, const void* W, const void* R, dsp_epilogue_t epi,
                        void* D, void* stream);

/* Attention core over the packed projection qkv [tok, 3C] ([q | k | v] columns, head j
 * at columns j*Dh.. of each part; R8): for every sequence and head
 *   O_j = softmax(q_j k_j^T / sqrt(Dh)) v_j     (R6, R7: no mask, no bias)
 * written to o [tok, C] (heads concatenated).  `dim` selects the sequences in the
 * local layout [B, T_loc, S_loc, C] (tok = B*T_loc*S_loc): DSP_DIM_S = spatial (one
 * sequence of length S_loc per (b,t)), DSP_DIM_T = temporal (one sequence of length
 * T_loc per (b,s)).  bf16: tcgen05/TMEM flash-attention kernel (online softmax in fp32,
 * P rounded to bf16 for the PV product); f32: SIMT check path. */
dsp_status_t dsp_attention_core(dsp_ctx_t ctx, dsp_dtype_t dtype, int64_t B, int64_t T_loc,
                                int64_t S_loc, int64_t C, int32_t num_heads, dsp_dim_t dim,
                                const void* qkv, void* o, void* stream);

/* ---- the NCCL transport of the dynamic switch, piece by piece (§3.1; SURVEY §8a "The
 * switch as an exact index map").  dsp_switch(impl = NCCL) is exactly
 *   dsp_switch_pack -> ncclAlltoAll(send, recv, chunk bytes per peer) -> dsp_switch_unpack
 * (each copy skipped there when it is an identity).  Chunk order of send / recv: one chunk
 * of B*(T/N)*(S/N)*C*elem bytes per peer, peers in rank order, each chunk [b][t'][s'][c]:
 *   T->S pack:   send[q][b][t'][s'][c] = x_local[b][t'][q*S/N + s'][c]     (x_local [B,T/N,S,C])
 *   T->S unpack: y_local[b][r*T/N + t'][s'][c] = recv[r][b][t'][s'][c]     (y_local [B,T,S/N,C])
 *   S->T pack:   send[r][b][t'][s'][c] = x_local[b][r*T/N + t'][s'][c]     (x_local [B,T,S/N,C])
 *   S->T unpack: y_local[b][t'][q*S/N + s'][c] = recv[q][b][t'][s'][c]     (y_local [B,T/N,S,C])
 * where recv on rank q holds, in slot r, the chunk rank r packed for q.  Local (no
 * communication), always launch one strided-run copy kernel.  Buffers: shard size
 * B*T*S*C*elem/N bytes each, device, 16-B aligned, non-overlapping.
 * Errors: as dsp_switch (SAME_DIM, BAD_DIM, DIVISIBILITY, ALIGNMENT, ALIAS), NULL, CUDA. */
dsp_status_t dsp_switch_pack(dsp_ctx_t ctx, const dsp_shape_t* shape, dsp_dim_t from_dim, dsp_dim_t to_dim,
                             const void* x_local, void* send, void* stream);
dsp_status_t dsp_switch_unpack(dsp_ctx_t ctx, const dsp_shape_t* shape, dsp_dim_t from_dim, dsp_dim_t to_dim,
                               const void* recv, void* y_local, void* stream);

/* The unpack of dsp_gather: `gathered` is the rank-major [N][local shard] buffer an
 * all-gather of the shards produces; x_global [B,T,S,C] receives shard r at its place along
 * `dim`.  Local, one strided-run copy kernel (always launched).  Errors: as dsp_split. */
dsp_status_t dsp_gather_unpack(dsp_ctx_t ctx, const dsp_shape_t* shape, dsp_dim_t dim, const void* gathered,
                               void* x_global, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DSP_KERNELS_H_ */
