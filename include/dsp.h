/*
 * dsp.h — C ABI of the B200-native Dynamic Sequence Parallelism (DSP) hot path.
 *
 * Paper: "DSP: Dynamic Sequence Parallelism for Multi-Dimensional Transformers"
 * (arXiv 2403.10266).  Citations: P:n = line n of PAPER.md, S:n = line n of
 * SPEC.md (interfaces only), R<k> = reading k in DESIGN.md §Readings.
 *
 * What the library computes (§3.1 System Design): the forward of one
 * spatial-temporal (ST) transformer block whose activation X[B,T,S,C] (row-major,
 * C innermost) is sharded over N ranks along ONE sequence dimension.  Spatial
 * attention runs locally on T-shards; a dynamic switch ("a single AlltoAll
 * operation ... when transitioning between computation stages") re-shards
 * T->S; temporal attention and the MLP run locally on S-shards; a second switch
 * goes back S->T ("two AlltoAll operations in total").
 *
 * Conventions (apply to every call unless stated):
 *  - Pointers: arguments named *_dev / x_* / y_* / w_* / out / residual are DEVICE
 *    pointers; arguments named *_host are HOST pointers (pinned memory recommended).
 *    All device pointers must be 16-byte aligned.
 *  - Layout: activations are contiguous row-major [B, T_local, S_local, C].  Rank r
 *    holds the r-th contiguous chunk of the sharded axis (R11).  Weights use
 *    the nn.Linear [out, in] layout; inside w_qkv rows [0,C) are q, [C,2C) k, [2C,3C) v
 *    and head j owns rows j*Dh..(j+1)*Dh-1 of each (R8).
 *  - Shapes: dsp_shape_t holds the GLOBAL shape and must be identical on all ranks.
 *  - Dtypes: DSP_BF16 is the product path (bf16 storage, fp32 accumulation/softmax);
 *    DSP_F32 is the fp32 check path (SIMT kernels, for the 1e-4 gate).
 *  - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *    stream-ordered and asynchronous unless marked HOST-ONLY or SYNCHRONOUS; there is
 *    no host synchronisation and no allocation on the hot path.
 *  - Ownership: the caller owns every buffer (allocate with torch or cudaMalloc).  A
 *    context BORROWS the NCCL communicator and peer pointers; it owns host state only.
 *  - Collective calls (dsp_gather, dsp_switch, dsp_st_block_forward*) must be entered
 *    by all N ranks in the same order with identical shape / dims / impl.
 *    Argument validation depends only on those identical arguments, so every rank
 *    returns the same error BEFORE any communication is enqueued.
 *  - Errors: every call returns dsp_status_t; nothing throws across the ABI.  Detail
 *    text for the last non-OK status of a context: dsp_last_error(ctx).  CUDA / NCCL
 *    failures map to DSP_ERR_CUDA / DSP_ERR_NCCL.
 *  - Determinism: split/switch/gather move bytes only and are bit-exact.  Compute
 *    kernels use no atomics and no split-K: outputs are run-to-run deterministic and
 *    independent of N (each output element's reduction order depends only on C, Dh, L).
 */
#ifndef DSP_H_
#define DSP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dsp_ctx* dsp_ctx_t;

typedef enum {
  DSP_OK = 0,
  DSP_ERR_NULL = 1,          /* a required pointer is NULL */
  DSP_ERR_SHAPE = 2,         /* invalid shape (non-positive extent, C % num_heads != 0) */
  DSP_ERR_DIVISIBILITY = 3,  /* N does not divide T or S (R12) */
  DSP_ERR_SAME_DIM = 4,      /* switch from a dim to itself */
  DSP_ERR_BAD_DIM = 5,       /* dim is not DSP_DIM_T / DSP_DIM_S */
  DSP_ERR_UNSUPPORTED = 6,   /* valid request this build does not implement (reason in dsp_last_error) */
  DSP_ERR_ALIGNMENT = 7,     /* pointer not 16-B aligned or row bytes not a multiple of 16 */
  DSP_ERR_ALIAS = 8,         /* input and output buffers overlap where they must not */
  DSP_ERR_WORKSPACE = 9,     /* workspace missing or smaller than dsp_workspace_bytes() */
  DSP_ERR_CUDA = 10,         /* CUDA runtime / launch failure */
  DSP_ERR_NCCL = 11,         /* NCCL failure or NCCL not available for world > 1 */
  DSP_ERR_STATE = 12,        /* context misuse (wrong device, peer buffers not set, ...) */
  DSP_ERR_PEER_TIMEOUT = 13  /* a P2P barrier gave up waiting for a peer (dsp_ctx_check_errors) */
} dsp_status_t;

typedef enum { DSP_DIM_T = 1, DSP_DIM_S = 2 } dsp_dim_t;   /* axis index in [B,T,S,C] */
typedef enum { DSP_BF16 = 0, DSP_F32 = 1 } dsp_dtype_t;
/* Switch transport.  Explicit choice, no heuristic dispatch.
 * NCCL : pack kernel -> ncclAlltoAll (bytes) -> unpack kernel (identity sides skipped).
 * P2P  : direct NVLink stores into the peers' symmetric buffers + signal-pad barriers.
 * FUSED: (dsp_st_block_forward only) no separate switch: the spatial out-projection
 *        epilogue stores every output row directly at its final address in the S-shard
 *        owner's buffer, and the FC2 epilogue stores directly into the T-shard owner's
 *        y_local, over the peer mappings (the NVLink transfer overlaps the GEMM tiles);
 *        one signal-pad barrier after each of the two GEMMs -- with prepared weights split
 *        into the neighbouring kernels: the GEMM's last CTA arrives (release-stores the epoch
 *        into every peer's pad) and the next kernel that reads the rows (the LN2 partials pass;
 *        in dsp_st_model_forward the next block's LN1 partials pass) waits per row only for the
 *        rank that sent it, so no barrier kernel runs (the last block of a stack keeps its S->T
 *        barrier).  Needs the peer buffers of DSP_SWITCH_P2P; dsp_switch treats FUSED as P2P. */
typedef enum { DSP_SWITCH_NCCL = 0, DSP_SWITCH_P2P = 1, DSP_SWITCH_FUSED = 2 } dsp_switch_impl_t;

/* GLOBAL shape of the activation; identical on all ranks. */
typedef struct {
  int64_t B, T, S, C;
  int32_t num_heads;
  dsp_dtype_t dtype;
} dsp_shape_t;

/* Weights of one ST block (MHA + MLP, LayerNorm before each layer, residuals),
 * all device pointers in shape->dtype, nn.Linear [out,in] layout, no biases (R4). */
typedef struct {
  const void *ln1_w, *ln1_b, *w_qkv_s /*[3C,C]*/, *w_o_s /*[C,C]*/;
  const void *ln2_w, *ln2_b, *w_qkv_t /*[3C,C]*/, *w_o_t /*[C,C]*/;
  const void *ln3_w, *ln3_b, *w_fc1 /*[4C,C]*/, *w_fc2 /*[C,4C]*/;
  float ln_eps;                                    /* 1e-5 (R3) */
  /* NULL: the block runs three LayerNorm kernels.  Otherwise a buffer filled by
   * dsp_st_block_prepare() from THESE weights (bf16 only): every LayerNorm is folded into
   * the GEMM that consumes it (R30).  Stale if the weights change after preparing. */
  const void* prepared;
  /* Optional cross-attention stage of the ST-DiT block (NULL ln_c_w = none):
   *   y2 <- y2 + CA(LN_c(y2), ctx_tokens)   between the temporal stage and the MLP,
   * local on the S-shards (every rank holds the full context).  Weights as dsp_cross_attn
   * (w_q_c [C, C], w_kv_c [2C, C] rows [k | v], w_o_c [C, C]); ctx_tokens [B, ctx_len, C];
   * bf16 only. */
  const void *ln_c_w, *ln_c_b, *w_q_c, *w_kv_c, *w_o_c;
  const void* ctx_tokens;
  int64_t ctx_len;
  /* Optional Latte pair (R38, "basically follows Latte"; NULL w_fc1_s = none):
   *   y1 <- y1 + W2_s gelu_tanh(W1_s LN_m(y1))   right after the spatial attention, on the
   * T-shards (position-wise: local).  ln_m_w / ln_m_b [C], w_fc1_s [4C, C], w_fc2_s [C, 4C]; bf16;
   * not with the FUSED transport. */
  const void *ln_m_w, *ln_m_b, *w_fc1_s, *w_fc2_s;
  /* Optional temporal positional embedding (R37; NULL = none): pe_t [T, C] (all T frames, every
   * rank) added to the residual stream after the spatial part, y1[b,t,s] += pe_t[t], on the
   * S-shards (each holds all frames of its columns).  Latte adds it before the first temporal
   * block: set it on the first block of a stack only. */
  const void* pe_t;
} dsp_block_weights_t;

/* ---------------------------------------------------------------- lifecycle */

/* Create a context on CUDA device `device` for rank `rank` of `world`.
 * nccl_comm: an ncclComm_t BORROWED from torch's ProcessGroupNCCL (_comm_ptr());
 * may be NULL when world == 1.  Never destroyed by dsp.  NCCL symbols are resolved at
 * run time from the libnccl.so.2 already loaded in the process (or $DSP_NCCL_LIBRARY).
 * Errors: NULL (out), SHAPE (world < 1, rank out of range), NCCL (world > 1 and no
 * comm or NCCL not loadable), CUDA (bad device).  SYNCHRONOUS. */
dsp_status_t dsp_ctx_create(void* nccl_comm, int rank, int world, int device, dsp_ctx_t* out);
/* Destroy host state of the context.  Does not free caller buffers or the comm. */
dsp_status_t dsp_ctx_destroy(dsp_ctx_t ctx);

/* HOST-ONLY, pure: bytes of workspace dsp_st_block_forward needs per rank:
 * tok_r * 6C * elem + 256 where tok_r = B*T*S/world (h: C, qkv+o / MLP hidden: 4C,
 * S-sharded activation: C; the switch send/recv buffers alias dead regions). */
size_t dsp_workspace_bytes(const dsp_shape_t* shape, int world);
/* Attach caller-owned device workspace (kept by pointer, not copied). */
dsp_status_t dsp_ctx_set_workspace(dsp_ctx_t ctx, void* workspace_dev, size_t bytes);

/* P2P switch only.  peer_base_dev[i] / peer_signal_dev[i] (HOST arrays of `world`
 * device pointers, copied into the context) are rank i's symmetric data buffer and
 * signal pad as mapped in THIS process (torch symmetric memory buffer_ptrs /
 * signal_pad_ptrs, or cudaIpc mappings).  Every rank's data buffer has `bytes` bytes at
 * the same offsets; signal pads need >= DSP_SIGNAL_PAD_BYTES bytes, zero-initialised, used
 * by nothing else.  Pad layout (uint64 slots): [0, 8) the barrier epoch peer i last arrived
 * at, [8] this rank's own barrier counter (device-resident and advanced by the barrier kernel,
 * so barriers captured in a CUDA graph stay correct on every replay), [9] the first timeout
 * record (see dsp_ctx_check_errors).
 * The switch destination (or the block's internal buffers) must lie inside the local
 * data buffer peer_base_dev[rank].  For tests, several "virtual ranks" may share one
 * device: pass one context per virtual rank. */
#define DSP_SIGNAL_PAD_BYTES 128
dsp_status_t dsp_ctx_set_peer_buffers(dsp_ctx_t ctx, void* const* peer_base_dev,
                                      void* const* peer_signal_dev, size_t bytes);

/* TEST INFRASTRUCTURE.  on != 0: the NCCL transport's collectives (the all-to-all of
 * dsp_switch / dsp_switch_nd / the blocks with impl NCCL, the all-gather of dsp_gather) are
 * emulated over the peer mappings instead of calling NCCL: signal-pad barrier, one kernel that
 * pulls every peer's piece (recv[r] = peer r's send chunk for this rank; stage[r] = peer r's
 * x_local), barrier.  Everything else of the NCCL code path (pack, unpack, workspace staging)
 * runs unchanged.  For N "virtual ranks" sharing one device (NCCL refuses two ranks per GPU);
 * the staged send buffer (the workspace, or x_local when the pack is an identity) must lie in
 * the registered symmetric buffer.  Errors: NULL, STATE (no peer buffers). */
dsp_status_t dsp_ctx_set_collective_emulation(dsp_ctx_t ctx, int on);

/* Wall-clock bound of every P2P signal-pad barrier wait (default 120 s, or
 * $DSP_BARRIER_TIMEOUT_S at context creation; <= 0 waits forever).  A barrier that times out
 * records (epoch, peer) in its pad and lets the stream continue -- the switch's data is then
 * invalid and dsp_ctx_check_errors() reports it; nothing traps, so the CUDA context survives a
 * slow peer (checkpointing, GC) as long as it arrives within the bound.  HOST-ONLY. */
dsp_status_t dsp_ctx_set_barrier_timeout(dsp_ctx_t ctx, double seconds);

/* Health check.  SYNCHRONOUS (reads 8 bytes from the device; call between steps, off the
 * hot path).  Returns PEER_TIMEOUT if any P2P barrier of this rank timed out (detail names
 * the barrier epoch and the peer), NCCL if the borrowed communicator reports an asynchronous
 * error (ncclCommGetAsyncError), else OK. */
dsp_status_t dsp_ctx_check_errors(dsp_ctx_t ctx);

/* Instrumentation (off the hot path).  Stage ids of dsp_st_block_forward, in order. */
typedef enum {
  DSP_STAGE_LN1 = 0, DSP_STAGE_QKV_S, DSP_STAGE_ATTN_S, DSP_STAGE_PROJ_S, DSP_STAGE_SWITCH_TS,
  DSP_STAGE_LN2, DSP_STAGE_QKV_T, DSP_STAGE_ATTN_T, DSP_STAGE_PROJ_T, DSP_STAGE_LN3,
  DSP_STAGE_FC1, DSP_STAGE_FC2, DSP_STAGE_SWITCH_ST, DSP_NUM_STAGES
} dsp_stage_t;
/* events: HOST array of 2*DSP_NUM_STAGES cudaEvent_t (caller-owned) or NULL to disable.
 * When set, dsp_st_block_forward records events[2*i] / events[2*i+1] on its stream
 * around stage i (both recorded even when a stage is skipped, e.g. switches at N=1).
 * NULL entries are skipped, so a caller can time one stage per pass: every event record
 * is a point where the next kernel's programmatic dependent launch cannot overlap. */
dsp_status_t dsp_ctx_set_stage_events(dsp_ctx_t ctx, void* const* events, int n_events);
/* Stage clocks (instrumentation; off by default).  clocks_dev: device buffer of
 * 2*DSP_NUM_STAGES uint64, or NULL to switch off.  While set, every kernel dsp_st_block_forward
 * launches inside stage i records, with one atomic per CTA, the earliest %globaltimer (ns) at
 * which one of its CTAs passed its dependency wait into clocks[2i] (atomicMin) and the latest
 * CTA exit into clocks[2i+1] (atomicMax) -- the stage's span inside an unperturbed (e.g. graph-
 * replayed) block, with programmatic dependent launch intact.  The caller resets the buffer
 * (clocks[2i] = UINT64_MAX, clocks[2i+1] = 0) before each block; stages without a kernel (folded
 * LayerNorms, switches at N = 1, NCCL / copy kernels) keep the reset values.  The pointer is
 * baked into captured graphs.  Errors: NULL, ALIGNMENT (8 B). */
dsp_status_t dsp_ctx_set_stage_clocks(dsp_ctx_t ctx, void* clocks_dev);
/* Instrumentation taps (test infrastructure; off by default): when set, dsp_st_block_forward
 * copies an intermediate of the block into `dst` (device, >= the local shard bytes) with a
 * stream-ordered D2D copy (also captured into CUDA graphs):
 *   DSP_TAP_Y1: y1 = x + MHA_S(LN1 x) after the T->S switch, S-sharded [B, T, S/N, C];
 *   DSP_TAP_Y2: y2 (after the temporal stage, and the cross stage if any), [B, T, S/N, C].
 * Slice independence then lets a test check each stage of the production launch
 * against the oracle on sampled frames / columns.  dst NULL switches a tap off.
 * Errors: NULL, SHAPE (unknown point), ALIGNMENT; a too-small buffer fails the block call
 * with WORKSPACE. */
typedef enum { DSP_TAP_Y1 = 0, DSP_TAP_Y2 = 1, DSP_NUM_TAPS = 2 } dsp_tap_t;
dsp_status_t dsp_ctx_set_tap(dsp_ctx_t ctx, dsp_tap_t point, void* dst, size_t bytes);
/* Number of this library's own kernels launched through ctx since creation (NCCL kernels
 * and cudaMemcpy excluded).  HOST-ONLY. */
int64_t dsp_ctx_launch_count(dsp_ctx_t ctx);

const char* dsp_status_str(dsp_status_t status);
const char* dsp_last_error(dsp_ctx_t ctx);   /* "" if none; valid until the next call */
int dsp_abi_version(void);                   /* DSP_ABI_VERSION */
#define DSP_ABI_VERSION 6  /* 2: dsp_block_weights_t.prepared, block preparation; 3: optional cross stage;
                              4: device-resident barrier epochs, barrier timeout + error check,
                              exported switch pack / unpack and gather unpack; 5: Ulysses block,
                              stage clocks, taps, collective emulation; 6: Latte pair, temporal
                              positional embedding, dsp_adaln_fold */

/* ----------------------------------------------------------- layout (bytes) */

/* x_local <- chunk `rank` of x_global along `dim` (R11).  Local, bit-exact.
 * x_global [B,T,S,C] device; x_local [B,T/N,S,C] (dim T) or [B,T,S/N,C] (dim S).
 * Errors: BAD_DIM, DIVISIBILITY, ALIGNMENT, ALIAS (overlap). */
dsp_status_t dsp_split(dsp_ctx_t ctx, const dsp_shape_t* shape, dsp_dim_t dim,
                       const void* x_global, void* x_local, void* stream);

/* x_global <- concatenation in rank order along `dim`.  COLLECTIVE.
 * ncclAllGather of the local shards; when the rank-major [N][local] order equals the
 * global layout (dim T with B == 1) it lands directly in x_global, otherwise it lands
 * in the workspace (>= B*T*S*C*elem bytes) and an unpack kernel scatters the runs.
 * N == 1: a device copy.  Errors: as dsp_split; WORKSPACE; NCCL. */
dsp_status_t dsp_gather(dsp_ctx_t ctx, const dsp_shape_t* shape, dsp_dim_t dim,
                        const void* x_local, void* x_global, void* stream);

/* The dynamic switch (§3.1; Fig. 2).  COLLECTIVE.
 * Pre: x_local is the `from_dim` chunk `rank` of a global X.  Post: y_local is the
 * `to_dim` chunk `rank` of the same X, bit-identical bytes.  For from=T,to=S:
 *   y[b, r*Tn + t', s', c] = (chunk received from rank r)[b, t', s', c], i.e.
 *   Y_q[b,t,s',c] = X[b,t,q*Sn+s',c]   (SURVEY §8a "The switch as an exact index map").
 * Volume: (N-1)*B*(T/N)*(S/N)*C elements sent and received per rank.
 * impl NCCL: uses the workspace (>= 2*B*T*S*C/N*elem bytes) for pack/recv staging.
 * impl P2P : y_local must lie inside the registered symmetric buffer.
 * N == 1: a device copy (no-op if x == y).
 * Errors: SAME_DIM, BAD_DIM, DIVISIBILITY, ALIGNMENT (C*elem % 16), ALIAS
 * (x overlaps y, N > 1), WORKSPACE, STATE (P2P without peer buffers), NCCL. */
dsp_status_t dsp_switch(dsp_ctx_t ctx, const dsp_shape_t* shape, dsp_dim_t from_dim,
                        dsp_dim_t to_dim, const void* x_local, void* y_local,
                        dsp_switch_impl_t impl, void* stream);

/* HOST-ONLY, pure: off-rank bytes one switch sends and receives per rank,
 * (N-1)*B*(T/N)*(S/N)*C*elem each (self-chunk excluded). */
dsp_status_t dsp_switch_volume(const dsp_shape_t* shape, int world,
                               int64_t* bytes_sent_per_rank, int64_t* bytes_recv_per_rank);

/* HOST-ONLY, pure: the byte-run plan of one switch on `rank` — the host logic every
 * transport executes.  A switch moves n0*n1*n2 runs of run_bytes contiguous bytes;
 * run (i0,i1,i2) (i0 = peer, i1 = b, i2 = t') is read at
 *   src_off = i0*src_stride[0] + i1*src_stride[1] + i2*src_stride[2]
 * of this rank's x_local and written to
 *   dst_off = i1*dst_stride[1] + i2*dst_stride[2] + dst_peer_off
 * of PEER i0's y_local, where dst_peer_off = rank*dst_stride[0] (the slot this rank
 * fills on every peer).  The NCCL transport realises it as pack (to chunk order
 * [peer][b][t'][s'][c]) + AlltoAll + unpack; the P2P transport stores directly. */
typedef struct {
  int64_t n[3];
  int64_t run_bytes;
  int64_t src_stride[3];
  int64_t dst_stride[3];
  int64_t dst_peer_off;
  int32_t pack_is_identity;     /* chunk order == x_local layout (no pack kernel) */
  int32_t unpack_is_identity;   /* chunk order == y_local layout (no unpack kernel) */
} dsp_switch_plan_t;
dsp_status_t dsp_switch_plan(const dsp_shape_t* shape, int world, int rank,
                             dsp_dim_t from_dim, dsp_dim_t to_dim, dsp_switch_plan_t* plan);

/* --------------------------------------------------- local attention stages */

/* out = (residual ? residual : 0) + MHA_S(h): spatial multi-head self-attention, one
 * sequence over S per (b, t), on a T-sharded h_local [B, T/N, S, C].
 * MHA(h) = concat_j softmax(q_j k_j^T / sqrt(Dh)) v_j  * w_o^T with [q|k|v] = h w_qkv^T
 * (R6-R8).  No LayerNorm inside.  Local (no communication).  Uses the workspace for
 * qkv and O (tok_r * 4C * elem bytes).  out may equal residual; out must not overlap h.
 * bf16: tcgen05 QKV GEMM -> tcgen05 FMHA -> tcgen05 out-proj GEMM (+residual epilogue).
 * Any sequence length >= 1 (lengths that neither divide nor are a multiple of 128 run with a
 * masked last key tile, DESIGN R33).
 * Errors: SHAPE (C % num_heads), UNSUPPORTED (bf16 needs Dh % 8 == 0, Dh <= 128 and
 * C % 32 == 0; see dsp_last_error), ALIAS, WORKSPACE, DIVISIBILITY. */
dsp_status_t dsp_spatial_attn(dsp_ctx_t ctx, const dsp_shape_t* shape, const void* h_local,
                              const void* w_qkv, const void* w_o, const void* residual,
                              void* out, void* stream);

/* As dsp_spatial_attn, temporal: one sequence over T per (b, s) on an S-sharded
 * h_local [B, T, S/N, C] (frame stride S/N*C elements). */
dsp_status_t dsp_temporal_attn(dsp_ctx_t ctx, const dsp_shape_t* shape, const void* h_local,
                               const void* w_qkv, const void* w_o, const void* residual,
                               void* out, void* stream);

/* ------------------------------------------------------------ the ST block */

/* One ST block (R1, R10, R13, R14), x_local and y_local both
 * T-sharded [B, T/N, S, C]:
 *   y1 = x + MHA_S(LN1 x)            local on T-shards          (y1 stored in y_local)
 *   switch T->S                      one all-to-all
 *   y2 = y1 + MHA_T(LN2 y1)          local on S-shards
 *   y  = y2 + MLP(LN3 y2)            MLP = gelu_tanh(. W1^T) W2^T (R5)
 *   switch S->T                      second all-to-all
 * COLLECTIVE.  x_local may equal y_local.  Workspace >= dsp_workspace_bytes().
 * N == 1: no switch is executed (both layouts coincide).
 * Errors: any of the above; WORKSPACE. */
dsp_status_t dsp_st_block_forward(dsp_ctx_t ctx, const dsp_shape_t* shape,
                                  const dsp_block_weights_t* w, const void* x_local,
                                  void* y_local, dsp_switch_impl_t impl, void* stream);

/* ------------------------------------------------- Ulysses schedule (A/B baseline)
 * The same ST block (identical weights, kernels and result) under DeepSpeed-Ulysses sequence
 * parallelism ("AlltoAll for query, key, value, and output"), the
 * comparison system of the paper's experiments, built on this library's kernels.
 * x_local / y_local are T-sharded [B, T/N, S, C] throughout (the activation never switches).
 * Each attention stage: local QKV GEMM -> three all-to-alls (q, k, v: sequence-sharded ->
 * head-sharded; rank g receives every token of heads [g*NH/N, (g+1)*NH/N)) -> attention over the
 * full sequence with NH/N heads -> one all-to-all (o: head-sharded -> sequence-sharded) ->
 * local out-projection + residual.  The MLP is local.  8 all-to-alls per block, each moving
 * (N-1)*M/N^2 elements per rank: 4x DSP's volume (Table 1: 8M/N vs 2M/N).
 * impl NCCL: one ncclAlltoAll per tensor (pack / unpack kernels around it); P2P: q, k, v in one
 * direct put and o in another (workspace inside the symmetric buffer).  N == 1: the DSP block.
 * Prepared weights (R30) supported; no cross stage.  Workspace >= dsp_ulysses_workspace_bytes
 * (11 * tok_r * C * elem + statistics).  COLLECTIVE.  Output is bitwise independent of N and
 * equal to dsp_st_block_forward at N = 1 (per-head attention, no reductions across ranks).
 * Errors: as dsp_st_block_forward; UNSUPPORTED (f32, N does not divide num_heads, cross stage,
 * impl FUSED), ALIGNMENT (C/N*elem % 16). */
size_t dsp_ulysses_workspace_bytes(const dsp_shape_t* shape, int world);  /* host-only */
dsp_status_t dsp_st_block_forward_ulysses(dsp_ctx_t ctx, const dsp_shape_t* shape, const dsp_block_weights_t* w,
                                          const void* x_local, void* y_local, dsp_switch_impl_t impl, void* stream);

/* ---------------------------------------------------------------- N-D switch
 * DSP on a multi-dimensional activation [d_0, ..., d_{n-2}, C] with any number of sequence
 * dims ("our method can generalize to all multi-dimensional transformers beyond the
 * demonstrated spatial-temporal transformer"; e.g. [B, T, H, W, C] with attention along T, H
 * and W separately).  Sharding convention as for the 4-D switch: rank r holds the r-th
 * contiguous chunk along the sharded dim (R11).  dims: HOST array of the GLOBAL extents,
 * outermost first, the last one is the channel dim (never sharded); elem_bytes: bytes per
 * element.  from_dim / to_dim in [0, ndim - 2], distinct. */
#define DSP_ND_MAX_DIMS 8
typedef struct {
  int64_t n[4];            /* loop extents: [peer, outer, rows of the outer switched dim, middle] */
  int64_t run_bytes;       /* contiguous bytes moved per run */
  int64_t src_stride[4];   /* bytes, in x_local */
  int64_t dst_stride[4];   /* bytes, in the destination's y_local; [0] = offset per source rank */
  int64_t dst_peer_off;    /* this rank's offset in every destination: rank * dst_stride[0] */
  int32_t pack_is_identity, unpack_is_identity;
} dsp_switch_nd_plan_t;
/* HOST-ONLY, pure: the byte plan of rank `rank`'s N-D switch.  Errors: NULL, SHAPE (ndim
 * outside [3, DSP_ND_MAX_DIMS], an extent < 1, elem_bytes < 1), BAD_DIM, SAME_DIM,
 * DIVISIBILITY (world does not divide d[from] or d[to]), ALIGNMENT (a run is not a multiple
 * of 16 bytes: needs d[max(from,to)] / world * prod(d after it) * elem_bytes % 16 == 0). */
dsp_status_t dsp_switch_nd_plan(const int64_t* dims, int ndim, int elem_bytes, int world, int rank,
                                int from_dim, int to_dim, dsp_switch_nd_plan_t* plan);
/* N-D dynamic switch: x_local = chunk `rank` of the global X along from_dim (extent
 * d[from]/world there), y_local = chunk `rank` along to_dim, bit-identical bytes.  Transport
 * as dsp_switch (NCCL: pack -> ncclAlltoAll -> unpack through the context workspace, which
 * must hold 2 local shards unless pack/unpack are identities; P2P: y_local inside the
 * registered symmetric buffer).  x, y 16-B aligned, non-overlapping (world > 1).
 * COLLECTIVE.  Errors: as dsp_switch_nd_plan, plus NULL, ALIAS, WORKSPACE, STATE, NCCL, CUDA. */
dsp_status_t dsp_switch_nd(dsp_ctx_t ctx, const int64_t* dims, int ndim, int elem_bytes, int from_dim,
                           int to_dim, const void* x_local, void* y_local, dsp_switch_impl_t impl, void* stream);

/* ---------------------------------------------------------------- cross-attention
 * ST-DiT's conditioning layer ("spatial-temporal and cross attention"): every local
 * token of sample b attends to sample b's Lc context tokens (e.g. caption embeddings), which
 * every rank holds in full -- position-independent, so it is local under any DSP sharding.
 *   out = (residual ? residual : 0) + CA(h),  CA(h) = softmax(q k^T / sqrt(Dh)) v  per head, w_o
 *   q = h w_q^T,  [k | v] = ctx_tokens w_kv^T  (w_kv [2C, C] rows [k | v], head j rows j*Dh.., R8)
 * h, residual, out: [B, T_loc, S_loc, C] local tokens (either sharding; LN applied by the caller);
 * ctx_tokens: [B, Lc, C] (already projected to C); bf16 only.  Keys beyond Lc in the last
 * 128-key tile are masked; any number of local tokens per sample (a ragged last query tile is
 * clipped).  Needs workspace >= dsp_cross_workspace_bytes.  Not collective.  Errors: NULL, SHAPE, DIVISIBILITY,
 * UNSUPPORTED, ALIGNMENT, ALIAS (out overlaps h; out == residual is allowed), WORKSPACE, CUDA. */
size_t dsp_cross_workspace_bytes(const dsp_shape_t* shape, int world, int64_t Lc);  /* host-only */
dsp_status_t dsp_cross_attn(dsp_ctx_t ctx, const dsp_shape_t* shape, const void* h_local, const void* ctx_tokens,
                            int64_t Lc, const void* w_q, const void* w_kv, const void* w_o, const void* residual,
                            void* out, void* stream);

/* ---------------------------------------------------------------- N-D block
 * Multi-dimensional transformer block on x [d_0, ..., d_{n-2}, C] with attention
 * along each of the dims attn_dims[0..n_stages-1] in that order (pre-LN + residual, R1-R8),
 * then the MLP (ratio 4, tanh-GELU):  for k in attn_dims: x += MHA_k(LN_k x);  y = x + MLP(LN x).
 * DSP schedule (generalised): x_local / y_local are chunk `rank` along shard_dim; stages
 * along other dims are local; before the stage along shard_dim ONE N-D switch to the dim
 * attended just before it, and after the MLP one switch back -- two per block, none
 * if shard_dim is not attended.  shard_dim != attn_dims[0].  dsp_st_block_forward is the
 * case [B, T, S, C], attn_dims = {S, T}, shard_dim = T (raw weights).  Workspace >=
 * dsp_nd_workspace_bytes.  COLLECTIVE.  Errors: NULL, SHAPE (ndim, dims, heads, stages),
 * BAD_DIM (a dim outside [0, n-2], repeated, or shard_dim == attn_dims[0]), DIVISIBILITY,
 * UNSUPPORTED (bf16 attention length / head-dim limits as dsp_spatial_attn), ALIGNMENT,
 * ALIAS, WORKSPACE, STATE, NCCL, CUDA. */
typedef struct { const void *ln_w, *ln_b, *w_qkv /*[3C, C]*/, *w_o /*[C, C]*/; } dsp_attn_weights_t;
typedef struct { const void *ln_w, *ln_b, *w_fc1 /*[4C, C]*/, *w_fc2 /*[C, 4C]*/; } dsp_mlp_weights_t;
size_t dsp_nd_workspace_bytes(const int64_t* dims, int ndim, dsp_dtype_t dtype, int world);  /* host-only */
dsp_status_t dsp_nd_block_forward(dsp_ctx_t ctx, const int64_t* dims, int ndim, int num_heads, dsp_dtype_t dtype,
                                  int n_stages, const int* attn_dims, const dsp_attn_weights_t* attn,
                                  const dsp_mlp_weights_t* mlp, float ln_eps, int shard_dim, const void* x_local,
                                  void* y_local, dsp_switch_impl_t impl, void* stream);

/* Forward of a stack of L ST blocks, y = block_{L-1}( ... block_0(x)) (BASELINE configs[2]:
 * the 28-layer ST-DiT-XL/2-shaped model), x and y T-sharded as for one block (x may
 * equal y; blocks 1.. run in place on y).  w: HOST array of L block-weight structs.  With
 * prepared weights (R30), block l + 1 folds LN1 from per-row LayerNorm partials of its input: at
 * N == 1 those block l's FC2 epilogue wrote (no statistics pass between blocks), at N > 1 the
 * same bits recomputed after the switch -- the output is bitwise independent of N.  Workspace as for one block (reused by every layer).  COLLECTIVE (2 switches per
 * layer).  Errors: as dsp_st_block_forward; SHAPE (L < 1); NULL. */
dsp_status_t dsp_st_model_forward(dsp_ctx_t ctx, const dsp_shape_t* shape, const dsp_block_weights_t* const* w,
                                  int L, const void* x_local, void* y_local, dsp_switch_impl_t impl, void* stream);

/* adaLN-Zero conditioning of one block for ONE sample (R36, DiT as cited by P:137):
 *   y = x + gate_k * F_k(LN_k(x) * (1 + scale_k) + shift_k)   for each sublayer k
 * with k = spatial attention, temporal attention, MLP, and the Latte pair's spatial MLP.  At B = 1
 * (the paper's batch) this is the plain block with modulated weights:
 *   gamma_k' = gamma_k (1 + scale_k),  beta_k' = beta_k (1 + scale_k) + shift_k,
 *   W_out_k' = diag(gate_k) W_out_k    (W_out = w_o_s, w_o_t, w_fc2, w_fc2_s),
 * which this call writes (bf16) into the buffers `out` points to: out->ln1_w/ln1_b, ln2_w/ln2_b,
 * ln3_w/ln3_b, w_o_s, w_o_t, w_fc2 (and ln_m_w/ln_m_b, w_fc2_s when w->w_fc1_s is set) -- the
 * caller owns them (same sizes as the inputs) and copies every other pointer of *w into *out.
 * The conditioned block is then dsp_st_block_forward(out) (prepare it again when preparing).
 * mod: device f32 [4][3][C] = (shift, scale, gate) for sublayers (spatial attention, temporal
 * attention, MLP, spatial MLP).  Once per sampling step per block; enqueued on `stream`.
 * Errors: NULL, UNSUPPORTED (f32, B != 1), ALIGNMENT, CUDA. */
dsp_status_t dsp_adaln_fold(dsp_ctx_t ctx, const dsp_shape_t* shape, const dsp_block_weights_t* w, const float* mod,
                            const dsp_block_weights_t* out, void* stream);

/* Bytes of the prepared-weights buffer for one bf16 block of this shape (0 for f32). */
size_t dsp_block_prepared_bytes(const dsp_shape_t* shape);

/* LayerNorm folding of one block's weights (R30), a one-time step per set of
 * weights (inference: weights are constant across the sampling steps).  With
 * LN(x) = (x - mean) * rstd * gamma + beta (R3) and a bias-free linear W [N, K]:
 *   LN(x) W^T = rstd * (x (W o gamma)^T - mean * u) + v,  u = (W o gamma) 1,  v = W beta,
 * so the GEMM reads the raw activation and applies rstd, mean, u, v in its epilogue.
 * Writes into `prepared` (device, caller-owned, 256-B aligned, >= dsp_block_prepared_bytes):
 *   [3C, C] bf16 w_qkv_s o ln1_w | [3C, C] bf16 w_qkv_t o ln2_w | [4C, C] bf16 w_fc1 o ln3_w
 *   (each 256-B aligned) | f32 u_s[3C] v_s[3C] u_t[3C] v_t[3C] u_1[4C] v_1[4C] | with a cross
 *   stage (ln_c_w set): [C, C] bf16 w_q_c o ln_c_w | f32 u_c[C] v_c[C] (LN_c statistics then come
 *   from the temporal out-projection's partials).
 * Enqueued on `stream`.  Errors: NULL, UNSUPPORTED (f32, C % 8 != 0, C > 3072, or more than 12
 * LayerNorm partials per row: C / BN > 12 with BN the out-projection tile width),
 * WORKSPACE (prepared_bytes too small), ALIGNMENT, CUDA. */
dsp_status_t dsp_st_block_prepare(dsp_ctx_t ctx, const dsp_shape_t* shape, const dsp_block_weights_t* w,
                                  void* prepared, size_t prepared_bytes, void* stream);

/* End-to-end variant through HOST buffers: copies x_local_host -> x_dev (H2D), runs
 * dsp_st_block_forward(x_dev -> y_dev), copies y_dev -> y_local_host (D2H), all on
 * `stream`; returns after enqueueing (synchronise the stream before reading y_host).
 * x_dev / y_dev are caller-owned device staging buffers of the local shard size
 * (may be equal).  COLLECTIVE. */
dsp_status_t dsp_st_block_forward_host(dsp_ctx_t ctx, const dsp_shape_t* shape,
                                       const dsp_block_weights_t* w,
                                       const void* x_local_host, void* y_local_host,
                                       void* x_dev, void* y_dev,
                                       dsp_switch_impl_t impl, void* stream);

/* Pipelined end-to-end path for a stream of n independent inputs (serving): for each i,
 * H2D x_local_host[i] -> x_dev[i % 2] on a context-owned copy-in stream, the block on `stream`
 * (x_dev[i % 2] -> y_dev[i % 2]), D2H y_dev[i % 2] -> y_local_host[i] on a context-owned
 * copy-out stream.  Events order every reuse of a staging buffer, so the copies of steps
 * i + 1 and i - 1 overlap the block of step i (PCIe is full duplex).  x_dev[2], y_dev[2]:
 * HOST arrays of four distinct, non-overlapping device buffers of the local shard size;
 * x_local_host / y_local_host: HOST arrays of n host pointers (pinned for overlap).  Work the
 * caller enqueued on `stream` before the call completes before the first copy; `stream`
 * completes only after the last D2H, so synchronising `stream` means every y is on the host.
 * COLLECTIVE (n blocks, same n on all ranks).  Errors: as dsp_st_block_forward; NULL; SHAPE
 * (n < 0); ALIAS (staging buffers overlap). */
dsp_status_t dsp_st_block_forward_host_pipelined(dsp_ctx_t ctx, const dsp_shape_t* shape,
                                                 const dsp_block_weights_t* w, int n,
                                                 const void* const* x_local_host, void* const* y_local_host,
                                                 void* const* x_dev, void* const* y_dev,
                                                 dsp_switch_impl_t impl, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DSP_H_ */
