// api.cu — the C ABI (include/dsp.h, include/dsp_kernels.h): validation, the switch
// plan, transports (NCCL / P2P) and the composition of the ST block forward.
// Every step of the path runs in this library's kernels (or NCCL); there is no host
// compute and no CPU fallback.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "dsp_internal.h"

using namespace dsp;

namespace {

thread_local std::string g_no_ctx_error;

dsp_status_t fail(dsp_ctx_t ctx, dsp_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->last_error = buf;
  else g_no_ctx_error = buf;
  return st;
}

dsp_status_t cuda_fail(dsp_ctx_t ctx, cudaError_t e, const char* what, const std::string& why = "") {
  if (e == cudaErrorNotSupported)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "%s: %s", what, why.empty() ? "unsupported" : why.c_str());
  return fail(ctx, DSP_ERR_CUDA, "%s: %s%s%s", what, cudaGetErrorString(e), why.empty() ? "" : " — ", why.c_str());
}

#define DSP_CUDA(ctx, expr, what)                        \
  do {                                                   \
    std::string _why;                                    \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, what, _why); \
  } while (0)
#define DSP_TRY(expr)                 \
  do {                                \
    dsp_status_t _s = (expr);         \
    if (_s != DSP_OK) return _s;      \
  } while (0)

constexpr double kDefaultBarrierTimeoutS = 120.0;

int64_t elem_bytes(dsp_dtype_t d) { return d == DSP_BF16 ? 2 : 4; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool overlap(const void* a, int64_t na, const void* b, int64_t nb) {
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + (uintptr_t)nb && y < x + (uintptr_t)na;
}

dsp_status_t check_shape(dsp_ctx_t ctx, const dsp_shape_t* s) {
  if (!s) return fail(ctx, DSP_ERR_NULL, "shape is NULL");
  if (s->B < 1 || s->T < 1 || s->S < 1 || s->C < 1 || s->num_heads < 1)
    return fail(ctx, DSP_ERR_SHAPE, "non-positive extent in shape (B=%lld T=%lld S=%lld C=%lld heads=%d)",
                (long long)s->B, (long long)s->T, (long long)s->S, (long long)s->C, s->num_heads);
  if (s->dtype != DSP_BF16 && s->dtype != DSP_F32) return fail(ctx, DSP_ERR_SHAPE, "unknown dtype %d", (int)s->dtype);
  if ((s->C * elem_bytes(s->dtype)) % 16)
    return fail(ctx, DSP_ERR_ALIGNMENT, "C*elem = %lld bytes is not a multiple of 16", (long long)(s->C * elem_bytes(s->dtype)));
  return DSP_OK;
}

dsp_status_t check_dim(dsp_ctx_t ctx, int d) {
  if (d != DSP_DIM_T && d != DSP_DIM_S) return fail(ctx, DSP_ERR_BAD_DIM, "dim %d is not DSP_DIM_T (1) or DSP_DIM_S (2)", d);
  return DSP_OK;
}

dsp_status_t check_div(dsp_ctx_t ctx, const dsp_shape_t* s, int world) {
  if (world < 1) return fail(ctx, DSP_ERR_SHAPE, "world %d < 1", world);
  if (s->T % world || s->S % world)
    return fail(ctx, DSP_ERR_DIVISIBILITY, "N=%d must divide T=%lld and S=%lld", world, (long long)s->T, (long long)s->S);
  return DSP_OK;
}

dsp_status_t check_ctx(dsp_ctx_t ctx) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != ctx->device)
    return fail(ctx, DSP_ERR_STATE, "current CUDA device %d is not the context device %d", dev, ctx->device);
  return DSP_OK;
}

int64_t shard_bytes(const dsp_shape_t* s, int world) { return s->B * s->T * s->S * s->C * elem_bytes(s->dtype) / world; }

int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

// Block workspace layout (bytes).  act = tok_r * C * elem.
//   [0, act)          h: LN output (unprepared path) / switch scratch
//   [act, 5 act)      big: qkv [tok,3C] + o [tok,C] | MLP hidden [tok,4C] | switch send/recv
//   [5 act, 6 act)    ys: S-sharded activation (N > 1)
//   stats             [tok] float2 (mean, rstd) of a LayerNorm input (prepared path)
//   parts             [tok, C / BN] float2 per-row partials from the out-projection epilogues
struct BlockWs {
  int64_t act, h, big, ys, stats, parts, total;
};
BlockWs block_ws(const dsp_shape_t* s, int world) {
  BlockWs w{};
  const int64_t tok = s->B * s->T * s->S / world, C = s->C, e = elem_bytes(s->dtype);
  w.act = tok * C * e;
  w.h = 0;
  w.big = w.act;
  w.ys = 5 * w.act;
  w.stats = align256(6 * w.act);
  w.parts = w.stats + align256(tok * 8);
  w.total = w.parts + align256(tok * (C / gemm_part_cols(C)) * 8) + 256;
  return w;
}

// Prepared (LayerNorm-folded) weights of one bf16 block: W o gamma for the three
// LayerNorm -> linear pairs and their per-output-column u = (W o gamma) 1, v = W beta.
struct PrepLayout {
  int64_t wf_s, wf_t, wf_1, uv, wf_c, uv_c, wf_1s, uv_1s, total;
};
PrepLayout prep_layout(int64_t C) {
  PrepLayout p{};
  p.wf_s = 0;
  p.wf_t = align256(3 * C * C * 2);
  p.wf_1 = p.wf_t + align256(3 * C * C * 2);
  p.uv = p.wf_1 + align256(4 * C * C * 2);
  p.wf_c = p.uv + align256(20 * C * 4);     // cross stage q projection (filled when ln_c_w is set)
  p.uv_c = p.wf_c + align256(C * C * 2);
  p.wf_1s = p.uv_c + align256(2 * C * 4);   // Latte pair spatial FC1 (filled when w_fc1_s is set, R38)
  p.uv_1s = p.wf_1s + align256(4 * C * C * 2);
  p.total = p.uv_1s + align256(8 * C * 4);
  return p;
}

// bf16 tensor-core path constraints for one attention stage over sequences of length L
dsp_status_t check_bf16_attn(dsp_ctx_t ctx, const dsp_shape_t* s, int64_t L) {
  if (s->C % s->num_heads) return fail(ctx, DSP_ERR_SHAPE, "C=%lld not divisible by num_heads=%d", (long long)s->C, s->num_heads);
  const int64_t Dh = s->C / s->num_heads;
  if (s->dtype == DSP_F32) {
    if (Dh > 128) return fail(ctx, DSP_ERR_UNSUPPORTED, "fp32 check path supports Dh <= 128 (Dh=%lld)", (long long)Dh);
    return DSP_OK;
  }
  if (Dh % 8 || Dh > 128) return fail(ctx, DSP_ERR_UNSUPPORTED, "bf16 attention needs Dh %% 8 == 0 and Dh <= 128 (Dh=%lld)", (long long)Dh);
  if (s->C % 32) return fail(ctx, DSP_ERR_UNSUPPORTED, "bf16 path needs C %% 32 == 0 (C=%lld)", (long long)s->C);
  (void)L;  // any length: divisors of 128 are packed per tile, others masked in the last key tile
  return DSP_OK;
}

// ---------------------------------------------------------------- switch plan
void make_plan(const dsp_shape_t* s, int N, int rank, int from, dsp_switch_plan_t* p) {
  const int64_t e = elem_bytes(s->dtype), row = s->C * e, Tn = s->T / N, Sn = s->S / N, B = s->B, T = s->T, S = s->S;
  memset(p, 0, sizeof(*p));
  p->n[0] = N; p->n[1] = B; p->n[2] = Tn;
  p->run_bytes = Sn * row;
  if (from == DSP_DIM_T) {  // x [B,Tn,S,C] -> y [B,T,Sn,C]
    p->src_stride[0] = Sn * row; p->src_stride[1] = Tn * S * row; p->src_stride[2] = S * row;
    p->dst_stride[0] = Tn * Sn * row; p->dst_stride[1] = T * Sn * row; p->dst_stride[2] = Sn * row;
    p->pack_is_identity = (N == 1 || B * Tn == 1);
    p->unpack_is_identity = (N == 1 || B == 1);
  } else {                  // x [B,T,Sn,C] -> y [B,Tn,S,C]
    p->src_stride[0] = Tn * Sn * row; p->src_stride[1] = T * Sn * row; p->src_stride[2] = Sn * row;
    p->dst_stride[0] = Sn * row; p->dst_stride[1] = Tn * S * row; p->dst_stride[2] = S * row;
    p->pack_is_identity = (N == 1 || B == 1);
    p->unpack_is_identity = (N == 1 || B * Tn == 1);
  }
  p->dst_peer_off = rank * p->dst_stride[0];
}

dsp_status_t validate_switch(dsp_ctx_t ctx, const dsp_shape_t* s, int world, int from, int to) {
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_dim(ctx, from));
  DSP_TRY(check_dim(ctx, to));
  if (from == to) return fail(ctx, DSP_ERR_SAME_DIM, "switch from a dim to itself (S:283)");
  return check_div(ctx, s, world);
}

bool in_region(const void* p, int64_t n, const void* base, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p), b = reinterpret_cast<uintptr_t>(base);
  return a >= b && a + (uintptr_t)n <= b + bytes;
}

// NCCL transport layouts: send / recv hold one chunk per peer, [peer][i1][i2][i3][run bytes].
// pack: x_local -> send (level 0 = destination peer); unpack: recv (level 0 = source rank) ->
// y_local at that rank's slot.  The plan's strides are identical on every rank, so the same
// dst strides place a received chunk.
struct ChunkCopies {
  RunCopy pack, unpack;
  int64_t chunk;  // bytes per peer
};
ChunkCopies chunk_copies(const RunCopy& rc) {
  ChunkCopies c;
  c.chunk = rc.n[1] * rc.n[2] * rc.n[3] * rc.run_bytes;
  c.pack = rc;
  c.unpack = rc;
  c.pack.ds[0] = c.chunk; c.pack.ds[1] = rc.n[2] * rc.n[3] * rc.run_bytes; c.pack.ds[2] = rc.n[3] * rc.run_bytes;
  c.pack.ds[3] = rc.run_bytes;
  for (int i = 0; i < 4; ++i) c.unpack.ss[i] = c.pack.ds[i];
  return c;
}

RunCopy plan_runs(const dsp_switch_plan_t& p) {
  RunCopy rc;
  for (int i = 0; i < 3; ++i) { rc.n[i] = p.n[i]; rc.ss[i] = p.src_stride[i]; rc.ds[i] = p.dst_stride[i]; }
  rc.run_bytes = p.run_bytes;
  return rc;
}

// Emulated collectives (virtual ranks on one device, dsp_ctx_set_collective_emulation): the
// contract of ncclAlltoAll / ncclAllGather on byte buffers -- recv[r] = peer r's send[rank] /
// stage[r] = peer r's x_local -- realised as barrier, one kernel pulling every peer's piece over
// the peer mappings, barrier.  `src` must lie inside the registered symmetric buffer (the same
// offset on every rank).  Test infrastructure for the NCCL transport's code path (NCCL cannot put
// two ranks on one GPU); never selected implicitly.
dsp_status_t emulated_gather_pieces(dsp_ctx_t ctx, const void* src, int64_t src_stride_rank, int64_t piece,
                                    void* dst, cudaStream_t st, const char* what) {
  const int N = ctx->world;
  if (!ctx->has_peers) return fail(ctx, DSP_ERR_STATE, "%s: collective emulation needs peer buffers", what);
  void* base = ctx->peer_base.p[ctx->rank];
  if (!in_region(src, src_stride_rank * (N - 1) + piece, base, ctx->peer_bytes))
    return fail(ctx, DSP_ERR_UNSUPPORTED, "%s: emulated collective source is not inside the symmetric buffer", what);
  const int64_t src_off = static_cast<const uint8_t*>(src) - static_cast<uint8_t*>(base) + ctx->rank * src_stride_rank;
  RunCopy rc;
  rc.n[0] = N;
  rc.run_bytes = piece;
  rc.ds[0] = piece;
  DSP_CUDA(ctx, launch_p2p_barrier(ctx->peer_signal, ctx->rank, N, ctx->barrier_timeout_ns, st), "emulated collective entry");
  DSP_CUDA(ctx, launch_p2p_pull(ctx->peer_base, src_off, dst, rc, ctx->num_sms, st), "emulated collective pull");
  DSP_CUDA(ctx, launch_p2p_barrier(ctx->peer_signal, ctx->rank, N, ctx->barrier_timeout_ns, st), "emulated collective exit");
  ctx->launches += 3;
  return DSP_OK;
}

// Execute a switch plan (4-level strided runs, level 0 = peer): P2P = entry barrier, direct
// stores of every run at its final address in the peer's buffer, exit barrier; NCCL = pack into
// per-peer chunks (skipped when identity) -> ncclAlltoAll (bytes) -> unpack (skipped when identity).
dsp_status_t do_switch_plan(dsp_ctx_t ctx, const RunCopy& rc, int64_t dst_peer_off, bool pack_identity,
                            bool unpack_identity, int64_t bytes, const void* x, void* y, dsp_switch_impl_t impl,
                            cudaStream_t st, void* scratch_send, void* scratch_recv) {
  const int N = ctx->world;
  if (impl == DSP_SWITCH_P2P) {
    if (!ctx->has_peers) return fail(ctx, DSP_ERR_STATE, "P2P switch without dsp_ctx_set_peer_buffers");
    void* base = ctx->peer_base.p[ctx->rank];
    if (!in_region(y, bytes, base, ctx->peer_bytes))
      return fail(ctx, DSP_ERR_UNSUPPORTED, "P2P switch destination is not inside the registered symmetric buffer");
    const int64_t y_off = static_cast<uint8_t*>(y) - static_cast<uint8_t*>(base);
    DSP_CUDA(ctx, launch_p2p_barrier(ctx->peer_signal, ctx->rank, N, ctx->barrier_timeout_ns, st), "p2p entry barrier");
    DSP_CUDA(ctx, launch_p2p_put(x, ctx->peer_base, y_off + dst_peer_off, rc, ctx->num_sms, st), "p2p put");
    DSP_CUDA(ctx, launch_p2p_barrier(ctx->peer_signal, ctx->rank, N, ctx->barrier_timeout_ns, st), "p2p exit barrier");
    ctx->launches += 3;
    return DSP_OK;
  }
  if (!ctx->emulate_collectives && (!ctx->nccl.ok || !ctx->comm))
    return fail(ctx, DSP_ERR_NCCL, "NCCL switch without a communicator");
  const ChunkCopies cc = chunk_copies(rc);
  const int64_t chunk = cc.chunk;
  const void* send = x;
  void* recv = y;
  if (!pack_identity) {
    DSP_CUDA(ctx, launch_run_copy(x, scratch_send, cc.pack, ctx->num_sms, st), "switch pack");
    ctx->launches += 1;
    send = scratch_send;
  }
  if (!unpack_identity) recv = scratch_recv;
  int r;
  if (ctx->emulate_collectives) {
    DSP_TRY(emulated_gather_pieces(ctx, send, chunk, chunk, recv, st, "switch"));
    r = 0;
  } else if (ctx->nccl.AlltoAll) {
    r = ctx->nccl.AlltoAll(send, recv, (size_t)chunk, kNcclUint8, ctx->comm, st);
  } else {
    r = ctx->nccl.GroupStart();
    for (int q = 0; q < N && r == 0; ++q) {
      r = ctx->nccl.Send(static_cast<const uint8_t*>(send) + q * chunk, chunk, kNcclUint8, q, ctx->comm, st);
      if (!r) r = ctx->nccl.Recv(static_cast<uint8_t*>(recv) + q * chunk, chunk, kNcclUint8, q, ctx->comm, st);
    }
    int r2 = ctx->nccl.GroupEnd();
    if (!r) r = r2;
  }
  if (r) return fail(ctx, DSP_ERR_NCCL, "ncclAlltoAll: %s", ctx->nccl.GetErrorString(r));
  if (!unpack_identity) {
    DSP_CUDA(ctx, launch_run_copy(recv, y, cc.unpack, ctx->num_sms, st), "switch unpack");
    ctx->launches += 1;
  }
  return DSP_OK;
}

dsp_status_t do_switch(dsp_ctx_t ctx, const dsp_shape_t* s, int from, const void* x, void* y, dsp_switch_impl_t impl,
                       cudaStream_t st, void* scratch_send, void* scratch_recv) {
  const int N = ctx->world;
  const int64_t bytes = shard_bytes(s, N);
  if (N == 1) {
    if (x != y) DSP_CUDA(ctx, cudaMemcpyAsync(y, x, bytes, cudaMemcpyDeviceToDevice, st), "switch copy (N=1)");
    return DSP_OK;
  }
  dsp_switch_plan_t p;
  make_plan(s, N, ctx->rank, from, &p);
  return do_switch_plan(ctx, plan_runs(p), p.dst_peer_off, p.pack_is_identity, p.unpack_is_identity, bytes, x, y, impl, st,
                        scratch_send, scratch_recv);
}

inline void mark(dsp_ctx_t ctx, int stage, int end, cudaStream_t st) {
  // stage clocks: every kernel launched inside the stage records its span into the stage's slot
  if (stage >= 0) t_clk = (!end && ctx->stage_clk) ? ctx->stage_clk + 2 * stage : nullptr;
  if (ctx->has_stage_events && stage >= 0 && ctx->stage_events[2 * stage + end]) {
    // inside a stream capture the record becomes an external event node of the graph, so a
    // replayed graph timestamps the stage boundary
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    cudaEventRecordWithFlags((cudaEvent_t)ctx->stage_events[2 * stage + end], st,
                             cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault);
  }
}

// one attention stage: out = (res ? res : 0) + MHA_dim(h); scratch qkv [tok,3C], o [tok,C].
// stage0 >= 0: record stage events for (QKV, ATTN, PROJ) = stage0, stage0+1, stage0+2.
// o_tseq != nullptr (temporal stage of the block): when the shape allows (tseq_ok), q | k | v are
// written sequence-major (TSEQ, dsp_internal.h) into qkv -- which must then hold tseq_bytes --
// and the attention output goes to o_tseq instead of o.
dsp_status_t attn_stage(dsp_ctx_t ctx, const dsp_shape_t* s, int64_t T_loc, int64_t S_loc, int dim, const void* h,
                        const void* w_qkv, const void* w_o, const void* res, void* out, void* qkv, void* o,
                        cudaStream_t st, int stage0 = -1, const EpiVec* ln = nullptr,
                        const RemoteMap* remote = nullptr, float2* part_out = nullptr, void* o_tseq = nullptr) {
  const int64_t tok = s->B * T_loc * S_loc, C = s->C;
#ifdef DSP_NO_TSEQ
  o_tseq = nullptr;  // A/B: token-major q | k | v for the temporal stage too
#endif
  const bool tseq = o_tseq && dim == DSP_DIM_T && s->dtype == DSP_BF16 && tseq_ok(s->B, T_loc, S_loc, C, s->num_heads);
  if (tseq) o = o_tseq;
  const int epi = res ? DSP_EPI_RESIDUAL : DSP_EPI_NONE;
  const int sq = stage0, sa = stage0 < 0 ? -1 : stage0 + 1, sp = stage0 < 0 ? -1 : stage0 + 2;
  if (s->dtype == DSP_BF16) {
    std::string why;
    mark(ctx, sq, 0, st);
    // ln != nullptr: h is the raw (un-normalised) input and w_qkv the LN-folded weight
    const TseqShape ts{(int)s->B, (int)T_loc, (int)S_loc, s->num_heads, (int)C};
    cudaError_t e = tseq ? launch_gemm_bf16_tseq(h, w_qkv, ln, qkv, ts, tok, C, ctx->num_sms, st, &why)
                    : ln ? launch_gemm_bf16_ln(h, w_qkv, *ln, qkv, tok, 3 * C, C, false, ctx->num_sms, st, &why)
                         : launch_gemm_bf16(h, w_qkv, nullptr, qkv, tok, 3 * C, C, DSP_EPI_NONE, ctx->num_sms, st, &why);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "qkv projection", why);
    mark(ctx, sq, 1, st);
    mark(ctx, sa, 0, st);
    e = tseq ? launch_fmha_bf16_tseq(qkv, o, s->B, T_loc, S_loc, C, s->num_heads, ctx->num_sms, st, &why)
             : launch_fmha_bf16(qkv, o, s->B, T_loc, S_loc, C, s->num_heads, dim, ctx->num_sms, st, &why);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "attention core", why);
    mark(ctx, sa, 1, st);
    mark(ctx, sp, 0, st);
    // remote != nullptr: switch fused into this epilogue (rows stored at their owner rank)
    e = remote     ? launch_gemm_bf16_remote(o, w_o, res, *remote, tok, C, C, ctx->num_sms, st, &why)
        : part_out ? launch_gemm_bf16_res_stats(o, w_o, res, out, tok, C, C, part_out, ctx->num_sms, st, &why)
                   : launch_gemm_bf16(o, w_o, res, out, tok, C, C, epi, ctx->num_sms, st, &why);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "output projection", why);
    mark(ctx, sp, 1, st);
  } else {
    mark(ctx, sq, 0, st);
    DSP_CUDA(ctx, launch_gemm_f32((const float*)h, (const float*)w_qkv, nullptr, (float*)qkv, tok, 3 * C, C, DSP_EPI_NONE, st), "qkv projection f32");
    mark(ctx, sq, 1, st);
    mark(ctx, sa, 0, st);
    DSP_CUDA(ctx, launch_attn_f32((const float*)qkv, (float*)o, s->B, T_loc, S_loc, C, s->num_heads, dim, st), "attention f32");
    mark(ctx, sa, 1, st);
    mark(ctx, sp, 0, st);
    DSP_CUDA(ctx, launch_gemm_f32((const float*)o, (const float*)w_o, (const float*)res, (float*)out, tok, C, C, epi, st), "output projection f32");
    mark(ctx, sp, 1, st);
  }
  if (tok > 0) ctx->launches += 3;
  return DSP_OK;
}

dsp_status_t linear(dsp_ctx_t ctx, dsp_dtype_t dt, int64_t M, int64_t N, int64_t K, const void* A, const void* W,
                    const void* R, int epi, void* D, cudaStream_t st) {
  if (dt == DSP_BF16) {
    std::string why;
    cudaError_t e = launch_gemm_bf16(A, W, R, D, M, N, K, epi, ctx->num_sms, st, &why);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "linear", why);
  } else {
    DSP_CUDA(ctx, launch_gemm_f32((const float*)A, (const float*)W, (const float*)R, (float*)D, M, N, K, epi, st), "linear f32");
  }
  if (M > 0) ctx->launches += 1;
  return DSP_OK;
}

}  // namespace

extern "C" {

int dsp_abi_version(void) { return DSP_ABI_VERSION; }

const char* dsp_status_str(dsp_status_t s) {
  switch (s) {
    case DSP_OK: return "DSP_OK";
    case DSP_ERR_NULL: return "DSP_ERR_NULL";
    case DSP_ERR_SHAPE: return "DSP_ERR_SHAPE";
    case DSP_ERR_DIVISIBILITY: return "DSP_ERR_DIVISIBILITY";
    case DSP_ERR_SAME_DIM: return "DSP_ERR_SAME_DIM";
    case DSP_ERR_BAD_DIM: return "DSP_ERR_BAD_DIM";
    case DSP_ERR_UNSUPPORTED: return "DSP_ERR_UNSUPPORTED";
    case DSP_ERR_ALIGNMENT: return "DSP_ERR_ALIGNMENT";
    case DSP_ERR_ALIAS: return "DSP_ERR_ALIAS";
    case DSP_ERR_WORKSPACE: return "DSP_ERR_WORKSPACE";
    case DSP_ERR_CUDA: return "DSP_ERR_CUDA";
    case DSP_ERR_NCCL: return "DSP_ERR_NCCL";
    case DSP_ERR_STATE: return "DSP_ERR_STATE";
    case DSP_ERR_PEER_TIMEOUT: return "DSP_ERR_PEER_TIMEOUT";
  }
  return "DSP_ERR_UNKNOWN";
}

const char* dsp_last_error(dsp_ctx_t ctx) { return ctx ? ctx->last_error.c_str() : g_no_ctx_error.c_str(); }

dsp_status_t dsp_ctx_create(void* nccl_comm, int rank, int world, int device, dsp_ctx_t* out) {
  if (!out) return fail(nullptr, DSP_ERR_NULL, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(nullptr, DSP_ERR_SHAPE, "bad rank %d / world %d", rank, world);
  dsp_ctx* c = new dsp_ctx();
  c->rank = rank; c->world = world; c->device = device; c->comm = nccl_comm;
  {
    const char* t = std::getenv("DSP_BARRIER_TIMEOUT_S");
    const double sec = t ? std::atof(t) : kDefaultBarrierTimeoutS;
    c->barrier_timeout_ns = sec > 0 ? (uint64_t)(sec * 1e9) : 0;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    fail(nullptr, DSP_ERR_CUDA, "device %d: %s", device, cudaGetErrorString(e));
    delete c;
    return DSP_ERR_CUDA;
  }
  if (nccl_comm) {
    std::string err;
    if (!nccl_load(&c->nccl, &err)) {
      fail(nullptr, DSP_ERR_NCCL, "%s", err.c_str());
      delete c;
      return DSP_ERR_NCCL;
    }
  }
  *out = c;
  return DSP_OK;
}

dsp_ctx::~dsp_ctx() {
  for (int b = 0; b < 2; ++b)
    for (void* e : {ev_in[b], ev_xfree[b], ev_out[b], ev_yfree[b]})
      if (e) cudaEventDestroy((cudaEvent_t)e);
  if (h2d_stream) cudaStreamDestroy((cudaStream_t)h2d_stream);
  for (void* e : wg_ev)
    if (e) cudaEventDestroy((cudaEvent_t)e);
  if (wg_stream) cudaStreamDestroy((cudaStream_t)wg_stream);
  if (d2h_stream) cudaStreamDestroy((cudaStream_t)d2h_stream);
}

dsp_status_t dsp_ctx_destroy(dsp_ctx_t ctx) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  delete ctx;
  return DSP_OK;
}

size_t dsp_workspace_bytes(const dsp_shape_t* s, int world) {
  if (!s || world < 1 || s->B < 1 || s->T < 1 || s->S < 1 || s->C < 1) return 0;
  return (size_t)block_ws(s, world).total;
}

dsp_status_t dsp_ctx_set_stage_events(dsp_ctx_t ctx, void* const* events, int n) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  if (!events) {
    ctx->has_stage_events = false;
    return DSP_OK;
  }
  if (n != 2 * DSP_NUM_STAGES) return fail(ctx, DSP_ERR_SHAPE, "need %d events", 2 * DSP_NUM_STAGES);
  for (int i = 0; i < n; ++i) ctx->stage_events[i] = events[i];
  ctx->has_stage_events = true;
  return DSP_OK;
}

dsp_status_t dsp_ctx_set_stage_clocks(dsp_ctx_t ctx, void* clocks_dev) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  if (clocks_dev && (reinterpret_cast<uintptr_t>(clocks_dev) & 7)) return fail(ctx, DSP_ERR_ALIGNMENT, "clock buffer not 8-B aligned");
  ctx->stage_clk = static_cast<unsigned long long*>(clocks_dev);
  return DSP_OK;
}

dsp_status_t dsp_ctx_set_tap(dsp_ctx_t ctx, dsp_tap_t point, void* dst, size_t bytes) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  if (point < 0 || point >= DSP_NUM_TAPS) return fail(ctx, DSP_ERR_SHAPE, "unknown tap %d", (int)point);
  if (dst && !aligned16(dst)) return fail(ctx, DSP_ERR_ALIGNMENT, "tap buffer not 16-B aligned");
  ctx->tap[point] = dst;
  ctx->tap_bytes[point] = dst ? bytes : 0;
  return DSP_OK;
}

int64_t dsp_ctx_launch_count(dsp_ctx_t ctx) { return ctx ? ctx->launches : -1; }

dsp_status_t dsp_ctx_set_workspace(dsp_ctx_t ctx, void* ws, size_t bytes) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  if (ws && !aligned16(ws)) return fail(ctx, DSP_ERR_ALIGNMENT, "workspace not 16-B aligned");
  ctx->ws = ws;
  ctx->ws_bytes = ws ? bytes : 0;
  return DSP_OK;
}

dsp_status_t dsp_ctx_set_peer_buffers(dsp_ctx_t ctx, void* const* base, void* const* sig, size_t bytes) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  if (!base || !sig) return fail(ctx, DSP_ERR_NULL, "peer pointer arrays are NULL");
  if (ctx->world > kMaxPeers) return fail(ctx, DSP_ERR_UNSUPPORTED, "P2P switch supports world <= %d", kMaxPeers);
  for (int i = 0; i < ctx->world; ++i) {
    if (!base[i] || !sig[i]) return fail(ctx, DSP_ERR_NULL, "peer %d pointer is NULL", i);
    if (!aligned16(base[i]) || !aligned16(sig[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "peer %d pointer not 16-B aligned", i);
    ctx->peer_base.p[i] = base[i];
    ctx->peer_signal.p[i] = sig[i];
  }
  ctx->peer_bytes = bytes;
  ctx->has_peers = true;
  return DSP_OK;
}

dsp_status_t dsp_switch_volume(const dsp_shape_t* s, int world, int64_t* sent, int64_t* recv) {
  DSP_TRY(check_shape(nullptr, s));
  DSP_TRY(check_div(nullptr, s, world));
  if (!sent || !recv) return fail(nullptr, DSP_ERR_NULL, "output pointer is NULL");
  const int64_t v = (int64_t)(world - 1) * s->B * (s->T / world) * (s->S / world) * s->C * elem_bytes(s->dtype);
  *sent = v;
  *recv = v;
  return DSP_OK;
}

dsp_status_t dsp_switch_plan(const dsp_shape_t* s, int world, int rank, dsp_dim_t from, dsp_dim_t to,
                             dsp_switch_plan_t* plan) {
  DSP_TRY(validate_switch(nullptr, s, world, from, to));
  if (!plan) return fail(nullptr, DSP_ERR_NULL, "plan is NULL");
  if (rank < 0 || rank >= world) return fail(nullptr, DSP_ERR_SHAPE, "rank %d out of range", rank);
  make_plan(s, world, rank, from, plan);
  return DSP_OK;
}

dsp_status_t dsp_split(dsp_ctx_t ctx, const dsp_shape_t* s, dsp_dim_t dim, const void* xg, void* xl, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_dim(ctx, dim));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!xg || !xl) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (!aligned16(xg) || !aligned16(xl)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const int N = ctx->world, r = ctx->rank;
  const int64_t e = elem_bytes(s->dtype), row = s->C * e, B = s->B, T = s->T, S = s->S, Tn = T / N, Sn = S / N;
  if (overlap(xg, B * T * S * row, xl, B * T * S * row / N)) return fail(ctx, DSP_ERR_ALIAS, "x_local overlaps x_global");
  RunCopy rc{};
  if (dim == DSP_DIM_T) {
    rc.n[0] = 1; rc.n[1] = B; rc.n[2] = 1; rc.run_bytes = Tn * S * row;
    rc.ss[1] = T * S * row; rc.ds[1] = Tn * S * row;
    xg = static_cast<const uint8_t*>(xg) + r * Tn * S * row;
  } else {
    rc.n[0] = 1; rc.n[1] = B; rc.n[2] = T; rc.run_bytes = Sn * row;
    rc.ss[1] = T * S * row; rc.ss[2] = S * row; rc.ds[1] = T * Sn * row; rc.ds[2] = Sn * row;
    xg = static_cast<const uint8_t*>(xg) + r * Sn * row;
  }
  DSP_CUDA(ctx, launch_run_copy(xg, xl, rc, ctx->num_sms, (cudaStream_t)stream), "split");
  ctx->launches += 1;
  return DSP_OK;
}

// Unpack of the all-gathered [N][local] rank-major buffer into the global layout.
static RunCopy gather_runs(const dsp_shape_t* s, int N, int dim) {
  const int64_t e = elem_bytes(s->dtype), row = s->C * e, B = s->B, T = s->T, S = s->S, Tn = T / N, Sn = S / N;
  const int64_t local = B * T * S * row / N;
  RunCopy rc{};
  if (dim == DSP_DIM_T) {
    rc.n[0] = N; rc.n[1] = B; rc.n[2] = 1; rc.run_bytes = Tn * S * row;
    rc.ss[0] = local; rc.ss[1] = Tn * S * row; rc.ds[0] = Tn * S * row; rc.ds[1] = T * S * row;
  } else {
    rc.n[0] = N; rc.n[1] = B; rc.n[2] = T; rc.run_bytes = Sn * row;
    rc.ss[0] = local; rc.ss[1] = T * Sn * row; rc.ss[2] = Sn * row;
    rc.ds[0] = Sn * row; rc.ds[1] = T * S * row; rc.ds[2] = S * row;
  }
  return rc;
}

static dsp_status_t check_layout_call(dsp_ctx_t ctx, const dsp_shape_t* s, int dim, const void* a, const void* b) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_dim(ctx, dim));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!a || !b) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (!aligned16(a) || !aligned16(b)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  return DSP_OK;
}

dsp_status_t dsp_gather(dsp_ctx_t ctx, const dsp_shape_t* s, dsp_dim_t dim, const void* xl, void* xg, void* stream) {
  DSP_TRY(check_layout_call(ctx, s, dim, xl, xg));
  const int N = ctx->world;
  const int64_t local = shard_bytes(s, N);
  cudaStream_t st = (cudaStream_t)stream;
  if (overlap(xg, local * N, xl, local)) return fail(ctx, DSP_ERR_ALIAS, "x_local overlaps x_global");
  if (N == 1) {
    DSP_CUDA(ctx, cudaMemcpyAsync(xg, xl, local, cudaMemcpyDeviceToDevice, st), "gather copy (N=1)");
    return DSP_OK;
  }
  if (!ctx->emulate_collectives && (!ctx->nccl.ok || !ctx->comm))
    return fail(ctx, DSP_ERR_NCCL, "gather without a communicator");
  const bool identity = (dim == DSP_DIM_T) ? (s->B == 1) : (s->B * s->T == 1);
  void* stage = xg;
  if (!identity) {
    if (!ctx->ws || ctx->ws_bytes < (size_t)(local * N)) return fail(ctx, DSP_ERR_WORKSPACE, "gather needs %lld bytes of workspace", (long long)(local * N));
    if (overlap(ctx->ws, local * N, xl, local) || overlap(ctx->ws, local * N, xg, local * N))
      return fail(ctx, DSP_ERR_ALIAS, "x_local / x_global overlap the workspace the gather stages through");
    stage = ctx->ws;
  }
  if (ctx->emulate_collectives) {
    DSP_TRY(emulated_gather_pieces(ctx, xl, 0, local, stage, st, "gather"));
  } else {
    int r = ctx->nccl.AllGather(xl, stage, (size_t)local, kNcclUint8, ctx->comm, st);
    if (r) return fail(ctx, DSP_ERR_NCCL, "ncclAllGather: %s", ctx->nccl.GetErrorString(r));
  }
  if (!identity) {
    DSP_CUDA(ctx, launch_run_copy(stage, xg, gather_runs(s, N, dim), ctx->num_sms, st), "gather unpack");
    ctx->launches += 1;
  }
  return DSP_OK;
}

dsp_status_t dsp_gather_unpack(dsp_ctx_t ctx, const dsp_shape_t* s, dsp_dim_t dim, const void* gathered, void* xg,
                               void* stream) {
  DSP_TRY(check_layout_call(ctx, s, dim, gathered, xg));
  const int64_t total = shard_bytes(s, 1);
  if (overlap(gathered, total, xg, total)) return fail(ctx, DSP_ERR_ALIAS, "gathered overlaps x_global");
  DSP_CUDA(ctx, launch_run_copy(gathered, xg, gather_runs(s, ctx->world, dim), ctx->num_sms, (cudaStream_t)stream),
           "gather unpack");
  ctx->launches += 1;
  return DSP_OK;
}

// Building blocks of the NCCL transport (include/dsp_kernels.h): the pack / unpack kernels of
// dsp_switch, always launched (an identity side is a contiguous copy here).
static dsp_status_t switch_chunk_call(dsp_ctx_t ctx, const dsp_shape_t* s, int from, int to, const void* a, void* b,
                                      bool pack, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(validate_switch(ctx, s, ctx->world, from, to));
  if (!a || !b) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (!aligned16(a) || !aligned16(b)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const int64_t bytes = shard_bytes(s, ctx->world);
  if (overlap(a, bytes, b, bytes)) return fail(ctx, DSP_ERR_ALIAS, "source and destination overlap");
  dsp_switch_plan_t p;
  make_plan(s, ctx->world, ctx->rank, from, &p);
  const ChunkCopies cc = chunk_copies(plan_runs(p));
  DSP_CUDA(ctx, launch_run_copy(a, b, pack ? cc.pack : cc.unpack, ctx->num_sms, (cudaStream_t)stream),
           pack ? "switch pack" : "switch unpack");
  ctx->launches += 1;
  return DSP_OK;
}

dsp_status_t dsp_switch_pack(dsp_ctx_t ctx, const dsp_shape_t* s, dsp_dim_t from, dsp_dim_t to, const void* x_local,
                             void* send, void* stream) {
  return switch_chunk_call(ctx, s, from, to, x_local, send, true, stream);
}

dsp_status_t dsp_switch_unpack(dsp_ctx_t ctx, const dsp_shape_t* s, dsp_dim_t from, dsp_dim_t to, const void* recv,
                               void* y_local, void* stream) {
  return switch_chunk_call(ctx, s, from, to, recv, y_local, false, stream);
}

dsp_status_t dsp_ctx_set_collective_emulation(dsp_ctx_t ctx, int on) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  if (on && !ctx->has_peers) return fail(ctx, DSP_ERR_STATE, "collective emulation needs dsp_ctx_set_peer_buffers");
  ctx->emulate_collectives = on != 0;
  return DSP_OK;
}

dsp_status_t dsp_ctx_set_barrier_timeout(dsp_ctx_t ctx, double seconds) {
  if (!ctx) return fail(nullptr, DSP_ERR_NULL, "context is NULL");
  ctx->barrier_timeout_ns = seconds > 0 ? (uint64_t)(seconds * 1e9) : 0;
  return DSP_OK;
}

dsp_status_t dsp_ctx_check_errors(dsp_ctx_t ctx) {
  DSP_TRY(check_ctx(ctx));
  if (ctx->has_peers) {
    uint64_t rec = 0;
    const uint64_t* slot = static_cast<const uint64_t*>(ctx->peer_signal.p[ctx->rank]) + kPadError;
    DSP_CUDA(ctx, cudaMemcpy(&rec, slot, sizeof(rec), cudaMemcpyDeviceToHost), "read barrier error record");
    if (rec)
      return fail(ctx, DSP_ERR_PEER_TIMEOUT, "P2P barrier %llu timed out waiting for rank %u (timeout %.1f s)",
                  (unsigned long long)(rec >> 16), (unsigned)(rec & 0xff), ctx->barrier_timeout_ns * 1e-9);
  }
  if (ctx->comm && ctx->nccl.CommGetAsyncError) {
    int async = 0;
    int r = ctx->nccl.CommGetAsyncError(ctx->comm, &async);
    if (r) return fail(ctx, DSP_ERR_NCCL, "ncclCommGetAsyncError: %s", ctx->nccl.GetErrorString(r));
    if (async) return fail(ctx, DSP_ERR_NCCL, "communicator async error: %s", ctx->nccl.GetErrorString(async));
  }
  return DSP_OK;
}

// N-D plan (see include/dsp.h).  With a = from, b = to, inner = prod(d after max(a, b)) * elem:
//   a < b: runs of (d_b/N)*inner bytes over (peer q, outer, i_a in [0, d_a/N), middle); peer q
//          gets the i_b block q; lands at i_a + rank*d_a/N in q's [.., d_a, .., d_b/N, ..];
//   a > b: runs of (d_a/N)*inner bytes over (peer q, outer, i_b in block q, middle); lands at
//          i_b - q*d_b/N, with the run at offset rank*(d_a/N)*inner, in q's [.., d_b/N, .., d_a, ..].
static dsp_status_t make_plan_nd(dsp_ctx_t ctx, const int64_t* d, int nd, int e, int N, int rank, int a, int b,
                                 dsp_switch_nd_plan_t* p) {
  if (!d || !p) return fail(ctx, DSP_ERR_NULL, "NULL argument");
  if (nd < 3 || nd > DSP_ND_MAX_DIMS) return fail(ctx, DSP_ERR_SHAPE, "ndim %d outside [3, %d]", nd, DSP_ND_MAX_DIMS);
  if (e < 1 || N < 1) return fail(ctx, DSP_ERR_SHAPE, "elem_bytes %d / world %d < 1", e, N);
  for (int i = 0; i < nd; ++i)
    if (d[i] < 1) return fail(ctx, DSP_ERR_SHAPE, "extent %d is %lld", i, (long long)d[i]);
  if (a < 0 || a > nd - 2 || b < 0 || b > nd - 2) return fail(ctx, DSP_ERR_BAD_DIM, "switch dims must be in [0, %d]", nd - 2);
  if (a == b) return fail(ctx, DSP_ERR_SAME_DIM, "switch from a dim to itself (S:283)");
  if (rank < 0 || rank >= N) return fail(ctx, DSP_ERR_SHAPE, "rank %d outside [0, %d)", rank, N);
  if (d[a] % N || d[b] % N) return fail(ctx, DSP_ERR_DIVISIBILITY, "world %d does not divide d[%d]=%lld / d[%d]=%lld", N, a,
                                        (long long)d[a], b, (long long)d[b]);
  const int lo = a < b ? a : b, hi = a < b ? b : a;
  int64_t outer = 1, mid = 1, inner = e;
  for (int i = 0; i < lo; ++i) outer *= d[i];
  for (int i = lo + 1; i < hi; ++i) mid *= d[i];
  for (int i = hi + 1; i < nd; ++i) inner *= d[i];
  const int64_t ra = d[a] / N, rb = d[b] / N;
  memset(p, 0, sizeof(*p));
  p->n[0] = N; p->n[1] = outer; p->n[3] = mid;
  if (a < b) {  // x [outer, d_a/N, mid, d_b, inner] -> y [outer, d_a, mid, d_b/N, inner]
    p->n[2] = ra;
    p->run_bytes = rb * inner;
    p->src_stride[0] = rb * inner; p->src_stride[1] = ra * mid * d[b] * inner;
    p->src_stride[2] = mid * d[b] * inner; p->src_stride[3] = d[b] * inner;
    p->dst_stride[1] = d[a] * mid * rb * inner; p->dst_stride[2] = mid * rb * inner; p->dst_stride[3] = rb * inner;
    p->dst_stride[0] = ra * p->dst_stride[2];
  } else {      // x [outer, d_b, mid, d_a/N, inner] -> y [outer, d_b/N, mid, d_a, inner]
    p->n[2] = rb;
    p->run_bytes = ra * inner;
    p->src_stride[0] = rb * mid * ra * inner; p->src_stride[1] = d[b] * mid * ra * inner;
    p->src_stride[2] = mid * ra * inner; p->src_stride[3] = ra * inner;
    p->dst_stride[1] = rb * mid * d[a] * inner; p->dst_stride[2] = mid * d[a] * inner; p->dst_stride[3] = d[a] * inner;
    p->dst_stride[0] = ra * inner;
  }
  p->dst_peer_off = rank * p->dst_stride[0];
  if (p->run_bytes % 16) return fail(ctx, DSP_ERR_ALIGNMENT, "switch runs of %lld bytes are not 16-B multiples", (long long)p->run_bytes);
  // pack is an identity when peer q's runs already sit contiguously at q * chunk in x; unpack
  // when the received [source rank][outer][rows][middle] layout is y's own layout
  const int64_t R = p->run_bytes, chunk = p->n[1] * p->n[2] * p->n[3] * R;
  auto same = [&](const int64_t* st) {
    return (p->n[3] == 1 || st[3] == R) && (p->n[2] == 1 || st[2] == p->n[3] * R) &&
           (p->n[1] == 1 || st[1] == p->n[2] * p->n[3] * R) && st[0] == chunk;
  };
  p->pack_is_identity = N == 1 || same(p->src_stride);
  p->unpack_is_identity = N == 1 || same(p->dst_stride);
  return DSP_OK;
}

dsp_status_t dsp_switch_nd_plan(const int64_t* dims, int ndim, int elem_bytes, int world, int rank, int from_dim,
                                int to_dim, dsp_switch_nd_plan_t* plan) {
  return make_plan_nd(nullptr, dims, ndim, elem_bytes, world, rank, from_dim, to_dim, plan);
}

dsp_status_t dsp_switch_nd(dsp_ctx_t ctx, const int64_t* dims, int ndim, int elem_bytes, int from_dim, int to_dim,
                           const void* x, void* y, dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_ctx(ctx));
  dsp_switch_nd_plan_t p;
  DSP_TRY(make_plan_nd(ctx, dims, ndim, elem_bytes, ctx->world, ctx->rank, from_dim, to_dim, &p));
  if (impl != DSP_SWITCH_NCCL && impl != DSP_SWITCH_P2P && impl != DSP_SWITCH_FUSED)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "unknown switch impl %d", (int)impl);
  if (impl == DSP_SWITCH_FUSED) impl = DSP_SWITCH_P2P;
  if (!x || !y) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (!aligned16(x) || !aligned16(y)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const int N = ctx->world;
  int64_t bytes = elem_bytes;
  for (int i = 0; i < ndim; ++i) bytes *= dims[i];
  bytes /= N;
  cudaStream_t st = (cudaStream_t)stream;
  if (N == 1) {
    if (x != y) DSP_CUDA(ctx, cudaMemcpyAsync(y, x, bytes, cudaMemcpyDeviceToDevice, st), "switch copy (N=1)");
    return DSP_OK;
  }
  if (overlap(x, bytes, y, bytes)) return fail(ctx, DSP_ERR_ALIAS, "x_local overlaps y_local");
  void* send = nullptr;
  void* recv = nullptr;
  if (impl == DSP_SWITCH_NCCL) {
    const int64_t need = (p.pack_is_identity ? 0 : bytes) + (p.unpack_is_identity ? 0 : bytes);
    if (need && (!ctx->ws || ctx->ws_bytes < (size_t)need))
      return fail(ctx, DSP_ERR_WORKSPACE, "switch needs %lld bytes of workspace", (long long)need);
    if (need && (overlap(ctx->ws, need, x, bytes) || overlap(ctx->ws, need, y, bytes)))
      return fail(ctx, DSP_ERR_ALIAS, "x_local / y_local overlap the workspace the NCCL switch stages through");
    send = ctx->ws;
    recv = static_cast<uint8_t*>(ctx->ws) + (p.pack_is_identity ? 0 : bytes);
  }
  RunCopy rc;
  for (int i = 0; i < 4; ++i) { rc.n[i] = p.n[i]; rc.ss[i] = p.src_stride[i]; rc.ds[i] = p.dst_stride[i]; }
  rc.run_bytes = p.run_bytes;
  return do_switch_plan(ctx, rc, p.dst_peer_off, p.pack_is_identity, p.unpack_is_identity, bytes, x, y, impl, st, send,
                        recv);
}

dsp_status_t dsp_switch(dsp_ctx_t ctx, const dsp_shape_t* s, dsp_dim_t from, dsp_dim_t to, const void* x, void* y,
                        dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(validate_switch(ctx, s, ctx->world, from, to));
  if (impl != DSP_SWITCH_NCCL && impl != DSP_SWITCH_P2P && impl != DSP_SWITCH_FUSED)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "unknown switch impl %d", (int)impl);
  if (impl == DSP_SWITCH_FUSED) impl = DSP_SWITCH_P2P;  // a standalone switch has nothing to fuse with
  if (!x || !y) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (!aligned16(x) || !aligned16(y)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const int64_t bytes = shard_bytes(s, ctx->world);
  if (ctx->world > 1 && overlap(x, bytes, y, bytes)) return fail(ctx, DSP_ERR_ALIAS, "x_local overlaps y_local");
  void* send = nullptr;
  void* recv = nullptr;
  if (ctx->world > 1 && impl == DSP_SWITCH_NCCL) {
    dsp_switch_plan_t p;
    make_plan(s, ctx->world, ctx->rank, from, &p);
    const int64_t need = (p.pack_is_identity ? 0 : bytes) + (p.unpack_is_identity ? 0 : bytes);
    if (need && (!ctx->ws || ctx->ws_bytes < (size_t)need))
      return fail(ctx, DSP_ERR_WORKSPACE, "switch needs %lld bytes of workspace", (long long)need);
    if (need && (overlap(ctx->ws, need, x, bytes) || overlap(ctx->ws, need, y, bytes)))
      return fail(ctx, DSP_ERR_ALIAS, "x_local / y_local overlap the workspace the NCCL switch stages through");
    send = ctx->ws;
    recv = static_cast<uint8_t*>(ctx->ws) + (p.pack_is_identity ? 0 : bytes);
  }
  return do_switch(ctx, s, from, x, y, impl, (cudaStream_t)stream, send, recv);
}

static dsp_status_t attn_public(dsp_ctx_t ctx, const dsp_shape_t* s, int dim, const void* h, const void* wqkv,
                                const void* wo, const void* res, void* out, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!h || !wqkv || !wo || !out) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  const int N = ctx->world;
  const int64_t T_loc = dim == DSP_DIM_S ? s->T / N : s->T, S_loc = dim == DSP_DIM_S ? s->S : s->S / N;
  DSP_TRY(check_bf16_attn(ctx, s, dim == DSP_DIM_S ? S_loc : T_loc));
  const int64_t e = elem_bytes(s->dtype), tok = s->B * T_loc * S_loc, act = tok * s->C * e;
  if (!aligned16(h) || !aligned16(out) || (res && !aligned16(res))) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  if (overlap(h, act, out, act)) return fail(ctx, DSP_ERR_ALIAS, "out overlaps h");
  if (res && res != out && overlap(res, act, out, act)) return fail(ctx, DSP_ERR_ALIAS, "out partially overlaps residual");
  const int64_t need = tok * 4 * s->C * e;
  if (!ctx->ws || ctx->ws_bytes < (size_t)need) return fail(ctx, DSP_ERR_WORKSPACE, "attention needs %lld bytes of workspace", (long long)need);
  void* qkv = ctx->ws;
  void* o = static_cast<uint8_t*>(ctx->ws) + tok * 3 * s->C * e;
  return attn_stage(ctx, s, T_loc, S_loc, dim, h, wqkv, wo, res, out, qkv, o, (cudaStream_t)stream);
}

dsp_status_t dsp_spatial_attn(dsp_ctx_t ctx, const dsp_shape_t* s, const void* h, const void* wqkv, const void* wo,
                              const void* res, void* out, void* stream) {
  return attn_public(ctx, s, DSP_DIM_S, h, wqkv, wo, res, out, stream);
}

dsp_status_t dsp_temporal_attn(dsp_ctx_t ctx, const dsp_shape_t* s, const void* h, const void* wqkv, const void* wo,
                               const void* res, void* out, void* stream) {
  return attn_public(ctx, s, DSP_DIM_T, h, wqkv, wo, res, out, stream);
}

// One block.  Chaining flags of dsp_st_model_forward (prepared weights):
//   ln1_from_parts: the LN1 statistics of x are combined from per-row partials: at N == 1 those
//                   the previous block's FC2 epilogue left in the workspace (no pass at all), at
//                   N > 1 recomputed bitwise by launch_row_partials (the rows crossed a switch);
//   emit_parts:     the FC2 epilogue writes the per-row partials of y for the next block's LN1
//                   (N == 1).
static dsp_status_t block_forward(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w, const void* x,
                                  void* y, dsp_switch_impl_t impl, void* stream, bool ln1_from_parts,
                                  bool emit_parts) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!w || !x || !y) return fail(ctx, DSP_ERR_NULL, "NULL argument");
  const void* wp[12] = {w->ln1_w, w->ln1_b, w->w_qkv_s, w->w_o_s, w->ln2_w, w->ln2_b,
                        w->w_qkv_t, w->w_o_t, w->ln3_w, w->ln3_b, w->w_fc1, w->w_fc2};
  for (int i = 0; i < 12; ++i) {
    if (!wp[i]) return fail(ctx, DSP_ERR_NULL, "weight %d is NULL", i);
    if (!aligned16(wp[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "weight %d not 16-B aligned", i);
  }
  if (!aligned16(x) || !aligned16(y)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const bool cross = w->ln_c_w != nullptr;
  if (cross) {
    const void* cp[6] = {w->ln_c_w, w->ln_c_b, w->w_q_c, w->w_kv_c, w->w_o_c, w->ctx_tokens};
    for (int i = 0; i < 6; ++i)
      if (!cp[i] || !aligned16(cp[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "cross weight %d NULL or not 16-B aligned", i);
    if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "the cross stage runs on the bf16 path");
    if (w->ctx_len < 1) return fail(ctx, DSP_ERR_SHAPE, "ctx_len %lld < 1", (long long)w->ctx_len);
    if (s->B * w->ctx_len > s->B * s->T * s->S / ctx->world)
      return fail(ctx, DSP_ERR_UNSUPPORTED, "context longer than the local tokens per sample");
  }
  const bool latte = w->w_fc1_s != nullptr;
  if (latte) {
    const void* lp[4] = {w->ln_m_w, w->ln_m_b, w->w_fc1_s, w->w_fc2_s};
    for (int i = 0; i < 4; ++i)
      if (!lp[i] || !aligned16(lp[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "Latte weight %d NULL or not 16-B aligned", i);
    if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "the Latte pair runs on the bf16 path");
    if (impl == DSP_SWITCH_FUSED && ctx->world > 1)
      return fail(ctx, DSP_ERR_UNSUPPORTED, "the Latte pair does not run with the fused switch");
  }
  if (w->pe_t && (s->dtype != DSP_BF16 || !aligned16(w->pe_t) || s->C % 8))
    return fail(ctx, DSP_ERR_UNSUPPORTED, "temporal positional embedding: bf16, 16-B aligned, C %% 8 == 0");
  if (w->prepared && s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "prepared weights exist for the bf16 path only");
  if (w->prepared && (s->C % 8 || s->C > 256 * kRowStatsMaxV || s->C / gemm_part_cols(s->C) > kMaxParts))
    return fail(ctx, DSP_ERR_UNSUPPORTED, "prepared path needs C %% 8 == 0, C <= %d and C / BN <= %d",
                256 * kRowStatsMaxV, kMaxParts);
  const int N = ctx->world;
  if (impl != DSP_SWITCH_NCCL && impl != DSP_SWITCH_P2P && impl != DSP_SWITCH_FUSED)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "unknown switch impl %d", (int)impl);
  DSP_TRY(check_bf16_attn(ctx, s, s->S));
  DSP_TRY(check_bf16_attn(ctx, s, s->T));
  const int64_t e = elem_bytes(s->dtype), C = s->C, tok = s->B * s->T * s->S / N, act = tok * C * e;
  const size_t need = dsp_workspace_bytes(s, N);
  if (!ctx->ws || ctx->ws_bytes < need) return fail(ctx, DSP_ERR_WORKSPACE, "block needs %zu bytes of workspace", need);
  if (x != y && overlap(x, act, y, act)) return fail(ctx, DSP_ERR_ALIAS, "x_local partially overlaps y_local");
  if (overlap(ctx->ws, need, x, act) || overlap(ctx->ws, need, y, act)) return fail(ctx, DSP_ERR_ALIAS, "workspace overlaps x/y");
  for (int t = 0; t < DSP_NUM_TAPS; ++t)
    if (ctx->tap[t] && ctx->tap_bytes[t] < (size_t)act) return fail(ctx, DSP_ERR_WORKSPACE, "tap %d needs %lld bytes", t, (long long)act);
  const BlockWs L = block_ws(s, N);
  uint8_t* ws = static_cast<uint8_t*>(ctx->ws);
  void* h = ws + L.h;                // [tok, C]
  uint8_t* big = ws + L.big;         // [tok, 4C]: qkv + o | MLP hidden | switch scratch
  void* qkv = big;
  void* o = big + 3 * act;
  void* ys = ws + L.ys;              // [tok, C] S-sharded activation (N > 1)
  const bool fused = N > 1 && impl == DSP_SWITCH_FUSED;
  RemoteMap rm_ts{}, rm_st{};
  if (N > 1 && (impl == DSP_SWITCH_P2P || fused)) {
    if (!ctx->has_peers) return fail(ctx, DSP_ERR_STATE, "P2P block without dsp_ctx_set_peer_buffers");
    void* base = ctx->peer_base.p[ctx->rank];
    if (!in_region(ys, act, base, ctx->peer_bytes) || !in_region(y, act, base, ctx->peer_bytes))
      return fail(ctx, DSP_ERR_UNSUPPORTED, "P2P block needs the workspace and y_local inside the symmetric buffer");
    if (fused) {
      if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "fused switch needs the bf16 path");
      const int64_t ys_off = static_cast<uint8_t*>(ys) - static_cast<uint8_t*>(base);
      const int64_t y_off = static_cast<uint8_t*>(y) - static_cast<uint8_t*>(base);
      rm_ts = RemoteMap{ctx->peer_base, ys_off, 1, ctx->rank, (int)s->B, (int)s->T, (int)s->S, (int)(s->T / N), (int)(s->S / N)};
      rm_st = RemoteMap{ctx->peer_base, y_off, 2, ctx->rank, (int)s->B, (int)s->T, (int)s->S, (int)(s->T / N), (int)(s->S / N)};
      // prepared weights: the T->S barrier is split -- PROJ_S's last CTA arrives, the LN2 partials
      // pass waits per row for the rank that sent it (f1: no barrier launch, rows consumed as
      // their sender finishes)
      rm_ts.signals = ctx->peer_signal;
      rm_ts.world = N;
      rm_ts.arrive = w->prepared != nullptr && !w->pe_t;
      // a stack of prepared blocks (dsp_st_model_forward): the S->T barrier is split too -- FC2's last
      // CTA arrives, the next block's LN1 partials pass waits per row; the last block keeps the barrier
      rm_st.signals = ctx->peer_signal;
      rm_st.world = N;
      rm_st.arrive = w->prepared != nullptr && emit_parts;
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  const float eps = w->ln_eps;
  const int64_t Tn = s->T / N, Sn = s->S / N;
  // Prepared weights (dsp_st_block_prepare): every LayerNorm is folded into the GEMM that
  // consumes it.  LN1: row statistics of x; LN2 (N == 1) and LN3: combined in the consuming
  // epilogue from per-row partials the out-projection epilogues write; LN2 at N > 1: row
  // statistics after the switch (the rows moved).
  const bool fold = w->prepared != nullptr;
  const PrepLayout P = prep_layout(C);
  const uint8_t* prep = static_cast<const uint8_t*>(w->prepared);
  const float* uv = fold ? reinterpret_cast<const float*>(prep + P.uv) : nullptr;
  float2* stats = reinterpret_cast<float2*>(ws + L.stats);
  float2* parts = reinterpret_cast<float2*>(ws + L.parts);
  const int nparts = (int)(C / gemm_part_cols(C));
  EpiVec ev1{}, ev2{}, ev3{};
  // LN statistics from per-row partials are the same bits at every N: at N > 1 the rows reach
  // their consumer through a switch without their producer's partials, so launch_row_partials
  // recomputes them bitwise (SURVEY §8c.4 (i) N-invariance).
  const bool chain_in = fold && ln1_from_parts, chain_out = fold && N == 1 && emit_parts;
  const int part_cnt = (int)(C / nparts);
  if (fold) {
    ev1.row_stats = stats; ev1.col_u = uv; ev1.col_v = uv + 3 * C;
    if (chain_in) {
      ev1.row_stats = nullptr;
      ev1.part_in = parts; ev1.nparts_in = nparts; ev1.part_cnt = part_cnt; ev1.eps = eps;
    }
    ev2.col_u = uv + 6 * C; ev2.col_v = uv + 9 * C;
    ev3.col_u = uv + 12 * C; ev3.col_v = uv + 16 * C;
    ev3.part_in = parts; ev3.nparts_in = nparts; ev3.part_cnt = part_cnt; ev3.eps = eps;
    ev2.part_in = parts; ev2.nparts_in = nparts; ev2.part_cnt = part_cnt; ev2.eps = eps;
  }
  const void* wf_s = fold ? prep + P.wf_s : nullptr;
  const void* wf_t = fold ? prep + P.wf_t : nullptr;
  const void* wf_1 = fold ? prep + P.wf_1 : nullptr;
  // a1: LN1 (prepared: row statistics of x only)
  mark(ctx, DSP_STAGE_LN1, 0, st);
  if (chain_in && N > 1) {  // the previous block's FC2 partials stayed on the other side of its switch
    // (fused: the previous block's FC2 arrived instead of a barrier; wait per row for its sender)
    const PeerWait st_wait = fused ? PeerWait{static_cast<const uint64_t*>(ctx->peer_signal.p[ctx->rank]), 2, (int)s->T,
                                              (int)Tn, (int)Sn, (int)s->S, (int)Sn, ctx->barrier_timeout_ns}
                                   : PeerWait{};
    DSP_CUDA(ctx, launch_row_partials(tok, C, part_cnt, x, parts, st, st_wait, ctx->num_sms), "LN1 partials");
    ctx->launches += 1;
  } else if (!chain_in) {
    if (fold) DSP_CUDA(ctx, launch_row_stats(tok, C, x, eps, stats, st), "LN1 stats");
    else DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, x, w->ln1_w, w->ln1_b, eps, h, st), "LN1");
    ctx->launches += 1;
  }
  mark(ctx, DSP_STAGE_LN1, 1, st);
  // a2-a4: y1 = x + MHA_S(LN1 x), local on T-shards, stored in y (N == 1 prepared: + LN2 partials)
  DSP_TRY(attn_stage(ctx, s, Tn, s->S, DSP_DIM_S, fold ? x : h, fold ? wf_s : w->w_qkv_s, w->w_o_s, x, y, qkv, o,
                     st, DSP_STAGE_QKV_S, fold ? &ev1 : nullptr, fused ? &rm_ts : nullptr,
                     fold && (N == 1 || latte) ? parts : nullptr));
  if (latte) {  // R38: y1 += W2_s gelu(W1_s LN_m(y1)), local on the T-shards (LN_m from PROJ_S's partials)
    std::string why;
    cudaError_t e2;
    if (fold) {
      const float* uv1s = reinterpret_cast<const float*>(prep + P.uv_1s);
      EpiVec evm{};
      evm.col_u = uv1s; evm.col_v = uv1s + 4 * C;
      evm.part_in = parts; evm.nparts_in = nparts; evm.part_cnt = part_cnt; evm.eps = eps;
      e2 = launch_gemm_bf16_ln(y, prep + P.wf_1s, evm, big, tok, 4 * C, C, true, ctx->num_sms, st, &why);
    } else {
      DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, y, w->ln_m_w, w->ln_m_b, eps, h, st), "LN_m");
      ctx->launches += 1;
      e2 = launch_gemm_bf16(h, w->w_fc1_s, nullptr, big, tok, 4 * C, C, DSP_EPI_GELU, ctx->num_sms, st, &why);
    }
    if (e2 == cudaSuccess)  // (+ the partials LN2 folds at N == 1)
      e2 = fold && N == 1 ? launch_gemm_bf16_res_stats(big, w->w_fc2_s, y, y, tok, C, 4 * C, parts, ctx->num_sms, st, &why)
                          : launch_gemm_bf16(big, w->w_fc2_s, y, y, tok, C, 4 * C, DSP_EPI_RESIDUAL, ctx->num_sms, st, &why);
    if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "Latte spatial MLP", why);
    ctx->launches += 2;
  }
  // a5: switch T -> S (fused: the out-projection already stored every row at its owner)
  void* cur = y;
  mark(ctx, DSP_STAGE_SWITCH_TS, 0, st);
  PeerWait ts_wait{};
  if (fused && rm_ts.arrive) {  // split barrier: the LN2 partials pass below waits per sending rank
    ts_wait = PeerWait{static_cast<const uint64_t*>(ctx->peer_signal.p[ctx->rank]), 1, (int)s->T, (int)Tn, (int)Sn,
                       (int)s->S, (int)Sn, ctx->barrier_timeout_ns};
    cur = ys;
  } else if (fused) {
    DSP_CUDA(ctx, launch_p2p_barrier(ctx->peer_signal, ctx->rank, N, ctx->barrier_timeout_ns, st), "fused switch barrier");
    ctx->launches += 1;
    cur = ys;
  } else if (N > 1) {
    DSP_TRY(do_switch(ctx, s, DSP_DIM_T, y, ys, impl, st, big, big + act));
    cur = ys;
  }
  mark(ctx, DSP_STAGE_SWITCH_TS, 1, st);
  if (w->pe_t) {  // R37: y1 += pe_t[t] on the S-shards (every frame of the local columns)
    DSP_CUDA(ctx, launch_add_temporal_pe(cur, w->pe_t, s->B, s->T, Sn, C, st), "temporal positional embedding");
    ctx->launches += 1;
  }
  if (ctx->tap[DSP_TAP_Y1]) DSP_CUDA(ctx, cudaMemcpyAsync(ctx->tap[DSP_TAP_Y1], cur, act, cudaMemcpyDeviceToDevice, st), "tap y1");
  // a6-a9: y2 = y1 + MHA_T(LN2 y1), local on S-shards (in place; prepared: + LN3 partials)
  mark(ctx, DSP_STAGE_LN2, 0, st);
  if (!fold) {
    DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, cur, w->ln2_w, w->ln2_b, eps, h, st), "LN2");
    ctx->launches += 1;
  } else if (N > 1 || w->pe_t) {  // the rows moved, or pe changed them: their partials again
    DSP_CUDA(ctx, launch_row_partials(tok, C, part_cnt, cur, parts, st, ts_wait, ctx->num_sms), "LN2 partials");
    ctx->launches += 1;
  }
#ifdef DSP_LN2_ROWSTATS  // A/B experiment: LN2 statistics by a row-statistics pass instead of partials
  if (fold) {
    DSP_CUDA(ctx, launch_row_stats(tok, C, cur, eps, stats, st), "LN2 stats");
    ev2.row_stats = stats;
  }
#endif
  mark(ctx, DSP_STAGE_LN2, 1, st);
  // (temporal q | k | v sequence-major in big, the attention output in h: both free here)
  DSP_TRY(attn_stage(ctx, s, s->T, Sn, DSP_DIM_T, fold ? cur : h, fold ? wf_t : w->w_qkv_t, w->w_o_t, cur, cur, qkv,
                     o, st, DSP_STAGE_QKV_T, fold ? &ev2 : nullptr, nullptr, fold ? parts : nullptr, h));
  if (cross) {  // ST-DiT cross stage: y2 += CA(LN_c(y2), ctx) on the S-shards, in place
    const int64_t Lq = s->T * (s->S / N), Lc = w->ctx_len;
    uint8_t* q = big;
    uint8_t* oc = big + act;
    uint8_t* kvb = big + 2 * act;  // B * Lc <= tok rows of [k | v]
    std::string why;
    cudaError_t e2;
    if (fold) {  // LN_c folded into the q projection; its statistics from PROJ_T's partials (R30)
      EpiVec evc{};
      const float* uvc = reinterpret_cast<const float*>(prep + P.uv_c);
      evc.col_u = uvc; evc.col_v = uvc + C;
      evc.part_in = parts; evc.nparts_in = nparts; evc.part_cnt = (int)(C / nparts); evc.eps = eps;
      e2 = launch_gemm_bf16_ln(cur, prep + P.wf_c, evc, q, tok, C, C, false, ctx->num_sms, st, &why);
    } else {
      DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, cur, w->ln_c_w, w->ln_c_b, eps, h, st), "LN_c");
      e2 = launch_gemm_bf16(h, w->w_q_c, nullptr, q, tok, C, C, DSP_EPI_NONE, ctx->num_sms, st, &why);
    }
    if (e2 == cudaSuccess)
      e2 = launch_gemm_bf16(w->ctx_tokens, w->w_kv_c, nullptr, kvb, s->B * Lc, 2 * C, C, DSP_EPI_NONE, ctx->num_sms, st, &why);
    if (e2 == cudaSuccess) e2 = launch_fmha_cross_bf16(q, kvb, oc, s->B, Lq, Lc, C, s->num_heads, ctx->num_sms, st, &why);
    // the cross output projection rewrites the rows LN3 normalises: it writes their partials (R30)
    if (e2 == cudaSuccess)
      e2 = fold ? launch_gemm_bf16_res_stats(oc, w->w_o_c, cur, cur, tok, C, C, parts, ctx->num_sms, st, &why)
                : launch_gemm_bf16(oc, w->w_o_c, cur, cur, tok, C, C, DSP_EPI_RESIDUAL, ctx->num_sms, st, &why);
    if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "cross stage", why);
    ctx->launches += fold ? 4 : 5;
  }
  if (ctx->tap[DSP_TAP_Y2]) DSP_CUDA(ctx, cudaMemcpyAsync(ctx->tap[DSP_TAP_Y2], cur, act, cudaMemcpyDeviceToDevice, st), "tap y2");
  // a10: y = y2 + W2 gelu(W1 LN3 y2) (in place)
  mark(ctx, DSP_STAGE_LN3, 0, st);
  if (!fold) {
    DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, cur, w->ln3_w, w->ln3_b, eps, h, st), "LN3");
    ctx->launches += 1;
  }
  mark(ctx, DSP_STAGE_LN3, 1, st);
  mark(ctx, DSP_STAGE_FC1, 0, st);
  if (fold) {
    std::string why;
    cudaError_t e2 = launch_gemm_bf16_ln(cur, wf_1, ev3, big, tok, 4 * C, C, true, ctx->num_sms, st, &why);
    if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "FC1 (LN3 folded)", why);
    if (tok > 0) ctx->launches += 1;
  } else {
    DSP_TRY(linear(ctx, s->dtype, tok, 4 * C, C, h, w->w_fc1, nullptr, DSP_EPI_GELU, big, st));
  }
  mark(ctx, DSP_STAGE_FC1, 1, st);
  mark(ctx, DSP_STAGE_FC2, 0, st);
  if (fused) {  // FC2 epilogue stores y = y2 + MLP rows straight into the T-shard owners' y_local
    std::string why;
    cudaError_t e2 = launch_gemm_bf16_remote(big, w->w_fc2, cur, rm_st, tok, C, 4 * C, ctx->num_sms, st, &why);
    if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "FC2 (switch fused)", why);
    ctx->launches += 1;
  } else if (chain_out) {  // + LN partials of y for the next block's LN1
    std::string why;
    cudaError_t e2 = launch_gemm_bf16_res_stats(big, w->w_fc2, cur, cur, tok, C, 4 * C, parts, ctx->num_sms, st, &why);
    if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "FC2 (+LN partials)", why);
    if (tok > 0) ctx->launches += 1;
  } else {
    DSP_TRY(linear(ctx, s->dtype, tok, C, 4 * C, big, w->w_fc2, cur, DSP_EPI_RESIDUAL, cur, st));
  }
  mark(ctx, DSP_STAGE_FC2, 1, st);
  // a11: switch S -> T back into y
  mark(ctx, DSP_STAGE_SWITCH_ST, 0, st);
  if (fused && !rm_st.arrive) {
    DSP_CUDA(ctx, launch_p2p_barrier(ctx->peer_signal, ctx->rank, N, ctx->barrier_timeout_ns, st), "fused switch barrier");
    ctx->launches += 1;
  } else if (N > 1 && !fused) {
    DSP_TRY(do_switch(ctx, s, DSP_DIM_S, ys, y, impl, st, big, big + act));
  }
  mark(ctx, DSP_STAGE_SWITCH_ST, 1, st);
  return DSP_OK;
}

dsp_status_t dsp_st_block_forward(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w, const void* x,
                                  void* y, dsp_switch_impl_t impl, void* stream) {
  return block_forward(ctx, s, w, x, y, impl, stream, false, false);
}

// ------------------------------------------------------------------ Ulysses
// DeepSpeed-Ulysses on the same kernels ("AlltoAll for query, key, value, and output"):
// the activation stays T-sharded; every attention stage projects q, k, v locally, exchanges
// them sequence-sharded -> head-sharded (rank g receives the full sequence of head group g,
// channels [g*C/N, (g+1)*C/N) of each of q, k, v), attends over the full sequence with NH/N
// heads, and exchanges o back head-sharded -> sequence-sharded before the local out-projection.
// 4 all-to-alls per attention stage, 8 per block (Table 1: 8M/N) against DSP's 2.
struct UlyssesWs {
  int64_t act, h, qkv, qkvh, oh, o, send, recv, stats, parts, total;
};
static UlyssesWs ulysses_ws(const dsp_shape_t* s, int world) {
  UlyssesWs w{};
  const int64_t tok = s->B * s->T * s->S / world, C = s->C, e = elem_bytes(s->dtype);
  w.act = tok * C * e;
  w.h = 0;
  w.qkv = w.act;        // [tok, 3C] local projection (and, with qkvh, the MLP hidden [tok, 4C])
  w.qkvh = 4 * w.act;   // [B*T*S, 3C/N] head-sharded q | k | v of this rank's head group
  w.oh = 7 * w.act;     // [B*T*S, C/N] attention output of the head group
  w.o = 8 * w.act;      // [tok, C] attention output, sequence-sharded again
  w.send = 9 * w.act;   // NCCL staging
  w.recv = 10 * w.act;
  w.stats = align256(11 * w.act);
  w.parts = w.stats + align256(tok * 8);
  w.total = w.parts + align256(tok * (C / gemm_part_cols(C)) * 8) + 256;
  return w;
}

// q, k, v (columns [p*C, (p+1)*C) of qkv [B, T/N, S, 3C]) -> qkvh [B, T, S, 3C/N]: run (g, b, row)
// of C/N elements goes to rank g's qkvh row (b, rank*T/N*S + row), column p*C/N.  NCCL: one
// all-to-all per part (q, k, v: three, as DeepSpeed-Ulysses); P2P: the three parts in one put.
static dsp_status_t ulysses_exchange_qkv(dsp_ctx_t ctx, const dsp_shape_t* s, const uint8_t* qkv, uint8_t* qkvh,
                                  dsp_switch_impl_t impl, cudaStream_t st, void* send, void* recv) {
  const int N = ctx->world;
  const int64_t e = elem_bytes(s->dtype), C = s->C, Cn = C / N, Tn = s->T / N, S = s->S, T = s->T, B = s->B;
  const int parts = impl == DSP_SWITCH_P2P ? 3 : 1;
  RunCopy rc;
  rc.n[0] = N; rc.n[1] = B; rc.n[2] = Tn * S; rc.n[3] = parts;
  rc.run_bytes = Cn * e;
  rc.ss[0] = Cn * e; rc.ss[1] = Tn * S * 3 * C * e; rc.ss[2] = 3 * C * e; rc.ss[3] = C * e;
  rc.ds[0] = Tn * S * 3 * Cn * e; rc.ds[1] = T * S * 3 * Cn * e; rc.ds[2] = 3 * Cn * e; rc.ds[3] = Cn * e;
  const int64_t total = B * T * S * 3 * Cn * e;
  for (int p = 0; p < 3; p += parts)
    DSP_TRY(do_switch_plan(ctx, rc, ctx->rank * rc.ds[0], false, false, total - p * Cn * e, qkv + p * C * e,
                           qkvh + p * Cn * e, impl, st, send, recv));
  return DSP_OK;
}

// oh [B, T, S, C/N] (this rank's head group, every token) -> o [B, T/N, S, C] of the token's owner,
// columns [rank*C/N, (rank+1)*C/N): the fourth all-to-all.
static dsp_status_t ulysses_exchange_o(dsp_ctx_t ctx, const dsp_shape_t* s, const uint8_t* oh, uint8_t* o,
                                dsp_switch_impl_t impl, cudaStream_t st, void* send, void* recv) {
  const int N = ctx->world;
  const int64_t e = elem_bytes(s->dtype), C = s->C, Cn = C / N, Tn = s->T / N, S = s->S, T = s->T, B = s->B;
  RunCopy rc;
  rc.n[0] = N; rc.n[1] = B; rc.n[2] = Tn * S; rc.n[3] = 1;
  rc.run_bytes = Cn * e;
  rc.ss[0] = Tn * S * Cn * e; rc.ss[1] = T * S * Cn * e; rc.ss[2] = Cn * e;
  rc.ds[0] = Cn * e; rc.ds[1] = Tn * S * C * e; rc.ds[2] = C * e;
  return do_switch_plan(ctx, rc, ctx->rank * rc.ds[0], false, false, B * Tn * S * C * e, oh, o, impl, st, send, recv);
}

// One Ulysses attention stage on the T-sharded activation: out = res + MHA_dim(LN(res)).
// ln != nullptr: prepared weights (LN folded into the QKV GEMM); else h holds LN(res) already.
static dsp_status_t ulysses_attn_stage(dsp_ctx_t ctx, const dsp_shape_t* s, int dim, const void* a_in, const void* res,
                                void* out, const void* w_qkv, const void* w_o, const EpiVec* ln, float2* part_out,
                                uint8_t* ws, const UlyssesWs& L, dsp_switch_impl_t impl, cudaStream_t st, int stage0) {
  const int N = ctx->world;
  const int64_t C = s->C, Cn = C / N, tok = s->B * s->T * s->S / N;
  uint8_t *qkv = ws + L.qkv, *qkvh = ws + L.qkvh, *oh = ws + L.oh, *o = ws + L.o;
  std::string why;
  mark(ctx, stage0, 0, st);
  cudaError_t e = ln ? launch_gemm_bf16_ln(a_in, w_qkv, *ln, qkv, tok, 3 * C, C, false, ctx->num_sms, st, &why)
                     : launch_gemm_bf16(a_in, w_qkv, nullptr, qkv, tok, 3 * C, C, DSP_EPI_NONE, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "qkv projection", why);
  ctx->launches += 1;
  mark(ctx, stage0, 1, st);
  mark(ctx, stage0 + 1, 0, st);
  DSP_TRY(ulysses_exchange_qkv(ctx, s, qkv, qkvh, impl, st, ws + L.send, ws + L.recv));
  // the full sequence (all T frames, all S positions) of NH/N heads
  e = launch_fmha_bf16(qkvh, oh, s->B, s->T, s->S, Cn, s->num_heads / N, dim, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "attention core (head group)", why);
  ctx->launches += 1;
  DSP_TRY(ulysses_exchange_o(ctx, s, oh, o, impl, st, ws + L.send, ws + L.recv));
  mark(ctx, stage0 + 1, 1, st);
  mark(ctx, stage0 + 2, 0, st);
  e = part_out ? launch_gemm_bf16_res_stats(o, w_o, res, out, tok, C, C, part_out, ctx->num_sms, st, &why)
               : launch_gemm_bf16(o, w_o, res, out, tok, C, C, DSP_EPI_RESIDUAL, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "output projection", why);
  ctx->launches += 1;
  mark(ctx, stage0 + 2, 1, st);
  return DSP_OK;
}

size_t dsp_ulysses_workspace_bytes(const dsp_shape_t* s, int world) {
  if (!s || world < 1 || s->B < 1 || s->T < 1 || s->S < 1 || s->C < 1) return 0;
  return (size_t)ulysses_ws(s, world).total;
}

dsp_status_t dsp_st_block_forward_ulysses(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w,
                                                     const void* x, void* y, dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!w || !x || !y) return fail(ctx, DSP_ERR_NULL, "NULL argument");
  const int N = ctx->world;
  if (N == 1) return block_forward(ctx, s, w, x, y, impl, stream, false, false);  // no exchange at N = 1
  if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "the Ulysses schedule runs on the bf16 path");
  if (impl != DSP_SWITCH_NCCL && impl != DSP_SWITCH_P2P)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "Ulysses supports the NCCL and P2P transports");
  if (s->num_heads % N) return fail(ctx, DSP_ERR_UNSUPPORTED, "Ulysses needs N | num_heads (N=%d, heads=%d)", N, s->num_heads);
  if (((s->C / N) * 2) % 16) return fail(ctx, DSP_ERR_ALIGNMENT, "Ulysses needs C/N*2 %% 16 == 0");
  if (w->ln_c_w) return fail(ctx, DSP_ERR_UNSUPPORTED, "the Ulysses block has no cross stage");
  if (w->w_fc1_s || w->pe_t)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "the Ulysses block has no Latte pair / temporal positional embedding");
  const void* wp[12] = {w->ln1_w, w->ln1_b, w->w_qkv_s, w->w_o_s, w->ln2_w, w->ln2_b,
                        w->w_qkv_t, w->w_o_t, w->ln3_w, w->ln3_b, w->w_fc1, w->w_fc2};
  for (int i = 0; i < 12; ++i)
    if (!wp[i] || !aligned16(wp[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "weight %d NULL or not 16-B aligned", i);
  if (!aligned16(x) || !aligned16(y)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  DSP_TRY(check_bf16_attn(ctx, s, 128));  // the projections run at the full width C
  // the attention core runs on C/N channels (NH/N heads): only its head-dim limits apply
  // (C/N need not be a GEMM tile multiple: C = 1152 at N = 8 gives 144)
  const bool fold = w->prepared != nullptr;
  const int64_t C = s->C, tok = s->B * s->T * s->S / N, act = tok * C * 2;
  const UlyssesWs L = ulysses_ws(s, N);
  if (!ctx->ws || ctx->ws_bytes < (size_t)L.total) return fail(ctx, DSP_ERR_WORKSPACE, "Ulysses block needs %lld bytes of workspace", (long long)L.total);
  if (x != y && overlap(x, act, y, act)) return fail(ctx, DSP_ERR_ALIAS, "x_local partially overlaps y_local");
  if (overlap(ctx->ws, L.total, x, act) || overlap(ctx->ws, L.total, y, act)) return fail(ctx, DSP_ERR_ALIAS, "workspace overlaps x/y");
  if (impl == DSP_SWITCH_P2P) {
    if (!ctx->has_peers) return fail(ctx, DSP_ERR_STATE, "P2P Ulysses without dsp_ctx_set_peer_buffers");
    if (!in_region(ctx->ws, L.total, ctx->peer_base.p[ctx->rank], ctx->peer_bytes))
      return fail(ctx, DSP_ERR_UNSUPPORTED, "P2P Ulysses needs the workspace inside the symmetric buffer");
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = static_cast<uint8_t*>(ctx->ws);
  const float eps = w->ln_eps;
  const PrepLayout P = prep_layout(C);
  const uint8_t* prep = static_cast<const uint8_t*>(w->prepared);
  const float* uv = fold ? reinterpret_cast<const float*>(prep + P.uv) : nullptr;
  float2* stats = reinterpret_cast<float2*>(ws + L.stats);
  float2* parts = reinterpret_cast<float2*>(ws + L.parts);
  const int nparts = (int)(C / gemm_part_cols(C));
  EpiVec ev1{}, ev2{}, ev3{};
  if (fold) {  // R30: as the DSP block at N = 1 (the rows never move, so every partial stays local)
    ev1.row_stats = stats; ev1.col_u = uv; ev1.col_v = uv + 3 * C;
    ev2.col_u = uv + 6 * C; ev2.col_v = uv + 9 * C;
    ev3.col_u = uv + 12 * C; ev3.col_v = uv + 16 * C;
    for (EpiVec* ev : {&ev2, &ev3}) {
      ev->part_in = parts; ev->nparts_in = nparts; ev->part_cnt = (int)(C / nparts); ev->eps = eps;
    }
  }
  void* h = ws + L.h;
  mark(ctx, DSP_STAGE_LN1, 0, st);
  if (fold) DSP_CUDA(ctx, launch_row_stats(tok, C, x, eps, stats, st), "LN1 stats");
  else DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, x, w->ln1_w, w->ln1_b, eps, h, st), "LN1");
  ctx->launches += 1;
  mark(ctx, DSP_STAGE_LN1, 1, st);
  DSP_TRY(ulysses_attn_stage(ctx, s, DSP_DIM_S, fold ? x : h, x, y, fold ? prep + P.wf_s : w->w_qkv_s, w->w_o_s,
                             fold ? &ev1 : nullptr, fold ? parts : nullptr, ws, L, impl, st, DSP_STAGE_QKV_S));
  mark(ctx, DSP_STAGE_LN2, 0, st);
  if (!fold) {
    DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, y, w->ln2_w, w->ln2_b, eps, h, st), "LN2");
    ctx->launches += 1;
  }
  mark(ctx, DSP_STAGE_LN2, 1, st);
  DSP_TRY(ulysses_attn_stage(ctx, s, DSP_DIM_T, fold ? y : h, y, y, fold ? prep + P.wf_t : w->w_qkv_t, w->w_o_t,
                             fold ? &ev2 : nullptr, fold ? parts : nullptr, ws, L, impl, st, DSP_STAGE_QKV_T));
  mark(ctx, DSP_STAGE_LN3, 0, st);
  if (!fold) {
    DSP_CUDA(ctx, launch_layer_norm(s->dtype, tok, C, y, w->ln3_w, w->ln3_b, eps, h, st), "LN3");
    ctx->launches += 1;
  }
  mark(ctx, DSP_STAGE_LN3, 1, st);
  uint8_t* hid = ws + L.qkv;  // [tok, 4C] over qkv and the front of qkvh
  std::string why;
  mark(ctx, DSP_STAGE_FC1, 0, st);
  cudaError_t e = fold ? launch_gemm_bf16_ln(y, prep + P.wf_1, ev3, hid, tok, 4 * C, C, true, ctx->num_sms, st, &why)
                       : launch_gemm_bf16(h, w->w_fc1, nullptr, hid, tok, 4 * C, C, DSP_EPI_GELU, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "FC1", why);
  mark(ctx, DSP_STAGE_FC1, 1, st);
  mark(ctx, DSP_STAGE_FC2, 0, st);
  e = launch_gemm_bf16(hid, w->w_fc2, y, y, tok, C, 4 * C, DSP_EPI_RESIDUAL, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "FC2", why);
  mark(ctx, DSP_STAGE_FC2, 1, st);
  ctx->launches += 2;
  return DSP_OK;
}

dsp_status_t dsp_st_model_forward(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* const* w, int L,
                                  const void* x, void* y, dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (L < 1) return fail(ctx, DSP_ERR_SHAPE, "L = %d < 1", L);
  if (!w) return fail(ctx, DSP_ERR_NULL, "NULL weights array");
  for (int l = 0; l < L; ++l)
    if (!w[l]) return fail(ctx, DSP_ERR_NULL, "weights of layer %d are NULL", l);
  for (int l = 0; l < L; ++l) {
    // LN1 of block l + 1 from block l's FC2 partials when both sides are prepared (N == 1)
    const bool in = l > 0 && w[l - 1]->prepared && w[l]->prepared;
    const bool out = l + 1 < L && w[l]->prepared && w[l + 1]->prepared;
    DSP_TRY(block_forward(ctx, s, w[l], l == 0 ? x : y, y, impl, stream, in, out));
  }
  return DSP_OK;
}

size_t dsp_cross_workspace_bytes(const dsp_shape_t* s, int world, int64_t Lc) {
  if (!s || world < 1 || s->B < 1 || s->T < 1 || s->S < 1 || s->C < 1 || Lc < 1) return 0;
  const int64_t tok = s->B * s->T * s->S / world;
  return (size_t)((2 * tok + 2 * s->B * Lc) * s->C * elem_bytes(s->dtype) + 512);  // q | o | kv
}

dsp_status_t dsp_cross_attn(dsp_ctx_t ctx, const dsp_shape_t* s, const void* h, const void* ctx_tokens, int64_t Lc,
                            const void* w_q, const void* w_kv, const void* w_o, const void* residual, void* out,
                            void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!h || !ctx_tokens || !w_q || !w_kv || !w_o || !out) return fail(ctx, DSP_ERR_NULL, "NULL argument");
  if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "cross attention runs on the bf16 path");
  if (Lc < 1) return fail(ctx, DSP_ERR_SHAPE, "context length %lld < 1", (long long)Lc);
  const int64_t C = s->C, N = ctx->world, tok = s->B * s->T * s->S / N, Lq = tok / s->B;
  {
    const dsp_shape_t hs{1, 1, 1, C, s->num_heads, s->dtype};
    DSP_TRY(check_bf16_attn(ctx, &hs, 128));
  }
  const void* bufs[8] = {h, ctx_tokens, w_q, w_kv, w_o, residual, out, ctx->ws};
  for (int i = 0; i < 8; ++i)
    if (bufs[i] && !aligned16(bufs[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const size_t need = dsp_cross_workspace_bytes(s, (int)N, Lc);
  if (!ctx->ws || ctx->ws_bytes < need) return fail(ctx, DSP_ERR_WORKSPACE, "cross attention needs %zu bytes of workspace", need);
  const int64_t act = tok * C * 2;
  if (overlap(out, act, h, act)) return fail(ctx, DSP_ERR_ALIAS, "out overlaps h");
  uint8_t* ws = static_cast<uint8_t*>(ctx->ws);
  void* q = ws;
  void* o = ws + act;
  void* kv = ws + 2 * act;
  cudaStream_t st = (cudaStream_t)stream;
  std::string why;
  cudaError_t e = launch_gemm_bf16(h, w_q, nullptr, q, tok, C, C, DSP_EPI_NONE, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cross q projection", why);
  e = launch_gemm_bf16(ctx_tokens, w_kv, nullptr, kv, s->B * Lc, 2 * C, C, DSP_EPI_NONE, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cross kv projection", why);
  e = launch_fmha_cross_bf16(q, kv, o, s->B, Lq, Lc, C, s->num_heads, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cross attention core", why);
  e = launch_gemm_bf16(o, w_o, residual, out, tok, C, C, residual ? DSP_EPI_RESIDUAL : DSP_EPI_NONE, ctx->num_sms, st,
                       &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cross output projection", why);
  ctx->launches += 4;
  return DSP_OK;
}

size_t dsp_nd_workspace_bytes(const int64_t* dims, int ndim, dsp_dtype_t dtype, int world) {
  if (!dims || ndim < 3 || ndim > DSP_ND_MAX_DIMS || world < 1) return 0;
  int64_t tok = 1;
  for (int i = 0; i < ndim - 1; ++i) {
    if (dims[i] < 1) return 0;
    tok *= dims[i];
  }
  if (dims[ndim - 1] < 1) return 0;
  return (size_t)(6 * (tok / world) * dims[ndim - 1] * elem_bytes(dtype) + 256);  // h | qkv + o / hidden | ys
}

dsp_status_t dsp_nd_block_forward(dsp_ctx_t ctx, const int64_t* d, int nd, int num_heads, dsp_dtype_t dtype,
                                  int n_stages, const int* order, const dsp_attn_weights_t* attn,
                                  const dsp_mlp_weights_t* mlp, float eps, int shard_dim, const void* x, void* y,
                                  dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!d || !order || !attn || !mlp || !x || !y) return fail(ctx, DSP_ERR_NULL, "NULL argument");
  if (nd < 3 || nd > DSP_ND_MAX_DIMS) return fail(ctx, DSP_ERR_SHAPE, "ndim %d outside [3, %d]", nd, DSP_ND_MAX_DIMS);
  if (dtype != DSP_BF16 && dtype != DSP_F32) return fail(ctx, DSP_ERR_SHAPE, "unknown dtype");
  for (int i = 0; i < nd; ++i)
    if (d[i] < 1) return fail(ctx, DSP_ERR_SHAPE, "extent %d is %lld", i, (long long)d[i]);
  const int N = ctx->world;
  const int64_t C = d[nd - 1], e = elem_bytes(dtype);
  if (num_heads < 1 || C % num_heads) return fail(ctx, DSP_ERR_SHAPE, "C=%lld not divisible by num_heads=%d", (long long)C, num_heads);
  if (n_stages < 1 || n_stages > nd - 1) return fail(ctx, DSP_ERR_SHAPE, "n_stages %d outside [1, %d]", n_stages, nd - 1);
  if (shard_dim < 0 || shard_dim > nd - 2) return fail(ctx, DSP_ERR_BAD_DIM, "shard_dim %d outside [0, %d]", shard_dim, nd - 2);
  int alt = -1;  // the dim the activation is switched to before the stage along shard_dim
  for (int i = 0; i < n_stages; ++i) {
    if (order[i] < 0 || order[i] > nd - 2) return fail(ctx, DSP_ERR_BAD_DIM, "attention dim %d outside [0, %d]", order[i], nd - 2);
    for (int j = 0; j < i; ++j)
      if (order[j] == order[i]) return fail(ctx, DSP_ERR_BAD_DIM, "attention dim %d repeated", order[i]);
    if (order[i] == shard_dim) {
      if (i == 0) return fail(ctx, DSP_ERR_BAD_DIM, "the first attended dim cannot be the sharded one");
      alt = order[i - 1];
    }
  }
  if (d[shard_dim] % N || (alt >= 0 && d[alt] % N))
    return fail(ctx, DSP_ERR_DIVISIBILITY, "world %d does not divide the sharded dims", N);
  {
    const dsp_shape_t hs{1, 1, 1, C, num_heads, dtype};
    for (int i = 0; i < n_stages; ++i) DSP_TRY(check_bf16_attn(ctx, &hs, d[order[i]]));
  }
  const void* wp[4] = {mlp->ln_w, mlp->ln_b, mlp->w_fc1, mlp->w_fc2};
  for (int i = 0; i < 4; ++i)
    if (!wp[i] || !aligned16(wp[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "MLP weight %d NULL or not 16-B aligned", i);
  for (int i = 0; i < n_stages; ++i) {
    const void* a[4] = {attn[i].ln_w, attn[i].ln_b, attn[i].w_qkv, attn[i].w_o};
    for (int j = 0; j < 4; ++j)
      if (!a[j] || !aligned16(a[j])) return fail(ctx, DSP_ERR_ALIGNMENT, "stage %d weight %d NULL or not 16-B aligned", i, j);
  }
  if (!aligned16(x) || !aligned16(y)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  int64_t tok = 1;
  for (int i = 0; i < nd - 1; ++i) tok *= d[i];
  tok /= N;
  const int64_t act = tok * C * e;
  const size_t need = dsp_nd_workspace_bytes(d, nd, dtype, N);
  if (!ctx->ws || ctx->ws_bytes < need) return fail(ctx, DSP_ERR_WORKSPACE, "N-D block needs %zu bytes of workspace", need);
  if (x != y && overlap(x, act, y, act)) return fail(ctx, DSP_ERR_ALIAS, "x_local partially overlaps y_local");
  if (overlap(ctx->ws, need, x, act) || overlap(ctx->ws, need, y, act)) return fail(ctx, DSP_ERR_ALIAS, "workspace overlaps x/y");
  uint8_t* ws = static_cast<uint8_t*>(ctx->ws);
  void* h = ws;
  uint8_t* big = ws + act;          // qkv [tok, 3C] + o [tok, C] | MLP hidden [tok, 4C] | switch scratch
  void* qkv = big;
  void* o = big + 3 * act;
  void* ys = ws + 5 * act;          // the activation while it is sharded on `alt`
  if (N > 1 && impl == DSP_SWITCH_P2P) {
    if (!ctx->has_peers) return fail(ctx, DSP_ERR_STATE, "P2P block without dsp_ctx_set_peer_buffers");
    void* base = ctx->peer_base.p[ctx->rank];
    if (!in_region(ys, act, base, ctx->peer_bytes) || !in_region(y, act, base, ctx->peer_bytes))
      return fail(ctx, DSP_ERR_UNSUPPORTED, "P2P block needs the workspace and y_local inside the symmetric buffer");
  } else if (N > 1 && impl != DSP_SWITCH_NCCL) {
    return fail(ctx, DSP_ERR_UNSUPPORTED, "the N-D block supports the NCCL and P2P switch transports");
  }
  cudaStream_t st = (cudaStream_t)stream;
  auto nd_switch = [&](const void* src, void* dst, int from, int to) -> dsp_status_t {
    dsp_switch_nd_plan_t p;
    DSP_TRY(make_plan_nd(ctx, d, nd, (int)e, N, ctx->rank, from, to, &p));
    RunCopy rc;
    for (int i = 0; i < 4; ++i) { rc.n[i] = p.n[i]; rc.ss[i] = p.src_stride[i]; rc.ds[i] = p.dst_stride[i]; }
    rc.run_bytes = p.run_bytes;
    return do_switch_plan(ctx, rc, p.dst_peer_off, p.pack_is_identity, p.unpack_is_identity, act, src, dst, impl, st,
                          big, big + act);
  };
  int64_t ld[DSP_ND_MAX_DIMS];
  for (int i = 0; i < nd; ++i) ld[i] = d[i];
  int cur = shard_dim;
  ld[cur] /= N;
  const void* in = x;
  void* buf = nullptr;  // the buffer the activation lives in after the first stage (y or ys)
  for (int i = 0; i < n_stages; ++i) {
    const int k = order[i];
    if (k == cur && N > 1) {  // switch before the stage along the sharded dim
      DSP_TRY(nd_switch(in, ys, cur, alt));
      ld[cur] = d[cur];
      cur = alt;
      ld[cur] = d[cur] / N;
      in = ys;
      buf = ys;
    }
    int64_t before = 1, after = 1;
    for (int j = 0; j < k; ++j) before *= ld[j];
    for (int j = k + 1; j < nd - 1; ++j) after *= ld[j];
    const int64_t L = ld[k];
    void* out = buf ? buf : y;
    DSP_CUDA(ctx, launch_layer_norm(dtype, tok, C, in, attn[i].ln_w, attn[i].ln_b, eps, h, st), "N-D block LN");
    ctx->launches += 1;
    // attention along k: sequences of length L at a stride of `after` rows, `before` outer groups
    const dsp_shape_t s2{after == 1 ? 1 : before, 1, 1, C, num_heads, dtype};
    if (after == 1) DSP_TRY(attn_stage(ctx, &s2, before, L, DSP_DIM_S, h, attn[i].w_qkv, attn[i].w_o, in, out, qkv, o, st));
    else DSP_TRY(attn_stage(ctx, &s2, L, after, DSP_DIM_T, h, attn[i].w_qkv, attn[i].w_o, in, out, qkv, o, st));
    in = out;
    buf = out;
  }
  void* cur_buf = buf;  // n_stages >= 1, so the activation is in y or ys
  DSP_CUDA(ctx, launch_layer_norm(dtype, tok, C, cur_buf, mlp->ln_w, mlp->ln_b, eps, h, st), "N-D block LN (MLP)");
  ctx->launches += 1;
  DSP_TRY(linear(ctx, dtype, tok, 4 * C, C, h, mlp->w_fc1, nullptr, DSP_EPI_GELU, big, st));
  DSP_TRY(linear(ctx, dtype, tok, C, 4 * C, big, mlp->w_fc2, cur_buf, DSP_EPI_RESIDUAL, cur_buf, st));
  if (cur != shard_dim && N > 1) DSP_TRY(nd_switch(cur_buf, y, cur, shard_dim));
  return DSP_OK;
}

size_t dsp_block_prepared_bytes(const dsp_shape_t* s) {
  if (!s || s->C < 1 || s->dtype != DSP_BF16) return 0;
  return (size_t)prep_layout(s->C).total;
}

dsp_status_t dsp_adaln_fold(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w, const float* mod,
                            const dsp_block_weights_t* out, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  if (!w || !mod || !out) return fail(ctx, DSP_ERR_NULL, "NULL argument");
  if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "adaLN fold: bf16 weights only");
  if (s->B != 1) return fail(ctx, DSP_ERR_UNSUPPORTED, "adaLN fold is per sample: B must be 1 (B = %lld)", (long long)s->B);
  const int64_t C = s->C;
  const bool latte = w->w_fc1_s != nullptr;
  // sublayer k: (LN gamma, beta, output weight [C, K]) and where the modulated copies go (R36)
  const AdaFold jobs[4] = {
      {w->ln1_w, w->ln1_b, w->w_o_s, (void*)out->ln1_w, (void*)out->ln1_b, (void*)out->w_o_s, mod, C},
      {w->ln2_w, w->ln2_b, w->w_o_t, (void*)out->ln2_w, (void*)out->ln2_b, (void*)out->w_o_t, mod + 3 * C, C},
      {w->ln3_w, w->ln3_b, w->w_fc2, (void*)out->ln3_w, (void*)out->ln3_b, (void*)out->w_fc2, mod + 6 * C, 4 * C},
      {w->ln_m_w, w->ln_m_b, w->w_fc2_s, (void*)out->ln_m_w, (void*)out->ln_m_b, (void*)out->w_fc2_s, mod + 9 * C, 4 * C}};
  const int nj = latte ? 4 : 3;
  for (int j = 0; j < nj; ++j) {
    const void* ptr[6] = {jobs[j].gamma, jobs[j].beta, jobs[j].W, jobs[j].gamma_out, jobs[j].beta_out, jobs[j].W_out};
    for (int i = 0; i < 6; ++i)
      if (!ptr[i]) return fail(ctx, DSP_ERR_NULL, "adaLN fold: sublayer %d tensor %d is NULL", j, i);
  }
  DSP_CUDA(ctx, launch_adaln_fold(nj, jobs, C, (cudaStream_t)stream), "adaLN fold");
  ctx->launches += 1;
  return DSP_OK;
}

dsp_status_t dsp_st_block_prepare(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w, void* prep,
                                  size_t prep_bytes, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  if (!w || !prep) return fail(ctx, DSP_ERR_NULL, "NULL argument");
  if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "prepared weights exist for the bf16 path only");
  const int64_t C = s->C;
  if (C % 8 || C > 256 * kRowStatsMaxV || C / gemm_part_cols(C) > kMaxParts)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "prepared path needs C %% 8 == 0, C <= %d and C / BN <= %d (C=%lld)",
                256 * kRowStatsMaxV, kMaxParts, (long long)C);
  const PrepLayout P = prep_layout(C);
  if (prep_bytes < (size_t)P.total) return fail(ctx, DSP_ERR_WORKSPACE, "prepared buffer needs %lld bytes", (long long)P.total);
  if (reinterpret_cast<uintptr_t>(prep) % 256) return fail(ctx, DSP_ERR_ALIGNMENT, "prepared buffer must be 256-B aligned");
  const void* wp[9] = {w->ln1_w, w->ln1_b, w->w_qkv_s, w->ln2_w, w->ln2_b, w->w_qkv_t, w->ln3_w, w->ln3_b, w->w_fc1};
  for (int i = 0; i < 9; ++i)
    if (!wp[i]) return fail(ctx, DSP_ERR_NULL, "weight %d is NULL", i);
  uint8_t* p = static_cast<uint8_t*>(prep);
  float* uv = reinterpret_cast<float*>(p + P.uv);
  float* uvc = reinterpret_cast<float*>(p + P.uv_c);
  float* uv1s = reinterpret_cast<float*>(p + P.uv_1s);
  LnFold jobs[4] = {{w->w_qkv_s, w->ln1_w, w->ln1_b, p + P.wf_s, uv, uv + 3 * C, 3 * C},
                    {w->w_qkv_t, w->ln2_w, w->ln2_b, p + P.wf_t, uv + 6 * C, uv + 9 * C, 3 * C},
                    {w->w_fc1, w->ln3_w, w->ln3_b, p + P.wf_1, uv + 12 * C, uv + 16 * C, 4 * C},
                    {w->w_q_c, w->ln_c_w, w->ln_c_b, p + P.wf_c, uvc, uvc + C, C}};
  const bool cross = w->ln_c_w && w->ln_c_b && w->w_q_c;
  DSP_CUDA(ctx, launch_fold_ln_weights(cross ? 4 : 3, jobs, C, (cudaStream_t)stream), "fold LN weights");
  ctx->launches += 1;
  if (w->w_fc1_s) {  // Latte pair: LN_m folded into the spatial FC1 (R38)
    if (!w->ln_m_w || !w->ln_m_b) return fail(ctx, DSP_ERR_NULL, "Latte pair without ln_m_w / ln_m_b");
    const LnFold lj = {w->w_fc1_s, w->ln_m_w, w->ln_m_b, p + P.wf_1s, uv1s, uv1s + 4 * C, 4 * C};
    DSP_CUDA(ctx, launch_fold_ln_weights(1, &lj, C, (cudaStream_t)stream), "fold LN_m weights");
    ctx->launches += 1;
  }
  return DSP_OK;
}

dsp_status_t dsp_st_block_forward_host(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w,
                                       const void* xh, void* yh, void* xd, void* yd, dsp_switch_impl_t impl,
                                       void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!xh || !yh || !xd || !yd) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  const int64_t act = shard_bytes(s, ctx->world);
  cudaStream_t st = (cudaStream_t)stream;
  DSP_CUDA(ctx, cudaMemcpyAsync(xd, xh, act, cudaMemcpyHostToDevice, st), "H2D x");
  DSP_TRY(dsp_st_block_forward(ctx, s, w, xd, yd, impl, stream));
  DSP_CUDA(ctx, cudaMemcpyAsync(yh, yd, act, cudaMemcpyDeviceToHost, st), "D2H y");
  return DSP_OK;
}

dsp_status_t dsp_st_block_forward_host_pipelined(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w,
                                                 int n, const void* const* xh, void* const* yh, void* const* xd,
                                                 void* const* yd, dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (n < 0) return fail(ctx, DSP_ERR_SHAPE, "n = %d < 0", n);
  if (n == 0) return DSP_OK;
  if (!xh || !yh || !xd || !yd || !xd[0] || !xd[1] || !yd[0] || !yd[1]) return fail(ctx, DSP_ERR_NULL, "NULL buffer array");
  for (int i = 0; i < n; ++i)
    if (!xh[i] || !yh[i]) return fail(ctx, DSP_ERR_NULL, "NULL host buffer %d", i);
  const int64_t act = shard_bytes(s, ctx->world);
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      if (overlap(xd[a], act, yd[b], act)) return fail(ctx, DSP_ERR_ALIAS, "x_dev[%d] overlaps y_dev[%d]", a, b);
  if (overlap(xd[0], act, xd[1], act) || overlap(yd[0], act, yd[1], act))
    return fail(ctx, DSP_ERR_ALIAS, "the two staging buffers of a pair overlap");
  if (!ctx->h2d_stream) {
    cudaStream_t a, b;
    DSP_CUDA(ctx, cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "copy-in stream");
    ctx->h2d_stream = a;
    DSP_CUDA(ctx, cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking), "copy-out stream");
    ctx->d2h_stream = b;
    for (int k = 0; k < 2; ++k)
      for (void** e : {&ctx->ev_in[k], &ctx->ev_xfree[k], &ctx->ev_out[k], &ctx->ev_yfree[k]}) {
        cudaEvent_t ev;
        DSP_CUDA(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "pipeline event");
        *e = ev;
      }
  }
  cudaStream_t st = (cudaStream_t)stream, hs = (cudaStream_t)ctx->h2d_stream, ds = (cudaStream_t)ctx->d2h_stream;
  auto ev = [](void* e) { return (cudaEvent_t)e; };
  // the staging buffers may still be in use by work the caller enqueued earlier on `stream`
  DSP_CUDA(ctx, cudaEventRecord(ev(ctx->ev_xfree[0]), st), "pipeline start");
  DSP_CUDA(ctx, cudaStreamWaitEvent(hs, ev(ctx->ev_xfree[0]), 0), "pipeline start");
  DSP_CUDA(ctx, cudaStreamWaitEvent(ds, ev(ctx->ev_xfree[0]), 0), "pipeline start");
  for (int i = 0; i < n; ++i) {
    const int b = i & 1;
    if (i >= 2) DSP_CUDA(ctx, cudaStreamWaitEvent(hs, ev(ctx->ev_xfree[b]), 0), "wait x_dev free");
    DSP_CUDA(ctx, cudaMemcpyAsync(xd[b], xh[i], act, cudaMemcpyHostToDevice, hs), "H2D x");
    DSP_CUDA(ctx, cudaEventRecord(ev(ctx->ev_in[b]), hs), "x ready");
    DSP_CUDA(ctx, cudaStreamWaitEvent(st, ev(ctx->ev_in[b]), 0), "wait x ready");
    if (i >= 2) DSP_CUDA(ctx, cudaStreamWaitEvent(st, ev(ctx->ev_yfree[b]), 0), "wait y_dev free");
    DSP_TRY(dsp_st_block_forward(ctx, s, w, xd[b], yd[b], impl, stream));
    DSP_CUDA(ctx, cudaEventRecord(ev(ctx->ev_xfree[b]), st), "x consumed");
    DSP_CUDA(ctx, cudaEventRecord(ev(ctx->ev_out[b]), st), "y ready");
    DSP_CUDA(ctx, cudaStreamWaitEvent(ds, ev(ctx->ev_out[b]), 0), "wait y ready");
    DSP_CUDA(ctx, cudaMemcpyAsync(yh[i], yd[b], act, cudaMemcpyDeviceToHost, ds), "D2H y");
    DSP_CUDA(ctx, cudaEventRecord(ev(ctx->ev_yfree[b]), ds), "y copied");
  }
  // `stream` completes only after every result has reached the host
  DSP_CUDA(ctx, cudaStreamWaitEvent(st, ev(ctx->ev_yfree[(n - 1) & 1]), 0), "pipeline end");
  if (n >= 2) DSP_CUDA(ctx, cudaStreamWaitEvent(st, ev(ctx->ev_yfree[n & 1]), 0), "pipeline end");
  return DSP_OK;
}

dsp_status_t dsp_layer_norm(dsp_ctx_t ctx, dsp_dtype_t dt, int64_t rows, int64_t C, const void* x, const void* g,
                            const void* b, float eps, void* y, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!x || !g || !b || !y) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (rows < 0 || C < 1) return fail(ctx, DSP_ERR_SHAPE, "bad LN shape");
  if (dt != DSP_BF16 && dt != DSP_F32) return fail(ctx, DSP_ERR_SHAPE, "unknown dtype");
  if (dt == DSP_BF16 && (C * 2) % 16) return fail(ctx, DSP_ERR_ALIGNMENT, "bf16 LN needs C %% 8 == 0");
  DSP_CUDA(ctx, launch_layer_norm(dt, rows, C, x, g, b, eps, y, (cudaStream_t)stream), "layer_norm");
  if (rows > 0) ctx->launches += 1;
  return DSP_OK;
}

dsp_status_t dsp_linear(dsp_ctx_t ctx, dsp_dtype_t dt, int64_t M, int64_t N, int64_t K, const void* A, const void* W,
                        const void* R, dsp_epilogue_t epi, void* D, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!A || !W || !D || (epi == DSP_EPI_RESIDUAL && !R)) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (M < 0 || N < 1 || K < 1) return fail(ctx, DSP_ERR_SHAPE, "bad linear shape");
  if (epi != DSP_EPI_NONE && epi != DSP_EPI_RESIDUAL && epi != DSP_EPI_GELU) return fail(ctx, DSP_ERR_UNSUPPORTED, "unknown epilogue");
  if (dt != DSP_BF16 && dt != DSP_F32) return fail(ctx, DSP_ERR_SHAPE, "unknown dtype");
  const int64_t e = elem_bytes(dt);
  if (overlap(D, M * N * e, A, M * K * e) || overlap(D, M * N * e, W, N * K * e)) return fail(ctx, DSP_ERR_ALIAS, "D overlaps A or W");
  if (dt == DSP_BF16) {
    if (K % 8 || N % 32) return fail(ctx, DSP_ERR_UNSUPPORTED, "bf16 linear needs K %% 8 == 0 and N %% 32 == 0");
    if (!aligned16(A) || !aligned16(W) || !aligned16(D) || (R && !aligned16(R))) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  }
  return linear(ctx, dt, M, N, K, A, W, R, epi, D, (cudaStream_t)stream);
}

dsp_status_t dsp_attention_core(dsp_ctx_t ctx, dsp_dtype_t dt, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C,
                                int32_t NH, dsp_dim_t dim, const void* qkv, void* o, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_dim(ctx, dim));
  if (!qkv || !o) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  dsp_shape_t s{B, T_loc, S_loc, C, NH, dt};
  DSP_TRY(check_shape(ctx, &s));
  DSP_TRY(check_bf16_attn(ctx, &s, dim == DSP_DIM_S ? S_loc : T_loc));
  if (!aligned16(qkv) || !aligned16(o)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == DSP_BF16) {
    std::string why;
    cudaError_t e = launch_fmha_bf16(qkv, o, B, T_loc, S_loc, C, NH, dim, ctx->num_sms, st, &why);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "attention core", why);
  } else {
    DSP_CUDA(ctx, launch_attn_f32((const float*)qkv, (float*)o, B, T_loc, S_loc, C, NH, dim, st), "attention f32");
  }
  ctx->launches += 1;
  return DSP_OK;
}

}  // extern "C"

// ===================================================================== training path (f4)
// include/dsp_train.h.  Forward-train = the raw block forward keeping its activations; backward =
// the chain rule of oracle/backward.py in reverse stage order on the same shards, the switches run
// in the opposite direction (a permutation's adjoint is its inverse).
namespace {

struct TrainWs {
  int64_t dz, big, dh, dyb, dob, dqacc, dvec, lnpart, wpart, wt, send, recv, total;
};

int64_t wgrad_part_bytes(int64_t M, int64_t N, int64_t K, int num_sms) {
  return (int64_t)wgrad_splits(M, N, K, num_sms) * M * N * 4;
}

TrainWs train_ws(const dsp_shape_t* s, int world, int num_sms) {
  TrainWs w{};
  const int64_t tok = s->B * s->T * s->S / world, C = s->C, act = tok * C * 2;
  int64_t o = 0;
  auto take = [&](int64_t bytes) { const int64_t r = o; o += align256(bytes); return r; };
  w.dz = take(act);
  w.big = take(4 * act);
  w.dh = take(act);
  w.dyb = take(act);
  w.dob = take(act);
  w.dqacc = take(tok * C * 4);
  w.dvec = take(tok * s->num_heads * 4);
  w.lnpart = take(ln_bwd_scratch_bytes(tok, C));
  int64_t wp = 0;
  const int64_t shapes[4][2] = {{3 * C, C}, {C, C}, {4 * C, C}, {C, 4 * C}};
  for (auto& sh : shapes) wp = std::max(wp, wgrad_part_bytes(sh[0], sh[1], tok, num_sms));
  w.wpart = take(wp);
  w.wt = take(16 * C * C * 2);  // the six transposed weights (dgrad on the K-major GEMM path; WtOff)
  w.send = take(act);
  w.recv = take(act);
  w.total = o;
  return w;
}

dsp_train_saved_layout_t saved_layout(const dsp_shape_t* s, int world) {
  dsp_train_saved_layout_t L{};
  const int64_t tok = s->B * s->T * s->S / world, C = s->C, act = tok * C * 2, lse = tok * s->num_heads * 4;
  int64_t o = 0;
  auto take = [&](int64_t bytes) { const int64_t r = o; o += align256(bytes); return r; };
  L.h1 = take(act);
  L.qkv_s = take(3 * act);
  L.o_s = take(act);
  L.lse_s = take(lse);
  L.y1s = take(act);
  L.h2 = take(act);
  L.qkv_t = take(3 * act);
  L.o_t = take(act);
  L.lse_t = take(lse);
  L.y2 = take(act);
  L.h3 = take(act);
  L.u = take(4 * act);
  L.g = take(4 * act);
  L.total = o;
  return L;
}

dsp_status_t check_train_call(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_shape(ctx, s));
  DSP_TRY(check_div(ctx, s, ctx->world));
  if (!w) return fail(ctx, DSP_ERR_NULL, "weights NULL");
  if (s->dtype != DSP_BF16) return fail(ctx, DSP_ERR_UNSUPPORTED, "the training path is bf16");
  if (s->C % s->num_heads || s->C / s->num_heads != 72)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "the training path needs head dim 72 (C / num_heads)");
  const int64_t Tl = s->T, Sl = s->S;
  auto okL = [](int64_t L) { return L % 128 == 0 || 128 % L == 0; };
  if (!okL(Tl) || !okL(Sl)) return fail(ctx, DSP_ERR_UNSUPPORTED, "training path: T and S must divide or be multiples of 128");
  if (w->prepared || w->ln_c_w || w->w_fc1_s || w->pe_t)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "training path: raw weights only (no prepared / cross / Latte / pe extras)");
  const void* wp[12] = {w->ln1_w, w->ln1_b, w->w_qkv_s, w->w_o_s, w->ln2_w, w->ln2_b,
                        w->w_qkv_t, w->w_o_t, w->ln3_w, w->ln3_b, w->w_fc1, w->w_fc2};
  for (int i = 0; i < 12; ++i) {
    if (!wp[i]) return fail(ctx, DSP_ERR_NULL, "weight %d is NULL", i);
    if (!aligned16(wp[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "weight %d not 16-B aligned", i);
  }
  const size_t need = dsp_train_workspace_bytes(s, ctx->world);
  if (!ctx->ws || ctx->ws_bytes < need) return fail(ctx, DSP_ERR_WORKSPACE, "training needs %zu bytes of workspace", need);
  return DSP_OK;
}

dsp_status_t check_train_impl(dsp_ctx_t ctx, dsp_switch_impl_t impl) {
  if (impl != DSP_SWITCH_NCCL && impl != DSP_SWITCH_P2P)
    return fail(ctx, DSP_ERR_UNSUPPORTED, "training path: switch impl NCCL or P2P (the fused epilogues are forward-only)");
  return DSP_OK;
}

// dW[N, K] (+)= dY[M, N]^T X[M, K] through the split-K partials in `part`
dsp_status_t wgrad(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* dY, const void* X, float* dW,
                   int accumulate, float* part, cudaStream_t st) {
  std::string why;
  const int ks = wgrad_splits(N, K, M, ctx->num_sms);
  cudaError_t e = launch_gemm_bf16_wgrad(dY, X, part, N, K, M, ks, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "wgrad GEMM", why);
  e = launch_wgrad_reduce(part, ks, N * K, dW, accumulate, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "wgrad reduce");
  ctx->launches += 2;
  return DSP_OK;
}

// element offsets of the transposed weights in ws.wt (C^2 units): fc2, fc1, o_t, qkv_t, o_s, qkv_s
struct WtOff {
  static constexpr int64_t fc2 = 0, fc1 = 4, o_t = 8, qkv_t = 9, o_s = 12, qkv_s = 13;
};

// W^T [K, N] of W [N, K] (the dgrad's K-major operand)
dsp_status_t transpose_w(dsp_ctx_t ctx, const void* W, int64_t N, int64_t K, void* wt, cudaStream_t st) {
  cudaError_t e = launch_transpose_bf16(W, wt, N, K, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "weight transpose");
  ctx->launches += 1;
  return DSP_OK;
}

// dX = dY W: wt == nullptr reads W as an MN-major operand; else wt holds W^T for the forward's
// K-major GEMM, transposed here unless wt_ready (the block backward transposes them up front)
dsp_status_t dgrad(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* dY, const void* W, const void* u,
                   void* dX, cudaStream_t st, void* wt = nullptr, bool wt_ready = false) {
  std::string why;
  cudaError_t e;
  if (wt) {
    if (!wt_ready) DSP_TRY(transpose_w(ctx, W, N, K, wt, st));
    e = launch_gemm_bf16_dgrad_kmajor(dY, wt, u, dX, M, K, N, u ? EPI_GELU_BWD : DSP_EPI_NONE, ctx->num_sms, st, &why);
  } else {  // W read as an MN-major operand
    e = launch_gemm_bf16_dgrad(dY, W, u, dX, M, K, N, u ? EPI_GELU_BWD : DSP_EPI_NONE, ctx->num_sms, st, &why);
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "dgrad GEMM", why);
  ctx->launches += 1;
  return DSP_OK;
}

dsp_status_t ln_bwd(dsp_ctx_t ctx, int64_t rows, int64_t C, const void* x, const void* gamma, const void* dh,
                    const void* dres, void* dx, float* dgamma, float* dbeta, float* part, cudaStream_t st) {
  cudaError_t e = launch_ln_bwd(rows, C, x, gamma, dh, dres, dx, part, dgamma, dbeta, 1, 1e-5f, ctx->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "layer_norm backward");
  ctx->launches += 3;
  return DSP_OK;
}

// Weight-gradient GEMMs beside the dgrad chain: each wgrad is forked onto the context's side stream
// when its inputs are ready and joined back before the main stream overwrites what it reads (the
// side stream runs them in order, so waiting for wgrad k also covers every earlier one).
struct Side {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, done[7] = {};
};
dsp_status_t side_init(dsp_ctx_t ctx, Side* sd) {
  if (!ctx->wg_stream) {
    cudaStream_t s;
    DSP_CUDA(ctx, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "side stream");
    ctx->wg_stream = s;
    for (auto& e : ctx->wg_ev) {
      cudaEvent_t ev;
      DSP_CUDA(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "side events");
      e = ev;
    }
  }
  sd->s = (cudaStream_t)ctx->wg_stream;
  sd->fork = (cudaEvent_t)ctx->wg_ev[0];
  for (int i = 0; i < 7; ++i) sd->done[i] = (cudaEvent_t)ctx->wg_ev[i + 1];
  return DSP_OK;
}
// wgrad k on the side stream once the main stream (st) has produced its inputs
dsp_status_t side_wgrad(dsp_ctx_t ctx, const Side& sd, int k, int64_t M, int64_t N, int64_t K, const void* dY,
                        const void* X, float* dW, float* part, cudaStream_t st) {
  static const bool off = [] { const char* e = std::getenv("DSP_BWD_SIDE"); return e && e[0] == '0'; }();
  if (off) return wgrad(ctx, M, N, K, dY, X, dW, 1, part, st);  // A/B: everything on the caller's stream
  DSP_CUDA(ctx, cudaEventRecord(sd.fork, st), "fork");
  DSP_CUDA(ctx, cudaStreamWaitEvent(sd.s, sd.fork, 0), "fork wait");
  DSP_TRY(wgrad(ctx, M, N, K, dY, X, dW, 1, part, sd.s));
  DSP_CUDA(ctx, cudaEventRecord(sd.done[k], sd.s), "wgrad done");
  return DSP_OK;
}
dsp_status_t side_join(dsp_ctx_t ctx, const Side& sd, int k, cudaStream_t st) {
  static const bool off = [] { const char* e = std::getenv("DSP_BWD_SIDE"); return e && e[0] == '0'; }();
  if (off) return DSP_OK;
  DSP_CUDA(ctx, cudaStreamWaitEvent(st, sd.done[k], 0), "join");
  return DSP_OK;
}
// fn(stream) on the side stream after what st has issued so far, completion recorded as done[k]
template <class F>
dsp_status_t side_run(dsp_ctx_t ctx, const Side& sd, int k, cudaStream_t st, F&& fn) {
  static const bool off = [] { const char* e = std::getenv("DSP_BWD_SIDE"); return e && e[0] == '0'; }();
  if (off) return fn(st);
  DSP_CUDA(ctx, cudaEventRecord(sd.fork, st), "fork");
  DSP_CUDA(ctx, cudaStreamWaitEvent(sd.s, sd.fork, 0), "fork wait");
  DSP_TRY(fn(sd.s));
  DSP_CUDA(ctx, cudaEventRecord(sd.done[k], sd.s), "side done");
  return DSP_OK;
}

// one attention stage's backward: from dout (gradient of the stage output, also the residual
// gradient) and the saved h / qkv / o / lse, dres_out = dout + LN^T(W_qkv^T (attn^T (W_o^T dout))).
// Side-stream wgrads k_o (W_o) and k_o + 1 (W_qkv); join_big: the wgrad that last read ws.big.
dsp_status_t attn_stage_bwd(dsp_ctx_t ctx, const dsp_shape_t* s, int64_t T_loc, int64_t S_loc, int dim,
                            const void* zin, const void* ln_w, const void* w_qkv, const void* w_o, const void* h,
                            const void* qkv, const void* o, const float* lse, const void* dout, void* dres_out,
                            float* g_lnw, float* g_lnb, float* g_qkv, float* g_o, const TrainWs& L, uint8_t* ws,
                            cudaStream_t st, const Side& sd, int k_o, int join_big, void* wt_o, void* wt_qkv) {
  const int64_t tok = s->B * T_loc * S_loc, C = s->C;
  void* dob = ws + L.dob;
  void* dqkv = ws + L.big;
  void* dh = ws + L.dh;
  float* part = reinterpret_cast<float*>(ws + L.wpart);
  DSP_TRY(dgrad(ctx, tok, C, C, dout, w_o, nullptr, dob, st, wt_o, true));          // dO = dout W_o
  DSP_TRY(side_wgrad(ctx, sd, k_o, tok, C, C, dout, o, g_o, part, st));             // dW_o += dout^T O
  DSP_TRY(side_join(ctx, sd, join_big, st));                                        // ws.big free
  std::string why;
  cudaError_t e = launch_fmha_bwd_bf16(qkv, o, dob, lse, dqkv, reinterpret_cast<float*>(ws + L.dvec),
                                       reinterpret_cast<float*>(ws + L.dqacc), s->B, T_loc, S_loc, C, s->num_heads,
                                       dim, ctx->num_sms, st, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "attention backward", why);
  ctx->launches += 4;
  DSP_TRY(dgrad(ctx, tok, 3 * C, C, dqkv, w_qkv, nullptr, dh, st, wt_qkv, true));   // dh = dqkv W_qkv
  DSP_TRY(side_wgrad(ctx, sd, k_o + 1, tok, 3 * C, C, dqkv, h, g_qkv, part, st));   // dW_qkv += dqkv^T h
  if (dres_out == dout) DSP_TRY(side_join(ctx, sd, k_o, st));                       // in place over dout
  return ln_bwd(ctx, tok, C, zin, ln_w, dh, dout, dres_out, g_lnw, g_lnb, reinterpret_cast<float*>(ws + L.lnpart), st);
}

}  // namespace

extern "C" {

dsp_status_t dsp_train_saved_layout(const dsp_shape_t* s, int world, dsp_train_saved_layout_t* out) {
  if (!s || !out) return fail(nullptr, DSP_ERR_NULL, "NULL argument");
  if (world < 1 || s->B < 1 || s->T < 1 || s->S < 1 || s->C < 1 || s->num_heads < 1)
    return fail(nullptr, DSP_ERR_SHAPE, "bad shape or world");
  *out = saved_layout(s, world);
  return DSP_OK;
}

size_t dsp_train_workspace_bytes(const dsp_shape_t* s, int world) {
  if (!s || world < 1) return 0;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (size_t)train_ws(s, world, sms).total;
}

dsp_status_t dsp_st_block_forward_train(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w,
                                        const void* x, void* y, void* saved, dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_train_call(ctx, s, w));
  DSP_TRY(check_train_impl(ctx, impl));
  if (!x || !y || !saved) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (!aligned16(x) || !aligned16(y) || (reinterpret_cast<uintptr_t>(saved) & 255))
    return fail(ctx, DSP_ERR_ALIGNMENT, "x, y 16-B and saved 256-B aligned");
  const int N = ctx->world;
  const int64_t C = s->C, tok = s->B * s->T * s->S / N, act = tok * C * 2, Tn = s->T / N, Sn = s->S / N;
  const dsp_train_saved_layout_t SL = saved_layout(s, N);
  const TrainWs L = train_ws(s, N, ctx->num_sms);
  uint8_t* sv = static_cast<uint8_t*>(saved);
  uint8_t* ws = static_cast<uint8_t*>(ctx->ws);
  if (overlap(saved, SL.total, x, act) || overlap(saved, SL.total, y, act)) return fail(ctx, DSP_ERR_ALIAS, "saved overlaps x/y");
  if (overlap(ctx->ws, L.total, x, act) || overlap(ctx->ws, L.total, y, act) || overlap(ctx->ws, L.total, saved, SL.total))
    return fail(ctx, DSP_ERR_ALIAS, "workspace overlaps x/y/saved");
  cudaStream_t st = (cudaStream_t)stream;
  std::string why;
  cudaError_t e;
  auto run = [&](cudaError_t err, const char* what) -> dsp_status_t {
    if (err != cudaSuccess) return cuda_fail(ctx, err, what, why);
    ctx->launches += 1;
    return DSP_OK;
  };
  // spatial stage on the T-shard (y1 -> dz scratch when it must be switched)
  void* y1 = N == 1 ? static_cast<void*>(sv + SL.y1s) : static_cast<void*>(ws + L.dz);
  DSP_TRY(run(launch_layer_norm(DSP_BF16, tok, C, x, w->ln1_w, w->ln1_b, 1e-5f, sv + SL.h1, st), "LN1"));
  DSP_TRY(run(launch_gemm_bf16(sv + SL.h1, w->w_qkv_s, nullptr, sv + SL.qkv_s, tok, 3 * C, C, DSP_EPI_NONE, ctx->num_sms, st, &why), "QKV_S"));
  DSP_TRY(run(launch_fmha_bf16(sv + SL.qkv_s, sv + SL.o_s, s->B, Tn, s->S, C, s->num_heads, DSP_DIM_S, ctx->num_sms, st, &why,
                               reinterpret_cast<float*>(sv + SL.lse_s)), "ATTN_S"));
  DSP_TRY(run(launch_gemm_bf16(sv + SL.o_s, w->w_o_s, x, y1, tok, C, C, DSP_EPI_RESIDUAL, ctx->num_sms, st, &why), "PROJ_S"));
  if (N > 1) DSP_TRY(do_switch(ctx, s, DSP_DIM_T, y1, sv + SL.y1s, impl, st, ws + L.send, ws + L.recv));
  // temporal stage + MLP on the S-shard
  DSP_TRY(run(launch_layer_norm(DSP_BF16, tok, C, sv + SL.y1s, w->ln2_w, w->ln2_b, 1e-5f, sv + SL.h2, st), "LN2"));
  DSP_TRY(run(launch_gemm_bf16(sv + SL.h2, w->w_qkv_t, nullptr, sv + SL.qkv_t, tok, 3 * C, C, DSP_EPI_NONE, ctx->num_sms, st, &why), "QKV_T"));
  DSP_TRY(run(launch_fmha_bf16(sv + SL.qkv_t, sv + SL.o_t, s->B, s->T, Sn, C, s->num_heads, DSP_DIM_T, ctx->num_sms, st, &why,
                               reinterpret_cast<float*>(sv + SL.lse_t)), "ATTN_T"));
  DSP_TRY(run(launch_gemm_bf16(sv + SL.o_t, w->w_o_t, sv + SL.y1s, sv + SL.y2, tok, C, C, DSP_EPI_RESIDUAL, ctx->num_sms, st, &why), "PROJ_T"));
  DSP_TRY(run(launch_layer_norm(DSP_BF16, tok, C, sv + SL.y2, w->ln3_w, w->ln3_b, 1e-5f, sv + SL.h3, st), "LN3"));
  DSP_TRY(run(launch_gemm_bf16_gelu_aux(sv + SL.h3, w->w_fc1, sv + SL.g, sv + SL.u, tok, 4 * C, C, ctx->num_sms, st, &why), "FC1"));
  void* z = N == 1 ? y : static_cast<void*>(ws + L.dz);
  e = launch_gemm_bf16(sv + SL.g, w->w_fc2, sv + SL.y2, z, tok, C, 4 * C, DSP_EPI_RESIDUAL, ctx->num_sms, st, &why);
  DSP_TRY(run(e, "FC2"));
  if (N > 1) DSP_TRY(do_switch(ctx, s, DSP_DIM_S, z, y, impl, st, ws + L.send, ws + L.recv));
  return DSP_OK;
}

dsp_status_t dsp_st_block_backward(dsp_ctx_t ctx, const dsp_shape_t* s, const dsp_block_weights_t* w, const void* saved,
                                   const void* x, const void* dy, void* dx, const dsp_block_grads_t* g,
                                   dsp_switch_impl_t impl, void* stream) {
  DSP_TRY(check_train_call(ctx, s, w));
  DSP_TRY(check_train_impl(ctx, impl));
  if (!x || !dy || !dx || !saved || !g) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  float* gp[12] = {g->ln1_w, g->ln1_b, g->w_qkv_s, g->w_o_s, g->ln2_w, g->ln2_b,
                   g->w_qkv_t, g->w_o_t, g->ln3_w, g->ln3_b, g->w_fc1, g->w_fc2};
  for (int i = 0; i < 12; ++i)
    if (!gp[i] || !aligned16(gp[i])) return fail(ctx, DSP_ERR_ALIGNMENT, "gradient %d NULL or not 16-B aligned", i);
  if (!aligned16(x) || !aligned16(dy) || !aligned16(dx)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const int N = ctx->world;
  const int64_t C = s->C, tok = s->B * s->T * s->S / N, act = tok * C * 2, Tn = s->T / N, Sn = s->S / N;
  const dsp_train_saved_layout_t SL = saved_layout(s, N);
  const TrainWs L = train_ws(s, N, ctx->num_sms);
  if (dx != dy && overlap(dx, act, dy, act)) return fail(ctx, DSP_ERR_ALIAS, "dx partially overlaps dy");
  if (overlap(ctx->ws, L.total, dx, act) || overlap(ctx->ws, L.total, dy, act) || overlap(ctx->ws, L.total, x, act))
    return fail(ctx, DSP_ERR_ALIAS, "workspace overlaps x/dy/dx");
  if (overlap(saved, SL.total, dx, act)) return fail(ctx, DSP_ERR_ALIAS, "dx overlaps saved");
  if (overlap(ctx->ws, L.total, saved, SL.total)) return fail(ctx, DSP_ERR_ALIAS, "workspace overlaps saved");
  for (int i = 0; i < 12; ++i)
    if (overlap(ctx->ws, L.total, gp[i], 4)) return fail(ctx, DSP_ERR_ALIAS, "gradient %d inside the workspace", i);
  const uint8_t* sv = static_cast<const uint8_t*>(saved);
  uint8_t* ws = static_cast<uint8_t*>(ctx->ws);
  cudaStream_t st = (cudaStream_t)stream;
  float* part = reinterpret_cast<float*>(ws + L.wpart);
  struct NoPdl {  // the backward's kernels launch without programmatic dependent launch (dsp_internal.h)
    bool prev = t_no_pdl;
    NoPdl() {
      static const bool keep = [] { const char* e = std::getenv("DSP_BWD_PDL"); return e && e[0] == '1'; }();
      t_no_pdl = !keep;  // A/B: DSP_BWD_PDL=1 keeps PDL
    }
    ~NoPdl() { t_no_pdl = prev; }
  } no_pdl;
  // 1. dz = switch_{T->S}(dy): the adjoint of the forward's closing S->T switch
  const void* dz = dy;
  if (N > 1) {
    DSP_TRY(do_switch(ctx, s, DSP_DIM_T, dy, ws + L.dz, impl, st, ws + L.send, ws + L.recv));
    dz = ws + L.dz;
  }
  Side sd;
  DSP_TRY(side_init(ctx, &sd));
  // the dgrads' transposed weights: W2^T here, the other five on the side stream ahead of its wgrads
  // (event done[6]), so they run beside the first dgrad instead of in front of each
  const int64_t C2 = C * C;
  auto wt = [&](int64_t off) -> void* { return ws + L.wt + off * C2 * 2; };  // bf16, WtOff units
  DSP_TRY(transpose_w(ctx, w->w_fc2, C, 4 * C, wt(WtOff::fc2), st));
  DSP_TRY(side_run(ctx, sd, 6, st, [&](cudaStream_t ss) -> dsp_status_t {
    DSP_TRY(transpose_w(ctx, w->w_fc1, 4 * C, C, wt(WtOff::fc1), ss));
    DSP_TRY(transpose_w(ctx, w->w_o_t, C, C, wt(WtOff::o_t), ss));
    DSP_TRY(transpose_w(ctx, w->w_qkv_t, 3 * C, C, wt(WtOff::qkv_t), ss));
    DSP_TRY(transpose_w(ctx, w->w_o_s, C, C, wt(WtOff::o_s), ss));
    return transpose_w(ctx, w->w_qkv_s, 3 * C, C, wt(WtOff::qkv_s), ss);
  }));
  // 2. MLP backward: du = (dz W2) * gelu'(u); dW2 += dz^T g; dh3 = du W1; dW1 += du^T h3 (wgrads 0, 1 aside)
  void* du = ws + L.big;
  DSP_TRY(side_wgrad(ctx, sd, 0, tok, C, 4 * C, dz, sv + SL.g, g->w_fc2, part, st));
  DSP_TRY(dgrad(ctx, tok, C, 4 * C, dz, w->w_fc2, sv + SL.u, du, st, wt(WtOff::fc2), true));
  DSP_TRY(side_wgrad(ctx, sd, 1, tok, 4 * C, C, du, sv + SL.h3, g->w_fc1, part, st));
  DSP_TRY(side_join(ctx, sd, 6, st));  // the five transposes done
  DSP_TRY(dgrad(ctx, tok, 4 * C, C, du, w->w_fc1, nullptr, ws + L.dh, st, wt(WtOff::fc1), true));
  // dy2 = dz + LN3^T dh3
  void* dy2 = ws + L.dyb;
  DSP_TRY(ln_bwd(ctx, tok, C, sv + SL.y2, w->ln3_w, ws + L.dh, dz, dy2, g->ln3_w, g->ln3_b,
                 reinterpret_cast<float*>(ws + L.lnpart), st));
  // 3. temporal stage backward on the S-shard: dy1s = dy2 + LN2^T(...) (in place over dy2)
  DSP_TRY(attn_stage_bwd(ctx, s, s->T, Sn, DSP_DIM_T, sv + SL.y1s, w->ln2_w, w->w_qkv_t, w->w_o_t, sv + SL.h2,
                         sv + SL.qkv_t, sv + SL.o_t, reinterpret_cast<const float*>(sv + SL.lse_t), dy2, dy2,
                         g->ln2_w, g->ln2_b, g->w_qkv_t, g->w_o_t, L, ws, st, sd, 2, 1, wt(WtOff::o_t),
                         wt(WtOff::qkv_t)));
  // 4. dy1 = switch_{S->T}(dy1s): the adjoint of the forward's T->S switch
  void* dy1 = dy2;
  if (N > 1) {
    DSP_TRY(side_join(ctx, sd, 0, st));  // wgrad FC2 read dz
    DSP_TRY(do_switch(ctx, s, DSP_DIM_S, dy2, ws + L.dz, impl, st, ws + L.send, ws + L.recv));
    dy1 = ws + L.dz;
  }
  // 5. spatial stage backward on the T-shard: dx = dy1 + LN1^T(...)
  DSP_TRY(attn_stage_bwd(ctx, s, Tn, s->S, DSP_DIM_S, x, w->ln1_w, w->w_qkv_s, w->w_o_s, sv + SL.h1, sv + SL.qkv_s,
                         sv + SL.o_s, reinterpret_cast<const float*>(sv + SL.lse_s), dy1, dx, g->ln1_w, g->ln1_b,
                         g->w_qkv_s, g->w_o_s, L, ws, st, sd, 4, 3, wt(WtOff::o_s), wt(WtOff::qkv_s)));
  return side_join(ctx, sd, 5, st);  // every weight gradient done before the call returns (stream order)
}

dsp_status_t dsp_grads_reduce(dsp_ctx_t ctx, float* buf, int64_t n, int zero_shard, float* out, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!buf || (zero_shard && !out)) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  const int N = ctx->world;
  if (n < 0 || (zero_shard && n % N)) return fail(ctx, DSP_ERR_SHAPE, "n %% world != 0 for the ZeRO shard");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t shard = n / N;
  if (N == 1) {
    if (zero_shard && out != buf) DSP_CUDA(ctx, cudaMemcpyAsync(out, buf, n * 4, cudaMemcpyDeviceToDevice, st), "grads copy");
    return DSP_OK;
  }
  if (ctx->emulate_collectives) return fail(ctx, DSP_ERR_UNSUPPORTED, "gradient reduction under collective emulation");
  if (!ctx->nccl.ok || !ctx->comm) return fail(ctx, DSP_ERR_NCCL, "gradient reduction without a communicator");
  constexpr int kF32 = 7, kSum = 0;  // ncclFloat32, ncclSum
  int r;
  if (zero_shard) {
    if (!ctx->nccl.ReduceScatter) return fail(ctx, DSP_ERR_NCCL, "ncclReduceScatter unavailable");
    r = ctx->nccl.ReduceScatter(buf, out, (size_t)shard, kF32, kSum, ctx->comm, st);
  } else {
    if (!ctx->nccl.AllReduce) return fail(ctx, DSP_ERR_NCCL, "ncclAllReduce unavailable");
    r = ctx->nccl.AllReduce(buf, buf, (size_t)n, kF32, kSum, ctx->comm, st);
  }
  if (r) return fail(ctx, DSP_ERR_NCCL, "gradient reduction: %s", ctx->nccl.GetErrorString(r));
  return DSP_OK;
}

// ---- building blocks
dsp_status_t dsp_linear_dgrad(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* dY, const void* W,
                              const void* u, void* dX, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!dY || !W || !dX) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (M < 0 || N < 1 || K < 1) return fail(ctx, DSP_ERR_SHAPE, "bad dgrad shape");
  if (K % 128 || N % 8) return fail(ctx, DSP_ERR_UNSUPPORTED, "dgrad needs K %% 128 == 0 and N %% 8 == 0");
  if (!aligned16(dY) || !aligned16(W) || !aligned16(dX) || (u && !aligned16(u))) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  if (overlap(dX, M * K * 2, dY, M * N * 2) || overlap(dX, M * K * 2, W, N * K * 2)) return fail(ctx, DSP_ERR_ALIAS, "dX overlaps dY or W");
  return dgrad(ctx, M, N, K, dY, W, u, dX, (cudaStream_t)stream);
}

size_t dsp_wgrad_workspace_bytes(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K) {
  const int sms = ctx ? ctx->num_sms : 148;
  return (size_t)wgrad_part_bytes(N, K, M, sms);
}

dsp_status_t dsp_linear_wgrad(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* dY, const void* X, float* dW,
                              int accumulate, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!dY || !X || !dW) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (M < 1 || N < 1 || K < 1) return fail(ctx, DSP_ERR_SHAPE, "bad wgrad shape");
  if (N % 64 || K % 128) return fail(ctx, DSP_ERR_UNSUPPORTED, "wgrad needs N %% 64 == 0 and K %% 128 == 0");
  if (!aligned16(dY) || !aligned16(X) || !aligned16(dW)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const size_t need = dsp_wgrad_workspace_bytes(ctx, M, N, K);
  if (!ctx->ws || ctx->ws_bytes < need) return fail(ctx, DSP_ERR_WORKSPACE, "wgrad needs %zu bytes of workspace", need);
  if (overlap(ctx->ws, need, dW, N * K * 4)) return fail(ctx, DSP_ERR_ALIAS, "dW overlaps the workspace");
  return wgrad(ctx, M, N, K, dY, X, dW, accumulate, static_cast<float*>(ctx->ws), (cudaStream_t)stream);
}

dsp_status_t dsp_linear_gelu_aux(dsp_ctx_t ctx, int64_t M, int64_t N, int64_t K, const void* A, const void* W, void* G,
                                 void* U, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!A || !W || !G || !U) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (M < 0 || N < 1 || K < 1) return fail(ctx, DSP_ERR_SHAPE, "bad linear shape");
  if (K % 8 || N % 32) return fail(ctx, DSP_ERR_UNSUPPORTED, "needs K %% 8 == 0 and N %% 32 == 0");
  if (!aligned16(A) || !aligned16(W) || !aligned16(G) || !aligned16(U)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  std::string why;
  cudaError_t e = launch_gemm_bf16_gelu_aux(A, W, G, U, M, N, K, ctx->num_sms, (cudaStream_t)stream, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gelu aux GEMM", why);
  if (M > 0) ctx->launches += 1;
  return DSP_OK;
}

dsp_status_t dsp_layer_norm_bwd(dsp_ctx_t ctx, int64_t rows, int64_t C, const void* x, const void* gamma, const void* dh,
                                const void* dres, float eps, void* dx, float* dgb, void* stream) {
  DSP_TRY(check_ctx(ctx));
  if (!x || !gamma || !dh || !dx || !dgb) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  if (rows < 0 || C < 8 || C % 8 || C > 2048) return fail(ctx, DSP_ERR_UNSUPPORTED, "LN backward needs C %% 8 == 0, C <= 2048");
  const size_t need = (size_t)ln_bwd_scratch_bytes(rows, C);
  if (!ctx->ws || ctx->ws_bytes < need) return fail(ctx, DSP_ERR_WORKSPACE, "LN backward needs %zu bytes of workspace", need);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_ln_bwd(rows, C, x, gamma, dh, dres, dx, static_cast<float*>(ctx->ws), dgb, dgb + C, 1, eps,
                                ctx->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "layer_norm backward");
  ctx->launches += 3;
  return DSP_OK;
}

dsp_status_t dsp_attention_core_lse(dsp_ctx_t ctx, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C, int32_t NH,
                                    dsp_dim_t dim, const void* qkv, void* o, float* lse, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_dim(ctx, dim));
  if (!qkv || !o || !lse) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  dsp_shape_t s{B, T_loc, S_loc, C, NH, DSP_BF16};
  DSP_TRY(check_shape(ctx, &s));
  DSP_TRY(check_bf16_attn(ctx, &s, dim == DSP_DIM_S ? S_loc : T_loc));
  if (!aligned16(qkv) || !aligned16(o) || !aligned16(lse)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  std::string why;
  cudaError_t e = launch_fmha_bf16(qkv, o, B, T_loc, S_loc, C, NH, dim, ctx->num_sms, (cudaStream_t)stream, &why, lse);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "attention core", why);
  ctx->launches += 1;
  return DSP_OK;
}

size_t dsp_attention_bwd_workspace_bytes(int64_t tok, int64_t C, int32_t NH) {
  return (size_t)(align256(tok * NH * 4) + align256(tok * C * 4));
}

dsp_status_t dsp_attention_core_bwd(dsp_ctx_t ctx, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C, int32_t NH,
                                    dsp_dim_t dim, const void* qkv, const void* o, const void* dout, const float* lse,
                                    void* dqkv, void* stream) {
  DSP_TRY(check_ctx(ctx));
  DSP_TRY(check_dim(ctx, dim));
  if (!qkv || !o || !dout || !lse || !dqkv) return fail(ctx, DSP_ERR_NULL, "NULL buffer");
  dsp_shape_t s{B, T_loc, S_loc, C, NH, DSP_BF16};
  DSP_TRY(check_shape(ctx, &s));
  if (!aligned16(qkv) || !aligned16(o) || !aligned16(dout) || !aligned16(dqkv)) return fail(ctx, DSP_ERR_ALIGNMENT, "buffers must be 16-B aligned");
  const int64_t tok = B * T_loc * S_loc;
  const size_t need = dsp_attention_bwd_workspace_bytes(tok, C, NH);
  if (!ctx->ws || ctx->ws_bytes < need) return fail(ctx, DSP_ERR_WORKSPACE, "attention backward needs %zu bytes of workspace", need);
  uint8_t* ws = static_cast<uint8_t*>(ctx->ws);
  std::string why;
  cudaError_t e = launch_fmha_bwd_bf16(qkv, o, dout, lse, dqkv, reinterpret_cast<float*>(ws),
                                       reinterpret_cast<float*>(ws + align256(tok * NH * 4)), B, T_loc, S_loc, C, NH, dim,
                                       ctx->num_sms, (cudaStream_t)stream, &why);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "attention backward", why);
  ctx->launches += 4;
  return DSP_OK;
}

}  // extern "C"
