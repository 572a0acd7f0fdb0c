// dsp_internal.h — library-internal declarations (context, launchers, NCCL shim).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "dsp.h"
#include "dsp_kernels.h"
#include "dsp_train.h"

namespace dsp {

constexpr int kMaxPeers = 8;  // one NVLink/NVSwitch box
// signal pad slots (uint64) of the P2P barrier (switch.cu): [0, kMaxPeers) peer arrivals,
// kPadEpoch own barrier counter, kPadError first timeout record; DSP_SIGNAL_PAD_BYTES in dsp.h
constexpr int kPadEpoch = kMaxPeers, kPadError = kMaxPeers + 1;
// kPadCount: CTAs of a signalling kernel that have finished (the last one arrives for the rank)
constexpr int kPadCount = kMaxPeers + 2;

// ---- NCCL, resolved at run time from the libnccl.so.2 torch already loaded ----
struct NcclApi {
  bool ok = false;
  int (*AlltoAll)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*CommGetAsyncError)(void*, int*) = nullptr;
  // gradient reduction (dsp_grads_reduce): (send, recv, count, ncclFloat32, ncclSum, comm, stream)
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*ReduceScatter)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
};
bool nccl_load(NcclApi* api, std::string* err);
constexpr int kNcclUint8 = 1;  // ncclUint8 in nccl.h

struct PeerPtrs {
  void* p[kMaxPeers];
};

// strided byte-run copy: run (i0,i1,i2) of run_bytes from src + sum(i*ss) to dst + sum(i*ds)
// Strided run copy: runs (i0, i1, i2, i3) over extents n[], each run_bytes contiguous bytes at
// src + sum(i_k * ss[k]) -> dst + sum(i_k * ds[k]) (level 0 selects the peer in a P2P put).
struct RunCopy {
  int64_t n[4] = {1, 1, 1, 1};
  int64_t run_bytes = 0;
  int64_t ss[4] = {0, 0, 0, 0}, ds[4] = {0, 0, 0, 0};
};

// Stage clock of the launches the current thread issues next ([2] u64 in device memory, or NULL):
// block_forward points it at the stage's slot of dsp_ctx_set_stage_clocks' buffer, the
// launchers pass it to their kernels (clk_start / clk_end in sm100.cuh).
extern thread_local unsigned long long* t_clk;

// ---- launchers (return cudaGetLastError() after the launch) ----
cudaError_t launch_gemm_bf16(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N, int64_t K,
                             int epi, int num_sms, cudaStream_t st, std::string* why);
cudaError_t launch_fmha_bf16(const void* qkv, void* o, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C, int NH,
                             int dim, int num_sms, cudaStream_t st, std::string* why, float* lse = nullptr);
// FMHA backward (f4) over the same token-major q | k | v views: dqkv [tok, 3C] (bf16; padding-free)
// from qkv, o, do [tok, C], lse [tok][NH] (log2 domain, written by the forward with lse != nullptr);
// dvec [tok][NH] (f32) and dq_acc [tok, C] (f32, zeroed here when the sequence spans several key
// tiles) are scratch.  Dh == 72; sequence length L % 128 == 0 or 128 % L == 0.
cudaError_t launch_fmha_bwd_bf16(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                                 float* dvec, float* dq_acc, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C,
                                 int NH, int dim, int num_sms, cudaStream_t st, std::string* why);
// the backward's SIMT helpers (bwd.cu)
// out (+)= sum_s part[s] (n floats); out1 != nullptr: elements >= split_at go to out1 instead
cudaError_t launch_wgrad_reduce(const float* part, int nparts, int64_t n, float* out, int accumulate, cudaStream_t st,
                                int64_t split_at = 0, float* out1 = nullptr);
int ln_bwd_blocks(int64_t rows, int num_sms);
int64_t ln_bwd_scratch_bytes(int64_t rows, int64_t C);  // row statistics + column partials
// dx = dres + LN^T dh; dgamma (+)= sum dh xhat, dbeta (+)= sum dh (three launches: rows, column chunks, sum)
cudaError_t launch_ln_bwd(int64_t rows, int64_t C, const void* x, const void* gamma, const void* dh, const void* dres,
                          void* dx, float* scratch, float* dgamma, float* dbeta, int accumulate, float eps,
                          int num_sms, cudaStream_t st);
cudaError_t launch_attn_bwd_dvec(int64_t tok, int NH, int Dh, const void* o, const void* dout, float* dvec,
                                 cudaStream_t st);
cudaError_t launch_dq_convert(int64_t tok, int64_t C, const float* dq_acc, void* dqkv, cudaStream_t st);
// out [Cc, R] = in [R, Cc]^T (bf16; Cc % 8 == 0, R even)
cudaError_t launch_transpose_bf16(const void* in, void* out, int64_t R, int64_t Cc, cudaStream_t st);
// dgrad on pre-transposed weights: D[M, N] = epi(A[M, K] Wt[N, K]^T) -- the forward GEMM's K-major path
// (BN by gemm_bn_for, narrow tail tiles), epi = DSP_EPI_NONE or EPI_GELU_BWD (R = u [M, N])
cudaError_t launch_gemm_bf16_dgrad_kmajor(const void* A, const void* Wt, const void* R, void* D, int64_t M, int64_t N,
                                          int64_t K, int epi, int num_sms, cudaStream_t st, std::string* why);
// temporal attention reading q | k | v from the TSEQ layout (launch_gemm_bf16_tseq); o [tok, C]
cudaError_t launch_fmha_bf16_tseq(const void* qkv_tseq, void* o, int64_t B, int64_t T, int64_t S_loc, int64_t C,
                                  int NH, int num_sms, cudaStream_t st, std::string* why);
// cross-attention: queries q [B*Lq, C], context keys / values kv [B*Lc, 2C] ([k | v])
cudaError_t launch_fmha_cross_bf16(const void* q, const void* kv, void* o, int64_t B, int64_t Lq, int64_t Lc,
                                   int64_t C, int NH, int num_sms, cudaStream_t st, std::string* why);
cudaError_t launch_gemm_f32(const float* A, const float* W, const float* R, float* D, int64_t M, int64_t N, int64_t K,
                            int epi, cudaStream_t st);
cudaError_t launch_attn_f32(const float* qkv, float* o, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C, int NH,
                            int dim, cudaStream_t st);
cudaError_t launch_layer_norm(int dtype, int64_t rows, int64_t C, const void* x, const void* g, const void* b,
                              float eps, void* y, cudaStream_t st);
cudaError_t launch_run_copy(const void* src, void* dst, const RunCopy& rc, int num_sms, cudaStream_t st);
// P2P: run (i0=peer,i1,i2) stored to peer_base.p[i0] + dst_off + i1*ds[1] + i2*ds[2]
cudaError_t launch_p2p_put(const void* src, const PeerPtrs& peer_base, int64_t dst_off, const RunCopy& rc,
                           int num_sms, cudaStream_t st);
// pull: run (i0=peer,i1,i2,i3) read from peer_base.p[i0] + src_off + i1*ss[1] + ... into dst + sum(i*ds)
cudaError_t launch_p2p_pull(const PeerPtrs& peer_base, int64_t src_off, void* dst, const RunCopy& rc, int num_sms,
                            cudaStream_t st);
cudaError_t launch_p2p_barrier(const PeerPtrs& signals, int rank, int world, uint64_t timeout_ns, cudaStream_t st);

// LayerNorm folded into the following GEMM (bf16 path)
struct LnFold {
  const void* W;      // [N, K] bf16 weight of the linear layer
  const void* gamma;  // [K] bf16
  const void* beta;   // [K] bf16
  void* Wf;           // [N, K] bf16 out: W * gamma
  float* u;           // [N] out: row sums of Wf
  float* v;           // [N] out: W beta
  int64_t N;
};
cudaError_t launch_row_stats(int64_t rows, int64_t C, const void* x, float eps, void* stats, cudaStream_t st);
// per-row wait of a consumer of rows that arrived through a fused switch: mode 1 (after T->S):
// the S-sharded rows [B, T, S_loc], row (b, t, s) sent by rank t / Tn; mode 2 (after S->T): the
// T-sharded rows [B, Tn, S], row (b, t, s) sent by rank s / Sn.  Waits until that rank's arrival
// (slot [src] of this rank's pad) reaches this rank's current epoch.  pad == nullptr: no wait.
struct PeerWait {
  const uint64_t* pad;
  int mode, T, Tn, S_loc, S, Sn;
  uint64_t timeout_ns;
};
// per-row LayerNorm partials over `seg`-column segments, bitwise = the residual epilogue's (R30)
cudaError_t launch_row_partials(int64_t rows, int64_t C, int seg, const void* x, float2* parts, cudaStream_t st,
                                const PeerWait& pw = PeerWait{}, int num_sms = 148);
// R37: x [B, T, S_loc, C] += pe [T, C] (bf16, in place)
cudaError_t launch_add_temporal_pe(void* x, const void* pe, int64_t B, int64_t T, int64_t S_loc, int64_t C,
                                   cudaStream_t st);
// R36: one sublayer's adaLN-Zero fold: gamma_out = gamma (1 + scale), beta_out = beta (1 + scale) + shift,
// W_out = diag(gate) W (W [C, K]); mod = [3][C] f32 (shift, scale, gate)
struct AdaFold {
  const void *gamma, *beta, *W;
  void *gamma_out, *beta_out, *W_out;
  const float* mod;
  int64_t K;
};
cudaError_t launch_adaln_fold(int njobs, const AdaFold* jobs, int64_t C, cudaStream_t st);
cudaError_t launch_fold_ln_weights(int njobs, const LnFold* jobs, int64_t K, cudaStream_t st);
// GEMM epilogue codes beyond the public dsp_epilogue_t
enum { EPI_LN = 3, EPI_LN_GELU = 4, EPI_RES_REMOTE = 5, EPI_TSEQ = 6, EPI_LN_TSEQ = 7,
       // backward (f4): D = acc * gelu'(R) (R = the saved FC1 pre-activation u); D = gelu(acc) with
       // the raw acc also stored to R (forward-train FC1: u and g in one pass); fp32 partial store
       EPI_GELU_BWD = 8, EPI_GELU_AUX = 9, EPI_F32 = 10 };
// Operand majors of the backward GEMMs (bit 0: A is MN-major, stored [K][M]; bit 1: W is MN-major,
// stored [K][N]).  dgrad dX = dY W uses W [N_fwd, K_fwd] as an MN-major B; wgrad dW = dY^T X
// reads both token-major activations as MN-major operands (no transposes in HBM).
enum { MAJ_K = 0, MAJ_A_MN = 1, MAJ_B_MN = 2 };
// dgrad: D[M, N] = epi(A[M, K] . Wt) with W stored [K, N] (N contiguous); epi = DSP_EPI_NONE or
// EPI_GELU_BWD (R = u [M, N]); N % 128 == 0
cudaError_t launch_gemm_bf16_dgrad(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N,
                                   int64_t K, int epi, int num_sms, cudaStream_t st, std::string* why);
// wgrad: part[s][M, N] (fp32) = sum over the s-th token range of dY[tok, M]^T X[tok, N]; ksplit
// ranges (ksplit = wgrad_splits(...)); M % 64 == 0, N % 128 == 0
int wgrad_splits(int64_t M, int64_t N, int64_t K, int num_sms);
cudaError_t launch_gemm_bf16_wgrad(const void* dY, const void* X, float* part, int64_t M, int64_t N, int64_t K,
                                   int ksplit, int num_sms, cudaStream_t st, std::string* why);
// forward-train FC1: G = gelu(A W^T) and U = A W^T (both bf16 [M, N])
cudaError_t launch_gemm_bf16_gelu_aux(const void* A, const void* W, void* G, void* U, int64_t M, int64_t N,
                                      int64_t K, int num_sms, cudaStream_t st, std::string* why);
// Sequence-major temporal layout of q | k | v ("TSEQ", written by the temporal QKV GEMM, read by
// the temporal FMHA): element (part, b, h, s, t, d) at ((((part*B + b)*NH + h)*S_loc + s)*T + t)*kTseqDP
// + d, d < Dh = kTseqDh; columns Dh..DP-1 are zero.  Every temporal sequence (b, h, s) is one
// contiguous block of T rows (T = 128: 20 KB), so the FMHA's tiles are single contiguous reads
// instead of T token rows S_loc * 3C elements apart (T = 128, S_loc = 4096: a 3.6 GB span per tile,
// which bounds the token-major gathers at ~2.6 TB/s).  Used for T >= 64 (tseq_ok).
constexpr int kTseqDh = 72, kTseqDP = 80;
struct TseqShape {
  int B, T, S_loc, NH, C;
};
int64_t tseq_bytes(const TseqShape& t);  // 3 * B * NH * S_loc * T * DP * 2
// the shapes the TSEQ path supports: bf16, Dh == kTseqDh, S_loc % 128 == 0, 3C % 144 == 0
bool tseq_ok(int64_t B, int64_t T, int64_t S_loc, int64_t C, int NH);
cudaError_t launch_gemm_bf16_tseq(const void* A, const void* W, const struct EpiVec* ln, void* qkv_tseq,
                                  const TseqShape& ts, int64_t M, int64_t K, int num_sms, cudaStream_t st,
                                  std::string* why);
// Residual epilogue whose output rows go straight to their owner rank after a switch
// (switch fused into the GEMM): mode 1 = T->S (rows of [B,Tn,S] -> peers' [B,T,Sn]),
// mode 2 = S->T (rows of [B,T,Sn] -> peers' [B,Tn,S]).  Row bytes = C * 2.
struct RemoteMap {
  PeerPtrs base;
  int64_t dst_off;  // offset of the destination buffer inside every peer's symmetric buffer
  int mode, rank, B, T, S, Tn, Sn;
  // arrive != 0: the kernel's last CTA to finish arrives at the signal-pad barrier for this rank
  // (the first half of p2p_barrier_kernel: epoch + 1, release-stored into every peer's slot
  // [rank]) once every CTA's rows are stored -- the consumer then waits only for the peers whose
  // rows it reads (launch_row_partials with a PeerWait) instead of a barrier launch.
  PeerPtrs signals;
  int arrive, world;
};
cudaError_t launch_gemm_bf16_remote(const void* A, const void* W, const void* R, const RemoteMap& rm, int64_t M,
                                    int64_t N, int64_t K, int num_sms, cudaStream_t st, std::string* why);
// Epilogue vectors.  LN-folded GEMM (EPI_LN*): per-row statistics either as (mean, rstd) in
// row_stats, or (row_stats == nullptr) combined in the epilogue from part_in: nparts_in
// per-row partials (mean_p, M2_p) over part_cnt columns each, written by the residual
// epilogue of the GEMM that produced the rows (part_out, one partial per gemm_part_cols(N) columns).
struct EpiVec {
  const float2* row_stats;  // [M] (mean, rstd)
  const float* col_u;       // [N]
  const float* col_v;       // [N]
  const float2* part_in;    // [M, nparts_in] (mean_p, M2_p)
  int nparts_in, part_cnt;
  float eps;
  float2* part_out;         // residual epilogue: [M, N / gemm_part_cols(N)] partials of the stored (bf16) rows
  unsigned long long* clk;  // stage clock (set by run_gemm from t_clk)
  TseqShape tseq;           // EPI_*TSEQ: the temporal layout's shape
};
// BN (output-tile width) the GEMM dispatch picks for N output columns
int gemm_bn_for(int64_t N);
// columns per LayerNorm partial the residual epilogue writes (one per BN-wide tile: 192 at C = 1152)
int gemm_part_cols(int64_t N);
// most per-row LayerNorm partials an LN-folded epilogue combines
constexpr int kMaxParts = 24;
constexpr int kRowStatsMaxV = 12;  // row statistics kernel: C <= 256 * 12 = 3072
cudaError_t launch_gemm_bf16_res_stats(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N,
                                       int64_t K, float2* part_out, int num_sms, cudaStream_t st, std::string* why);
cudaError_t launch_gemm_bf16_ln(const void* A, const void* Wf, const EpiVec& ev, void* D, int64_t M, int64_t N,
                                int64_t K, bool gelu, int num_sms, cudaStream_t st, std::string* why);

// Launch with programmatic dependent launch (and optionally a cluster).  Every kernel
// launched this way calls griddep_wait() before touching dependent memory.  DSP_PDL=0
// disables the attribute (A/B experiments).
// launches of the current host thread made with PDL off (the block backward: its side-stream weight
// gradients and early-launched dependents compete for the SMs; measured 1.96 vs 2.05 ms, same box)
extern thread_local bool t_no_pdl;
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DSP_PDL");
    return !(e && e[0] == '0');
  }();
  return on && !t_no_pdl;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, unsigned cluster,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

bool make_tmap_bf16(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                    const uint32_t* box, CUtensorMapSwizzle swz, std::string* why);
// f32 tensor map (the FMHA backward's dQ reduce-add target)
bool make_tmap_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                   const uint32_t* box, std::string* why, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE);

}  // namespace dsp

struct dsp_ctx {
  int rank = 0, world = 1, device = 0, num_sms = 148;
  void* comm = nullptr;  // borrowed ncclComm_t
  dsp::NcclApi nccl;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  dsp::PeerPtrs peer_base{}, peer_signal{};
  bool has_peers = false;
  size_t peer_bytes = 0;
  int64_t launches = 0;            // own kernels launched (instrumentation)
  void* stage_events[2 * DSP_NUM_STAGES] = {};
  bool has_stage_events = false;
  unsigned long long* stage_clk = nullptr;  // [DSP_NUM_STAGES][2] device buffer (dsp_ctx_set_stage_clocks)
  void* tap[DSP_NUM_TAPS] = {};    // instrumentation: copies of intermediates (dsp_ctx_set_tap)
  size_t tap_bytes[DSP_NUM_TAPS] = {};
  uint64_t barrier_timeout_ns = 0;
  bool emulate_collectives = false;  // virtual ranks: NCCL all-to-all / all-gather emulated over peer mappings  // P2P barrier wall-clock timeout (0 = none); DSP_BARRIER_TIMEOUT_S
  // pipelined host path (dsp_st_block_forward_host_pipelined): copy-in / copy-out streams and
  // per-staging-buffer events, created on first use, destroyed with the context
  void* h2d_stream = nullptr;
  void* d2h_stream = nullptr;
  void* ev_in[2] = {};      // x_dev[b] filled (copy-in stream)
  void* ev_xfree[2] = {};   // x_dev[b] consumed by the block (compute stream)
  void* ev_out[2] = {};     // y_dev[b] written by the block (compute stream)
  void* ev_yfree[2] = {};   // y_dev[b] copied out (copy-out stream)
  // block backward: the weight-gradient GEMMs run on a side stream beside the dgrad chain
  void* wg_stream = nullptr;
  void* wg_ev[8] = {};       // [0] fork, [1..6] wgrad k done
  std::string last_error;
  ~dsp_ctx();
};
