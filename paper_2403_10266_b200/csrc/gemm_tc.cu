// gemm_tc.cu — persistent warp-specialised tcgen05 GEMM for sm_100a, CTA-pair (2-SM) MMA.
//
// D[M,N] = epi(A[M,K] * W[N,K]^T), bf16 in / fp32 accumulate in TMEM / bf16 out.
// Used for every dense contraction of the ST block:
// QKV projection (plain), out-projection (+residual), FC1 (+GELU), FC2 (+residual).
//
// Why CTA pairs: with single-CTA 128xBN tiles every operand byte crosses the SM's shared
// memory twice (TMA write + UMMA read), which caps the tensor pipe near 60% of peak on
// B200.  A cluster of 2 CTAs computes a 256xBN tile with tcgen05.mma.cta_group::2: each
// CTA stages its own 128 rows of A and HALF of the BN rows of W, so per-SM smem traffic
// per MMA drops by ~30% at BN=192/256.
//
// Roles (256 threads per CTA, grid = 2 x min(tiles, #SMs/2), static round-robin tiles):
//   warp 0      TMA producer (both CTAs): A rows [m0+128r, +128) and W rows
//               [n0 + r*BN/2, +BN/2) per 64-wide k-block into a STAGES-deep ring; the
//               bytes complete on the LEADER's full barrier.
//   warp 1      TMEM allocator (both CTAs, cta_group::2) and, in the leader only, the MMA
//               issuer: 4 x tcgen05.mma (M=256, N=BN, K=16) per k-block into one of two
//               TMEM accumulators; multicast commits free the smem stage in both CTAs and,
//               after the last k-block, signal both epilogues.
//   warps 4-7   epilogue (both CTAs): tcgen05.ld 32 columns at a time (thread = accumulator
//               row), fused residual / GELU, bf16 pack, 16-B global stores; then arrive on
//               the leader's accumulator-empty barrier.
// Tiles are rasterised n-fastest: concurrently running pairs share A row blocks and the
// (L2-resident, <= 21 MB) weight matrix, so A streams from HBM once even when it is larger
// than L2 (FC2: A = 151 MB at the single-block config).
// No split-K, no atomics: each output's reduction order depends only on K (N-invariance).
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "dsp_internal.h"
#include "sm100.cuh"

namespace dsp {

thread_local unsigned long long* t_clk = nullptr;
thread_local bool t_no_pdl = false;

namespace {

#ifndef DSP_GEMM_EPI_WG
// epilogue warpgroups of the LN-folded + GELU epilogue (FC1): its per-element work keeps one
// warpgroup behind the MMA (block FC1 135 -> 124 us with two); the lighter epilogues measured
// 2-3 % slower with two (A/B: -DDSP_GEMM_EPI_WG=1)
#define DSP_GEMM_EPI_WG 2
#endif
constexpr int BM = 128;  // rows per CTA (256 per pair)
constexpr int BK = 64;   // 64 bf16 = 128 B = one SW128 atom row

template <int BN, int EPI, int MAJ = MAJ_K>
struct GemmCfg {
  static constexpr bool A_MN = (MAJ & MAJ_A_MN) != 0;  // A staged as BM/64 MN-major SW128 boxes {64 rows, BK}
  static constexpr bool B_MN = (MAJ & MAJ_B_MN) != 0;  // W staged as BNH/64 MN-major boxes
  static_assert(!B_MN || (BN / 2) % 64 == 0, "an MN-major W half-tile is whole 64-column atoms");
  static constexpr bool AUX = EPI == EPI_GELU_BWD;      // R tile staged by TMA like the residual
  static constexpr bool F32 = EPI == EPI_F32;           // fp32 partials, per-thread-row stores
  static constexpr int BNH = BN / 2;                    // W rows staged per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BNH * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // store/residual box width (columns): SW128 at 64, SW64 at 32, SW32 at 16 (BN = 144)
  static constexpr int EB = BN % 64 == 0 ? 64 : BN % 32 == 0 ? 32 : 16;
  // epilogue staging: the residual epilogue stages the whole 128 x BN tile (the residual tile
  // lands there by TMA); the others use a ring of two boxes (store of box i overlaps box i+1),
  // which leaves room for one more mainloop stage at BN = 256
  static constexpr bool TSEQ = EPI == EPI_TSEQ || EPI == EPI_LN_TSEQ;  // temporal q|k|v layout, per-head boxes
  static constexpr bool RING = EPI != DSP_EPI_RESIDUAL && EPI != EPI_RES_REMOTE && !TSEQ && !AUX && !F32;
  static constexpr int E_BYTES = TSEQ ? (BN / kTseqDh) * 128 * kTseqDP * 2 : F32 ? 0 : RING ? 2 * 128 * EB * 2 : BN * 256;
  static constexpr int CW = BN % 32 == 0 ? 32 : 16;      // accumulator columns per TMEM load in the epilogue
  static constexpr int E_BOX = 128 * EB * 2;
  static constexpr int NBOX = BN / EB;  // staging boxes per tile (stored / reloaded one by one)
  // a narrow tail tile is a whole number of EB-column boxes (MN-major W: whole 64-column atoms,
  // not cut; fp32 partials: split-K instead)
  static constexpr int SPLIT_MAX = (B_MN || F32) ? 1 : NBOX;
  // epilogue warpgroups (TMA epilogues: two, each owning every other box; the remote-row
  // epilogue of the fused switch: one)
  static constexpr int EPI_WG = EPI == EPI_LN_GELU ? DSP_GEMM_EPI_WG : 1;
  static constexpr int THREADS = 128 + 128 * EPI_WG;
  static constexpr int STAGES = (216 * 1024 - E_BYTES) / STAGE_BYTES > 8 ? 8 : (216 * 1024 - E_BYTES) / STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int EPI_VEC_BYTES = 2 * 2 * BN * 4 + 2 * 128 * 8;  // per-accumulator u, v and row stats (LN-folded)
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE_BYTES + E_BYTES + 256 /*barriers*/ + EPI_VEC_BYTES;
};

__device__ __forceinline__ float gelu_tanh_f(float u) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * u * (1.f + fast_tanh(k0 * (u + k1 * u * u * u)));
}
// d/du gelu_tanh(u) = 0.5 (1 + t) + 0.5 u (1 - t^2) k0 (1 + 3 k1 u^2), t = tanh(k0 (u + k1 u^3))
__device__ __forceinline__ float gelu_tanh_grad_f(float u) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = fast_tanh(k0 * (u + k1 * u * u * u));
  return 0.5f * (1.f + t) + 0.5f * u * (1.f - t * t) * k0 * (1.f + 3.f * k1 * u * u);
}

// Static tile schedule over P pairs: `full` BN-wide tiles; when the last wave is partial (rem =
// full % P tiles) and its tiles cut into `split` narrower ones (split | BN/EB, so a narrow tile is
// whole epilogue boxes) fit in one wave (rem * split <= P), tiles [head, num_tiles) are those
// narrow tiles, split-major per parent tile.  head is a multiple of P, so every pair gets at most
// one narrow tile, as its last.
struct TileSched {
  int head, split, num_tiles;
};
// most narrow tiles one BN-wide tile may be cut into; 1 for a residual epilogue that writes
// LayerNorm partials (one partial per BN-wide tile, R30)
template <int BN, int EPI, int MAJ = MAJ_K>
__host__ __device__ inline int gemm_split_max(const EpiVec& ev) {
  return ((EPI == DSP_EPI_RESIDUAL && ev.part_out != nullptr) || GemmCfg<BN, EPI, MAJ>::TSEQ)
             ? 1
             : GemmCfg<BN, EPI, MAJ>::SPLIT_MAX;
}
__host__ __device__ inline TileSched make_tile_sched(int full, int P, int smax) {
  TileSched t{full, 1, full};
  const int rem = full % P;
#ifdef DSP_GEMM_NO_SPLIT
  return t;  // A/B experiments only
#endif
  if (rem == 0) return t;
  for (int sp = smax; sp > 1; --sp) {
    if (smax % sp || rem * sp > P) continue;
    t.split = sp;
    t.head = full - rem;
    t.num_tiles = t.head + rem * sp;
    break;
  }
  return t;
}

// LayerNorm statistics (mean, rstd) of row r from its producer's per-row partials (mean_p, M2_p)
// over part_cnt columns each (R30): Chan et al. combination of equal-count partials, in column
// order.  The row's partials are contiguous: loaded as 16-B vectors up to 24 partials.
template <int KV>
__device__ __forceinline__ float2 ln_combine(const EpiVec& ev, const float4 (&pv)[KV]) {
  const int np = ev.nparts_in;
  float mean = 0.f, m2 = 0.f;
#pragma unroll
  for (int i = 0; i < KV; ++i)
    if (2 * i < np) {
      mean += pv[i].x;
      mean += pv[i].z;
    }
  mean /= np;
#pragma unroll
  for (int i = 0; i < KV; ++i)
    if (2 * i < np) {
      const float d0 = pv[i].x - mean, d1 = pv[i].z - mean;
      m2 += pv[i].y + ev.part_cnt * d0 * d0;
      m2 += pv[i].w + ev.part_cnt * d1 * d1;
    }
  return make_float2(mean, rsqrtf(m2 / (float)(np * ev.part_cnt) + ev.eps));
}
__device__ __forceinline__ bool ln_parts_vec(const EpiVec& ev, int kv) {
  return (ev.nparts_in & 1) == 0 && ev.nparts_in <= 2 * kv && (reinterpret_cast<uintptr_t>(ev.part_in) & 15) == 0;
}
template <int KV>
__device__ __forceinline__ void ln_parts_load(const EpiVec& ev, int r, float4 (&pv)[KV]) {
  const float4* pp = reinterpret_cast<const float4*>(ev.part_in + (size_t)r * ev.nparts_in);
#pragma unroll
  for (int i = 0; i < KV; ++i)
    if (2 * i < ev.nparts_in) pv[i] = __ldg(pp + i);
}
// LayerNorm statistics (mean, rstd) of row r from its producer's per-row partials (mean_p, M2_p)
// over part_cnt columns each (R30): Chan et al. combination of equal-count partials, in column
// order.  The row's partials are contiguous: loaded as 16-B vectors up to 24 partials.
__device__ __forceinline__ float2 ln_stats_from_parts(const EpiVec& ev, int r) {
  constexpr int kVec = 12;
  if (ln_parts_vec(ev, kVec)) {
    float4 pv[kVec];
    ln_parts_load(ev, r, pv);
    return ln_combine(ev, pv);
  }
  const int np = ev.nparts_in;
  const float2* pp = ev.part_in + (size_t)r * np;
  float mean = 0.f, m2 = 0.f;
  for (int i = 0; i < np; ++i) mean += pp[i].x;
  mean /= np;
  for (int i = 0; i < np; ++i) {
    const float2 pv = pp[i];
    const float d = pv.x - mean;
    m2 += pv.y + ev.part_cnt * d * d;
  }
  return make_float2(mean, rsqrtf(m2 / (float)(np * ev.part_cnt) + ev.eps));
}

template <int BN, int EPI, int MAJ>
__global__ void __launch_bounds__(GemmCfg<BN, EPI, MAJ>::THREADS, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmD,
                        const __grid_constant__ CUtensorMap tmR,
                        const __nv_bfloat16* __restrict__ R, __nv_bfloat16* D, int M, int N, int K,
                        int ksplit, const EpiVec ev, const RemoteMap rm) {
  using Cfg = GemmCfg<BN, EPI, MAJ>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sE = smem + STAGES * Cfg::STAGE_BYTES;  // epilogue staging tile (residual in, output out)
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + Cfg::E_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* r_full = tempty + 2;  // [NBOX]: residual box b of the current tile landed
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(r_full + Cfg::NBOX);
  static_assert((2 * STAGES + 4 + Cfg::NBOX) * 8 + 4 <= 256, "barrier region");
  float* evec = reinterpret_cast<float*>(sE + Cfg::E_BYTES + 256);  // [2 acc][u | v][BN]

  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();  // 0 = leader of the CTA pair
  const bool leader = rank == 0;
  const int tiles_m = (M + 2 * BM - 1) / (2 * BM);
  // a ragged last column tile only for the f32 wgrad partials (zero-filled W columns, guarded stores)
  const int tiles_n = Cfg::F32 ? (N + BN - 1) / BN : N / BN;
  const int num_kb = (K + BK - 1) / BK;
  const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
  // Tile schedule (static round robin over the pairs): the last, partial wave of BN-wide tiles
  // is cut into `split` narrower tiles when they then fit in one wave (gemm_tail_split), so the
  // idle pairs of that wave share its work.  Every output element is still one tile's K-ordered
  // accumulation: the bits do not depend on the tile width (N-invariance).
  // split-K (fp32 partials, ksplit > 1): tile t computes output tile t % (tiles_m * tiles_n) over
  // the k-blocks of range t / (tiles_m * tiles_n); concurrently running pairs share a token range
  const int tmn = tiles_m * tiles_n;
  const int kbs = (num_kb + ksplit - 1) / ksplit;
  const TileSched ts = make_tile_sched(tmn * ksplit, num_pairs, gemm_split_max<BN, EPI, MAJ>(ev));
  const int num_tiles = ts.num_tiles;
  auto geom = [&](int t, int& mrow, int& ncol, int& width) {
    int p = t, sub = 0;
    width = BN;
    if (t >= ts.head) {
      p = ts.head + (t - ts.head) / ts.split;
      sub = (t - ts.head) % ts.split;
      width = BN / ts.split;
    }
    p %= tmn;
    mrow = (p / tiles_n) * (2 * BM);
    ncol = (p % tiles_n) * BN + sub * width;
  };
  auto krange = [&](int t, int& kb0, int& kb1) {
    kb0 = ksplit > 1 ? (t / tmn) * kbs : 0;  // ksplit > 1 never has narrow tiles (SPLIT_MAX 1)
    kb1 = kb0 + kbs < num_kb ? kb0 + kbs : num_kb;
  };

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmW);
    tma_prefetch(&tmD);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * 128 * Cfg::EPI_WG);  // both CTAs' epilogue threads
    }
    for (int b = 0; b < Cfg::NBOX; ++b) mbar_init(&r_full[b], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc_2sm(tmem_holder, Cfg::TMEM_COLS);
    tmem_relinquish_2sm();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  griddep_launch_dependents();
  griddep_wait();
  clk_start(ev.clk);

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < num_tiles; tile += num_pairs) {
        int mrow, ncol, width;
        geom(tile, mrow, ncol, width);
        const int m0 = mrow + rank * BM;
        const int n0 = ncol + rank * (width / 2);
        const bool narrow = width != BN;
        const uint32_t bytes = 2 * (Cfg::A_BYTES + (width / 2) * BK * 2);
        int kb0, kb1;
        krange(tile, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
          if (Cfg::A_MN) {  // A stored [K][M]: BM/64 boxes {64 rows of M, BK k-rows}, 8 KB apart
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d_2sm(sA + stage * Cfg::A_BYTES + j * (BK * 128), &tmA, &full[stage], m0 + 64 * j, kb * BK);
          } else {
            tma_load_2d_2sm(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * BK, m0);
          }
          if (Cfg::B_MN) {
#pragma unroll
            for (int j = 0; j < Cfg::BNH / 64; ++j)
              tma_load_2d_2sm(sB + stage * Cfg::B_BYTES + j * (BK * 128), &tmW, &full[stage], n0 + 64 * j, kb * BK);
          } else {
            tma_load_2d_2sm(sB + stage * Cfg::B_BYTES, narrow ? &tmW2 : &tmW, &full[stage], kb * BK, n0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc_full = make_idesc_bf16(2 * BM, BN, Cfg::A_MN, Cfg::B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = pair; tile < num_tiles; tile += num_pairs, ++it) {
        const int acc = it & 1;
        const uint32_t idesc = tile < ts.head ? idesc_full : make_idesc_bf16(2 * BM, BN / ts.split, 0, 0);
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        int kb0, kb1;
        krange(tile, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
            const uint32_t b0 = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // K-major: the k-th 16-column slice is 32 B into each 128-B row; MN-major: 16 k-rows
              // (2 KB) down, 64-element MN groups BK * 128 B apart (LBO), 8-row groups 1 KB (SBO)
              const uint64_t ad = Cfg::A_MN ? make_sdesc(a0 + k * 2048, BK * 128, 1024, SW_128B)
                                            : make_sdesc(a0 + k * 32, 16, 1024, SW_128B);
              const uint64_t bd = Cfg::B_MN ? make_sdesc(b0 + k * 2048, BK * 128, 1024, SW_128B)
                                            : make_sdesc(b0 + k * 32, 16, 1024, SW_128B);
              umma_bf16_ss_2sm(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0));
            }
            umma_commit_2sm_mc(&empty[stage], 0x3);
            if (kb == kb1 - 1) umma_commit_2sm_mc(&tfull[acc], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4 && Cfg::TSEQ) {
   if constexpr (Cfg::TSEQ) {
    // Temporal-layout epilogue (EPI_TSEQ / EPI_LN_TSEQ): the tile's BN = HPT * Dh columns are
    // HPT whole heads of q, k or v; each head's 128 x Dh block is staged in sE as 128 rows of DP
    // elements (columns Dh..DP-1 zero, so every stored row is whole 32-B sectors) and stored by
    // one 5-D TMA box {DP, 1 (t), 128 (s), 1 (h), 1 (part*B + b)}: the CTA's 128 rows are 128
    // consecutive columns s of one (b, t) (S_loc % 128 == 0), T * DP elements apart in the layout
    // (dsp_internal.h TseqShape).  All BN accumulator columns are read from TMEM before one wait.
    constexpr bool kLn = EPI == EPI_LN_TSEQ;
    constexpr int HD = kTseqDh, HPT = BN / HD;
    static_assert(BN % HD == 0 && Cfg::CW == 16, "TSEQ tiles are whole heads, read 16 columns at a time");
    const int q = warp & 3;
    const int row = q * 32 + lane_id();
    const bool elected = threadIdx.x == 128;
    const uint32_t e0 = smem_u32(sE);
    const TseqShape tq = ev.tseq;
    constexpr int ROWB = kTseqDP * 2;  // staged row pitch (bytes)
#pragma unroll
    for (int hh = 0; hh < HPT; ++hh)  // the padding columns Dh..DP-1 of every staged row: zero, once
      for (int c = HD * 2; c < ROWB; c += 16) st_shared_v4(e0 + hh * (128 * ROWB) + row * ROWB + c, 0u, 0u, 0u, 0u);
    int it = 0;
    for (int tile = pair; tile < num_tiles; tile += num_pairs, ++it) {
      const int acc = it & 1;
      int m0, n0, width;
      geom(tile, m0, n0, width);
      m0 += rank * BM;
      float2 rstat = make_float2(0.f, 0.f);
      float* eu = evec + acc * 2 * BN;
      if (kLn) {
        if (m0 + row < M) rstat = ev.row_stats ? ev.row_stats[m0 + row] : ln_stats_from_parts(ev, m0 + row);
        for (int i = threadIdx.x - 128; i < BN; i += 128) {
          st_shared_f32(smem_u32(eu + i), ev.col_u[n0 + i]);
          st_shared_f32(smem_u32(eu + BN + i), ev.col_v[n0 + i]);
        }
      }
      if (elected) bulk_wait_group_read0();  // the previous tile's head boxes have left sE
      named_bar_sync(1, 128);               // (and u, v staged)
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      uint32_t va[BN];
#pragma unroll
      for (int c = 0; c < BN / 16; ++c)
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c * 16, *reinterpret_cast<uint32_t(*)[16]>(va + 16 * c));
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < BN / 16; ++c) {
        const uint32_t* v = va + 16 * c;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int col = c * 16 + g * 8, hh = col / HD, d = col - hh * HD;
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(v[8 * g + i]);
          if (kLn) {
            const float2 nm = make_float2(-rstat.x, -rstat.x), rs = make_float2(rstat.y, rstat.y);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const float4 uu = ld_shared_f32x4(smem_u32(eu + col + 4 * hf)),
                           vv = ld_shared_f32x4(smem_u32(eu + BN + col + 4 * hf));
              const float2 y0 = ffma2(rs, ffma2(nm, make_float2(uu.x, uu.y), make_float2(f[4 * hf], f[4 * hf + 1])),
                                      make_float2(vv.x, vv.y));
              const float2 y1 = ffma2(rs, ffma2(nm, make_float2(uu.z, uu.w), make_float2(f[4 * hf + 2], f[4 * hf + 3])),
                                      make_float2(vv.z, vv.w));
              f[4 * hf] = y0.x; f[4 * hf + 1] = y0.y; f[4 * hf + 2] = y1.x; f[4 * hf + 3] = y1.y;
            }
          }
          st_shared_v4(e0 + hh * (128 * ROWB) + row * ROWB + d * 2, pack_bf16x2(f[0], f[1]),
                       pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (elected) {
        const int ts_rows = tq.T * tq.S_loc;
        const int b = m0 / ts_rows, t = (m0 / tq.S_loc) % tq.T, s0 = m0 % tq.S_loc;
#pragma unroll
        for (int hh = 0; hh < HPT; ++hh) {
          const int gcol = n0 + hh * HD, part = gcol / tq.C, h = (gcol % tq.C) / HD;
          tma_store_5d(&tmD, sE + hh * (128 * ROWB), 0, t, s0, h, part * tq.B + b);
        }
        bulk_commit_group();
      }
      tc_fence_before();
      if (leader) mbar_arrive(&tempty[acc]);
      else mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
    }
    if (elected) bulk_wait_group_read0();
   }
  } else if (warp >= 4 && EPI != EPI_RES_REMOTE && !Cfg::F32) {
    // Bulk-tensor epilogue, EPI_WG warpgroups: warpgroup h (warps 4+4h .. 7+4h, TMEM lane quadrant
    // = warp % 4, thread = accumulator row) owns the tile's EB-column boxes b with b % EPI_WG == h.
    // Each thread adds its accumulator row into its box in place (SW128 layout: 16-B chunk c of
    // row r at c ^ (r & 7)); as soon as the warpgroup has finished a box, one of its threads
    // TMA-stores it (rows >= M are clipped).  Residual epilogue: box b's slot first receives the
    // residual box by TMA (issued while the previous tile's epilogue ran: once that tile's store of
    // the warpgroup's previous box has been read out of sE, the next tile's copy of that box is
    // loaded).  Other epilogues stage through one slot per warpgroup.  A LayerNorm partial is one
    // box of one row, so the partials' arithmetic does not depend on the warpgroup split.
    constexpr bool kRes = EPI == DSP_EPI_RESIDUAL;
    constexpr bool kStage = kRes || Cfg::AUX;   // an R tile (residual, or u for gelu') staged by TMA
    constexpr bool kDual = EPI == EPI_GELU_AUX;  // two stores per box: gelu(acc) -> D, acc -> R
    constexpr bool kLn = EPI == EPI_LN || EPI == EPI_LN_GELU;
    constexpr int WG = Cfg::EPI_WG;
    static_assert(!kDual || WG == 1, "the dual-store epilogue uses both ring slots per box");
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const int row = q * 32 + lane_id();
    const int etid = threadIdx.x - 128;
    const bool elected = (etid & 127) == 0;
    const uint32_t bar_wg = 2 + h;
    const uint32_t e0 = smem_u32(sE);
    int it = 0, nbox_done = 0;
    auto nbox_of = [&](int tile) { return tile < ts.head ? Cfg::NBOX : Cfg::NBOX / ts.split; };
    auto load_res_box = [&](int tile, int b) {
      if (b >= nbox_of(tile)) return;  // a narrow tail tile has fewer boxes
      int mrow, ncol, width;
      geom(tile, mrow, ncol, width);
      mbar_arrive_expect_tx(&r_full[b], Cfg::E_BOX);
      tma_load_2d(sE + b * Cfg::E_BOX, &tmR, &r_full[b], ncol + Cfg::EB * b, mrow + rank * BM);
    };
    if (kStage && elected && pair < num_tiles)
      for (int b = h; b < Cfg::NBOX; b += WG) load_res_box(pair, b);
    // LayerNorm folded (kLn): the next tile's row statistics (or its rows' partials, up to 8) are
    // loaded while this tile is processed, so their L2 latency is off the epilogue's critical path
    constexpr int kPF = 4;
    const bool pf_parts = kLn && !ev.row_stats && ln_parts_vec(ev, kPF);
    float4 pfv[kPF];
    float2 pfrs = make_float2(0.f, 0.f);
    auto prefetch = [&](int t) {
      int mr, nc, wd;
      geom(t, mr, nc, wd);
      const int r = mr + rank * BM + row;
      if (r >= M) return;
      if (ev.row_stats) pfrs = ev.row_stats[r];
      else if (pf_parts) ln_parts_load(ev, r, pfv);
    };
    if (kLn && h == 0 && pair < num_tiles) prefetch(pair);
    // ... and so are the next tile's per-column u, v (at most two columns per thread: BN <= 256)
    float pu[2] = {0.f, 0.f}, pvv[2] = {0.f, 0.f};
    auto prefetch_uv = [&](int t) {
      int mr, nc, wd;
      geom(t, mr, nc, wd);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = etid + k * 128 * WG;
        if (i < wd) {
          pu[k] = ev.col_u[nc + i];
          pvv[k] = ev.col_v[nc + i];
        }
      }
    };
    static_assert(!kLn || BN <= 2 * 128, "u, v prefetch covers two columns per epilogue thread");
    if (kLn && pair < num_tiles) prefetch_uv(pair);
    for (int tile = pair; tile < num_tiles; tile += num_pairs, ++it) {
      const int acc = it & 1;
      int m0, n0, width;
      geom(tile, m0, n0, width);
      m0 += rank * BM;
      const int nb = width / Cfg::EB;
      // LayerNorm folded into this GEMM: per-row (mean, rstd) of the raw input row; the tile's
      // per-column u, v staged in smem (one copy per accumulator: the other copy may still be
      // read by a slower warp of the previous tile)
      float2 rstat = make_float2(0.f, 0.f);
      float* eu = evec + acc * 2 * BN;
      float2* rsm = reinterpret_cast<float2*>(evec + 2 * 2 * BN) + acc * 128;  // row stats, shared by the WGs
      if (kLn) {
        if (h == 0) {
          if (m0 + row < M)
            rstat = ev.row_stats ? pfrs : pf_parts ? ln_combine(ev, pfv) : ln_stats_from_parts(ev, m0 + row);
          rsm[row] = rstat;
          if (tile + num_pairs < num_tiles) prefetch(tile + num_pairs);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = etid + k * 128 * WG;
          if (i < width) {
            st_shared_f32(smem_u32(eu + i), pu[k]);
            st_shared_f32(smem_u32(eu + BN + i), pvv[k]);
          }
        }
        if (tile + num_pairs < num_tiles) prefetch_uv(tile + num_pairs);
      }
      const bool has_next = tile + num_pairs < num_tiles;
      if (kLn) {
        named_bar_sync(1, 128 * WG);  // u, v and the row statistics staged
        rstat = rsm[row];
      }
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      // row statistics of the stored (bf16-rounded) values, shifted by the box's first one
      // (one LayerNorm partial per row per BN-wide tile; the residual epilogue runs one warpgroup,
      // so the row's boxes are summed in column order by one thread)
      const bool kStats = kRes && ev.part_out != nullptr;
      static_assert(!kStage || WG == 1, "the residual epilogue's row partials assume one warpgroup");
      float2 sh = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f), s2 = make_float2(0.f, 0.f);
      constexpr int CW = Cfg::CW;
      for (int b = h; b < nb; b += WG, ++nbox_done) {
        // staging slot: the residual tile's own box; else a ring of two slots (one warpgroup:
        // boxes alternate, so a store overlaps the next box) or one slot per warpgroup
        const int slot = kDual ? 0 : Cfg::RING ? (WG == 1 ? (nbox_done & 1) : h) : b;
        const uint32_t line = e0 + slot * Cfg::E_BOX + row * (Cfg::EB * 2);
#pragma unroll
        for (int cb = 0; cb < Cfg::EB / CW; ++cb) {
          const int col0 = b * Cfg::EB + cb * CW;
          uint32_t v[CW];
          if constexpr (CW == 32) tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col0, v);
          else tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col0, v);
          tmem_ld_wait();
          if (cb == 0) {
            if (kStage) mbar_wait(&r_full[b], it & 1);
            if (Cfg::RING) {  // the warpgroup's previous store out of this slot has been read
              if (elected) {
                if (WG == 1 && !kDual) bulk_wait_group_read1();
                else bulk_wait_group_read0();
              }
              named_bar_sync(bar_wg, 128);
            }
          }
#pragma unroll
          for (int u = 0; u < CW / 8; ++u) {
            const int j = cb * (CW / 8) + u;
            const uint32_t addr =
                line + ((Cfg::EB == 64 ? (j ^ (row & 7)) : Cfg::EB == 32 ? (j ^ ((row >> 1) & 3)) : (j ^ ((row >> 2) & 1)))
                        << 4);
            float f[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(v[8 * u + i]);
            if (kStage) {
              uint32_t r0, r1, r2, r3;
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
              const float r[8] = {bf16lo(r0), bf16hi(r0), bf16lo(r1), bf16hi(r1),
                                  bf16lo(r2), bf16hi(r2), bf16lo(r3), bf16hi(r3)};
              if (kRes) {
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] += r[i];
              } else {  // EPI_GELU_BWD: du = dg * gelu'(u)
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] *= gelu_tanh_grad_f(r[i]);
              }
            } else if (kDual) {  // u = acc (bf16) into the other ring slot, g = gelu(acc) below
              st_shared_v4(addr + ((slot ^ 1) - slot) * Cfg::E_BOX, pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                           pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
#pragma unroll
              for (int i = 0; i < 8; ++i) f[i] = gelu_tanh_f(f[i]);
            } else if (EPI == DSP_EPI_GELU) {
#pragma unroll
              for (int i = 0; i < 8; ++i) f[i] = gelu_tanh_f(f[i]);
            } else if (kLn) {
              // y = rstd * (x.(W o gamma) - mean * u) + W.beta   (u, v: per-column, broadcast loads)
              const uint32_t ua = smem_u32(eu + col0 + 8 * u), va = smem_u32(eu + BN + col0 + 8 * u);
              const float2 nm = make_float2(-rstat.x, -rstat.x), rs = make_float2(rstat.y, rstat.y);
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const float4 uu = ld_shared_f32x4(ua + 16 * hh), vv = ld_shared_f32x4(va + 16 * hh);
                const float2 y0 = ffma2(rs, ffma2(nm, make_float2(uu.x, uu.y), make_float2(f[4 * hh], f[4 * hh + 1])),
                                        make_float2(vv.x, vv.y));
                const float2 y1 = ffma2(rs, ffma2(nm, make_float2(uu.z, uu.w), make_float2(f[4 * hh + 2], f[4 * hh + 3])),
                                        make_float2(vv.z, vv.w));
                f[4 * hh] = y0.x; f[4 * hh + 1] = y0.y; f[4 * hh + 2] = y1.x; f[4 * hh + 3] = y1.y;
                if (EPI == EPI_LN_GELU) {
#pragma unroll
                  for (int t = 0; t < 4; ++t) f[4 * hh + t] = gelu_tanh_f(f[4 * hh + t]);
                }
              }
            }
            const uint32_t pk[4] = {pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                    pack_bf16x2(f[6], f[7])};
            st_shared_v4(addr, pk[0], pk[1], pk[2], pk[3]);
            if (kStats) {  // shifted sums of the STORED (bf16-rounded) row values (R30), packed pairs
              if (b == 0 && cb == 0 && u == 0) sh = make_float2(-bf16lo(pk[0]), -bf16lo(pk[0]));
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 d = fadd2(make_float2(bf16lo(pk[i]), bf16hi(pk[i])), sh);
                s1 = fadd2(s1, d);
                s2 = ffma2(d, d, s2);
              }
            }
          }
        }
        // box b of this tile complete in every row of the warpgroup
        fence_proxy_async_smem();
        named_bar_sync(bar_wg, 128);
        if (elected) {
          tma_store_2d(&tmD, sE + slot * Cfg::E_BOX, n0 + Cfg::EB * b, m0);
          if (kDual) tma_store_2d(&tmR, sE + (slot ^ 1) * Cfg::E_BOX, n0 + Cfg::EB * b, m0);
          bulk_commit_group();
          if (kStage && has_next && b >= WG) {
            bulk_wait_group_read1();  // box b-WG read out of sE: reload it for the next tile
            load_res_box(tile + num_pairs, b - WG);
          }
        }
      }
      if (kStats && m0 + row < M) {
        // explicit rounding steps: launch_row_partials (simt.cu) reproduces these bits for rows
        // that crossed a switch (a tile with partials is always BN wide: no narrow tail tiles)
        const float a = __fadd_rn(s1.x, s1.y), mp = __fmul_rn(a, 1.f / BN);
        ev.part_out[(size_t)(m0 + row) * tiles_n + n0 / BN] =
            make_float2(__fsub_rn(mp, sh.x), fmaxf(__fmaf_rn(-a, mp, __fadd_rn(s2.x, s2.y)), 0.f));
      }
      tc_fence_before();
      if (leader) mbar_arrive(&tempty[acc]);  // accumulator free for the tile after next
      else mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
      if (kStage && elected && has_next) {
        bulk_wait_group_read0();  // the warpgroup's boxes of the next tile not reloaded yet
        int last = -1;
        for (int b = h; b < nb; b += WG) last = b;
        for (int b = (last >= 0 ? last : h); b < Cfg::NBOX; b += WG) load_res_box(tile + num_pairs, b);
      }
    }
    if (elected) bulk_wait_group_read0();
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane_id();
    int it = 0;
    for (int tile = pair; tile < num_tiles; tile += num_pairs, ++it) {
      const int acc = it & 1;
      int m0, n0, width;
      geom(tile, m0, n0, width);
      m0 += rank * BM;
      const int grow = m0 + row;
      const bool live = grow < M;
      __nv_bfloat16* drow = D + (size_t)grow * N + n0;
      // fp32 partials of split-K range t / tmn: part[ks][M][N]
      float* frow = reinterpret_cast<float*>(D) + ((size_t)(tile / tmn) * M + grow) * N + n0;
      if (EPI == EPI_RES_REMOTE && live) {
        // switch fused into the epilogue: this row's owner rank q and row index there
        int64_t dst;
        int q;
        if (rm.mode == 1) {  // T-sharded [B,Tn,S] row -> S-shard owner's [B,T,Sn]
          const int64_t ts = (int64_t)rm.Tn * rm.S, b = grow / ts, rem = grow % ts, t = rem / rm.S, sx = rem % rm.S;
          q = (int)(sx / rm.Sn);
          dst = (b * rm.T + (int64_t)rm.rank * rm.Tn + t) * rm.Sn + sx % rm.Sn;
        } else {             // S-sharded [B,T,Sn] row -> T-shard owner's [B,Tn,S]
          const int64_t ts = (int64_t)rm.T * rm.Sn, b = grow / ts, rem = grow % ts, t = rem / rm.Sn, sx = rem % rm.Sn;
          q = (int)(t / rm.Tn);
          dst = (b * rm.Tn + t % rm.Tn) * rm.S + (int64_t)rm.rank * rm.Sn + sx;
        }
        drow = reinterpret_cast<__nv_bfloat16*>(static_cast<uint8_t*>(rm.base.p[q]) + rm.dst_off) + dst * N + n0;
      }
      // residual row segment is independent of the accumulator: fetch it before waiting
      constexpr bool kRes = EPI == DSP_EPI_RESIDUAL || EPI == EPI_RES_REMOTE;
      uint4 rv[kRes ? BN / 8 : 1];
      if (kRes && live) {
        const uint4* rp = reinterpret_cast<const uint4*>(R + (size_t)grow * N + n0);
#pragma unroll
        for (int j = 0; j < BN / 8; ++j)
          if (j * 8 < width) rv[j] = rp[j];
      }
      // LayerNorm folded into this GEMM: per-row (mean, rstd) of the raw input row; the tile's
      // per-column u, v staged once in smem (one copy per accumulator, so a slow warp of the
      // previous tile never sees them overwritten)
      float2 rstat = make_float2(0.f, 0.f);
      float* eu = evec + acc * 2 * BN;
      if (EPI == EPI_LN || EPI == EPI_LN_GELU) {
        if (live) rstat = ev.row_stats[grow];
        for (int i = threadIdx.x - 128; i < width; i += 128) {
          eu[i] = ev.col_u[n0 + i];
          eu[BN + i] = ev.col_v[n0 + i];
        }
        named_bar_sync(1, 128);
      }
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      constexpr int CW = Cfg::CW;
#pragma unroll
      for (int c = 0; c < BN / CW; ++c) {
        if (c * CW >= width) break;  // narrow tail tile
        if (Cfg::F32 && n0 + c * CW >= N) break;  // ragged last column tile (wgrad)
        uint32_t v[CW];
        if constexpr (CW == 32) tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c * CW, v);
        else tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c * CW, v);
        tmem_ld_wait();
        if (live) {
          float f[CW];
#pragma unroll
          for (int i = 0; i < CW; ++i) f[i] = __uint_as_float(v[i]);
          if (kRes) {
#pragma unroll
            for (int j = 0; j < CW / 8; ++j) {
              const uint4 r4 = rv[c * (CW / 8) + j];
              f[8 * j + 0] += bf16lo(r4.x);
              f[8 * j + 1] += bf16hi(r4.x);
              f[8 * j + 2] += bf16lo(r4.y);
              f[8 * j + 3] += bf16hi(r4.y);
              f[8 * j + 4] += bf16lo(r4.z);
              f[8 * j + 5] += bf16hi(r4.z);
              f[8 * j + 6] += bf16lo(r4.w);
              f[8 * j + 7] += bf16hi(r4.w);
            }
          } else if (EPI == DSP_EPI_GELU) {
#pragma unroll
            for (int i = 0; i < CW; ++i) f[i] = gelu_tanh_f(f[i]);
          } else if (EPI == EPI_LN || EPI == EPI_LN_GELU) {
            // y = rstd * (x.(W o gamma) - mean * u) + W.beta   (u, v: per-column, warp-uniform loads)
            const float4* u4 = reinterpret_cast<const float4*>(eu + c * CW);
            const float4* v4 = reinterpret_cast<const float4*>(eu + BN + c * CW);
#pragma unroll
            for (int q4 = 0; q4 < CW / 4; ++q4) {
              const float4 uu = u4[q4], vv = v4[q4];
              const float us[4] = {uu.x, uu.y, uu.z, uu.w}, vs[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                float y = fmaf(rstat.y, fmaf(-rstat.x, us[t], f[4 * q4 + t]), vs[t]);
                if (EPI == EPI_LN_GELU) y = gelu_tanh_f(y);
                f[4 * q4 + t] = y;
              }
            }
          }
          if constexpr (Cfg::F32) {
            float4* fp = reinterpret_cast<float4*>(frow + c * CW);
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) fp[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
          } else {
            uint4* dp = reinterpret_cast<uint4*>(drow + c * CW);
#pragma unroll
            for (int j = 0; j < CW / 8; ++j) {
              dp[j] = make_uint4(pack_bf16x2(f[8 * j], f[8 * j + 1]), pack_bf16x2(f[8 * j + 2], f[8 * j + 3]),
                                 pack_bf16x2(f[8 * j + 4], f[8 * j + 5]), pack_bf16x2(f[8 * j + 6], f[8 * j + 7]));
            }
          }
        }
      }
      tc_fence_before();
      if (leader) mbar_arrive(&tempty[acc]);
      else mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
    }
    if (EPI == EPI_RES_REMOTE && rm.arrive) __threadfence_system();  // this thread's peer stores, before the arrival
  }

  tc_fence_before();
  cluster_sync();
  if (EPI == EPI_RES_REMOTE && rm.arrive && threadIdx.x == 0) {
    // the last CTA to get here arrives at the signal-pad barrier for this rank (RemoteMap): every
    // CTA's epilogue threads fenced their peer stores at system scope before the cluster barrier
    uint64_t* pad = static_cast<uint64_t*>(rm.signals.p[rm.rank]);
    __threadfence_system();
    const unsigned long long done = atomicAdd(reinterpret_cast<unsigned long long*>(pad + kPadCount), 1ull);
    if (done == gridDim.x - 1) {
      __threadfence_system();
      pad[kPadCount] = 0;
      const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(pad + kPadEpoch) + 1;
      pad[kPadEpoch] = epoch;
      for (int i = 0; i < rm.world; ++i) {
        uint64_t* remote = static_cast<uint64_t*>(rm.signals.p[i]) + rm.rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote), "l"(epoch) : "memory");
      }
    }
  }
  clk_end(ev.clk);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, Cfg::TMEM_COLS);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

// bf16 tensor map, dims/strides innermost first (strides in bytes for dims >= 1).
bool make_tmap_bf16(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                    const uint32_t* box, CUtensorMapSwizzle swz, std::string* why) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    if (why) *why = "cuTensorMapEncodeTiled unavailable (driver entry point)";
    return false;
  }
  uint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (why) *why = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r);
    return false;
  }
  return true;
}

bool make_tmap_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                   const uint32_t* box, std::string* why, CUtensorMapSwizzle swz) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    if (why) *why = "cuTensorMapEncodeTiled unavailable (driver entry point)";
    return false;
  }
  uint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (why) *why = "cuTensorMapEncodeTiled (f32) failed with CUresult " + std::to_string((int)r);
    return false;
  }
  return true;
}

template <int BN, int EPI, int MAJ = MAJ_K>
static cudaError_t run_gemm(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N, int64_t K,
                            int num_sms, cudaStream_t st, std::string* why, const EpiVec& ev = EpiVec{},
                            const RemoteMap& rm = RemoteMap{}, int ksplit = 1) {
  using Cfg = GemmCfg<BN, EPI, MAJ>;
  CUtensorMap ta, tw, tw2, td, tr;
  // K-major operands: {K, rows}, box {BK, rows}; MN-major ({rows, K} in memory order): box {64, BK}
  uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, sa[1] = {(uint64_t)K * 2};
  uint64_t dw[2] = {(uint64_t)K, (uint64_t)N}, sw[1] = {(uint64_t)K * 2};
  uint64_t dd[2] = {(uint64_t)N, (uint64_t)M}, sd[1] = {(uint64_t)N * 2};
  uint32_t ba[2] = {BK, BM}, bw[2] = {BK, Cfg::BNH}, bd[2] = {Cfg::EB, BM};
  if (Cfg::A_MN) {
    da[0] = (uint64_t)M; da[1] = (uint64_t)K; sa[0] = (uint64_t)M * 2;
    ba[0] = 64; ba[1] = BK;
  }
  if (Cfg::B_MN) {
    dw[0] = (uint64_t)N; dw[1] = (uint64_t)K; sw[0] = (uint64_t)N * 2;
    bw[0] = 64; bw[1] = BK;
  }
  const CUtensorMapSwizzle esw = Cfg::EB == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : Cfg::EB == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                 : CU_TENSOR_MAP_SWIZZLE_32B;
  if (!make_tmap_bf16(&ta, A, 2, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B, why) ||
      !make_tmap_bf16(&tw, W, 2, dw, sw, bw, CU_TENSOR_MAP_SWIZZLE_128B, why))
    return cudaErrorInvalidValue;
  // grid: one pair per tile up to all pairs; a partial last wave becomes narrow tiles (TileSched)
  const int64_t full = ((M + 2 * BM - 1) / (2 * BM)) * (Cfg::F32 ? (N + BN - 1) / BN : N / BN) * ksplit;
  const int pmax = num_sms / 2;
  const int smax = gemm_split_max<BN, EPI, MAJ>(ev);
  TileSched tsh = make_tile_sched((int)full, pmax, smax);
  const int64_t pairs = full >= pmax ? pmax : (tsh.num_tiles < pmax ? tsh.num_tiles : pmax);
  tsh = make_tile_sched((int)full, (int)pairs, smax);  // what the kernel will compute
  tw2 = tw;
  if (tsh.split > 1) {
    uint32_t bw2[2] = {BK, (uint32_t)(Cfg::BNH / tsh.split)};
    if (!make_tmap_bf16(&tw2, W, 2, dw, sw, bw2, CU_TENSOR_MAP_SWIZZLE_128B, why)) return cudaErrorInvalidValue;
  }
  td = ta;
  tr = ta;
  if (Cfg::TSEQ) {  // 5-D store view of the temporal layout: {DP, T, S_loc, NH, 3B}
    const TseqShape& q = ev.tseq;
    const uint64_t row = kTseqDP * 2;
    uint64_t dt[5] = {(uint64_t)kTseqDP, (uint64_t)q.T, (uint64_t)q.S_loc, (uint64_t)q.NH, (uint64_t)(3 * q.B)};
    uint64_t st5[4] = {row, (uint64_t)q.T * row, (uint64_t)q.S_loc * q.T * row, (uint64_t)q.NH * q.S_loc * q.T * row};
    uint32_t bx[5] = {(uint32_t)kTseqDP, 1, BM, 1, 1};
    if (!make_tmap_bf16(&td, D, 5, dt, st5, bx, CU_TENSOR_MAP_SWIZZLE_NONE, why)) return cudaErrorInvalidValue;
  } else if (EPI != EPI_RES_REMOTE && !Cfg::F32) {
    if (!make_tmap_bf16(&td, D, 2, dd, sd, bd, esw, why)) return cudaErrorInvalidValue;
    if ((EPI == DSP_EPI_RESIDUAL || Cfg::AUX || EPI == EPI_GELU_AUX) && !make_tmap_bf16(&tr, R, 2, dd, sd, bd, esw, why))
      return cudaErrorInvalidValue;
  }
  auto kern = gemm_bf16_tc_kernel<BN, EPI, MAJ>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  EpiVec evc = ev;
  evc.clk = t_clk;
  return launch_k(kern, dim3((unsigned)(2 * pairs)), dim3(Cfg::THREADS), Cfg::SMEM, st, 2, ta, tw, tw2, td, tr, (const __nv_bfloat16*)R,
                  (__nv_bfloat16*)D, (int)M, (int)N, (int)K, ksplit, evc, rm);
}

template <int EPI>
static cudaError_t dispatch_bn(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N,
                               int64_t K, int num_sms, cudaStream_t st, std::string* why,
                               const EpiVec& ev = EpiVec{}, const RemoteMap& rm = RemoteMap{}) {
  switch (gemm_bn_for(N)) {
    case 256: return run_gemm<256, EPI>(A, W, R, D, M, N, K, num_sms, st, why, ev, rm);
    case 192: return run_gemm<192, EPI>(A, W, R, D, M, N, K, num_sms, st, why, ev, rm);
    case 144: return run_gemm<144, EPI>(A, W, R, D, M, N, K, num_sms, st, why, ev, rm);
    case 128: return run_gemm<128, EPI>(A, W, R, D, M, N, K, num_sms, st, why, ev, rm);
    case 64: return run_gemm<64, EPI>(A, W, R, D, M, N, K, num_sms, st, why, ev, rm);
    default: return run_gemm<32, EPI>(A, W, R, D, M, N, K, num_sms, st, why, ev, rm);
  }
}

int64_t tseq_bytes(const TseqShape& t) {
  return 3 * (int64_t)t.B * t.NH * t.S_loc * t.T * kTseqDP * 2;
}

bool tseq_ok(int64_t B, int64_t T, int64_t S_loc, int64_t C, int NH) {
  (void)B;
  // T >= 64: at T = 16 the token-major gathers already run near the HBM floor (32 us at configs[1])
  // and the head-at-a-time epilogue costs the QKV GEMM more than the attention gains
  return T >= 64 && NH > 0 && C % NH == 0 && C / NH == kTseqDh && S_loc % BM == 0 && (3 * C) % (2 * kTseqDh) == 0;
}

cudaError_t launch_gemm_bf16_tseq(const void* A, const void* W, const EpiVec* ln, void* qkv_tseq, const TseqShape& ts,
                                  int64_t M, int64_t K, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  if (!tseq_ok(ts.B, ts.T, ts.S_loc, ts.C, ts.NH) || M != (int64_t)ts.B * ts.T * ts.S_loc) {
    if (why) *why = "TSEQ layout: unsupported shape";
    return cudaErrorNotSupported;
  }
  EpiVec ev = ln ? *ln : EpiVec{};
  ev.tseq = ts;
  constexpr int BNT = 2 * kTseqDh;  // two heads per tile
  if (ln) return run_gemm<BNT, EPI_LN_TSEQ>(A, W, nullptr, qkv_tseq, M, 3 * ts.C, K, num_sms, st, why, ev);
  return run_gemm<BNT, EPI_TSEQ>(A, W, nullptr, qkv_tseq, M, 3 * ts.C, K, num_sms, st, why, ev);
}

cudaError_t launch_gemm_bf16_remote(const void* A, const void* W, const void* R, const RemoteMap& rm, int64_t M,
                                    int64_t N, int64_t K, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  return dispatch_bn<EPI_RES_REMOTE>(A, W, R, nullptr, M, N, K, num_sms, st, why, EpiVec{}, rm);
}

cudaError_t launch_gemm_bf16_ln(const void* A, const void* Wf, const EpiVec& ev, void* D, int64_t M, int64_t N,
                                int64_t K, bool gelu, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  if (gelu) return dispatch_bn<EPI_LN_GELU>(A, Wf, nullptr, D, M, N, K, num_sms, st, why, ev);
  return dispatch_bn<EPI_LN>(A, Wf, nullptr, D, M, N, K, num_sms, st, why, ev);
}

int gemm_part_cols(int64_t N) { return gemm_bn_for(N); }  // one partial per BN-wide tile

// ----------------------------------------------------------------- backward GEMMs (f4)
cudaError_t launch_gemm_bf16_dgrad(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N,
                                   int64_t K, int epi, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  if (N % 128 != 0 || K % 8 != 0) {
    if (why) *why = "dgrad GEMM: N % 128 == 0 and K % 8 == 0 required";
    return cudaErrorNotSupported;
  }
  const bool wide = N % 256 == 0;
  if (epi == EPI_GELU_BWD)
    return wide ? run_gemm<256, EPI_GELU_BWD, MAJ_B_MN>(A, W, R, D, M, N, K, num_sms, st, why)
                : run_gemm<128, EPI_GELU_BWD, MAJ_B_MN>(A, W, R, D, M, N, K, num_sms, st, why);
  if (epi == DSP_EPI_NONE)
    return wide ? run_gemm<256, DSP_EPI_NONE, MAJ_B_MN>(A, W, R, D, M, N, K, num_sms, st, why)
                : run_gemm<128, DSP_EPI_NONE, MAJ_B_MN>(A, W, R, D, M, N, K, num_sms, st, why);
  if (why) *why = "dgrad GEMM: unsupported epilogue";
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemm_bf16_dgrad_kmajor(const void* A, const void* Wt, const void* R, void* D, int64_t M, int64_t N,
                                          int64_t K, int epi, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  if (epi == EPI_GELU_BWD) return dispatch_bn<EPI_GELU_BWD>(A, Wt, R, D, M, N, K, num_sms, st, why);
  if (epi == DSP_EPI_NONE) return dispatch_bn<DSP_EPI_NONE>(A, Wt, R, D, M, N, K, num_sms, st, why);
  if (why) *why = "dgrad GEMM: unsupported epilogue";
  return cudaErrorInvalidValue;
}

// Split count for the wgrad GEMM: the output has few tiles (dW [3C, C] at C = 1152: 126 tiles of
// 256 x 128 for 74 CTA pairs) and a long reduction (all tokens), so the token range is cut into
// ksplit slices, the smallest count whose tiles fill >= 90 % of the last wave (at most 16, each
// slice >= 8 k-blocks); the fp32 partials are summed in slice order by launch_wgrad_reduce.
int wgrad_splits(int64_t M, int64_t N, int64_t K, int num_sms) {
  const int64_t bn = N % 256 == 0 || N > 256 ? 256 : 128;  // as launch_gemm_bf16_wgrad
  const int64_t tiles = ((M + 255) / 256) * ((N + bn - 1) / bn), pairs = num_sms / 2, nkb = (K + 63) / 64;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 16 && s <= nkb / 8; ++s) {
    const int64_t kbs = (nkb + s - 1) / s, se = (nkb + kbs - 1) / kbs;  // slices actually used
    if (se != s) continue;
    const int64_t units = tiles * s, waves = (units + pairs - 1) / pairs;
    const double eff = (double)units / (double)(waves * pairs);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
    if (eff >= 0.9) break;
  }
  return best;
}

cudaError_t launch_gemm_bf16_wgrad(const void* dY, const void* X, float* part, int64_t M, int64_t N, int64_t K,
                                   int ksplit, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0 || N == 0) return cudaSuccess;
  if (M % 64 != 0 || N % 128 != 0 || ksplit < 1) {
    if (why) *why = "wgrad GEMM: M % 64 == 0, N % 128 == 0 required";
    return cudaErrorNotSupported;
  }
  const int64_t nkb = (K + 63) / 64, kbs = (nkb + ksplit - 1) / ksplit;
  if ((nkb + kbs - 1) / kbs != ksplit) {  // every slice must own k-blocks (an empty one never completes)
    if (why) *why = "wgrad GEMM: ksplit leaves an empty token slice (use wgrad_splits)";
    return cudaErrorInvalidValue;
  }
  constexpr int MAJ = MAJ_A_MN | MAJ_B_MN;
  // BN = 256 (a ragged last column tile when 256 does not divide N: 10 % idle MMA columns at N = 1152)
  // halves the operand bytes each CTA pulls from L2 per MMA cycle against BN = 128 (measured 66 % vs
  // 88 % tensor-active: the 128-wide tiles are bound by L2 -> SM bandwidth)
  if (N % 256 == 0 || N > 256)
    return run_gemm<256, EPI_F32, MAJ>(dY, X, nullptr, part, M, N, K, num_sms, st, why, EpiVec{}, RemoteMap{}, ksplit);
  return run_gemm<128, EPI_F32, MAJ>(dY, X, nullptr, part, M, N, K, num_sms, st, why, EpiVec{}, RemoteMap{}, ksplit);
}

cudaError_t launch_gemm_bf16_gelu_aux(const void* A, const void* W, void* G, void* U, int64_t M, int64_t N,
                                      int64_t K, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  return dispatch_bn<EPI_GELU_AUX>(A, W, U, G, M, N, K, num_sms, st, why);
}

int gemm_bn_for(int64_t N) {
#ifdef DSP_GEMM_BN_1152
  if (N == 1152) return DSP_GEMM_BN_1152;  // A/B experiments only
#endif
#ifdef DSP_GEMM_BN_4608
  if (N == 4608) return DSP_GEMM_BN_4608;  // A/B experiments only
#endif
  // A function of N only (never of M): the tile width fixes how many LayerNorm partials a
  // residual epilogue writes, and the block must not depend on the shard size (N-invariance).
  // 144-wide tiles (8 column tiles at C = 1152, 6.9 waves of 74 pairs instead of 5.2 -> 6 at
  // 192) were measured slower on B200 (FC2 134 vs 128 us): the mainloop is bound by the bytes
  // staged per k-block, which do not shrink with BN (A is 16 KB either way).  Selectable with
  // -DDSP_GEMM_BN_1152=144 for experiments.
  if (N % 256 == 0) return 256;
  return N % 192 == 0 ? 192 : N % 128 == 0 ? 128 : N % 64 == 0 ? 64 : 32;
}

cudaError_t launch_gemm_bf16_res_stats(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N,
                                       int64_t K, float2* part_out, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  EpiVec ev{};
  ev.part_out = part_out;
  return dispatch_bn<DSP_EPI_RESIDUAL>(A, W, R, D, M, N, K, num_sms, st, why, ev);
}

cudaError_t launch_gemm_bf16(const void* A, const void* W, const void* R, void* D, int64_t M, int64_t N,
                             int64_t K, int epi, int num_sms, cudaStream_t st, std::string* why) {
  if (M == 0) return cudaSuccess;
  switch (epi) {
    case DSP_EPI_NONE:
      return dispatch_bn<DSP_EPI_NONE>(A, W, R, D, M, N, K, num_sms, st, why);
    case DSP_EPI_RESIDUAL:
      return dispatch_bn<DSP_EPI_RESIDUAL>(A, W, R, D, M, N, K, num_sms, st, why);
    case DSP_EPI_GELU:
      return dispatch_bn<DSP_EPI_GELU>(A, W, R, D, M, N, K, num_sms, st, why);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsp
