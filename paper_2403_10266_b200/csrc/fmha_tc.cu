// fmha_tc.cu — tcgen05/TMEM flash attention for the DSP spatial and temporal stages.
//
// For every sequence and head: O_j = softmax(q_j k_j^T / sqrt(Dh)) v_j (R6-R7),
// reading q/k/v straight out of the QKV projection output qkv[tok, 3C] (no head-split
// copy): a 5-D TMA map over each of the q / k / v column blocks does the head split,
// the sequence gather (spatial rows are contiguous; temporal rows have stride
// S_loc*3C) and the Dh=72 -> 80 zero padding (out-of-bounds fill).
//
// Tiles are 128 query rows x 128 key rows.  Sequences of length L >= 128 (L % 128 == 0)
// get one sequence per tile.  Shorter sequences (temporal T=16) are packed G = 128/L
// per tile, rows ordered sequence-major (r = seq*L + pos), so the attention mask is
// block-diagonal with contiguous LxL blocks: each softmax warp only reads, exponentiates
// and writes the 32 (or 64) key columns of its own diagonal blocks; the rest of P stays
// zero for the CTA's lifetime.
//
// Persistent kernel, 2 CTAs per SM (<= 113 KB smem, 256 TMEM columns, <= 128 regs each):
// one CTA's softmax overlaps the other CTA's TMA + MMA.  Roles per CTA (256 threads):
//   warp 0     TMA producer: Q per work item, K_j and V_j in single-stage slots with
//              separate full/empty barriers (K_{j+1} streams in during softmax_j).
//   warp 1     MMA issuer: S = Q K^T into TMEM; after softmax j: S_{j+1}, then O += P_j V_j
//              (P from smem, K-major; V from smem, MN-major).
//   warps 4-7  softmax + epilogue, thread = query row: two passes over 64-column halves
//              (max, then exp2 / row-sum / bf16 P), online softmax in fp32 with lazy
//              rescaling (the running max only moves when it grows by > 8 in log2
//              units), final O / l -> bf16 -> o[tok, C].
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>

#include "dsp_internal.h"
#include "sm100.cuh"

// fraction of the softmax exponentials computed with poly_exp2 on the FMA pipe
// Experimental schedules of the long-sequence kernel, both measured SLOWER on B200 at the
// spatial blk shape (pair kernel, lock-step: 100-105 us; ping-pong: 105-109; split rows:
// 107-112; split + ping-pong: 107-112) and therefore off by default.  The exp loop itself is
// the bound: scripts/micro/exp_loop.cu measures 3.8 exps/clk/SMSP with two warps per SMSP and
// 4.8 with four, against 32768 exps per SM per K/V step.
// Schedules measured SLOWER on B200 at the blk shapes and removed (git history has them):
// rows split over two softmax threads (4 warps/SMSP, max exchanged through smem): 107-112 us;
// ping-pong of the two query tiles' exp phases: 105-109 us; a 3-stage Q|K|V ring for
// single-K/V-tile sequences (temporal): 36.3 vs 32.8 us; a dedicated epilogue warpgroup (512
// threads, own O staging; the 128-register launch cap spills the softmax): 125 vs 102 us.
// The pair kernel (lock-step): 100-105 us.
#ifndef DSP_POLY_NUM
#define DSP_POLY_NUM 6  // with tensor-core row sums: 4/16 104.0 us, 5/16 105.8, 6/16 99.8, 7/16 100.4 (same box)
#endif
#ifndef DSP_POLY_DEN
#define DSP_POLY_DEN 16
#endif

namespace dsp {
namespace {

struct FmhaParams {
  int spatial;   // 1: sequences over S per frame; 0: over T per (b, s)
  int L;         // sequence length
  int G;         // sequences per tile (1 if L >= 128)
  int n_kv;      // kv tiles per sequence
  int n_qt;      // query tiles per sequence
  int n_outer;   // outer work units (frames / columns, or groups of G of them)
  int NH, Dh, C;
  int S_loc, T_loc, B;
  int items;     // n_outer * NH * n_qt
  int kv_last;   // valid keys in the last K/V tile (128 unless the key length is ragged: cross-attention)
  int cross;     // 1: cross-attention views (queries and keys from different tensors)
  int colfast;   // 1: item order column-fastest (outer before head), for the head-major TSEQ layout
  int walk_ch;   // backward: consecutive items per CTA chunk (BwdWalk; 0: one contiguous range per CTA)
  float scale_log2;
  __nv_bfloat16* o;
  float* lse;                 // optional [tok][NH]: log2-domain log-sum-exp of the scaled scores (training)
  unsigned long long* trace;  // DSP_FMHA_TRACE builds only: per-phase clock64 stamps of CTA 0
  unsigned long long* clk;    // stage clock (instrumentation, t_clk)
};

#ifdef DSP_FMHA_TRACE
#define FMHA_STAMP(buf, idx) \
  do { if ((buf) && blockIdx.x == 0 && lane_id() == 0 && (threadIdx.x & 127) == 0) (buf)[idx] = clock64(); } while (0)
#else
#define FMHA_STAMP(buf, idx) do { } while (0)
#endif

template <int NA, int RB>
struct FmhaCfg {
  static constexpr int DP = NA * 64 + RB;                       // padded head dim
  static constexpr int RB_BYTES = RB == 0 ? 0 : 1024 * ((128 * RB * 2 + 1023) / 1024);
  static constexpr int TILE = NA * 16384 + RB_BYTES;            // one 128-row operand tile
  static constexpr int TX = 128 * DP * 2;                        // TMA bytes per tile
  static constexpr int P_BYTES = 2 * 16384;
  // Q, K, V x 2 stages, P, barriers.  No alignment slack: dynamic smem starts right after the
  // 1 KB system-reserved block and is therefore 1024-B aligned (checked in the kernel), which
  // keeps two CTAs per SM at Dh = 72 (115,712 B available per CTA).
  static constexpr int SMEM = 5 * TILE /*Q,K,V0,V1*/ - TILE + P_BYTES + 256;
  static constexpr uint32_t RB_SW = RB == 16 ? SW_32B : SW_64B;
  static constexpr uint32_t RB_ROW = RB * 2;                     // bytes per row in the rem chunk
  static constexpr int CTAS_PER_SM = SMEM <= 113 * 1024 ? 2 : 1;  // Dh <= 96: two CTAs per SM
};

// TMA coordinates {h, x2, x3, x4} of the 128-row tile (query tile if kv < 0).
struct TileCoord {
  int h, x2, x3, x4;
};
__device__ __forceinline__ TileCoord tile_coord(const FmhaParams& p, int item, int kv) {
  const int qt = item % p.n_qt;
  const int rest = item / p.n_qt;
  TileCoord t;
  t.h = p.colfast ? rest / p.n_outer : rest % p.NH;
  const int outer = p.colfast ? rest % p.n_outer : rest / p.NH;
  if (p.G == 1) {
    t.x2 = (kv >= 0 ? kv : qt) * 128;
    if (p.spatial) { t.x3 = outer; t.x4 = 0; }
    else { t.x3 = outer % p.S_loc; t.x4 = outer / p.S_loc; }
  } else {
    t.x2 = 0;
    if (p.spatial) { t.x3 = outer * p.G; t.x4 = 0; }
    else { const int ng = (p.S_loc + p.G - 1) / p.G; t.x3 = (outer % ng) * p.G; t.x4 = outer / ng; }
  }
  return t;
}

// token index of tile row r (or -1 if the row is padding)
__device__ __forceinline__ long row_token(const FmhaParams& p, const TileCoord& t, int r) {
  int pos, outer;
  if (p.G == 1) { pos = t.x2 + r; outer = t.x3; }
  else { pos = r % p.L; outer = t.x3 + r / p.L; }
  if (p.spatial) {  // outer = frame b*T_loc + t
    if (outer >= p.B * p.T_loc) return -1;
    return (long)outer * p.S_loc + pos;
  }
  if (outer >= p.S_loc) return -1;  // outer = column s, t.x4 = b
  return ((long)t.x4 * p.T_loc + pos) * p.S_loc + outer;
}

template <int NA, int RB>
__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* ma, const CUtensorMap* mb, uint64_t* bar,
                                          const TileCoord& t) {
#pragma unroll
  for (int i = 0; i < NA; ++i) tma_load_5d(dst + i * 16384, ma, bar, 64 * i, t.h, t.x2, t.x3, t.x4);
  if (RB) tma_load_5d(dst + NA * 16384, mb, bar, 64 * NA, t.h, t.x2, t.x3, t.x4);
}

__device__ __forceinline__ float max8(const float* v) {
  const float a = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
  const float b = fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7]));
  return fmaxf(a, b);
}

// Geometry of the key columns one softmax thread touches.
struct SoftmaxGeom {
  int row;            // query row of this thread in the tile (= TMEM lane)
  uint32_t lane_off;  // TMEM lane offset of this warp's quadrant
  bool diag;          // block-diagonal packing (G > 1)
  int wc0, nhalf, hcols, L, my_blk;
  float sl2;          // log2(e) / sqrt(Dh)
};

__device__ __forceinline__ SoftmaxGeom make_geom(const FmhaParams& p, int warp, float sl2) {
  SoftmaxGeom g;
  const int q = warp & 3;
  g.row = q * 32 + lane_id();
  g.lane_off = (uint32_t)(q * 32) << 16;
  g.diag = p.G > 1;
  const int wcols = g.diag ? (p.L > 32 ? p.L : 32) : 128;
  g.wc0 = g.diag ? (q * 32 / wcols) * wcols : 0;
  g.nhalf = (wcols + 63) / 64;
  g.hcols = wcols < 64 ? wcols : 64;
  g.L = p.L;
  g.my_blk = g.row / (p.L < 128 ? p.L : 128);
  g.sl2 = sl2;
  return g;
}

// One online-softmax step on S_j (in TMEM at tS): row max, lazy O rescale (after PV_{j-1}
// completed, signalled on o_done), P_j = exp2(S*scale - m) as bf16 into the SW128 smem tile
// sP, running sum l.  Returns after the P stores are fenced for the async proxy.
// valid < 128 (non-diagonal tiles only): keys >= valid of this tile are padding of a ragged
// sequence (TMA zero fill) and are excluded (-inf) in both passes.
template <int DP>
__device__ __forceinline__ void softmax_tile(const SoftmaxGeom& G, uint32_t tS, uint32_t tO, uint8_t* sP, int j,
                                             float& m, float& l, uint64_t* o_done, uint32_t& no,
                                             int* store_pending = nullptr, uint32_t bar_id = 0, int valid = 128) {
  const int row = G.row;
  const uint32_t lane_off = G.lane_off;
  const bool diag = G.diag;
  const int wc0 = G.wc0, nhalf = G.nhalf, hcols = G.hcols, my_blk = G.my_blk;
  const float sl2 = G.sl2;
  uint8_t* prow = sP + row * 128;
  // pass 1: row max over this thread's valid columns
  float mx = -INFINITY;
  for (int hf = 0; hf < nhalf; ++hf) {
    float s[64];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (c * 32 < hcols) {
        uint32_t v[32];
        tmem_ld32(tS + lane_off + wc0 + hf * 64 + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = -INFINITY;
      }
    }
    if (diag) {
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if ((wc0 + hf * 64 + i) / G.L != my_blk) s[i] = -INFINITY;
    } else if (valid < 128) {
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (hf * 64 + i >= valid) s[i] = -INFINITY;
    }
    float t8[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) t8[a] = max8(s + 8 * a);
    mx = fmaxf(mx, max8(t8));
  }
  const float mx2 = mx * sl2;
  const bool bump = (j == 0) || (mx2 > m + 8.f);
  const float m_new = bump ? mx2 : m;
  const float alpha = (j == 0) ? 0.f : fast_exp2(m - m_new);
  m = m_new;
  if (j > 0) {
    mbar_wait(o_done, no & 1);  // PV_{j-1} done: O stable, P buffer free
    ++no;
    tc_fence_after();
    if (__any_sync(0xffffffffu, bump)) {
      const float a = bump ? alpha : 1.f;
#pragma unroll
      for (int c = 0; c < DP / 16; ++c) {
        uint32_t v[16];
        tmem_ld16(tO + lane_off + c * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * a);
        tmem_st16(tO + lane_off + c * 16, v);
      }
      tmem_st_wait();
    }
  }
  if (store_pending && *store_pending) {  // previous item's O TMA store must have read the P buffer
    if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
    named_bar_sync(bar_id, 128);
    *store_pending = 0;
  }
  // pass 2: exponentiate, row-sum, P (bf16) -> smem.  SW128 K-major: 16-B chunk c of
  // row r lives at chunk position c ^ (r & 7) of the row's 128-B line.  In the diagonal
  // mode the whole row is written (zeros outside this thread's window) so the buffer can
  // also serve as the O staging tile.
  float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const uint32_t prow_s = smem_u32(prow);
  if (diag) {
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int col = c * 8;
      if (col < wc0 || col >= wc0 + nhalf * hcols)
        st_shared_v4(prow_s + (c >> 3) * 16384 + (((c & 7) ^ (row & 7)) << 4), 0u, 0u, 0u, 0u);
    }
  }
  for (int hf = 0; hf < nhalf; ++hf) {
    const int col0 = wc0 + hf * 64;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (c * 32 < hcols) {
        uint32_t v[32];
        tmem_ld32(tS + lane_off + col0 + c * 32, v);
        tmem_ld_wait();
        float e[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x = __uint_as_float(v[i]);
          if (diag ? (col0 + c * 32 + i) / G.L != my_blk : col0 + c * 32 + i >= valid) x = -INFINITY;
          e[i] = fast_exp2(fmaf(x, sl2, -m_new));
          rs8[i & 7] += e[i];
        }
        const int colb = col0 + c * 32;  // multiple of 32
        const uint32_t line = prow_s + (colb >> 6) * 16384;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int chunk = ((colb & 63) >> 3) + u;
          st_shared_v4(line + ((chunk ^ (row & 7)) << 4), pack_bf16x2(e[8 * u + 0], e[8 * u + 1]),
                       pack_bf16x2(e[8 * u + 2], e[8 * u + 3]), pack_bf16x2(e[8 * u + 4], e[8 * u + 5]),
                       pack_bf16x2(e[8 * u + 6], e[8 * u + 7]));
        }
      }
    }
  }
  const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
  l = l * alpha + rs;
  fence_proxy_async_smem();
  tc_fence_before();
}

// Non-diagonal tiles (L >= 128): single pass with the whole 128-column S row in registers.
// All four TMEM loads are in flight before one wait; the exponentials are computed before
// waiting for PV_{j-1} (only the O rescale and the P store need it).
//
// ONES: V carries a column of ones at DP - 8 (written into each V tile by the patcher warp),
// so the P.V MMA accumulates the row sum l into O's column DP - 8 under the same lazy
// rescale as O; the softmax threads then skip the 128-term sum.
template <int DP, bool ONES = false>
__device__ __forceinline__ void softmax_tile_full(const SoftmaxGeom& G, uint32_t tS, uint32_t tO, uint8_t* sP, int j,
                                                  float& m, float& l, uint64_t* o_done, uint32_t& no,
                                                  unsigned long long* tr = nullptr, uint64_t* s_free = nullptr,
                                                  int* store_pending = nullptr, uint32_t bar_id = 0,
                                                  int valid = 128) {
  const int row = G.row;
  const uint32_t lane_off = G.lane_off;
  const float sl2 = G.sl2;
  uint32_t v[128];
  tmem_ld32(tS + lane_off + 0, *reinterpret_cast<uint32_t(*)[32]>(v + 0));
  tmem_ld32(tS + lane_off + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
  tmem_ld32(tS + lane_off + 64, *reinterpret_cast<uint32_t(*)[32]>(v + 64));
  tmem_ld32(tS + lane_off + 96, *reinterpret_cast<uint32_t(*)[32]>(v + 96));
  tmem_ld_wait();
  FMHA_STAMP(tr, 8);
  if (s_free) {  // the whole S row is in registers: the MMA may overwrite S with S_{j+1}
    tc_fence_before();
    mbar_arrive(s_free);
  }
  if (valid < 128) {  // ragged key length: keys >= valid of this tile are padding (TMA zero fill)
#pragma unroll
    for (int i = 0; i < 128; ++i)
      if (i >= valid) v[i] = __float_as_uint(-INFINITY);
  }
  const float mx = max_tree3<128>(reinterpret_cast<const float*>(v));
  FMHA_STAMP(tr, 9);
  const float mx2 = mx * sl2;
  const bool bump = (j == 0) || (mx2 > m + 8.f);
  const float m_new = bump ? mx2 : m;
  const float alpha = (j == 0) ? 0.f : fast_exp2(m - m_new);
  m = m_new;
  float2 rs4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t pk[64];
  const float2 sl2x2 = make_float2(sl2, sl2), mx2n = make_float2(-m_new, -m_new);
  FMHA_STAMP(tr, 10);
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    // x = s * scale*log2(e) - m on pairs; DSP_POLY_NUM/DSP_POLY_DEN of the pairs exponentiated on
    // the FMA pipe (poly_exp2_x2), the rest on the MUFU (ex2.approx)
    const float2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2x2, mx2n);
    float2 e;
    if ((i % DSP_POLY_DEN) < DSP_POLY_NUM) {
      e = poly_exp2_x2(x);
    } else {
      e.x = fast_exp2(x.x);
      e.y = fast_exp2(x.y);
    }
    if (!ONES) rs4[i & 3] = fadd2(rs4[i & 3], e);
    pk[i] = pack_bf16x2(e.x, e.y);
  }
  FMHA_STAMP(tr, 11);
  if (!ONES) {
    const float2 rsa = fadd2(fadd2(rs4[0], rs4[1]), fadd2(rs4[2], rs4[3]));
    l = l * alpha + (rsa.x + rsa.y);
  }
  FMHA_STAMP(tr, 1);
  if (j > 0) {
    mbar_wait(o_done, no & 1);  // PV_{j-1} done: O stable, P buffer free
    ++no;
    tc_fence_after();
    FMHA_STAMP(tr, 2);
    if (__any_sync(0xffffffffu, bump)) {
      const float a = bump ? alpha : 1.f;
#pragma unroll
      for (int c = 0; c < DP / 16; ++c) {
        uint32_t o[16];
        tmem_ld16(tO + lane_off + c * 16, o);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
        tmem_st16(tO + lane_off + c * 16, o);
      }
      tmem_st_wait();
    }
  }
  if (store_pending && *store_pending) {  // previous item's O TMA store must have read the P buffer
    if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
    named_bar_sync(bar_id, 128);
    *store_pending = 0;
  }
  // P (bf16) -> smem, SW128 K-major: 16-B chunk c of row r at chunk position c ^ (r & 7)
#ifdef DSP_P_GENERIC_STORE
  uint8_t* prow = sP + row * 128;
#pragma unroll
  for (int c = 0; c < 16; ++c)
    *reinterpret_cast<uint4*>(prow + (c >> 3) * 16384 + (((c & 7) ^ (row & 7)) << 4)) =
        make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
#else
  const uint32_t prow = smem_u32(sP) + row * 128;
#pragma unroll
  for (int c = 0; c < 16; ++c)
    st_shared_v4(prow + (c >> 3) * 16384 + (((c & 7) ^ (row & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                 pk[4 * c + 3]);
#endif
  fence_proxy_async_smem();
  FMHA_STAMP(tr, 12);
  tc_fence_before();
}

// Epilogue through TMA: O / l -> bf16 -> smem staging tile in the TMA box layout (the SW128
// 64-column chunks, then the SW32 / SW64 remainder), fence, named barrier over the 128
// threads of the tile, one elected thread issues the bulk tensor stores (columns >= Dh and
// padding rows are out of bounds and not written).  `o_free` is arrived as soon as O has
// been read from TMEM.  The staging buffer may only be rewritten after
// bulk_wait_group_read0() (tracked by store_pending).
template <int NA, int RB, int LCOL = -1>  // LCOL >= 0: the row sum l is O's column LCOL (ones column of V)
__device__ __forceinline__ void epilogue_tma_store(const FmhaParams& p, const CUtensorMap* to_a,
                                                   const CUtensorMap* to_b, uint8_t* stage, uint32_t tO,
                                                   uint32_t lane_off, int row, float l, uint32_t bar_id,
                                                   const TileCoord& t, uint64_t* o_free, int& store_pending,
                                                   float m) {
  constexpr int DP = NA * 64 + RB;
  const uint32_t st0 = smem_u32(stage);
  uint32_t ov[DP];  // all TMEM loads in flight before one wait
#pragma unroll
  for (int c = 0; c < DP / 16; ++c) tmem_ld16(tO + lane_off + c * 16, *reinterpret_cast<uint32_t(*)[16]>(ov + c * 16));
  tmem_ld_wait();
  const float lsum = LCOL >= 0 ? __uint_as_float(ov[LCOL < 0 ? 0 : LCOL]) : l;
  const float inv_l = 1.f / lsum;
  if (p.lse) {  // training: P = exp2(s * scale_log2 - lse2) reproduces this row's softmax (m, l consistent)
    const long tok = row_token(p, t, row);
    if (tok >= 0) p.lse[tok * p.NH + t.h] = m + __log2f(lsum);
  }
#pragma unroll
  for (int c = 0; c < DP / 16; ++c) {
    const uint32_t* o = ov + c * 16;
#pragma unroll
    for (int h8 = 0; h8 < 2; ++h8) {
      const int d = c * 16 + h8 * 8;
      const uint32_t* w = o + h8 * 8;
      const uint32_t a0 = pack_bf16x2(__uint_as_float(w[0]) * inv_l, __uint_as_float(w[1]) * inv_l);
      const uint32_t a1 = pack_bf16x2(__uint_as_float(w[2]) * inv_l, __uint_as_float(w[3]) * inv_l);
      const uint32_t a2 = pack_bf16x2(__uint_as_float(w[4]) * inv_l, __uint_as_float(w[5]) * inv_l);
      const uint32_t a3 = pack_bf16x2(__uint_as_float(w[6]) * inv_l, __uint_as_float(w[7]) * inv_l);
      uint32_t addr;
      if (d < NA * 64) {
        const int blk = d >> 6, ch = (d & 63) >> 3;
        addr = st0 + blk * 16384 + row * 128 + ((ch ^ (row & 7)) << 4);
      } else {
        const int ch = (d - NA * 64) >> 3;  // RB = 16: SW32 (2 chunks/row), RB = 32: SW64 (4 chunks/row)
        addr = RB == 16 ? st0 + NA * 16384 + row * 32 + ((ch ^ ((row >> 2) & 1)) << 4)
                        : st0 + NA * 16384 + row * 64 + ((ch ^ ((row >> 1) & 3)) << 4);
      }
      st_shared_v4(addr, a0, a1, a2, a3);
    }
  }
  tc_fence_before();
  mbar_arrive(o_free);
  fence_proxy_async_smem();
  named_bar_sync(bar_id, 128);
  if ((threadIdx.x & 127) == 0) {
#pragma unroll
    for (int i = 0; i < NA; ++i) tma_store_5d(to_a, stage + i * 16384, 64 * i, t.h, t.x2, t.x3, t.x4);
    if (RB) tma_store_5d(to_b, stage + NA * 16384, 64 * NA, t.h, t.x2, t.x3, t.x4);
    bulk_commit_group();
  }
  store_pending = 1;
}

// Block-diagonal tiles (G sequences of length L < 128 per tile, rows sequence-major): this
// thread's keys are the columns [lo, lo + L) of its diagonal block, inside the warp's 32-
// or 64-column window.  Single pass from registers, range-compare mask (no division), the
// full P row is written (zeros outside the block) so the buffer can stage O afterwards.
// PT: P goes to tensor memory instead (columns [0, 64) of this lane's S row, two bf16 per
// column: the A operand of a TS-form P.V), so the shared tile only stages O.
template <int W, bool PT>  // window width: 32 or 64 columns
__device__ __forceinline__ void softmax_tile_diag(const SoftmaxGeom& G, uint32_t tS, uint8_t* sP, float& m, float& l,
                                                  int* store_pending, uint32_t bar_id) {
  const int row = G.row;
  const int lo = G.my_blk * G.L, hi = lo + G.L;
  constexpr int wcols = W;
  uint32_t v[64];
  tmem_ld32(tS + G.lane_off + G.wc0, *reinterpret_cast<uint32_t(*)[32]>(v + 0));
  if (wcols > 32) tmem_ld32(tS + G.lane_off + G.wc0 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
  tmem_ld_wait();
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const int col = G.wc0 + i;
    if (i < wcols && col >= lo && col < hi) mx = fmaxf(mx, __uint_as_float(v[i]));
  }
  const float m_new = mx * G.sl2;
  float rs = 0.f;
  uint32_t pk[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c0 = G.wc0 + 2 * i;
    const float x0 = (2 * i < wcols && c0 >= lo && c0 < hi) ? fmaf(__uint_as_float(v[2 * i]), G.sl2, -m_new) : -INFINITY;
    const float x1 = (2 * i + 1 < wcols && c0 + 1 >= lo && c0 + 1 < hi)
                         ? fmaf(__uint_as_float(v[2 * i + 1]), G.sl2, -m_new) : -INFINITY;
    const float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
    rs += e0 + e1;
    pk[i] = pack_bf16x2(e0, e1);
  }
  m = m_new;
  l = rs;
  if (PT) {  // packed column c holds keys 2c, 2c+1; 32-key chunks outside the window are zero
    const int wch = G.wc0 >> 5;
    const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int ch = 0; ch < 4; ++ch)
      if (ch < wch || ch >= wch + W / 32) tmem_st16(tS + G.lane_off + ch * 16, z);
    tmem_st16(tS + G.lane_off + wch * 16, *reinterpret_cast<const uint32_t(*)[16]>(pk));
    if (W == 64) tmem_st16(tS + G.lane_off + wch * 16 + 16, *reinterpret_cast<const uint32_t(*)[16]>(pk + 16));
    tmem_st_wait();
    tc_fence_before();
    return;
  }
  if (store_pending && *store_pending) {  // previous item's O TMA store must have read the P buffer
    if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
    named_bar_sync(bar_id, 128);
    *store_pending = 0;
  }
  const uint32_t prow = smem_u32(sP) + row * 128;
  const int c0w = G.wc0 >> 3, ncw = wcols >> 3;  // window = chunks [c0w, c0w + ncw) of 8 keys
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    if (u < ncw) {
      const int c = c0w + u;
      st_shared_v4(prow + (c >> 3) * 16384 + (((c & 7) ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2],
                   pk[4 * u + 3]);
    }
  }
#pragma unroll
  for (int c = 0; c < 16; ++c)  // zeros outside the window
    if (c < c0w || c >= c0w + ncw)
      st_shared_v4(prow + (c >> 3) * 16384 + (((c & 7) ^ (row & 7)) << 4), 0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  tc_fence_before();
}

// O / l -> bf16 -> o[tok, h*Dh + d] for this thread's row (after the last PV completed).
template <int DP>
__device__ __forceinline__ void store_o(const FmhaParams& p, const TileCoord& t, int row, uint32_t tO,
                                        uint32_t lane_off, float l) {
  const long tok = row_token(p, t, row);
  const float inv_l = 1.f / l;
  __nv_bfloat16* orow = p.o + tok * p.C + t.h * p.Dh;
#pragma unroll
  for (int c = 0; c < DP / 16; ++c) {
    uint32_t v[16];
    tmem_ld16(tO + lane_off + c * 16, v);
    tmem_ld_wait();
    if (tok >= 0) {
#pragma unroll
      for (int h8 = 0; h8 < 2; ++h8) {
        const int d = c * 16 + h8 * 8;
        if (d < p.Dh) {
          const uint32_t* w = v + h8 * 8;
          uint4 o4 = make_uint4(pack_bf16x2(__uint_as_float(w[0]) * inv_l, __uint_as_float(w[1]) * inv_l),
                                pack_bf16x2(__uint_as_float(w[2]) * inv_l, __uint_as_float(w[3]) * inv_l),
                                pack_bf16x2(__uint_as_float(w[4]) * inv_l, __uint_as_float(w[5]) * inv_l),
                                pack_bf16x2(__uint_as_float(w[6]) * inv_l, __uint_as_float(w[7]) * inv_l));
          *reinterpret_cast<uint4*>(orow + d) = o4;
        }
      }
    }
  }
}

#ifdef DSP_FMHA_P_SMEM
constexpr bool kFmhaPTmem = false;  // A/B: block-diagonal P through shared memory (SS-form P.V)
#else
constexpr bool kFmhaPTmem = true;
#endif

template <int NA, int RB>
__global__ void __launch_bounds__(256, FmhaCfg<NA, RB>::CTAS_PER_SM)
    fmha_bf16_tc_kernel(const __grid_constant__ CUtensorMap tq_a, const __grid_constant__ CUtensorMap tq_b,
                        const __grid_constant__ CUtensorMap tk_a, const __grid_constant__ CUtensorMap tk_b,
                        const __grid_constant__ CUtensorMap tv_a, const __grid_constant__ CUtensorMap tv_b,
                        const __grid_constant__ CUtensorMap to_a, const __grid_constant__ CUtensorMap to_b,
                        const FmhaParams p) {
  using Cfg = FmhaCfg<NA, RB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();  // layout assumes a 1024-B aligned base
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::TILE;
  uint8_t* sV = sK + Cfg::TILE;      // 2 stages
  uint8_t* sP = sV + 2 * Cfg::TILE;  // 2 x [128 rows x 128 B] SW128, K-major
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + Cfg::P_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = bars + 3;
  uint64_t* v_full = bars + 4;   // [2]
  uint64_t* v_empty = bars + 6;  // [2]
  uint64_t* s_full = bars + 8;
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint64_t* o_free = bars + 11;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = warp_id();
  const int n = p.n_kv;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tq_a); tma_prefetch(&tk_a); tma_prefetch(&tv_a);
    if (RB) { tma_prefetch(&tq_b); tma_prefetch(&tk_b); tma_prefetch(&tv_b); }
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    mbar_init(o_free, 128);
    fence_barrier_init();
  }
  if (warp >= 4) {  // P starts (and, outside the diagonal blocks, stays) zero
    uint4* pz = reinterpret_cast<uint4*>(sP);
    for (int i = threadIdx.x - 128; i < Cfg::P_BYTES / 16; i += 128) pz[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  if (warp == 2) {
    tmem_alloc(tmem_holder, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  griddep_launch_dependents();
  griddep_wait();
  clk_start(p.clk);
  const uint32_t tS = tmem;        // 128 columns
  const uint32_t tO = tmem + 128;  // DP columns

  // two CTAs per SM: launch allocation 128 regs x 256 threads; 56 x 128 + 200 x 128 == 128 x 256
  // (the softmax warps hold a whole 128-key S row in registers on the non-diagonal path)
  if (warp == 0) {
    if constexpr (Cfg::CTAS_PER_SM == 2) setmaxnreg_dec<56>();
    if (elect_one()) {
      uint32_t nq = 0, nk = 0, nv = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        mbar_wait(q_empty, (nq & 1) ^ 1);
        ++nq;
        mbar_arrive_expect_tx(q_full, Cfg::TX);
        load_tile<NA, RB>(sQ, &tq_a, &tq_b, q_full, tile_coord(p, item, -1));
        for (int j = 0; j < n; ++j) {
          const TileCoord t = tile_coord(p, item, j);
          mbar_wait(k_empty, (nk & 1) ^ 1);
          ++nk;
          mbar_arrive_expect_tx(k_full, Cfg::TX);
          load_tile<NA, RB>(sK, &tk_a, &tk_b, k_full, t);
          const int vs = nv & 1;  // V is double-buffered: V_{j+1} streams in while PV_j runs
          mbar_wait(&v_empty[vs], ((nv >> 1) & 1) ^ 1);
          ++nv;
          mbar_arrive_expect_tx(&v_full[vs], Cfg::TX);
          load_tile<NA, RB>(sV + vs * Cfg::TILE, &tv_a, &tv_b, &v_full[vs], t);
        }
      }
    }
  } else if (warp == 1) {
    if constexpr (Cfg::CTAS_PER_SM == 2) setmaxnreg_dec<56>();
    constexpr uint32_t idS = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idPVa = make_idesc_bf16(128, 64, 0, 1);
    constexpr uint32_t idPVb = make_idesc_bf16(128, RB == 0 ? 16 : RB, 0, 1);
    const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV), p0 = smem_u32(sP);
    const bool p_tmem = kFmhaPTmem && p.G > 1;  // block-diagonal tiles (n == 1): P in TMEM
    uint32_t nq = 0, nk = 0, nv = 0, np = 0, nit = 0;
    auto issue_s = [&]() {
      mbar_wait(k_full, nk & 1);
      ++nk;
      tc_fence_after();
      if (elect_one()) {
        int step = 0;
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k, ++step)
            umma_bf16_ss(tS, make_sdesc(q0 + i * 16384 + k * 32, 16, 1024, SW_128B),
                         make_sdesc(k0 + i * 16384 + k * 32, 16, 1024, SW_128B), idS, step != 0);
        if (RB) {
#pragma unroll
          for (int k = 0; k < RB / 16; ++k, ++step)
            umma_bf16_ss(tS, make_sdesc(q0 + NA * 16384 + k * 32, 16, 8 * Cfg::RB_ROW, Cfg::RB_SW),
                         make_sdesc(k0 + NA * 16384 + k * 32, 16, 8 * Cfg::RB_ROW, Cfg::RB_SW), idS, step != 0);
        }
        umma_commit(s_full);
        umma_commit(k_empty);
      }
      __syncwarp();
    };
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++nit) {
      mbar_wait(q_full, nq & 1);
      ++nq;
      issue_s();
      if (n == 1 && elect_one()) umma_commit(q_empty);
      __syncwarp();
      for (int j = 0; j < n; ++j) {
        mbar_wait(p_full, np & 1);  // softmax consumed S_j and wrote P_j
        ++np;
        if (j + 1 < n) {
          issue_s();
          if (j + 2 == n && elect_one()) umma_commit(q_empty);
          __syncwarp();
        }
        const int vs = nv & 1;
        mbar_wait(&v_full[vs], (nv >> 1) & 1);
        ++nv;
        if (j == 0) mbar_wait(o_free, (nit & 1) ^ 1);  // previous item's epilogue has read O
        tc_fence_after();
        if (elect_one()) {
          const uint32_t vb = v0 + vs * Cfg::TILE;
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // 128 keys in steps of 16
            const uint64_t bdr = make_sdesc(vb + NA * 16384 + k * 16 * Cfg::RB_ROW, 16384, 8 * Cfg::RB_ROW, Cfg::RB_SW);
            if (p_tmem) {  // P_j in TMEM (S columns [0, 64)): 8 packed columns per 16 keys
#pragma unroll
              for (int i = 0; i < NA; ++i)
                umma_bf16_ts(tO + 64 * i, tS + 8 * k, make_sdesc(vb + i * 16384 + k * 2048, 16384, 1024, SW_128B), idPVa,
                             (j | k) != 0);
              if (RB) umma_bf16_ts(tO + 64 * NA, tS + 8 * k, bdr, idPVb, (j | k) != 0);
            } else {
              const uint64_t ad = make_sdesc(p0 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SW_128B);
#pragma unroll
              for (int i = 0; i < NA; ++i)
                umma_bf16_ss(tO + 64 * i, ad, make_sdesc(vb + i * 16384 + k * 2048, 16384, 1024, SW_128B), idPVa,
                             (j | k) != 0);
              if (RB) umma_bf16_ss(tO + 64 * NA, ad, bdr, idPVb, (j | k) != 0);
            }
          }
          umma_commit(o_done);
          umma_commit(&v_empty[vs]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    if constexpr (Cfg::CTAS_PER_SM == 2) setmaxnreg_dec<56>();
  } else {
    if constexpr (Cfg::CTAS_PER_SM == 2) setmaxnreg_inc<200>();
    const SoftmaxGeom G = make_geom(p, warp, p.scale_log2);
    uint32_t ns = 0, no = 0;
    int store_pending = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      float m = -INFINITY, l = 0.f;
      unsigned long long* tr = p.trace ? p.trace + ((size_t)(ns & 127) * 16) : nullptr;
      FMHA_STAMP(tr, 0);
      for (int j = 0; j < n; ++j) {
        mbar_wait(s_full, ns & 1);
        ++ns;
        tc_fence_after();
        FMHA_STAMP(tr, 1);
        if (G.diag) {  // n == 1 in this mode
          if (G.nhalf * G.hcols > 32) softmax_tile_diag<64, kFmhaPTmem>(G, tS, sP, m, l, &store_pending, 1);
          else softmax_tile_diag<32, kFmhaPTmem>(G, tS, sP, m, l, &store_pending, 1);
        } else {
          // whole S row in registers, MUFU + FMA-pipe exp2 (the pair kernel's softmax)
          softmax_tile_full<Cfg::DP, false>(G, tS, tO, sP, j, m, l, o_done, no, nullptr, nullptr, &store_pending, 1,
                                            j + 1 == n ? p.kv_last : 128);
        }
        FMHA_STAMP(tr, 2);
        mbar_arrive(p_full);
      }
      if (kFmhaPTmem && G.diag && store_pending) {  // the staging tile only holds O: free it here
        if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
        named_bar_sync(1, 128);
        store_pending = 0;
      }
      mbar_wait(o_done, no & 1);
      ++no;
      tc_fence_after();
      FMHA_STAMP(tr, 3);
      epilogue_tma_store<NA, RB>(p, &to_a, &to_b, sP, tO, G.lane_off, G.row, l, 1, tile_coord(p, item, -1), o_free,
                                 store_pending, m);
      FMHA_STAMP(tr, 4);
    }
    if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
  }

  tc_fence_before();
  __syncthreads();
  clk_end(p.clk);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------------------------
// Long sequences (L % 256 == 0): one CTA per SM works on TWO 128-row query tiles
// ("slots") of the same (sequence, head), sharing one K/V stream (2-stage ring).  TMEM
// (512 columns) holds S0, S1 (128 columns each) and O0, O1.  One softmax warpgroup per slot,
// thread = query row with the whole 128-key S row in registers; the tensor pipe runs
// S_{j+1} of a slot as soon as that slot holds S_j in registers, then both P_j V_j.
// ONES (Dh <= DP - 8): the row sums come from the tensor core (R31), see softmax_tile_full.
//   warp 0       TMA producer        warp 1       MMA issuer + TMEM allocator
//   warp 2       V patcher (ONES)    warp 3       idle
//   warps 4-7    slot 0 softmax      warps 8-11   slot 1 softmax
template <int NA, int RB>
struct PairCfg {
  using Base = FmhaCfg<NA, RB>;
  static constexpr int TILE = Base::TILE, TX = Base::TX, DP = Base::DP, P_BYTES = Base::P_BYTES;
  static constexpr int RED_BYTES = 2 * 2 * 2 * 128 * 4;   // [max | sum][slot][half][row] floats
  static constexpr int SMEM = 1024 + 6 * TILE /*Q0,Q1,K x2,V x2*/ + 2 * P_BYTES + RED_BYTES + 256;
  static constexpr bool OK = SMEM <= 227 * 1024;
  static constexpr int THREADS = 384;
};

template <int NA, int RB, bool ONES>
__global__ void __launch_bounds__(384, 1)
    fmha_pair_kernel(const __grid_constant__ CUtensorMap tq_a, const __grid_constant__ CUtensorMap tq_b,
                     const __grid_constant__ CUtensorMap tk_a, const __grid_constant__ CUtensorMap tk_b,
                     const __grid_constant__ CUtensorMap tv_a, const __grid_constant__ CUtensorMap tv_b,
                     const __grid_constant__ CUtensorMap to_a, const __grid_constant__ CUtensorMap to_b,
                     const FmhaParams p) {
  using Cfg = PairCfg<NA, RB>;
  using Base = FmhaCfg<NA, RB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                       // 2 tiles
  uint8_t* sK = sQ + 2 * Cfg::TILE;         // 2 stages
  uint8_t* sV = sK + 2 * Cfg::TILE;         // 2 stages
  uint8_t* sP = sV + 2 * Cfg::TILE;         // 2 x 32 KB
  float* red = reinterpret_cast<float*>(sP + 2 * Cfg::P_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * Cfg::P_BYTES + Cfg::RED_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;    // [2]
  uint64_t* k_empty = bars + 4;   // [2]
  uint64_t* v_full = bars + 6;    // [2]
  uint64_t* v_empty = bars + 8;   // [2]
  uint64_t* s_full = bars + 10;   // [2] per slot
  uint64_t* p_full = bars + 12;   // [2]
  uint64_t* o_done = bars + 14;   // [2]
  uint64_t* o_free = bars + 16;   // [2]
  uint64_t* s_free = bars + 18;   // [2] S row fully in registers
  uint64_t* v_ready = bars + 20;  // [2] ONES: V tile patched with its ones column
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 22);

  const int warp = warp_id();
  const int n = p.n_kv;
  const int npairs = p.items / 2;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tq_a); tma_prefetch(&tk_a); tma_prefetch(&tv_a);
    if (RB) { tma_prefetch(&tq_b); tma_prefetch(&tk_b); tma_prefetch(&tv_b); }
    for (int i = 0; i < 12; ++i) mbar_init(&bars[i], 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&p_full[t], 128);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_free[t], 128);
      mbar_init(&s_free[t], 128);
      mbar_init(&v_ready[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  griddep_launch_dependents();
  griddep_wait();
  clk_start(p.clk);

  // launch allocation is 168 regs x 384 threads; 56 x 128 + 224 x 256 == 168 x 384 exactly
  if (warp == 0) {
    setmaxnreg_dec<56>();
    if (elect_one()) {
      uint32_t nq = 0, kv = 0;
      for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
        mbar_wait_sleep(q_empty, (nq & 1) ^ 1);
        ++nq;
        mbar_arrive_expect_tx(q_full, 2 * Cfg::TX);
        load_tile<NA, RB>(sQ, &tq_a, &tq_b, q_full, tile_coord(p, 2 * ip, -1));
        load_tile<NA, RB>(sQ + Cfg::TILE, &tq_a, &tq_b, q_full, tile_coord(p, 2 * ip + 1, -1));
        for (int j = 0; j < n; ++j, ++kv) {
          const int st = kv & 1;
          const uint32_t ph = (kv >> 1) & 1;
          const TileCoord t = tile_coord(p, 2 * ip, j);
          mbar_wait_sleep(&k_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&k_full[st], Cfg::TX);
          load_tile<NA, RB>(sK + st * Cfg::TILE, &tk_a, &tk_b, &k_full[st], t);
          mbar_wait_sleep(&v_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&v_full[st], Cfg::TX);
          load_tile<NA, RB>(sV + st * Cfg::TILE, &tv_a, &tv_b, &v_full[st], t);
        }
      }
    }
  } else if (warp == 1) {
    setmaxnreg_dec<56>();
    {
      constexpr uint32_t idS = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idPVa = make_idesc_bf16(128, 64, 0, 1);
      constexpr uint32_t idPVb = make_idesc_bf16(128, RB == 0 ? 16 : RB, 0, 1);
      const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV), p0 = smem_u32(sP);
      auto issue_s = [&](int slot, int st) {  // S_slot = Q_slot K^T
        if (elect_one()) {
          const uint32_t qa = q0 + slot * Cfg::TILE, ka = k0 + st * Cfg::TILE, d = tmem + slot * 128;
          int step = 0;
#pragma unroll
          for (int i = 0; i < NA; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k, ++step)
              umma_bf16_ss(d, make_sdesc(qa + i * 16384 + k * 32, 16, 1024, SW_128B),
                           make_sdesc(ka + i * 16384 + k * 32, 16, 1024, SW_128B), idS, step != 0);
          if (RB) {
#pragma unroll
            for (int k = 0; k < RB / 16; ++k, ++step)
              umma_bf16_ss(d, make_sdesc(qa + NA * 16384 + k * 32, 16, 8 * Base::RB_ROW, Base::RB_SW),
                           make_sdesc(ka + NA * 16384 + k * 32, 16, 8 * Base::RB_ROW, Base::RB_SW), idS, step != 0);
          }
          umma_commit(&s_full[slot]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int slot, int st, bool acc0) {  // O_slot (+)= P_slot V
        if (elect_one()) {
          const uint32_t pa = p0 + slot * Cfg::P_BYTES, va = v0 + st * Cfg::TILE, o = tmem + 256 + slot * 128;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t ad = make_sdesc(pa + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SW_128B);
#pragma unroll
            for (int i = 0; i < NA; ++i)
              umma_bf16_ss(o + 64 * i, ad, make_sdesc(va + i * 16384 + k * 2048, 16384, 1024, SW_128B), idPVa,
                           acc0 || k != 0);
            if (RB)
              umma_bf16_ss(o + 64 * NA, ad,
                           make_sdesc(va + NA * 16384 + k * 16 * Base::RB_ROW, 16384, 8 * Base::RB_ROW, Base::RB_SW),
                           idPVb, acc0 || k != 0);
          }
          umma_commit(&o_done[slot]);
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) umma_commit(bar);
        __syncwarp();
      };
      uint32_t nq = 0, np0 = 0, np1 = 0, nf0 = 0, nf1 = 0, nit = 0, kvbase = 0;
      for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x, ++nit, kvbase += n) {
        mbar_wait(q_full, nq & 1);
        ++nq;
        const uint32_t kv0 = kvbase;
        mbar_wait(&k_full[kv0 & 1], (kv0 >> 1) & 1);
        tc_fence_after();
        issue_s(0, kv0 & 1);
        issue_s(1, kv0 & 1);
        commit(&k_empty[kv0 & 1]);
        if (n == 1) commit(q_empty);
        for (int j = 0; j < n; ++j) {
          const uint32_t kj = kvbase + j, kn = kj + 1;
          // S_{j+1} as soon as each slot has S_j in registers (overlaps its exp phase) ...
          if (j + 1 < n) {
            mbar_wait(&s_free[0], nf0 & 1);
            mbar_wait(&k_full[kn & 1], (kn >> 1) & 1);
            tc_fence_after();
            issue_s(0, kn & 1);
            mbar_wait(&s_free[1], nf1 & 1);
            tc_fence_after();
            issue_s(1, kn & 1);
            commit(&k_empty[kn & 1]);
            if (j + 2 == n) commit(q_empty);
          }
          ++nf0;
          ++nf1;
          // ... then O += P_j V_j once each slot has stored P_j
          mbar_wait(&p_full[0], np0 & 1);
          ++np0;
          mbar_wait(ONES ? &v_ready[kj & 1] : &v_full[kj & 1], (kj >> 1) & 1);
          if (j == 0) mbar_wait(&o_free[0], (nit & 1) ^ 1);
          tc_fence_after();
          issue_pv(0, kj & 1, j > 0);
          mbar_wait(&p_full[1], np1 & 1);
          ++np1;
          if (j == 0) mbar_wait(&o_free[1], (nit & 1) ^ 1);
          tc_fence_after();
          issue_pv(1, kj & 1, j > 0);
          commit(&v_empty[kj & 1]);
        }
      }
    }
  } else if (warp < 4) {
    setmaxnreg_dec<56>();
    if (ONES && warp == 2) {
      // V patcher: once a V tile has landed, set its column DP - 8 (zero-filled padding, since
      // Dh <= DP - 8) to 1.0 in every row, so P.V also produces the row sums (see softmax_tile_full)
      constexpr int CB = (RB - 8) * 2;  // byte offset of the ones column inside the RB chunk row
      uint32_t kv = 0;
      for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
        for (int j = 0; j < n; ++j, ++kv) {
          const int st = kv & 1;
          mbar_wait(&v_full[st], (kv >> 1) & 1);
          const uint32_t vb = smem_u32(sV + st * Cfg::TILE) + NA * 16384;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = lane_id() + 32 * i;
            const uint32_t ch = RB == 16 ? ((CB >> 4) ^ ((r >> 2) & 1)) : ((CB >> 4) ^ ((r >> 1) & 3));
            st_shared_u16(vb + r * Base::RB_ROW + (ch << 4) + (CB & 15), 0x3F80);  // bf16 1.0
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&v_ready[st]);
        }
      }
    }
  } else {
    setmaxnreg_inc<224>();
    const int slot = (warp - 4) >> 2;
    const SoftmaxGeom G = make_geom(p, warp, p.scale_log2);
    const uint32_t tS = tmem + slot * 128, tO = tmem + 256 + slot * 128;
    uint8_t* sPs = sP + slot * Cfg::P_BYTES;
    const uint32_t bar_id = 1 + slot;
    const bool store_leader = (threadIdx.x & 127) == 0;
    int store_pending = 0;
    uint32_t ns = 0, no = 0;
    for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n; ++j) {
        unsigned long long* tr = p.trace ? p.trace + ((size_t)(slot * 64 + (ns & 63)) * 16) : nullptr;
        FMHA_STAMP(tr, 0);
        mbar_wait(&s_full[slot], ns & 1);
        ++ns;
        tc_fence_after();
        FMHA_STAMP(tr, 3);
        softmax_tile_full<Cfg::DP, ONES>(G, tS, tO, sPs, j, m, l, &o_done[slot], no, tr, &s_free[slot], &store_pending,
                                         bar_id, j + 1 == n ? p.kv_last : 128);
        FMHA_STAMP(tr, 4);
        mbar_arrive(&p_full[slot]);
      }
      unsigned long long* te = p.trace ? p.trace + ((size_t)(slot * 64 + ((ns - 1) & 63)) * 16) : nullptr;
      FMHA_STAMP(te, 5);
      mbar_wait(&o_done[slot], no & 1);  // last PV done: O final, P buffer free
      ++no;
      tc_fence_after();
      FMHA_STAMP(te, 6);
      epilogue_tma_store<NA, RB, ONES ? Cfg::DP - 8 : -1>(p, &to_a, &to_b, sPs, tO, G.lane_off, G.row, l, bar_id,
                                 tile_coord(p, 2 * ip + slot, -1), &o_free[slot], store_pending, m);
      FMHA_STAMP(te, 7);
    }
    if (store_leader) bulk_wait_group_read0();
  }

  tc_fence_before();
  __syncthreads();
  clk_end(p.clk);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------
// Long sequences, P in tensor memory (the production spatial kernel; DSP_FMHA_PAIR_SMEM builds
// the shared-memory-P pair kernel above for A/B).  Same roles and two query tiles ("slots")
// per CTA as fmha_pair_kernel, but each slot's P_j (bf16) overwrites the first 64 columns of its
// own S_j in TMEM and P.V is the TS form (A = P from TMEM, B = V from smem).  Shared memory then
// carries only the TMA tiles and the MMA's Q / K / V operand reads: the pair kernel's 64 KB of P
// stores plus 64 KB of P operand reads per K/V step (more than the K/V/Q traffic itself) are
// gone.  Because P_j aliases S_j, S_{j+1} of a slot is issued right after PV_j of that slot;
// the MMA warp alternates slots (PV0_j, S0_{j+1}, PV1_j, S1_{j+1}), so one slot's exponentials
// overlap the other slot's tensor work (ping-pong).  When a slot sees S_j, every earlier MMA of
// the CTA has completed (tcgen05.commit tracks all prior MMAs), so PV_{j-1} is done: O can be
// rescaled in place and S's columns may be overwritten by P_j without further waits.
// TMEM: S0 [0,128), S1 [128,256), O0 [256, 256+DP), O1 [384, 384+DP).  ONES only (the row sums
// come from V's ones column, R31).
template <int NA, int RB>
struct PtCfg {
  using Base = FmhaCfg<NA, RB>;
  static constexpr int TILE = Base::TILE, TX = Base::TX, DP = Base::DP;
  static constexpr int KV_STAGES = 2;
  // Q0,Q1 | K x stages | V x stages | O staging x 2 | barriers
  static constexpr int SMEM = 1024 + (2 + 2 * KV_STAGES + 2) * TILE + 256;
  static constexpr bool OK = SMEM <= 227 * 1024 && RB > 0;
  static constexpr int THREADS = 384;
};

#ifndef DSP_PT_POLY_NUM
#define DSP_PT_POLY_NUM DSP_POLY_NUM
#endif

// One online-softmax step of the P-in-TMEM kernel (thread = query row, whole 128-key row):
// S_j -> registers, row max, lazy O rescale (R28), P_j = exp2(S*scale - m) as bf16 into TMEM
// columns [0, 64) of the same S tile (packed column c = keys 2c, 2c+1), chunk by chunk as the
// exponentials are produced.  valid < 128: keys >= valid are padding (masked to -inf).
template <int DP>
__device__ __forceinline__ void softmax_step_pt(const SoftmaxGeom& G, uint32_t tS, uint32_t tO, int j, float& m,
                                                int valid, unsigned long long* tr = nullptr) {
  const uint32_t lane_off = G.lane_off;
  const float sl2 = G.sl2;
  uint32_t v[128];
  tmem_ld32(tS + lane_off + 0, *reinterpret_cast<uint32_t(*)[32]>(v + 0));
  tmem_ld32(tS + lane_off + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
  tmem_ld32(tS + lane_off + 64, *reinterpret_cast<uint32_t(*)[32]>(v + 64));
  tmem_ld32(tS + lane_off + 96, *reinterpret_cast<uint32_t(*)[32]>(v + 96));
  tmem_ld_wait();
  FMHA_STAMP(tr, 8);
  if (valid < 128) {
#pragma unroll
    for (int i = 0; i < 128; ++i)
      if (i >= valid) v[i] = __float_as_uint(-INFINITY);
  }
  const float mx = max_tree3<128>(reinterpret_cast<const float*>(v));
  const float mx2 = mx * sl2;
  const bool bump = (j == 0) || (mx2 > m + 8.f);
  const float m_new = bump ? mx2 : m;
  const float alpha = (j == 0) ? 0.f : fast_exp2(m - m_new);
  m = m_new;
  FMHA_STAMP(tr, 9);
  if (j > 0 && __any_sync(0xffffffffu, bump)) {  // PV_{j-1} completed before S_j: O is stable
    const float a = bump ? alpha : 1.f;
#pragma unroll
    for (int c = 0; c < DP / 16; ++c) {
      uint32_t o[16];
      tmem_ld16(tO + lane_off + c * 16, o);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
      tmem_st16(tO + lane_off + c * 16, o);
    }
  }
  const float2 sl2x2 = make_float2(sl2, sl2), mx2n = make_float2(-m_new, -m_new);
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {  // 32 keys -> 16 packed P columns per chunk
    uint32_t pk[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = ch * 16 + u;
      const float2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2x2, mx2n);
      float2 e;
#ifdef DSP_PT_SPREAD  // A/B: FMA-pipe pairs spread evenly through each group of DEN
      if ((((i % DSP_POLY_DEN) * DSP_PT_POLY_NUM) % DSP_POLY_DEN) < DSP_PT_POLY_NUM) {
#else
      if ((i % DSP_POLY_DEN) < DSP_PT_POLY_NUM) {
#endif
        e = poly_exp2_x2(x);
      } else {
        e.x = fast_exp2(x.x);
        e.y = fast_exp2(x.y);
      }
      pk[u] = pack_bf16x2(e.x, e.y);
    }
    tmem_st16(tS + lane_off + ch * 16, pk);
  }
  FMHA_STAMP(tr, 11);
  tmem_st_wait();
  FMHA_STAMP(tr, 12);
  tc_fence_before();
}

template <int NA, int RB>
__global__ void __launch_bounds__(384, 1)
    fmha_pt_kernel(const __grid_constant__ CUtensorMap tq_a, const __grid_constant__ CUtensorMap tq_b,
                   const __grid_constant__ CUtensorMap tk_a, const __grid_constant__ CUtensorMap tk_b,
                   const __grid_constant__ CUtensorMap tv_a, const __grid_constant__ CUtensorMap tv_b,
                   const __grid_constant__ CUtensorMap to_a, const __grid_constant__ CUtensorMap to_b,
                   const FmhaParams p) {
  using Cfg = PtCfg<NA, RB>;
  using Base = FmhaCfg<NA, RB>;
  constexpr int KS = Cfg::KV_STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                        // 2 tiles
  uint8_t* sK = sQ + 2 * Cfg::TILE;          // KS stages
  uint8_t* sV = sK + KS * Cfg::TILE;         // KS stages
  uint8_t* sO = sV + KS * Cfg::TILE;         // 2 staging tiles (epilogue)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 2 * Cfg::TILE);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;             // [KS]
  uint64_t* k_empty = k_full + KS;         // [KS]
  uint64_t* v_full = k_empty + KS;         // [KS]
  uint64_t* v_empty = v_full + KS;         // [KS]
  uint64_t* v_ready = v_empty + KS;        // [KS] V patched with its ones column
  uint64_t* s_full = v_ready + KS;         // [2] per slot
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* o_done = p_full + 2;           // [2]
  uint64_t* o_free = o_done + 2;           // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = warp_id();
  const int n = p.n_kv;
  const int npairs = p.items / 2;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tq_a); tma_prefetch(&tk_a); tma_prefetch(&tv_a);
    tma_prefetch(&tq_b); tma_prefetch(&tk_b); tma_prefetch(&tv_b);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); mbar_init(&v_ready[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_free[t], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  griddep_launch_dependents();
  griddep_wait();
  clk_start(p.clk);

  // launch allocation is 168 regs x 384 threads; 56 x 128 + 224 x 256 == 168 x 384 exactly
  if (warp == 0) {
    setmaxnreg_dec<56>();
    if (elect_one()) {
      uint32_t nq = 0, kv = 0;
      for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
        mbar_wait_sleep(q_empty, (nq & 1) ^ 1);
        ++nq;
        mbar_arrive_expect_tx(q_full, 2 * Cfg::TX);
        load_tile<NA, RB>(sQ, &tq_a, &tq_b, q_full, tile_coord(p, 2 * ip, -1));
        load_tile<NA, RB>(sQ + Cfg::TILE, &tq_a, &tq_b, q_full, tile_coord(p, 2 * ip + 1, -1));
        for (int j = 0; j < n; ++j, ++kv) {
          const int st = kv % KS;
          const uint32_t ph = (kv / KS) & 1;
          const TileCoord t = tile_coord(p, 2 * ip, j);
          mbar_wait_sleep(&k_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&k_full[st], Cfg::TX);
          load_tile<NA, RB>(sK + st * Cfg::TILE, &tk_a, &tk_b, &k_full[st], t);
          mbar_wait_sleep(&v_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&v_full[st], Cfg::TX);
          load_tile<NA, RB>(sV + st * Cfg::TILE, &tv_a, &tv_b, &v_full[st], t);
        }
      }
    }
  } else if (warp == 1) {
    setmaxnreg_dec<56>();
    constexpr uint32_t idS = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idPVa = make_idesc_bf16(128, 64, 0, 1);
    constexpr uint32_t idPVb = make_idesc_bf16(128, RB, 0, 1);
    const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV);
    auto issue_s = [&](int slot, int st) {  // S_slot = Q_slot K^T
      if (elect_one()) {
        const uint32_t qa = q0 + slot * Cfg::TILE, ka = k0 + st * Cfg::TILE, d = tmem + slot * 128;
        int step = 0;
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k, ++step)
            umma_bf16_ss(d, make_sdesc(qa + i * 16384 + k * 32, 16, 1024, SW_128B),
                         make_sdesc(ka + i * 16384 + k * 32, 16, 1024, SW_128B), idS, step != 0);
#pragma unroll
        for (int k = 0; k < RB / 16; ++k, ++step)
          umma_bf16_ss(d, make_sdesc(qa + NA * 16384 + k * 32, 16, 8 * Base::RB_ROW, Base::RB_SW),
                       make_sdesc(ka + NA * 16384 + k * 32, 16, 8 * Base::RB_ROW, Base::RB_SW), idS, step != 0);
        umma_commit(&s_full[slot]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int slot, int st, bool acc0) {  // O_slot (+)= P_slot V (P from TMEM)
      if (elect_one()) {
        const uint32_t va = v0 + st * Cfg::TILE, o = tmem + 256 + slot * 128, ps = tmem + slot * 128;
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 keys = 8 packed P columns per step
#pragma unroll
          for (int i = 0; i < NA; ++i)
            umma_bf16_ts(o + 64 * i, ps + 8 * k, make_sdesc(va + i * 16384 + k * 2048, 16384, 1024, SW_128B), idPVa,
                         acc0 || k != 0);
          umma_bf16_ts(o + 64 * NA, ps + 8 * k,
                       make_sdesc(va + NA * 16384 + k * 16 * Base::RB_ROW, 16384, 8 * Base::RB_ROW, Base::RB_SW),
                       idPVb, acc0 || k != 0);
        }
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    uint32_t nq = 0, np0 = 0, np1 = 0, nit = 0, kvbase = 0;
    for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x, ++nit, kvbase += n) {
      mbar_wait(q_full, nq & 1);
      ++nq;
      {
        const uint32_t kv0 = kvbase;
        mbar_wait(&k_full[kv0 % KS], (kv0 / KS) & 1);
        tc_fence_after();
        issue_s(0, kv0 % KS);
        issue_s(1, kv0 % KS);
        commit(&k_empty[kv0 % KS]);
        if (n == 1) commit(q_empty);
      }
      for (int j = 0; j < n; ++j) {
        const uint32_t kj = kvbase + j, kn = kj + 1;
        const int sj = kj % KS, sn = kn % KS;
        // slot 0: O0 += P0_j V_j, then S0_{j+1} into the same TMEM (after PV0_j in issue order)
        mbar_wait(&p_full[0], np0 & 1);
        ++np0;
        mbar_wait(&v_ready[sj], (kj / KS) & 1);
        if (j == 0) mbar_wait(&o_free[0], (nit & 1) ^ 1);
        tc_fence_after();
        issue_pv(0, sj, j > 0);
        if (j + 1 == n) commit(&o_done[0]);
        if (j + 1 < n) {
          mbar_wait(&k_full[sn], (kn / KS) & 1);
          tc_fence_after();
          issue_s(0, sn);
        }
        // slot 1
        mbar_wait(&p_full[1], np1 & 1);
        ++np1;
        if (j == 0) mbar_wait(&o_free[1], (nit & 1) ^ 1);
        tc_fence_after();
        issue_pv(1, sj, j > 0);
        commit(&v_empty[sj]);
        if (j + 1 == n) commit(&o_done[1]);
        if (j + 1 < n) {
          issue_s(1, sn);
          commit(&k_empty[sn]);
          if (j + 2 == n) commit(q_empty);
        }
      }
    }
  } else if (warp < 4) {
    setmaxnreg_dec<56>();
    if (warp == 2) {
      // V patcher: once a V tile has landed, set its column DP - 8 (zero-filled padding, since
      // Dh <= DP - 8) to 1.0 in every row, so P.V also produces the row sums (R31)
      constexpr int CB = (RB - 8) * 2;  // byte offset of the ones column inside the RB chunk row
      uint32_t kv = 0;
      for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
        for (int j = 0; j < n; ++j, ++kv) {
          const int st = kv % KS;
          mbar_wait(&v_full[st], (kv / KS) & 1);
          const uint32_t vb = smem_u32(sV + st * Cfg::TILE) + NA * 16384;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = lane_id() + 32 * i;
            const uint32_t ch = RB == 16 ? ((CB >> 4) ^ ((r >> 2) & 1)) : ((CB >> 4) ^ ((r >> 1) & 3));
            st_shared_u16(vb + r * Base::RB_ROW + (ch << 4) + (CB & 15), 0x3F80);  // bf16 1.0
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&v_ready[st]);
        }
      }
    }
  } else {
    setmaxnreg_inc<224>();
    const int slot = (warp - 4) >> 2;
    const SoftmaxGeom G = make_geom(p, warp, p.scale_log2);
    const uint32_t tS = tmem + slot * 128, tO = tmem + 256 + slot * 128;
    uint8_t* sOs = sO + slot * Cfg::TILE;
    const uint32_t bar_id = 1 + slot;
    int store_pending = 0;
    uint32_t ns = 0, no = 0;
    for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
      float m = -INFINITY;
      for (int j = 0; j < n; ++j) {
        unsigned long long* tr = p.trace ? p.trace + ((size_t)(slot * 64 + (ns & 63)) * 16) : nullptr;
        FMHA_STAMP(tr, 0);
        mbar_wait(&s_full[slot], ns & 1);
        ++ns;
        tc_fence_after();
        FMHA_STAMP(tr, 3);
        softmax_step_pt<Cfg::DP>(G, tS, tO, j, m, j + 1 == n ? p.kv_last : 128, tr);
        mbar_arrive(&p_full[slot]);
        FMHA_STAMP(tr, 4);
      }
      mbar_wait(&o_done[slot], no & 1);  // last PV done: O final
      ++no;
      tc_fence_after();
      if (store_pending) {  // the previous item's O store must have read the staging tile
        if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
        named_bar_sync(bar_id, 128);
        store_pending = 0;
      }
      epilogue_tma_store<NA, RB, Cfg::DP - 8>(p, &to_a, &to_b, sOs, tO, G.lane_off, G.row, 0.f, bar_id,
                                              tile_coord(p, 2 * ip + slot, -1), &o_free[slot], store_pending, m);
    }
    if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
  }

  tc_fence_before();
  __syncthreads();
  clk_end(p.clk);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------
// Sequences of one 128-row tile (L <= 128 with one sequence per tile: the long video's T = 128
// temporal stage, ragged lengths), self-attention.  Each item (sequence, head) needs its own Q,
// K and V tiles exactly once, gathered by TMA from token rows far apart in HBM (T = 128: 128
// rows S_loc * 6912 B apart per tile), so the kernel is bound by how many bytes it keeps in
// flight: one CTA per SM with a KS-deep ring of {Q, K, V} stages (the loads of the next KS - 1
// items stream in while one is computed), two softmax/epilogue warpgroups ("slots") taking
// alternate items, and per-slot S and O in TMEM so item i + 1's Q K^T runs during item i's
// softmax.  P_i (bf16) overwrites the first 64 columns of its S in TMEM, P.V is the TS form,
// the row sums come from V's ones column (R31).
// TMEM: S0 [0,128), S1 [128,256), O0 [256, 256+DP), O1 [384, 384+DP).
//   warp 0 TMA producer   warp 1 MMA issuer + TMEM allocator   warp 2 V patcher   warp 3 idle
//   warps 4-7 slot 0 (even items)   warps 8-11 slot 1 (odd items)
#ifndef DSP_FMHA_SEQ_DIAG
#define DSP_FMHA_SEQ_DIAG 1  // block-diagonal tiles (T = 16: 8 sequences per tile) on fmha_seq_kernel too
#endif
constexpr bool kSeqDiag = DSP_FMHA_SEQ_DIAG != 0;
template <int NA, int RB>
struct SeqCfg {
  using Base = FmhaCfg<NA, RB>;
  static constexpr int TILE = Base::TILE, TX = Base::TX, DP = Base::DP;
  static constexpr int KS = 3;  // {Q, K, V} stages
  static constexpr int SMEM = 1024 + (3 * KS + 2) * TILE + 256;
  static constexpr bool OK = SMEM <= 227 * 1024 && RB > 0;
  static constexpr int THREADS = 384;
};

template <int NA, int RB>
__global__ void __launch_bounds__(384, 1)
    fmha_seq_kernel(const __grid_constant__ CUtensorMap tq_a, const __grid_constant__ CUtensorMap tq_b,
                    const __grid_constant__ CUtensorMap tk_a, const __grid_constant__ CUtensorMap tk_b,
                    const __grid_constant__ CUtensorMap tv_a, const __grid_constant__ CUtensorMap tv_b,
                    const __grid_constant__ CUtensorMap to_a, const __grid_constant__ CUtensorMap to_b,
                    const FmhaParams p) {
  using Cfg = SeqCfg<NA, RB>;
  using Base = FmhaCfg<NA, RB>;
  constexpr int KS = Cfg::KS, DP = Cfg::DP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQKV = smem;                      // stage st: Q, K, V tiles at (3 * st + part) * TILE
  uint8_t* sO = smem + 3 * KS * Cfg::TILE;   // 2 staging tiles (epilogue), one per slot
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 2 * Cfg::TILE);
  uint64_t* full = bars;                     // [KS] Q, K, V of the stage landed
  uint64_t* empty = full + KS;               // [KS] the stage's P.V has completed
  uint64_t* v_ready = empty + KS;            // [KS] V patched with its ones column
  uint64_t* s_full = v_ready + KS;           // [2] per slot
  uint64_t* p_full = s_full + 2;             // [2] (count 128)
  uint64_t* o_done = p_full + 2;             // [2]
  uint64_t* o_free = o_done + 2;             // [2] (count 128)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = warp_id();

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tq_a); tma_prefetch(&tk_a); tma_prefetch(&tv_a);
    tma_prefetch(&tq_b); tma_prefetch(&tk_b); tma_prefetch(&tv_b);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&v_ready[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_free[t], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  griddep_launch_dependents();
  griddep_wait();
  clk_start(p.clk);

  // launch allocation 168 regs x 384 threads; 56 x 128 + 224 x 256 == 168 x 384
  if (warp == 0) {
    setmaxnreg_dec<56>();
    if (elect_one()) {
      uint32_t k = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++k) {
        const int st = k % KS;
        mbar_wait_sleep(&empty[st], ((k / KS) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], 3 * Cfg::TX);
        uint8_t* b = sQKV + 3 * st * Cfg::TILE;
        load_tile<NA, RB>(b, &tq_a, &tq_b, &full[st], tile_coord(p, item, -1));
        const TileCoord t = tile_coord(p, item, 0);
        load_tile<NA, RB>(b + Cfg::TILE, &tk_a, &tk_b, &full[st], t);
        load_tile<NA, RB>(b + 2 * Cfg::TILE, &tv_a, &tv_b, &full[st], t);
      }
    }
  } else if (warp == 1) {
    setmaxnreg_dec<56>();
    constexpr uint32_t idS = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idPVa = make_idesc_bf16(128, 64, 0, 1);
    constexpr uint32_t idPVb = make_idesc_bf16(128, RB, 0, 1);
    const uint32_t b0 = smem_u32(sQKV);
    // The tensor pipe serves two independent streams -- S of the next item once its tiles have
    // landed, P.V of the previous item once its softmax is done -- so the issuer polls both
    // instead of blocking on one: P.V (which frees a {Q, K, V} stage for the producer) is
    // never held up behind the loads of a later item.
    auto issue_s = [&](uint32_t k) {  // S_slot = Q K^T of the k-th local item
      const int st = k % KS, slot = k & 1;
      tc_fence_after();
      if (elect_one()) {
        const uint32_t qa = b0 + 3 * st * Cfg::TILE, ka = qa + Cfg::TILE, d = tmem + slot * 128;
        int step = 0;
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk, ++step)
            umma_bf16_ss(d, make_sdesc(qa + i * 16384 + kk * 32, 16, 1024, SW_128B),
                         make_sdesc(ka + i * 16384 + kk * 32, 16, 1024, SW_128B), idS, step != 0);
#pragma unroll
        for (int kk = 0; kk < RB / 16; ++kk, ++step)
          umma_bf16_ss(d, make_sdesc(qa + NA * 16384 + kk * 32, 16, 8 * Base::RB_ROW, Base::RB_SW),
                       make_sdesc(ka + NA * 16384 + kk * 32, 16, 8 * Base::RB_ROW, Base::RB_SW), idS, step != 0);
        umma_commit(&s_full[slot]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](uint32_t k) {  // O_slot = P V (P from TMEM), then the stage is free
      const int st = k % KS, slot = k & 1;
      tc_fence_after();
      if (elect_one()) {
        const uint32_t va = b0 + (3 * st + 2) * Cfg::TILE, o = tmem + 256 + slot * 128, ps = tmem + slot * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 keys = 8 packed P columns per step
#pragma unroll
          for (int i = 0; i < NA; ++i)
            umma_bf16_ts(o + 64 * i, ps + 8 * kk, make_sdesc(va + i * 16384 + kk * 2048, 16384, 1024, SW_128B), idPVa,
                         kk != 0);
          umma_bf16_ts(o + 64 * NA, ps + 8 * kk,
                       make_sdesc(va + NA * 16384 + kk * 16 * Base::RB_ROW, 16384, 8 * Base::RB_ROW, Base::RB_SW),
                       idPVb, kk != 0);
        }
        umma_commit(&o_done[slot]);
        umma_commit(&empty[st]);
      }
      __syncwarp();
    };
    const uint32_t nloc = blockIdx.x < (unsigned)p.items ? (p.items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    uint32_t ks = 0, kp = 0;  // next item to issue S for / P.V for (kp <= ks)
    while (kp < nloc) {
      const uint32_t ks0 = ks, kp0 = kp;
      // S of item ks: its tiles landed, and its slot's previous item (ks - 2) has been stored
      // (its P.V done, O read), so S and O of the slot may be overwritten
      if (ks < nloc && ks < kp + 2 && mbar_try_wait(smem_u32(&full[ks % KS]), (ks / KS) & 1) &&
          mbar_try_wait(smem_u32(&o_free[ks & 1]), ((ks >> 1) & 1) ^ 1)) {
        issue_s(ks);
        ++ks;
      }
      if (kp < ks && mbar_try_wait(smem_u32(&p_full[kp & 1]), (kp >> 1) & 1) &&
          mbar_try_wait(smem_u32(&v_ready[kp % KS]), (kp / KS) & 1)) {
        issue_pv(kp);
        ++kp;
      }
      if (ks == ks0 && kp == kp0) __nanosleep(20);  // nothing ready: leave the issue slots to the softmax warps
    }
  } else if (warp < 4) {
    setmaxnreg_dec<56>();
    if (warp == 2) {
      // V patcher: once a V tile has landed, set its column DP - 8 (zero-filled padding, since
      // Dh <= DP - 8) to 1.0 in every row, so P.V also produces the row sums (R31)
      constexpr int CB = (RB - 8) * 2;  // byte offset of the ones column inside the RB chunk row
      uint32_t k = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++k) {
        const int st = k % KS;
        mbar_wait(&full[st], (k / KS) & 1);
        const uint32_t vb = smem_u32(sQKV + (3 * st + 2) * Cfg::TILE) + NA * 16384;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = lane_id() + 32 * i;
          const uint32_t ch = RB == 16 ? ((CB >> 4) ^ ((r >> 2) & 1)) : ((CB >> 4) ^ ((r >> 1) & 3));
          st_shared_u16(vb + r * Base::RB_ROW + (ch << 4) + (CB & 15), 0x3F80);  // bf16 1.0
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&v_ready[st]);
      }
    }
  } else {
    setmaxnreg_inc<224>();
    const int slot = (warp - 4) >> 2;
    const SoftmaxGeom G = make_geom(p, warp, p.scale_log2);
    const uint32_t tS = tmem + slot * 128, tO = tmem + 256 + slot * 128;
    uint8_t* sOs = sO + slot * Cfg::TILE;
    const uint32_t bar_id = 1 + slot;
    int store_pending = 0;
    uint32_t n = 0;
    uint32_t k = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++k) {
      if ((int)(k & 1) != slot) continue;
      mbar_wait(&s_full[slot], n & 1);
      tc_fence_after();
      float m = -INFINITY, l = 0.f;
      if (G.diag) {  // G = 128 / L sequences per tile: each thread only its diagonal block, l in fp32
        if (G.nhalf * G.hcols > 32) softmax_tile_diag<64, true>(G, tS, nullptr, m, l, nullptr, bar_id);
        else softmax_tile_diag<32, true>(G, tS, nullptr, m, l, nullptr, bar_id);
      } else {
        softmax_step_pt<DP>(G, tS, tO, 0, m, p.kv_last);
      }
      mbar_arrive(&p_full[slot]);
      mbar_wait(&o_done[slot], n & 1);  // P.V done: O final
      ++n;
      tc_fence_after();
      if (store_pending) {  // the previous item's O store must have read the staging tile
        if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
        named_bar_sync(bar_id, 128);
        store_pending = 0;
      }
      if (G.diag)
        epilogue_tma_store<NA, RB>(p, &to_a, &to_b, sOs, tO, G.lane_off, G.row, l, bar_id, tile_coord(p, item, -1),
                                   &o_free[slot], store_pending, m);
      else
        epilogue_tma_store<NA, RB, DP - 8>(p, &to_a, &to_b, sOs, tO, G.lane_off, G.row, 0.f, bar_id,
                                           tile_coord(p, item, -1), &o_free[slot], store_pending, m);
    }
    if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
  }

  tc_fence_before();
  __syncthreads();
  clk_end(p.clk);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------
// Long sequences, split-row softmax (an A/B variant, -DDSP_FMHA_SPLIT: at the blk shape it
// measured 110-113 us against fmha_pt_kernel's 101-104 us; 640 threads cap it at 96 registers,
// which spills, and the row max exchange adds a barrier per step).  As fmha_pt_kernel -- two query tiles ("slots") per CTA ping-ponging on the
// tensor pipe, P_j (bf16) over S_j in TMEM, TS-form P.V -- plus:
//  * every query row is exponentiated by TWO threads (one per 64-key half; 16 softmax warps,
//    four warpgroups: slot x half), which halves the per-step dependency chain of the softmax;
//    the two halves agree on the row max through shared memory (one named barrier per slot);
//  * Q lives in TMEM too (copied there once per item by the softmax threads), so S = Q K^T is a
//    TS-form MMA that reads only K from shared memory (the SS form needs 128 B/clk of smem,
//    all of it, at the tensor pipe's rate);
//  * a 3-deep K/V ring, and Q's smem tile is released as soon as it is in TMEM.
// TMEM: S0 [0,128), S1 [128,256), O0 [256,256+DP), Q0 [256+DP, 256+DP*3/2), O1 / Q1 at +128.
// Roles: warp 0 TMA, warp 1 MMA + TMEM alloc, warp 2 V patcher (ones column, R31), warp 3 idle,
// warps 4 + 4*(2*slot + half) .. +3 softmax (TMEM lane quadrant = warp % 4); the half-0
// warpgroup of each slot also runs the epilogue.
template <int NA, int RB>
struct SplitCfg {
  using Base = FmhaCfg<NA, RB>;
  static constexpr int TILE = Base::TILE, TX = Base::TX, DP = Base::DP;
  static constexpr int KV_STAGES = 3;
  static constexpr int RED_BYTES = 2 * 2 * 2 * 128 * 4;  // [parity][slot][half][row] row maxima
  static constexpr int SMEM = 1024 + (2 + 2 * KV_STAGES + 2) * TILE + RED_BYTES + 256;
  static constexpr bool OK = SMEM <= 227 * 1024 && RB > 0 && DP + DP / 2 <= 128;
  static constexpr int THREADS = 640;
};

template <int DP>
__device__ __forceinline__ void softmax_step_split(const SoftmaxGeom& G, int half, uint32_t tS, uint32_t tO, int j,
                                                   float& m, int valid, float* red_mine, const float* red_other,
                                                   uint32_t bar_id, unsigned long long* tr = nullptr) {
  const uint32_t lane_off = G.lane_off;
  const float sl2 = G.sl2;
  const int c0 = half * 64;  // this thread's key columns [c0, c0 + 64)
  uint32_t v[64];
  tmem_ld32(tS + lane_off + c0, *reinterpret_cast<uint32_t(*)[32]>(v + 0));
  tmem_ld32(tS + lane_off + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
  tmem_ld_wait();
  FMHA_STAMP(tr, 8);
  if (valid < 128) {
#pragma unroll
    for (int i = 0; i < 64; ++i)
      if (c0 + i >= valid) v[i] = __float_as_uint(-INFINITY);
  }
  const float mh = max_tree3<64>(reinterpret_cast<const float*>(v));
  *red_mine = mh;
  named_bar_sync(bar_id, 256);  // both halves' S loaded (P may now overwrite S) and maxima posted
  FMHA_STAMP(tr, 9);
  const float mx = fmaxf(mh, *red_other);
  const float mx2 = mx * sl2;
  const bool bump = (j == 0) || (mx2 > m + 8.f);
  const float m_new = bump ? mx2 : m;
  const float alpha = (j == 0) ? 0.f : fast_exp2(m - m_new);
  m = m_new;
  if (j > 0 && __any_sync(0xffffffffu, bump)) {  // PV_{j-1} completed before S_j: O is stable
    const float a = bump ? alpha : 1.f;
    constexpr int NC = DP / 16, NC0 = (NC + 1) / 2;  // 16-column chunks of O: half 0 takes the first NC0
    const int cb = half ? NC0 : 0, ce = half ? NC : NC0;
    for (int c = cb; c < ce; ++c) {
      uint32_t o[16];
      tmem_ld16(tO + lane_off + c * 16, o);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
      tmem_st16(tO + lane_off + c * 16, o);
    }
  }
  const float2 sl2x2 = make_float2(sl2, sl2), mx2n = make_float2(-m_new, -m_new);
#pragma unroll
  for (int ch = 0; ch < 2; ++ch) {  // 32 keys -> 16 packed P columns per chunk
    uint32_t pk[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = ch * 16 + u;
      const float2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2x2, mx2n);
      float2 e;
      if (((i + half * 32) % DSP_POLY_DEN) < DSP_PT_POLY_NUM) {
        e = poly_exp2_x2(x);
      } else {
        e.x = fast_exp2(x.x);
        e.y = fast_exp2(x.y);
      }
      pk[u] = pack_bf16x2(e.x, e.y);
    }
    tmem_st16(tS + lane_off + half * 32 + ch * 16, pk);
  }
  FMHA_STAMP(tr, 11);
  tmem_st_wait();
  FMHA_STAMP(tr, 12);
  tc_fence_before();
}

template <int NA, int RB>
__global__ void __launch_bounds__(640, 1)
    fmha_split_kernel(const __grid_constant__ CUtensorMap tq_a, const __grid_constant__ CUtensorMap tq_b,
                      const __grid_constant__ CUtensorMap tk_a, const __grid_constant__ CUtensorMap tk_b,
                      const __grid_constant__ CUtensorMap tv_a, const __grid_constant__ CUtensorMap tv_b,
                      const __grid_constant__ CUtensorMap to_a, const __grid_constant__ CUtensorMap to_b,
                      const FmhaParams p) {
  using Cfg = SplitCfg<NA, RB>;
  using Base = FmhaCfg<NA, RB>;
  constexpr int KS = Cfg::KV_STAGES, DP = Cfg::DP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                        // 2 tiles
  uint8_t* sK = sQ + 2 * Cfg::TILE;          // KS stages
  uint8_t* sV = sK + KS * Cfg::TILE;         // KS stages
  uint8_t* sO = sV + KS * Cfg::TILE;         // 2 staging tiles (epilogue)
  float* red = reinterpret_cast<float*>(sO + 2 * Cfg::TILE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 2 * Cfg::TILE + Cfg::RED_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;            // count 512: Q copied to TMEM by every softmax thread
  uint64_t* k_full = bars + 2;             // [KS]
  uint64_t* k_empty = k_full + KS;         // [KS]
  uint64_t* v_full = k_empty + KS;         // [KS]
  uint64_t* v_empty = v_full + KS;         // [KS]
  uint64_t* v_ready = v_empty + KS;        // [KS] V patched with its ones column
  uint64_t* q_tm = v_ready + KS;           // [2] Q_slot in TMEM (count 256)
  uint64_t* s_full = q_tm + 2;             // [2]
  uint64_t* p_full = s_full + 2;           // [2] (count 256)
  uint64_t* o_done = p_full + 2;           // [2]
  uint64_t* o_free = o_done + 2;           // [2] (count 128: the half-0 warpgroup)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = warp_id();
  const int n = p.n_kv;
  const int npairs = p.items / 2;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tq_a); tma_prefetch(&tk_a); tma_prefetch(&tv_a);
    tma_prefetch(&tq_b); tma_prefetch(&tk_b); tma_prefetch(&tv_b);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 512);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); mbar_init(&v_ready[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&q_tm[t], 256);
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 256);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_free[t], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  griddep_launch_dependents();
  griddep_wait();
  clk_start(p.clk);

  // launch allocation 96 regs x 640 threads = 61440, redistributed exactly: 32 x 128 + 112 x 512
  // (setmaxnreg.inc can only take registers this CTA's own setmaxnreg.dec released)
  if (warp == 0) {
    setmaxnreg_dec<32>();
    if (elect_one()) {
      uint32_t nq = 0, kv = 0;
      for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
        mbar_wait_sleep(q_empty, (nq & 1) ^ 1);
        ++nq;
        mbar_arrive_expect_tx(q_full, 2 * Cfg::TX);
        load_tile<NA, RB>(sQ, &tq_a, &tq_b, q_full, tile_coord(p, 2 * ip, -1));
        load_tile<NA, RB>(sQ + Cfg::TILE, &tq_a, &tq_b, q_full, tile_coord(p, 2 * ip + 1, -1));
        for (int j = 0; j < n; ++j, ++kv) {
          const int st = kv % KS;
          const uint32_t ph = (kv / KS) & 1;
          const TileCoord t = tile_coord(p, 2 * ip, j);
          mbar_wait_sleep(&k_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&k_full[st], Cfg::TX);
          load_tile<NA, RB>(sK + st * Cfg::TILE, &tk_a, &tk_b, &k_full[st], t);
          mbar_wait_sleep(&v_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&v_full[st], Cfg::TX);
          load_tile<NA, RB>(sV + st * Cfg::TILE, &tv_a, &tv_b, &v_full[st], t);
        }
      }
    }
  } else if (warp == 1) {
    setmaxnreg_dec<32>();
    constexpr uint32_t idS = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idPVa = make_idesc_bf16(128, 64, 0, 1);
    constexpr uint32_t idPVb = make_idesc_bf16(128, RB, 0, 1);
    const uint32_t k0 = smem_u32(sK), v0 = smem_u32(sV);
    auto issue_s = [&](int slot, int st) {  // S_slot = Q_slot (TMEM) K^T
      if (elect_one()) {
        const uint32_t ka = k0 + st * Cfg::TILE, d = tmem + slot * 128, qt = tmem + 256 + slot * 128 + DP;
        int step = 0;
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k, ++step)
            umma_bf16_ts(d, qt + 8 * step, make_sdesc(ka + i * 16384 + k * 32, 16, 1024, SW_128B), idS, step != 0);
#pragma unroll
        for (int k = 0; k < RB / 16; ++k, ++step)
          umma_bf16_ts(d, qt + 8 * step, make_sdesc(ka + NA * 16384 + k * 32, 16, 8 * Base::RB_ROW, Base::RB_SW), idS,
                       step != 0);
        umma_commit(&s_full[slot]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int slot, int st, bool acc0) {  // O_slot (+)= P_slot V (P from TMEM)
      if (elect_one()) {
        const uint32_t va = v0 + st * Cfg::TILE, o = tmem + 256 + slot * 128, ps = tmem + slot * 128;
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 keys = 8 packed P columns per step
#pragma unroll
          for (int i = 0; i < NA; ++i)
            umma_bf16_ts(o + 64 * i, ps + 8 * k, make_sdesc(va + i * 16384 + k * 2048, 16384, 1024, SW_128B), idPVa,
                         acc0 || k != 0);
          umma_bf16_ts(o + 64 * NA, ps + 8 * k,
                       make_sdesc(va + NA * 16384 + k * 16 * Base::RB_ROW, 16384, 8 * Base::RB_ROW, Base::RB_SW),
                       idPVb, acc0 || k != 0);
        }
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    uint32_t np0 = 0, np1 = 0, nit = 0, kvbase = 0;
    for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x, ++nit, kvbase += n) {
      {
        const uint32_t kv0 = kvbase;
        mbar_wait(&k_full[kv0 % KS], (kv0 / KS) & 1);
        mbar_wait(&q_tm[0], nit & 1);
        tc_fence_after();
        issue_s(0, kv0 % KS);
        mbar_wait(&q_tm[1], nit & 1);
        tc_fence_after();
        issue_s(1, kv0 % KS);
        commit(&k_empty[kv0 % KS]);
      }
      for (int j = 0; j < n; ++j) {
        const uint32_t kj = kvbase + j, kn = kj + 1;
        const int sj = kj % KS, sn = kn % KS;
        mbar_wait(&p_full[0], np0 & 1);
        ++np0;
        mbar_wait(&v_ready[sj], (kj / KS) & 1);
        if (j == 0) mbar_wait(&o_free[0], (nit & 1) ^ 1);
        tc_fence_after();
        issue_pv(0, sj, j > 0);
        if (j + 1 == n) commit(&o_done[0]);
        if (j + 1 < n) {
          mbar_wait(&k_full[sn], (kn / KS) & 1);
          tc_fence_after();
          issue_s(0, sn);
        }
        mbar_wait(&p_full[1], np1 & 1);
        ++np1;
        if (j == 0) mbar_wait(&o_free[1], (nit & 1) ^ 1);
        tc_fence_after();
        issue_pv(1, sj, j > 0);
        commit(&v_empty[sj]);
        if (j + 1 == n) commit(&o_done[1]);
        if (j + 1 < n) {
          issue_s(1, sn);
          commit(&k_empty[sn]);
        }
      }
    }
  } else if (warp < 4) {
    setmaxnreg_dec<32>();
    if (warp == 2) {  // V patcher: column DP - 8 of every V row := 1.0 (row sums by the tensor core, R31)
      constexpr int CB = (RB - 8) * 2;
      uint32_t kv = 0;
      for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
        for (int j = 0; j < n; ++j, ++kv) {
          const int st = kv % KS;
          mbar_wait(&v_full[st], (kv / KS) & 1);
          const uint32_t vb = smem_u32(sV + st * Cfg::TILE) + NA * 16384;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = lane_id() + 32 * i;
            const uint32_t ch = RB == 16 ? ((CB >> 4) ^ ((r >> 2) & 1)) : ((CB >> 4) ^ ((r >> 1) & 3));
            st_shared_u16(vb + r * Base::RB_ROW + (ch << 4) + (CB & 15), 0x3F80);  // bf16 1.0
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&v_ready[st]);
        }
      }
    }
  } else {
    setmaxnreg_inc<112>();
    const int wg = (warp - 4) >> 2;  // 0..3
    const int slot = wg >> 1, half = wg & 1;
    const SoftmaxGeom G = make_geom(p, warp, p.scale_log2);
    const int row = G.row;
    const uint32_t tS = tmem + slot * 128, tO = tmem + 256 + slot * 128, tQ = tO + DP;
    const uint32_t q_src = smem_u32(sQ + slot * Cfg::TILE);
    uint8_t* sOs = sO + slot * Cfg::TILE;
    const uint32_t bar_red = 1 + slot, bar_epi = 3 + slot;
    int store_pending = 0;
    uint32_t nq = 0, ns = 0, no = 0;
    for (int ip = blockIdx.x; ip < npairs; ip += gridDim.x) {
      // Q_slot -> TMEM (packed bf16 pairs: column c = dims 2c, 2c+1): half 0 the SW128 atoms,
      // half 1 the RB remainder chunk; then release the smem tile to the producer
      mbar_wait(q_full, nq & 1);
      ++nq;
      if (half == 0) {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
          uint32_t w[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t a = q_src + i * 16384 + row * 128 + ((c ^ (row & 7)) << 4);
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w[4 * c]), "=r"(w[4 * c + 1]), "=r"(w[4 * c + 2]), "=r"(w[4 * c + 3]) : "r"(a));
          }
          tmem_st16(tQ + G.lane_off + i * 32, *reinterpret_cast<const uint32_t(*)[16]>(w));
          tmem_st16(tQ + G.lane_off + i * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(w + 16));
        }
      } else {
        constexpr int NCH = RB / 8;  // 16-B chunks of the remainder row
        uint32_t w[16];
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const uint32_t sw = RB == 16 ? (c ^ ((row >> 2) & 1)) : (c ^ ((row >> 1) & 3));
          const uint32_t a = q_src + NA * 16384 + row * Base::RB_ROW + (sw << 4);
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w[4 * c]), "=r"(w[4 * c + 1]), "=r"(w[4 * c + 2]), "=r"(w[4 * c + 3]) : "r"(a));
        }
        if constexpr (RB == 16) {
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                           tQ + G.lane_off + NA * 32),
                       "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                       : "memory");
        } else {
          tmem_st16(tQ + G.lane_off + NA * 32, *reinterpret_cast<const uint32_t(*)[16]>(w));
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&q_tm[slot]);
      mbar_arrive(q_empty);
      float m = -INFINITY;
      for (int j = 0; j < n; ++j) {
        unsigned long long* tr = (p.trace && half == 0) ? p.trace + ((size_t)(slot * 64 + (ns & 63)) * 16) : nullptr;
        FMHA_STAMP(tr, 0);
        mbar_wait(&s_full[slot], ns & 1);
        tc_fence_after();
        FMHA_STAMP(tr, 3);
        float* rb = red + ((ns & 1) * 4 + slot * 2) * 128;
        ++ns;
        softmax_step_split<DP>(G, half, tS, tO, j, m, j + 1 == n ? p.kv_last : 128, rb + half * 128 + row,
                               rb + (1 - half) * 128 + row, bar_red, tr);
        mbar_arrive(&p_full[slot]);
        FMHA_STAMP(tr, 4);
      }
      mbar_wait(&o_done[slot], no & 1);  // last PV done: O final
      ++no;
      tc_fence_after();
      if (half == 0) {
        if (store_pending) {  // the previous item's O store must have read the staging tile
          if ((threadIdx.x & 127) == 0) bulk_wait_group_read0();
          named_bar_sync(bar_epi, 128);
          store_pending = 0;
        }
        epilogue_tma_store<NA, RB, DP - 8>(p, &to_a, &to_b, sOs, tO, G.lane_off, row, 0.f, bar_epi,
                                           tile_coord(p, 2 * ip + slot, -1), &o_free[slot], store_pending, m);
      }
    }
    if (half == 0 && (threadIdx.x & 127) == 0) bulk_wait_group_read0();
  }

  tc_fence_before();
  __syncthreads();
  clk_end(p.clk);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// 5-D tile views {Dh, NH, position, outer, outer2} of q, k, v (one per part) and of o
struct FmhaViews {
  const void* base[3];
  uint64_t dims[3][5], strides[3][4];
  uint64_t odims[5], ostr[4];
};

template <int NA, int RB>
cudaError_t run_fmha(const FmhaViews& vw, const FmhaParams& p, const uint32_t* box_rows, int num_sms,
                     cudaStream_t st, std::string* why) {
  using Cfg = FmhaCfg<NA, RB>;
  CUtensorMap m[6];
  for (int part = 0; part < 3; ++part) {
    const void* b = vw.base[part];
    const uint64_t* dims = vw.dims[part];
    const uint64_t* strides = vw.strides[part];
    uint32_t boxa[5] = {64, 1, box_rows[0], box_rows[1], 1};
    uint32_t boxb[5] = {(uint32_t)(RB ? RB : 16), 1, box_rows[0], box_rows[1], 1};
    if (!make_tmap_bf16(&m[2 * part], b, 5, dims, strides, boxa, CU_TENSOR_MAP_SWIZZLE_128B, why))
      return cudaErrorInvalidValue;
    if (RB) {
      if (!make_tmap_bf16(&m[2 * part + 1], b, 5, dims, strides, boxb,
                          RB == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B, why))
        return cudaErrorInvalidValue;
    } else {
      m[2 * part + 1] = m[2 * part];
    }
  }
  // output maps: the query-side tile view over o [tok, C]
  CUtensorMap mo[2];
  {
    const uint64_t* dims = vw.odims;
    const uint64_t* ostr = vw.ostr;
    uint32_t boxa[5] = {64, 1, box_rows[0], box_rows[1], 1};
    uint32_t boxb[5] = {(uint32_t)(RB ? RB : 16), 1, box_rows[0], box_rows[1], 1};
    if (!make_tmap_bf16(&mo[0], p.o, 5, dims, ostr, boxa, CU_TENSOR_MAP_SWIZZLE_128B, why)) return cudaErrorInvalidValue;
    if (RB) {
      if (!make_tmap_bf16(&mo[1], p.o, 5, dims, ostr, boxb,
                          RB == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B, why))
        return cudaErrorInvalidValue;
    } else {
      mo[1] = mo[0];
    }
  }
#if defined(DSP_FMHA_SPLIT)  // A/B only: measured slower than fmha_pt_kernel (110-113 vs 101-104 us)
  if constexpr (SplitCfg<NA, RB>::OK) {
    if (p.G == 1 && p.n_qt % 2 == 0 && p.Dh <= SplitCfg<NA, RB>::DP - 8) {
      auto kp = fmha_split_kernel<NA, RB>;
      static bool attr_sp = false;
      if (!attr_sp) {
        cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, SplitCfg<NA, RB>::SMEM);
        if (e != cudaSuccess) return e;
        attr_sp = true;
      }
      const int npairs = p.items / 2;
      const int grid = npairs < num_sms ? npairs : num_sms;
      return launch_k(kp, dim3(grid), dim3(SplitCfg<NA, RB>::THREADS), SplitCfg<NA, RB>::SMEM, st, 1, m[0], m[1], m[2],
                      m[3], m[4], m[5], mo[0], mo[1], p);
    }
  }
#endif
#ifndef DSP_FMHA_NO_SEQ
  if constexpr (SeqCfg<NA, RB>::OK) {
    if (p.n_kv == 1 && !p.cross && p.Dh <= SeqCfg<NA, RB>::DP - 8 && (p.G == 1 || kSeqDiag)) {
      auto kp = fmha_seq_kernel<NA, RB>;
      static bool attr_sq = false;
      if (!attr_sq) {
        cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, SeqCfg<NA, RB>::SMEM);
        if (e != cudaSuccess) return e;
        attr_sq = true;
      }
      const int grid = p.items < num_sms ? p.items : num_sms;
      return launch_k(kp, dim3(grid), dim3(SeqCfg<NA, RB>::THREADS), SeqCfg<NA, RB>::SMEM, st, 1, m[0], m[1], m[2],
                      m[3], m[4], m[5], mo[0], mo[1], p);
    }
  }
#endif
#ifndef DSP_FMHA_PAIR_SMEM
  if constexpr (PtCfg<NA, RB>::OK) {
    if (p.G == 1 && p.n_qt % 2 == 0 && p.Dh <= PtCfg<NA, RB>::DP - 8) {
      auto kp = fmha_pt_kernel<NA, RB>;
      static bool attr_pt = false;
      if (!attr_pt) {
        cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, PtCfg<NA, RB>::SMEM);
        if (e != cudaSuccess) return e;
        attr_pt = true;
      }
      const int npairs = p.items / 2;
      const int grid = npairs < num_sms ? npairs : num_sms;
      return launch_k(kp, dim3(grid), dim3(PtCfg<NA, RB>::THREADS), PtCfg<NA, RB>::SMEM, st, 1, m[0], m[1], m[2], m[3],
                      m[4], m[5], mo[0], mo[1], p);
    }
  }
#endif
  if constexpr (PairCfg<NA, RB>::OK) {
    if (p.G == 1 && p.n_qt % 2 == 0) {
      // row sums by the tensor core when the padded head dim leaves a free column for the ones
      const bool ones = RB > 0 && p.Dh <= PairCfg<NA, RB>::DP - 8;
      auto kp = ones ? fmha_pair_kernel<NA, RB, (RB > 0)> : fmha_pair_kernel<NA, RB, false>;
      static bool attr_p[2] = {false, false};
      if (!attr_p[ones]) {
        cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<NA, RB>::SMEM);
        if (e != cudaSuccess) return e;
        attr_p[ones] = true;
      }
      const int npairs = p.items / 2;
      const int grid = npairs < num_sms ? npairs : num_sms;
      return launch_k(kp, dim3(grid), dim3(PairCfg<NA, RB>::THREADS), PairCfg<NA, RB>::SMEM, st, 1, m[0], m[1], m[2],
                      m[3], m[4], m[5], mo[0], mo[1], p);
    }
  }
  auto kern = fmha_bf16_tc_kernel<NA, RB>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int slots = Cfg::CTAS_PER_SM * num_sms;
  const int grid = p.items < slots ? p.items : slots;
  return launch_k(kern, dim3(grid), dim3(256), Cfg::SMEM, st, 1, m[0], m[1], m[2], m[3], m[4], m[5], mo[0], mo[1], p);
}


// ===================================================================== backward (f4)
// FMHA backward for one sequence / head / 128-key tile per work item (P:17 attention, the gradient
// of oracle/backward.py attention_core_bwd): with the forward's log2-domain row normaliser lse2,
//   S^T = K Q^T,  P^T = exp2(S^T * scale_log2 - lse2[q]),  dP^T = V dO^T,
//   dS^T = P^T * (dP^T - D[q]) / sqrt(Dh)   (D = rowsum(dO * O), attn_bwd_dvec_kernel),
//   dV += P^T dO,  dK += dS^T Q,  dQ_j = dS K   for every 128-query tile j of the sequence.
// Keys are the TMEM lanes: a compute thread owns one key row of S^T / dP^T and writes its P^T row
// back into TMEM over the consumed S^T columns (the TS-form A of dV += P^T dO) and its dS^T row
// into shared memory (SW128 K-major over queries), which is the K-major A of dK += dS^T Q and,
// read as MN-major, the A of dQ = dS K.  dQ leaves per query tile by a TMA reduce-add (f32) into
// dq_acc when the sequence has several key tiles, else as one bf16 TMA store; dK, dV leave after
// the item's last query tile.  TMEM (512 columns): S^T [0,128), dP^T [128,256), dV [256,336),
// dK [336,416), dQ [416,496).  Roles (256 threads, one CTA per SM): warp 0 TMA producer (K, V
// per item; {Q, dO} per query tile, two stages), warp 1 TMEM allocator + MMA issuer, warps 4-7
// compute (P, dS, dQ / dK / dV epilogues).  Block-diagonal packing (G = 128 / L sequences per
// tile, temporal T = 16) masks P and dS outside each thread's own sequence.
#ifdef DSP_FMHA_BWD_TRACE  // per-step clock64 stamps of CTA 0 (scripts/fmha_bwd_trace.py)
#define BWD_STAMP(idx) \
  do { if (p.trace && blockIdx.x == 0 && g < 64) p.trace[g * 8 + (idx)] = clock64(); } while (0)
#else
#define BWD_STAMP(idx) do { } while (0)
#endif
struct BwdMaps {
  CUtensorMap q[2], k[2], v[2], dout[2], dq[2], dk[2], dv[2];
  CUtensorMap dq_acc[2];  // f32 reduce-add boxes: {32 columns, rows} SW128 (x2), {16 columns, rows} SW64
};

template <int NA, int RB>
struct BwdCfg {
  using Base = FmhaCfg<NA, RB>;
  static constexpr int TILE = Base::TILE, DP = Base::DP, TX = Base::TX;
  static constexpr int OFF_K = 0, OFF_V = TILE, OFF_Q = 2 * TILE;  // stage s: Q at OFF_Q + 2 s TILE, dO next
  static constexpr int OFF_DS = 6 * TILE;                            // dS^T: 2 x [128 keys][64 queries] SW128
  static constexpr int OFF_DQ = OFF_DS + 32768;                      // dQ f32 staging (3 swizzled boxes) / dK, dV bf16
  static constexpr int OFF_VEC = OFF_DQ + 128 * DP * 4;              // [2 buf][lse2 | D][128] f32
  static constexpr int OFF_BAR = OFF_VEC + 2 * 2 * 128 * 4;
  // no alignment slack: dynamic smem starts 1024-B aligned after the system-reserved block (checked)
  static constexpr int SMEM = OFF_BAR + 256;
  static constexpr bool OK = SMEM <= 227 * 1024 && RB == 16 && NA == 1;
  static_assert(2 * TILE <= 128 * DP * 4, "dK and dV staging fit in the dQ staging area");
  // warps 0-3: producer, MMA, idle x2; warps 4-19: four compute warpgroups; warps 20-23: epilogue
  static constexpr int NWG = 4, THREADS = 128 + 128 * NWG + 128;
};

__device__ __forceinline__ TileCoord bwd_coord(const FmhaParams& p, int outer, int h, int pt) {
  TileCoord t;
  t.h = h;
  if (p.G == 1) {
    t.x2 = pt * 128;
    if (p.spatial) { t.x3 = outer; t.x4 = 0; }
    else { t.x3 = outer % p.S_loc; t.x4 = outer / p.S_loc; }
  } else {
    t.x2 = 0;
    if (p.spatial) { t.x3 = outer * p.G; t.x4 = 0; }
    else { const int ng = (p.S_loc + p.G - 1) / p.G; t.x3 = (outer % ng) * p.G; t.x4 = outer / ng; }
  }
  return t;
}

// bf16 row of a [128][DP] tile -> the TMA box staging layout (SW128 64-column chunks, then the SW32
// remainder), scaled by `mul`
template <int NA, int RB, int D0 = 0, int D1 = NA * 64 + RB>  // columns [D0, D1) of the row; v[0] = column D0
__device__ __forceinline__ void stage_row_bf16(uint32_t st0, int row, const uint32_t* v, float mul) {
#pragma unroll
  for (int d = D0; d < D1; d += 8) {
    const uint32_t* w = v + (d - D0);
    const uint32_t a0 = pack_bf16x2(__uint_as_float(w[0]) * mul, __uint_as_float(w[1]) * mul);
    const uint32_t a1 = pack_bf16x2(__uint_as_float(w[2]) * mul, __uint_as_float(w[3]) * mul);
    const uint32_t a2 = pack_bf16x2(__uint_as_float(w[4]) * mul, __uint_as_float(w[5]) * mul);
    const uint32_t a3 = pack_bf16x2(__uint_as_float(w[6]) * mul, __uint_as_float(w[7]) * mul);
    uint32_t addr;
    if (d < NA * 64) {
      const int blk = d >> 6, ch = (d & 63) >> 3;
      addr = st0 + blk * 16384 + row * 128 + ((ch ^ (row & 7)) << 4);
    } else {
      const int ch = (d - NA * 64) >> 3;  // RB = 16: SW32, two chunks per 32-B row
      addr = st0 + NA * 16384 + row * 32 + ((ch ^ ((row >> 2) & 1)) << 4);
    }
    st_shared_v4(addr, a0, a1, a2, a3);
  }
}

// 16 columns [d0, d0 + 16) of a bf16 row into the TMA box staging layout (as stage_row_bf16)
template <int NA, int RB>
__device__ __forceinline__ void stage_cols16_bf16(uint32_t st0, int row, const uint32_t* v, int d0) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int d = d0 + 8 * h;
    const uint32_t* w = v + 8 * h;
    const uint32_t a0 = pack_bf16x2(__uint_as_float(w[0]), __uint_as_float(w[1]));
    const uint32_t a1 = pack_bf16x2(__uint_as_float(w[2]), __uint_as_float(w[3]));
    const uint32_t a2 = pack_bf16x2(__uint_as_float(w[4]), __uint_as_float(w[5]));
    const uint32_t a3 = pack_bf16x2(__uint_as_float(w[6]), __uint_as_float(w[7]));
    uint32_t addr;
    if (d < NA * 64) {
      const int blk = d >> 6, ch = (d & 63) >> 3;
      addr = st0 + blk * 16384 + row * 128 + ((ch ^ (row & 7)) << 4);
    } else {
      const int ch = (d - NA * 64) >> 3;  // RB = 16: SW32, two chunks per 32-B row
      addr = st0 + NA * 16384 + row * 32 + ((ch ^ ((row >> 2) & 1)) << 4);
    }
    st_shared_v4(addr, a0, a1, a2, a3);
  }
}

template <int NA, int RB>
__device__ __forceinline__ void store_tile(const CUtensorMap* ma, const CUtensorMap* mb, const uint8_t* src,
                                           const TileCoord& t) {
#pragma unroll
  for (int i = 0; i < NA; ++i) tma_store_5d(ma, src + i * 16384, 64 * i, t.h, t.x2, t.x3, t.x4);
  tma_store_5d(mb, src + NA * 16384, 64 * NA, t.h, t.x2, t.x3, t.x4);
}

// The backward's Q, K, V, dO tiles: DP / 16 boxes of [rows][16 columns], SW32, 4 KB apart.  One
// layout serves as the K-major operand (one box per 16-column k-step, SBO 256 B) and as an MN-major
// operand with N = DP in ONE instruction (16-column groups LBO = 4 KB apart, 8-row groups 256 B):
// the dV / dK / dQ products take one N = 80 MMA per 16-row k-step instead of N = 64 + N = 16.
template <int NA, int RB>
__device__ __forceinline__ void load_tile_sw32(uint8_t* dst, const CUtensorMap* mb, uint64_t* bar, const TileCoord& t) {
  constexpr int DP = NA * 64 + RB;
#pragma unroll
  for (int i = 0; i < DP / 16; ++i) tma_load_5d(dst + i * 4096, mb, bar, 16 * i, t.h, t.x2, t.x3, t.x4);
}

// Slot schedule shared by the producer and the MMA issuer (both walk it in the same order): item i
// keeps K, V in slot kv; query tile j uses slot o[j % 2]; item i + 1 puts K, V into o[nq % 2] (free
// once tile nq - 2 is done) and its query tiles use {kv, o[(nq - 1) % 2]}, both freed by the item's last
// products.  Per-slot use counters give the mbarrier phases.
struct SlotRing {
  int kv = 0, o[2] = {1, 2};
  uint32_t use[3] = {0, 0, 0};
  // reuse: the next item's first query tile is this item's last (BwdWalk), still in its slot, so
  // the next item starts in that slot and its second tile goes to this item's K, V slot
  __device__ __forceinline__ void next_item(int nq, bool reuse) {
    const int nkv = o[nq & 1], last = o[(nq - 1) & 1];
    o[0] = reuse ? last : kv;
    o[1] = reuse ? kv : last;
    kv = nkv;
  }
};

// A CTA's items: chunks of walk_ch consecutive items of the item list (key tile fastest), chunk c on
// CTA c mod grid (walk_ch = 1: plain grid stride; 0: one contiguous range per CTA).  Consecutive items
// of a chunk mostly share (sequence group, head) and differ in the key tile; such a follower walks its
// query tiles in the opposite order, its first tile being its predecessor's last: that tile's {Q, dO}
// stay in their slot and the item boundary waits for no load.  Concurrent CTAs still cover
// neighbouring key tiles of the same sequences (their {Q, dO} read once from HBM, then from L2).
struct BwdWalk {
  int item, end, chunk, ch, items, nq, n_kv;
  bool rev = false, reuse = false;  // query order of the current item; its first tile is the previous one's last
  __device__ __forceinline__ explicit BwdWalk(const FmhaParams& p)
      : ch(p.walk_ch), items(p.items), nq(p.n_qt), n_kv(p.n_kv) {
    if (ch > 0) {
      chunk = blockIdx.x;
      item = chunk * ch;
      end = min(item + ch, items);
    } else {
      item = (int)((long long)blockIdx.x * items / gridDim.x);
      end = (int)((long long)(blockIdx.x + 1) * items / gridDim.x);
    }
  }
  __device__ __forceinline__ bool valid() const { return item < end; }
  __device__ __forceinline__ int qt(int j) const { return rev ? nq - 1 - j : j; }
  __device__ __forceinline__ bool next_reuses() const {
    return nq > 1 && item + 1 < end && (item + 1) / n_kv == item / n_kv;
  }
  __device__ __forceinline__ void advance() {
    const bool r = next_reuses();
    rev = r && !rev;
    reuse = r;
    if (item + 1 < end || ch == 0) {
      ++item;
    } else {  // this CTA's next chunk
      chunk += gridDim.x;
      item = chunk * ch;
      end = min(item + ch, items);
    }
  }
};

template <int NA, int RB, bool DIAG>
__global__ void __launch_bounds__(BwdCfg<NA, RB>::THREADS, 1)
    fmha_bwd_kernel(const __grid_constant__ BwdMaps mp, const FmhaParams p, const float* __restrict__ lse,
                    const float* __restrict__ dvec, int accum) {
  using Cfg = BwdCfg<NA, RB>;
  using Base = FmhaCfg<NA, RB>;
  constexpr int DP = Cfg::DP;
  extern __shared__ uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();  // layout assumes a 1024-B aligned base
  uint8_t* smem = smem_raw;
  uint8_t* sK = smem + Cfg::OFF_K;
  uint8_t* sV = smem + Cfg::OFF_V;
  uint8_t* sDS = smem + Cfg::OFF_DS;
  uint8_t* sDQ = smem + Cfg::OFF_DQ;
  float* sVec = reinterpret_cast<float*>(smem + Cfg::OFF_VEC);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  // Three 40 KB slots (two tiles each) hold an item's {K, V} and its query tiles' {Q, dO}: the item's K, V
  // take one slot, its query tiles alternate in the other two, and the next item's K, V go into the slot
  // the last query tile does not use -- loaded while that tile is computed (SlotRing)
  uint64_t* slot_full = bars;       // [3]
  uint64_t* slot_empty = bars + 3;  // [3]
  uint64_t* s_full = bars + 6;
  uint64_t* p_full = bars + 7;   // count 128
  uint64_t* dq_full = bars + 8;
  uint64_t* dq_free = bars + 9;  // count 128
  uint64_t* kv_free = bars + 10; // count 128
  uint64_t* s_free = bars + 11;  // the compute warpgroups have read S^T / dP^T out of TMEM
  uint64_t* dp_full = bars + 12; // dP^T of the tile in TMEM (issued behind the previous tile's dV)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 13);

  const int warp = warp_id();
  if (warp == 0 && lane_id() == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(&slot_full[i], 1);
      mbar_init(&slot_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 128 * Cfg::NWG);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 128);
    mbar_init(kv_free, 128);
    mbar_init(s_free, 128 * Cfg::NWG);
    mbar_init(dp_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  griddep_launch_dependents();
  griddep_wait();
  clk_start(p.clk);

  const int nq = p.n_qt;
  auto decomp = [&](int item, int& outer, int& h, int& kvt) {
    kvt = item % p.n_kv;
    const int rest = item / p.n_kv;
    h = rest % p.NH;
    outer = rest / p.NH;
  };

  // 768 threads: every role fits the launch allocation of 80 registers (no setmaxnreg)
  if (warp == 0) {
    if (elect_one()) {
      SlotRing rg;
      auto fill = [&](int slot, const CUtensorMap* ma, const CUtensorMap* mb, const TileCoord& t) {
        mbar_wait_sleep(&slot_empty[slot], (rg.use[slot] & 1) ^ 1);
        ++rg.use[slot];
        mbar_arrive_expect_tx(&slot_full[slot], 2 * Cfg::TX);
        uint8_t* b = smem + slot * 2 * Cfg::TILE;
        load_tile_sw32<NA, RB>(b, ma, &slot_full[slot], t);
        load_tile_sw32<NA, RB>(b + Cfg::TILE, mb, &slot_full[slot], t);
      };
      BwdWalk wk(p);
      if (wk.valid()) {
        int outer, h, kvt;
        decomp(wk.item, outer, h, kvt);
        fill(rg.kv, &mp.k[1], &mp.v[1], bwd_coord(p, outer, h, kvt));
      }
      while (wk.valid()) {
        int outer, h, kvt;
        decomp(wk.item, outer, h, kvt);
        for (int j = wk.reuse ? 1 : 0; j < nq; ++j)
          fill(rg.o[j & 1], &mp.q[1], &mp.dout[1], bwd_coord(p, outer, h, wk.qt(j)));
        rg.next_item(nq, wk.next_reuses());
        wk.advance();
        if (wk.valid()) {  // the next item's K, V behind the last query tile
          int o2, h2, k2;
          decomp(wk.item, o2, h2, k2);
          fill(rg.kv, &mp.k[1], &mp.v[1], bwd_coord(p, o2, h2, k2));
        }
      }
    }
  } else if (warp == 1) {
    constexpr int DP = Cfg::DP;
    constexpr uint32_t idS = make_idesc_bf16(128, 128, 0, 0);       // S^T, dP^T
    constexpr uint32_t idK = make_idesc_bf16(128, DP, 0, 1);        // dV, dK: A K-major, B MN-major (N = 80)
    constexpr uint32_t idQ = make_idesc_bf16(128, DP, 1, 1);        // dQ: A (dS) MN-major, B (K) MN-major
    const uint32_t dsb = smem_u32(sDS);
    const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 336, tdQ = tmem + 416;
    // D[tmem] = X Y^T over the head dim: X, Y two [128][DP] tiles of SW32 boxes (one box per k-step)
    auto qk = [&](uint32_t d, uint32_t xa, uint32_t ya) {
#pragma unroll
      for (int kk = 0; kk < DP / 16; ++kk)
        umma_bf16_ss(d, make_sdesc(xa + kk * 4096, 16, 256, SW_32B), make_sdesc(ya + kk * 4096, 16, 256, SW_32B), idS,
                     kk != 0);
    };
    // MN-major B descriptor of a [128 rows = K][DP] tile, all DP columns, 16-row k-step kk
    auto bmn = [&](uint32_t base, int kk) { return make_sdesc(base + kk * 512, 4096, 256, SW_32B); };
    // Issue order: S^T/dP^T of tile g + 1 as soon as the compute warps have read tile g's out of TMEM
    // (s_free), BEFORE dV/dK/dQ of tile g, so tile g + 1's exponentials overlap tile g's products
    // (P^T and dS^T live in shared memory).  Across an item boundary the next K, V land only after
    // the item's last products (single K/V buffer), so there the order is the plain one.
    SlotRing rg;
    uint32_t cons[3] = {0, 0, 0};  // full-barrier waits per slot
    auto wait_slot = [&](int slot) {
      mbar_wait(&slot_full[slot], cons[slot] & 1);
      ++cons[slot];
    };
    // S^T of tile g + 1 goes out as soon as the compute warps have read tile g out of TMEM; dP^T of
    // tile g + 1 behind tile g's dV, which reads P^T from dP^T's columns (TS form: no smem for P)
    auto issue_s = [&](uint32_t gg, int j, bool first_of_item, bool reused) {
      const uint32_t qa = smem_u32(smem + rg.o[j & 1] * 2 * Cfg::TILE);
      const uint32_t kb = smem_u32(smem + rg.kv * 2 * Cfg::TILE);
      if (first_of_item) wait_slot(rg.kv);
      if (!reused) wait_slot(rg.o[j & 1]);  // a reused tile's {Q, dO} are in the slot already
      if (gg >= 1) mbar_wait(s_free, (gg - 1) & 1);  // S^T / dP^T of the previous tile read out of TMEM
      tc_fence_after();
      if (lane_id() == 0) { const uint32_t g = gg; BWD_STAMP(3); }
      if (elect_one()) {
        qk(tS, kb, qa);   // S^T = K Q^T
        umma_commit(s_full);
      }
      __syncwarp();
    };
    auto issue_dp = [&](int j) {
      const uint32_t da = smem_u32(smem + rg.o[j & 1] * 2 * Cfg::TILE) + Cfg::TILE;
      const uint32_t vb = smem_u32(smem + rg.kv * 2 * Cfg::TILE) + Cfg::TILE;
      if (elect_one()) {
        qk(tdP, vb, da);  // dP^T = V dO^T
        umma_commit(dp_full);
      }
      __syncwarp();
    };
    auto issue_bc = [&](uint32_t gg, int j, uint32_t itx, bool keep) {
      const int qs = rg.o[j & 1];
      const uint32_t qa = smem_u32(smem + qs * 2 * Cfg::TILE), da = qa + Cfg::TILE;
      const uint32_t kb = smem_u32(smem + rg.kv * 2 * Cfg::TILE);
      mbar_wait(p_full, gg & 1);
      if (lane_id() == 0) { const uint32_t g = gg; BWD_STAMP(4); }
      if (gg >= 1) mbar_wait(dq_free, (gg - 1) & 1);
      if (j == 0 && itx >= 1) mbar_wait(kv_free, (itx - 1) & 1);
      tc_fence_after();
      if (lane_id() == 0) { const uint32_t g = gg; BWD_STAMP(5); }
      if (elect_one()) {
        const uint32_t acc0 = j != 0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 queries per step
          // dV += P^T dO and dK += dS^T Q, both A operands packed in TMEM over dP^T's consumed columns:
          // compute warpgroup w's 32 queries at columns 32 w .. 32 w + 15 (P^T) and + 16 .. + 31 (dS^T)
          const uint32_t pa = tdP + 32 * (kk >> 1) + 8 * (kk & 1);
          umma_bf16_ts(tdV, pa, bmn(da, kk), idK, acc0 | (kk != 0));
          umma_bf16_ts(tdK, pa + 16, bmn(qa, kk), idK, acc0 | (kk != 0));
        }
        if (!keep) umma_commit(&slot_empty[qs]);  // Q and dO read (dV, dK issued): the producer may refill the slot
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ = dS K: 16 keys per step; dS MN-major (queries contiguous)
          umma_bf16_ss(tdQ, make_sdesc(dsb + kk * 2048, 16384, 1024, SW_128B), bmn(kb, kk), idQ, kk != 0);
        umma_commit(dq_full);
        if (j == nq - 1) umma_commit(&slot_empty[rg.kv]);  // the item's K, V read
      }
      __syncwarp();
    };
    uint32_t it = 0, g = 0;
    for (BwdWalk wk(p); wk.valid(); wk.advance(), ++it) {
      const bool rn = wk.next_reuses();  // the last tile's slot is kept for the next item
      issue_s(g, 0, true, wk.reuse);
      issue_dp(0);
      for (int j = 0; j < nq; ++j, ++g) {
        if (j + 1 < nq) issue_s(g + 1, j + 1, false, false);
        issue_bc(g, j, it, rn && j == nq - 1);
        if (j + 1 < nq) issue_dp(j + 1);
      }
      rg.next_item(nq, rn);
    }
  } else if (warp >= 4 && warp < 4 + 4 * Cfg::NWG) {
    // Four compute warpgroups share each key row (TMEM lane quadrant = warp % 4): warpgroup hw owns
    // queries [32 hw, 32 hw + 32) of S^T / dP^T, i.e. chunks (hw & 1) * 4 .. + 3 of the 64-query P^T /
    // dS^T smem tile hw >> 1.  Four warps per SMSP keep the TMEM-load latency of each covered.
    const int q4 = warp & 3, hw = (warp - 4) >> 2;
    const int row = q4 * 32 + lane_id();
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_off + hw * 32, tdP = tmem + 128 + lane_off + hw * 32;
    const uint32_t bar_wg = 1 + hw;  // named barrier of the own warpgroup (128)
    const float sl2 = p.scale_log2;
    const float sc = rsqrtf((float)p.Dh);
    // block-diagonal packing: this key row's sequence owns queries [qlo, qhi) of the warpgroup's 32
    const int qlo = p.G > 1 ? (row / p.L) * p.L - 32 * hw : 0;
    const int qhi = p.G > 1 ? qlo + p.L : 32;
    const uint32_t tile_off = (hw >> 1) * 16384 + row * 128;
    const uint32_t dsrow = smem_u32(sDS) + tile_off;
    // lse2 and D / sqrt(Dh) of the query this thread stages (threads row < 32 of each warpgroup: query
    // 32 hw + row), copied global -> smem by cp.async one tile ahead (no registers held across the tile,
    // the latency off the critical path); padding queries get lse2 = +inf (P = 0), D = 0
    auto fetch = [&](bool valid, int item, int j, uint32_t vbuf) {
      if (row >= 32) return;
      long tok = -1;
      int h = 0;
      if (valid) {
        int outer, kvt;
        decomp(item, outer, h, kvt);
        tok = row_token(p, bwd_coord(p, outer, h, j), 32 * hw + row);
      }
      if (tok >= 0) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(vbuf + row * 4), "l"(lse + tok * p.NH + h) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(vbuf + 512 + row * 4), "l"(dvec + tok * p.NH + h)
                     : "memory");
      } else {
        st_shared_f32(vbuf + row * 4, INFINITY);
        st_shared_f32(vbuf + 512 + row * 4, 0.f);
      }
    };
    uint32_t g = 0;
    BwdWalk wk(p);
    fetch(wk.valid(), wk.item, wk.qt(0), smem_u32(sVec + hw * 32));
    for (; wk.valid(); wk.advance()) {
      for (int j = 0; j < nq; ++j, ++g) {
        const uint32_t vb = smem_u32(sVec + (g & 1) * 256 + hw * 32);  // this warpgroup's 32 queries
        asm volatile("cp.async.wait_all;" ::: "memory");               // this tile's lse2 / D landed
        const uint32_t vnext = smem_u32(sVec + ((g + 1) & 1) * 256 + hw * 32);
        if (threadIdx.x == 128) BWD_STAMP(0);
        named_bar_sync(bar_wg, 128);
        // the next tile's values go to the other buffer (its readers finished before this barrier)
        if (j + 1 < nq) {
          fetch(true, wk.item, wk.qt(j + 1), vnext);
        } else {
          BwdWalk nx = wk;
          nx.advance();
          fetch(nx.valid(), nx.item, nx.qt(0), vnext);
        }
        mbar_wait(s_full, g & 1);
        tc_fence_after();
        if (threadIdx.x == 128) BWD_STAMP(1);
        if (threadIdx.x == 128 + 128 * (Cfg::NWG - 1)) BWD_STAMP(6);  // the last warpgroup saw S
        // phase 1: P from S^T (two 16-query chunks), packed bf16 (kept for dS and stored for dV)
        uint32_t pk[16], dk[16];
        const float2 sl22 = make_float2(sl2, sl2), sc2 = make_float2(sc, sc);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          uint32_t sv[16];
          tmem_ld16(tS + k * 16, sv);
          tmem_ld_wait();
#pragma unroll
          for (int i4 = 0; i4 < 4; ++i4) {
            const int q0 = k * 16 + 4 * i4;
            const float4 l4 = ld_shared_f32x4(vb + q0 * 4);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int e = 4 * i4 + 2 * h2;
              const float2 s2 = make_float2(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1]));
              const float2 nl = h2 ? make_float2(-l4.z, -l4.w) : make_float2(-l4.x, -l4.y);
              float2 x = ffma2(s2, sl22, nl);
              if (DIAG) {
                const int qc = q0 + 2 * h2;
                if (qc < qlo || qc >= qhi) x.x = -INFINITY;
                if (qc + 1 < qlo || qc + 1 >= qhi) x.y = -INFINITY;
              }
              pk[k * 8 + 2 * i4 + h2] = pack_bf16x2(fast_exp2(x.x), fast_exp2(x.y));
            }
          }
        }
        // phase 2: dS = P (dP / sqrt(Dh) - D / sqrt(Dh)) with the bf16 P the dV product uses
        mbar_wait(dp_full, g & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          uint32_t dv[16];
          tmem_ld16(tdP + k * 16, dv);
          tmem_ld_wait();
#pragma unroll
          for (int i4 = 0; i4 < 4; ++i4) {
            const int q0 = k * 16 + 4 * i4;
            const float4 d4 = ld_shared_f32x4(vb + 512 + q0 * 4);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int e = 4 * i4 + 2 * h2, kk = k * 8 + 2 * i4 + h2;
              const float2 p2 = make_float2(__uint_as_float(dv[e]), __uint_as_float(dv[e + 1]));
              const float2 nd = h2 ? make_float2(-d4.z, -d4.w) : make_float2(-d4.x, -d4.y);
              const float2 pe = make_float2(bf16lo(pk[kk]), bf16hi(pk[kk]));
              const float2 ds = fmul2(pe, ffma2(p2, sc2, nd));
              dk[kk] = pack_bf16x2(ds.x, ds.y);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(s_free);  // S^T / dP^T of this tile are in registers: the next tile's S may be issued
        tmem_st16(tdP, pk);       // P^T over this warpgroup's consumed dP^T columns (dV, TS form)
        tmem_st16(tdP + 16, dk);  // dS^T beside it (dK, TS form); dQ reads the smem copy (MN-major)
        // dS^T of the warpgroup's 32 queries -> smem (SW128 K-major over queries)
        if (g >= 1) mbar_wait(dq_full, (g - 1) & 1);  // the previous tile's products have read it
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ch = (hw & 1) * 4 + u;
          st_shared_v4(dsrow + ((ch ^ (row & 7)) << 4), dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
        }
        tmem_st_wait();
        tc_fence_before();
        fence_proxy_async_smem();
        if (threadIdx.x == 128) BWD_STAMP(2);
        if (threadIdx.x == 128 + 128 * (Cfg::NWG - 1)) BWD_STAMP(7);  // the last warpgroup's P done
        mbar_arrive(p_full);
      }
    }
  } else if (warp >= 4 + 4 * Cfg::NWG) {
    // Epilogue warpgroup (thread = TMEM lane = query row for dQ, key row for dK / dV): dQ of every
    // query tile leaves as three swizzled f32 TMA reduce-adds into dq_acc (several key tiles) or
    // as one bf16 TMA store (one key tile); dK, dV as bf16 TMA stores after the item's last tile.
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane_id();
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t tdV = tmem + 256 + lane_off, tdK = tmem + 336 + lane_off, tdQ = tmem + 416 + lane_off;
    const bool elected = threadIdx.x == 128 + 128 * Cfg::NWG;  // issues every bulk store / reduce of the CTA
    constexpr uint32_t kBarEpi = 1 + Cfg::NWG;
    const uint32_t s0 = smem_u32(sDQ);
    uint32_t g = 0;
    for (BwdWalk wk(p); wk.valid(); wk.advance()) {
      int outer, h, kvt;
      decomp(wk.item, outer, h, kvt);
      for (int j = 0; j < nq; ++j, ++g) {
        mbar_wait(dq_full, g & 1);
        tc_fence_after();
        const TileCoord tq = bwd_coord(p, outer, h, wk.qt(j));
        if (elected) bulk_wait_group_read0();  // the previous reduce / stores have read sDQ
        named_bar_sync(kBarEpi, 128);
        if (accum) {
          // f32 staging as three swizzled TMA boxes (conflict-free row writes): columns 0-31 and 32-63
          // SW128 (128 B rows), 64-79 SW64 (64 B rows); reduce-added into dq_acc.  16 columns per
          // TMEM load (register budget).
#pragma unroll
          for (int c = 0; c < DP / 16; ++c) {
            uint32_t qv[16];
            tmem_ld16(tdQ + c * 16, qv);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int col = c * 16 + k * 4;  // 4 floats = one 16-B chunk
              uint32_t addr;
              if (col < 64) addr = s0 + (col >> 5) * 16384 + row * 128 + ((((col & 31) >> 2) ^ (row & 7)) << 4);
              else addr = s0 + 32768 + row * 64 + ((((col - 64) >> 2) ^ ((row >> 1) & 3)) << 4);
              st_shared_v4(addr, qv[4 * k], qv[4 * k + 1], qv[4 * k + 2], qv[4 * k + 3]);
            }
          }
          tc_fence_before();
          mbar_arrive(dq_free);
          fence_proxy_async_smem();
          named_bar_sync(kBarEpi, 128);
          if (elected) {
            tma_reduce_add_5d(&mp.dq_acc[0], sDQ, 0, tq.h, tq.x2, tq.x3, tq.x4);
            tma_reduce_add_5d(&mp.dq_acc[0], sDQ + 16384, 32, tq.h, tq.x2, tq.x3, tq.x4);
            tma_reduce_add_5d(&mp.dq_acc[1], sDQ + 32768, 64, tq.h, tq.x2, tq.x3, tq.x4);
            bulk_commit_group();
          }
        } else {  // one key tile per sequence: dQ is final (bf16), 16 columns per TMEM load
#pragma unroll
          for (int c = 0; c < DP / 16; ++c) {
            uint32_t qv[16];
            tmem_ld16(tdQ + c * 16, qv);
            tmem_ld_wait();
            stage_cols16_bf16<NA, RB>(s0, row, qv, c * 16);
          }
          tc_fence_before();
          mbar_arrive(dq_free);
          fence_proxy_async_smem();
          named_bar_sync(kBarEpi, 128);
          if (elected) {
            store_tile<NA, RB>(&mp.dq[0], &mp.dq[1], sDQ, tq);
            bulk_commit_group();
          }
        }
        if (j == nq - 1) {  // dK, dV final: dq_full of the last tile covers every MMA of the item
          if (elected) bulk_wait_group_read0();
          named_bar_sync(kBarEpi, 128);
#pragma unroll
          for (int c = 0; c < 2 * (DP / 16); ++c) {  // dK then dV, 16 columns per TMEM load
            const int cc = c % (DP / 16);
            uint32_t kv[16];
            tmem_ld16((c < DP / 16 ? tdK : tdV) + cc * 16, kv);
            tmem_ld_wait();
            stage_cols16_bf16<NA, RB>(s0 + (c < DP / 16 ? 0 : Cfg::TILE), row, kv, cc * 16);
          }
          tc_fence_before();
          mbar_arrive(kv_free);
          fence_proxy_async_smem();
          named_bar_sync(kBarEpi, 128);
          if (elected) {
            const TileCoord tk = bwd_coord(p, outer, h, kvt);
            store_tile<NA, RB>(&mp.dk[0], &mp.dk[1], sDQ, tk);
            store_tile<NA, RB>(&mp.dv[0], &mp.dv[1], sDQ + Cfg::TILE, tk);
            bulk_commit_group();
          }
        }
      }
    }
    if (elected) bulk_wait_group0();  // reduce-adds and stores complete before the CTA retires
  }
  tc_fence_before();
  __syncthreads();
  clk_end(p.clk);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

static cudaError_t dispatch_dh(const FmhaViews& vw, const FmhaParams& p, const uint32_t* box_rows, int num_sms,
                               cudaStream_t st, std::string* why);

#ifdef DSP_FMHA_TRACE
unsigned long long* g_fmha_trace = nullptr;
extern "C" void* dsp_debug_fmha_trace() { return g_fmha_trace; }
#endif

cudaError_t launch_fmha_bf16(const void* qkv, void* o, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C, int NH,
                             int dim, int num_sms, cudaStream_t st, std::string* why, float* lse) {
  FmhaParams p{};
  p.lse = lse;
  p.NH = NH;
  p.Dh = (int)(C / NH);
  p.C = (int)C;
  p.S_loc = (int)S_loc;
  p.T_loc = (int)T_loc;
  p.B = (int)B;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.trace = nullptr;
  p.clk = t_clk;
#ifdef DSP_FMHA_TRACE
  {
    static unsigned long long* tbuf = nullptr;
    if (!tbuf) cudaMalloc(&tbuf, 2 * 64 * 16 * sizeof(unsigned long long));
    p.trace = tbuf;
    extern unsigned long long* g_fmha_trace;
    g_fmha_trace = tbuf;
  }
#endif
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)p.Dh));
  p.spatial = (dim == DSP_DIM_S);
  p.L = (int)(p.spatial ? S_loc : T_loc);
  if (p.L % 128 == 0) {
    p.G = 1;
    p.n_kv = p.L / 128;
    p.n_qt = p.L / 128;
  } else if (128 % p.L == 0) {
    p.G = 128 / p.L;
    p.n_kv = 1;
    p.n_qt = 1;
  } else {  // ragged length: one sequence per tile row block, last query tile clipped by the
            // TMA store, keys >= L of the last key tile masked
    p.G = 1;
    p.n_kv = (p.L + 127) / 128;
    p.n_qt = p.n_kv;
  }
  const uint64_t e = 2, rowb = 3 * (uint64_t)C * e;
  uint64_t dims[5], strides[4];
  // Rows of a tile run along x2 (position in the sequence), then x3 (next sequence).
  if (p.spatial) {  // {Dh, NH, S (pos), frames, 1}
    dims[0] = p.Dh; dims[1] = NH; dims[2] = S_loc; dims[3] = B * T_loc; dims[4] = 1;
    strides[0] = p.Dh * e; strides[1] = rowb; strides[2] = S_loc * rowb; strides[3] = B * T_loc * S_loc * rowb;
    const int64_t frames = B * T_loc;
    p.n_outer = (int)(p.G == 1 ? frames : (frames + p.G - 1) / p.G);
  } else {          // {Dh, NH, T (pos, stride S_loc rows), S (column, stride 1 row), B}
    dims[0] = p.Dh; dims[1] = NH; dims[2] = T_loc; dims[3] = S_loc; dims[4] = B;
    strides[0] = p.Dh * e; strides[1] = S_loc * rowb; strides[2] = rowb; strides[3] = T_loc * S_loc * rowb;
    p.n_outer = (int)(p.G == 1 ? B * S_loc : B * ((S_loc + p.G - 1) / p.G));
  }
  uint32_t box_rows[2] = {(uint32_t)(p.G == 1 ? 128 : p.L), (uint32_t)p.G};
  p.items = p.n_outer * NH * p.n_qt;
  p.kv_last = p.G == 1 ? p.L - 128 * (p.n_kv - 1) : 128;
  if (p.items == 0) return cudaSuccess;
  FmhaViews vw;
  const auto* base = static_cast<const __nv_bfloat16*>(qkv);
  for (int part = 0; part < 3; ++part) {  // q, k, v: column blocks [part*C, (part+1)*C) of qkv
    vw.base[part] = base + part * C;
    for (int i = 0; i < 5; ++i) vw.dims[part][i] = dims[i];
    for (int i = 0; i < 4; ++i) vw.strides[part][i] = strides[i];
  }
  for (int i = 0; i < 5; ++i) vw.odims[i] = dims[i];
  for (int i = 0; i < 4; ++i) vw.ostr[i] = i == 0 ? strides[0] : strides[i] / 3;  // o [tok, C]: row pitch C
  return dispatch_dh(vw, p, box_rows, num_sms, st, why);
}

cudaError_t launch_fmha_cross_bf16(const void* q, const void* kv, void* o, int64_t B, int64_t Lq, int64_t Lc,
                                   int64_t C, int NH, int num_sms, cudaStream_t st, std::string* why) {
  FmhaParams p{};
  p.NH = NH;
  p.Dh = (int)(C / NH);
  p.C = (int)C;
  p.B = (int)B;
  p.S_loc = (int)Lq;
  p.T_loc = 1;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.trace = nullptr;
  p.clk = t_clk;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)p.Dh));
  p.spatial = 1;  // queries of sample b = rows [b*Lq, (b+1)*Lq) of q; keys / values = rows of kv
  p.cross = 1;
  p.L = (int)Lq;
  p.G = 1;
  p.n_qt = (int)((Lq + 127) / 128);  // a ragged last query tile is clipped by the TMA store
  p.n_kv = (int)((Lc + 127) / 128);
  p.kv_last = (int)(Lc - 128 * (p.n_kv - 1));
  p.n_outer = (int)B;
  p.items = p.n_outer * NH * p.n_qt;
  if (Lc < 1) {
    if (why) *why = "cross attention needs at least one context token";
    return cudaErrorNotSupported;
  }
  if (p.items == 0) return cudaSuccess;
  const uint64_t e = 2;
  FmhaViews vw;
  vw.base[0] = q;
  vw.base[1] = kv;
  vw.base[2] = static_cast<const __nv_bfloat16*>(kv) + C;
  const uint64_t qd[5] = {(uint64_t)p.Dh, (uint64_t)NH, (uint64_t)Lq, (uint64_t)B, 1};
  const uint64_t qs[4] = {p.Dh * e, C * e, Lq * C * e, B * Lq * C * e};
  const uint64_t kd[5] = {(uint64_t)p.Dh, (uint64_t)NH, (uint64_t)Lc, (uint64_t)B, 1};
  const uint64_t ks[4] = {p.Dh * e, 2 * C * e, Lc * 2 * C * e, B * Lc * 2 * C * e};
  for (int i = 0; i < 5; ++i) {
    vw.dims[0][i] = qd[i];
    vw.dims[1][i] = vw.dims[2][i] = kd[i];
    vw.odims[i] = qd[i];
  }
  for (int i = 0; i < 4; ++i) {
    vw.strides[0][i] = qs[i];
    vw.strides[1][i] = vw.strides[2][i] = ks[i];
    vw.ostr[i] = qs[i];
  }
  const uint32_t box_rows[2] = {128, 1};
  return dispatch_dh(vw, p, box_rows, num_sms, st, why);
}

cudaError_t launch_fmha_bf16_tseq(const void* qkv_tseq, void* o, int64_t B, int64_t T, int64_t S_loc, int64_t C,
                                  int NH, int num_sms, cudaStream_t st, std::string* why) {
  // Same tiles and dims order {Dh, NH, T (pos), S (column), B} as the token-major temporal view,
  // only the strides differ (layout [part][b][h][s][t][DP]): a tile is one contiguous block.
  FmhaParams p{};
  p.NH = NH;
  p.Dh = (int)(C / NH);
  p.C = (int)C;
  p.S_loc = (int)S_loc;
  p.T_loc = (int)T;
  p.B = (int)B;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.trace = nullptr;
  p.clk = t_clk;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)p.Dh));
  p.spatial = 0;
  p.L = (int)T;
  if (p.Dh != kTseqDh) {
    if (why) *why = "TSEQ layout needs Dh == 72";
    return cudaErrorNotSupported;
  }
  if (p.L % 128 == 0) {
    p.G = 1; p.n_kv = p.L / 128; p.n_qt = p.n_kv;
  } else if (128 % p.L == 0) {
    p.G = 128 / p.L; p.n_kv = 1; p.n_qt = 1;
  } else {
    p.G = 1; p.n_kv = (p.L + 127) / 128; p.n_qt = p.n_kv;
  }
  const uint64_t e = 2, row = kTseqDP * e;
  const uint64_t dims[5] = {(uint64_t)p.Dh, (uint64_t)NH, (uint64_t)T, (uint64_t)S_loc, (uint64_t)B};
  const uint64_t strides[4] = {S_loc * T * row, row, T * row, NH * S_loc * T * row};
  p.n_outer = (int)(p.G == 1 ? B * S_loc : B * ((S_loc + p.G - 1) / p.G));
  uint32_t box_rows[2] = {(uint32_t)(p.G == 1 ? 128 : p.L), (uint32_t)p.G};
  p.items = p.n_outer * NH * p.n_qt;
  p.kv_last = p.G == 1 ? p.L - 128 * (p.n_kv - 1) : 128;
  if (p.items == 0) return cudaSuccess;
  FmhaViews vw;
  const auto* base = static_cast<const __nv_bfloat16*>(qkv_tseq);
  const uint64_t part_elems = (uint64_t)B * NH * S_loc * T * kTseqDP;
  for (int part = 0; part < 3; ++part) {
    vw.base[part] = base + part * part_elems;
    for (int i = 0; i < 5; ++i) vw.dims[part][i] = dims[i];
    for (int i = 0; i < 4; ++i) vw.strides[part][i] = strides[i];
  }
  // o [tok, C] token-major as for the standard view: {Dh, NH, T (stride S_loc rows), S, B}
  const uint64_t orow = C * e;
  const uint64_t ostr[4] = {p.Dh * e, S_loc * orow, orow, T * S_loc * orow};
  for (int i = 0; i < 5; ++i) vw.odims[i] = dims[i];
  for (int i = 0; i < 4; ++i) vw.ostr[i] = ostr[i];
  return dispatch_dh(vw, p, box_rows, num_sms, st, why);
}

static cudaError_t dispatch_dh(const FmhaViews& vw, const FmhaParams& p, const uint32_t* box_rows, int num_sms,
                               cudaStream_t st, std::string* why) {
  const int dp = ((p.Dh + 15) / 16) * 16;
  int na = dp / 64, rb = dp % 64;
  if (rb == 48) { na += 1; rb = 0; }
  if (na == 1 && rb == 16) return run_fmha<1, 16>(vw, p, box_rows, num_sms, st, why);  // Dh 72, 80
  if (na == 0 && rb == 16) return run_fmha<0, 16>(vw, p, box_rows, num_sms, st, why);  // Dh 8, 16
  if (na == 0 && rb == 32) return run_fmha<0, 32>(vw, p, box_rows, num_sms, st, why);  // Dh 24, 32
  if (na == 1 && rb == 0) return run_fmha<1, 0>(vw, p, box_rows, num_sms, st, why);    // Dh 40..64
  if (na == 1 && rb == 32) return run_fmha<1, 32>(vw, p, box_rows, num_sms, st, why);  // Dh 88, 96
  if (na == 2 && rb == 0) return run_fmha<2, 0>(vw, p, box_rows, num_sms, st, why);    // Dh 104..128
  if (why) *why = "bf16 attention supports head dims up to 128";
  return cudaErrorNotSupported;
}


cudaError_t launch_fmha_bwd_bf16(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                                 float* dvec, float* dq_acc, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C,
                                 int NH, int dim, int num_sms, cudaStream_t st, std::string* why) {
  using Cfg = BwdCfg<1, 16>;
  FmhaParams p{};
  p.NH = NH;
  p.Dh = (int)(C / NH);
  p.C = (int)C;
  p.S_loc = (int)S_loc;
  p.T_loc = (int)T_loc;
  p.B = (int)B;
  p.clk = t_clk;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)p.Dh));
  p.spatial = (dim == DSP_DIM_S);
  p.L = (int)(p.spatial ? S_loc : T_loc);
  if (NH <= 0 || C % NH != 0 || p.Dh != 72 || C > 2048) {
    if (why) *why = "attention backward: head dim 72 only (the paper's C = 1152, 16 heads), C <= 2048";
    return cudaErrorNotSupported;
  }
  if (p.L <= 0 || !(p.L % 128 == 0 || 128 % p.L == 0)) {
    if (why) *why = "attention backward: sequence length must divide or be a multiple of 128";
    return cudaErrorNotSupported;
  }
  const int64_t tok = B * T_loc * S_loc;
  if (tok == 0) return cudaSuccess;
  if (p.L % 128 == 0) {
    p.G = 1;
    p.n_kv = p.n_qt = p.L / 128;
  } else {
    p.G = 128 / p.L;
    p.n_kv = p.n_qt = 1;
  }
  const uint64_t e = 2, rowb = 3 * (uint64_t)C * e;
  uint64_t dims[5], strides[4];
  if (p.spatial) {
    dims[0] = p.Dh; dims[1] = NH; dims[2] = S_loc; dims[3] = B * T_loc; dims[4] = 1;
    strides[0] = p.Dh * e; strides[1] = rowb; strides[2] = S_loc * rowb; strides[3] = B * T_loc * S_loc * rowb;
    const int64_t frames = B * T_loc;
    p.n_outer = (int)(p.G == 1 ? frames : (frames + p.G - 1) / p.G);
  } else {
    dims[0] = p.Dh; dims[1] = NH; dims[2] = T_loc; dims[3] = S_loc; dims[4] = B;
    strides[0] = p.Dh * e; strides[1] = S_loc * rowb; strides[2] = rowb; strides[3] = T_loc * S_loc * rowb;
    p.n_outer = (int)(p.G == 1 ? B * S_loc : B * ((S_loc + p.G - 1) / p.G));
  }
  uint64_t ostr[4];
  for (int i = 0; i < 4; ++i) ostr[i] = i == 0 ? strides[0] : strides[i] / 3;  // [tok, C] views
  p.items = p.n_outer * NH * p.n_kv;
  const int accum = p.n_kv > 1;
  const uint32_t r0 = (uint32_t)(p.G == 1 ? 128 : p.L), r1 = (uint32_t)p.G;
  uint32_t boxa[5] = {64, 1, r0, r1, 1}, boxb[5] = {16, 1, r0, r1, 1};
  BwdMaps mp;
  const auto* qb = static_cast<const __nv_bfloat16*>(qkv);
  auto* db = static_cast<__nv_bfloat16*>(dqkv);
  auto pair = [&](CUtensorMap* m, const void* base, const uint64_t* s4) {
    return make_tmap_bf16(&m[0], base, 5, dims, s4, boxa, CU_TENSOR_MAP_SWIZZLE_128B, why) &&
           make_tmap_bf16(&m[1], base, 5, dims, s4, boxb, CU_TENSOR_MAP_SWIZZLE_32B, why);
  };
  if (!pair(mp.q, qb, strides) || !pair(mp.k, qb + C, strides) || !pair(mp.v, qb + 2 * C, strides) ||
      !pair(mp.dout, dout, ostr) || !pair(mp.dq, db, strides) || !pair(mp.dk, db + C, strides) ||
      !pair(mp.dv, db + 2 * C, strides))
    return cudaErrorInvalidValue;
  if (accum) {
    uint64_t fstr[4];
    for (int i = 0; i < 4; ++i) fstr[i] = 2 * ostr[i];
    uint32_t boxf0[5] = {32, 1, r0, r1, 1}, boxf1[5] = {16, 1, r0, r1, 1};
    if (!make_tmap_f32(&mp.dq_acc[0], dq_acc, 5, dims, fstr, boxf0, why, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap_f32(&mp.dq_acc[1], dq_acc, 5, dims, fstr, boxf1, why, CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
  } else {
    mp.dq_acc[0] = mp.dq_acc[1] = mp.q[0];  // unused
  }
#ifdef DSP_FMHA_BWD_TRACE
  {
    static unsigned long long* tbuf = nullptr;
    if (!tbuf) cudaMalloc(&tbuf, 64 * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(tbuf, 0, 64 * 8 * sizeof(unsigned long long), st);
    p.trace = tbuf;
    extern unsigned long long* g_fmha_trace;
    g_fmha_trace = tbuf;
  }
#endif
  cudaError_t err = launch_attn_bwd_dvec(tok, NH, p.Dh, o, dout, dvec, st);
  if (err != cudaSuccess) return err;
  if (accum && (err = cudaMemsetAsync(dq_acc, 0, (size_t)tok * C * sizeof(float), st)) != cudaSuccess) return err;
  auto kern = p.G > 1 ? fmha_bwd_kernel<1, 16, true> : fmha_bwd_kernel<1, 16, false>;
  static bool attr[2] = {false, false};
  if (!attr[p.G > 1]) {
    if ((err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM)) != cudaSuccess)
      return err;
    attr[p.G > 1] = true;
  }
  // item walk (BwdWalk): pairs of key tiles when a sequence has several (the second reuses the first's
  // last {Q, dO}: scripts/fmha_bwd_walk_ab.py measured 387 -> 384 us spatial; longer chunks lose L2
  // locality, 447-464 us); one contiguous range per CTA for one-tile sequences (consecutive items are
  // the heads of the same tokens: temporal 107 -> 102 us).  DSP_FMHA_BWD_CH overrides (A/B).
  static const int walk_env = [] { const char* e = std::getenv("DSP_FMHA_BWD_CH"); return e ? std::atoi(e) : -1; }();
  p.walk_ch = walk_env >= 0 ? walk_env : (p.n_qt > 1 ? 2 : 0);
  const int units = p.walk_ch > 0 ? (p.items + p.walk_ch - 1) / p.walk_ch : p.items;
  const int grid = units < num_sms ? units : num_sms;
  err = launch_k(kern, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, st, 1, mp, p, lse, (const float*)dvec, accum);
  if (err != cudaSuccess) return err;
  if (accum) return launch_dq_convert(tok, C, dq_acc, dqkv, st);
  return cudaSuccess;
}

}  // namespace dsp
