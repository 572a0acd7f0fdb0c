// fmha_tc.cu — tcgen05/TMEM flash attention for the DSP spatial and temporal stages.
//
// For every sequence and head: O_j = softmax(q_j k_j^T / sqrt(Dh)) v_j (R6-R7),
// reading q/k/v straight out of the QKV projection output qkv[tok, 3C] (no head-split
// copy): a 5-D TMA map {Dh, NH, x2, x3, x4} over each of the q / k / v column blocks
// does the head split, the sequence gather (spatial rows are contiguous, temporal rows
// have stride S_loc*3C) and the Dh=72 -> 80 zero padding (out-of-bounds fill).
//
// Tile = 128 query rows x 128 key rows.  Sequences shorter than 128 are packed G=128/L
// per tile with a block-diagonal mask (temporal T=16: 8 columns per tile, interleaved
// rows r = t*G + s; spatial S<128: G whole frames per tile).  L >= 128 must be a
// multiple of 128 (S=1024, 4096; T=128).
//
// Roles (256 threads, one work item = one 128-row query tile per CTA):
//   warp 0      TMA producer: Q once, then K_j / V_j into a 2-stage ring.
//   warp 1      MMA issuer: S_{j+1} = Q K_{j+1}^T (double-buffered in TMEM) is issued
//               while the softmax works on S_j; then O += P_j V_j (P from smem, V
//               MN-major from smem) accumulating in TMEM.
//   warps 4-7   softmax + epilogue: thread = query row; online softmax in fp32 with
//               lazy rescaling (the running max only moves when it grows by > 8 in
//               log2 units, so O is rarely rescaled); P rounded to bf16 into a SW128
//               K-major smem tile; final O / l -> bf16 -> o[tok, C].
#include <cuda_bf16.h>

#include <cmath>

#include "dsp_internal.h"
#include "sm100.cuh"

namespace dsp {
namespace {

enum FmhaMode : int { SP1 = 0, SPG = 1, TP1 = 2, TPG = 3 };

struct FmhaParams {
  int mode;
  int L;          // sequence length
  int G;          // sequences per tile (1 for L >= 128)
  int n_kv;       // kv tiles per sequence (L/128 or 1)
  int n_qt;       // query tiles per sequence
  int NH, Dh, C;
  int S_loc, T_loc, B;
  int items;      // total work items
  float scale_log2;
  __nv_bfloat16* o;
};

template <int NA, int RB>
struct FmhaCfg {
  static constexpr int DP = NA * 64 + RB;                       // padded head dim
  static constexpr int RB_BYTES = RB == 0 ? 0 : 1024 * ((128 * RB * 2 + 1023) / 1024);
  static constexpr int TILE = NA * 16384 + RB_BYTES;            // one 128-row operand tile
  static constexpr int TX = 128 * DP * 2;                        // TMA bytes per tile
  static constexpr int P_BYTES = 2 * 16384;
  static constexpr int SMEM = 1024 + TILE /*Q*/ + 4 * TILE /*K,V x2*/ + P_BYTES + 256;
  static constexpr uint32_t RB_SW = RB == 16 ? SW_32B : SW_64B;
  static constexpr uint32_t RB_ROW = RB * 2;                     // bytes per row in the rem chunk
};

__device__ __forceinline__ void tile_coords(const FmhaParams& p, int item, int kv, int& h, int& x2, int& x3,
                                            int& x4) {
  // item = (outer * NH + h) * n_qt + qt
  const int qt = item % p.n_qt;
  const int rest = item / p.n_qt;
  h = rest % p.NH;
  const int outer = rest / p.NH;
  const int row0 = (kv >= 0 ? kv : qt) * 128;
  switch (p.mode) {
    case SP1:  // outer = frame (b*T_loc+t); dims {Dh, NH, S_loc, B*T_loc, 1}
      x2 = row0; x3 = outer; x4 = 0; break;
    case SPG:  // outer = frame group
      x2 = 0; x3 = outer * p.G; x4 = 0; break;
    case TP1: {  // outer = b*S_loc + s; dims {Dh, NH, S_loc, T_loc, B}
      x2 = outer % p.S_loc; x3 = row0; x4 = outer / p.S_loc; break;
    }
    default: {  // TPG: outer = b*ceil(S_loc/G) + sg
      const int ng = (p.S_loc + p.G - 1) / p.G;
      x2 = (outer % ng) * p.G; x3 = 0; x4 = outer / ng; break;
    }
  }
}

template <int NA, int RB>
__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* ma, const CUtensorMap* mb, uint64_t* bar,
                                          int h, int x2, int x3, int x4) {
#pragma unroll
  for (int i = 0; i < NA; ++i) tma_load_5d(dst + i * 16384, ma, bar, 64 * i, h, x2, x3, x4);
  if (RB) tma_load_5d(dst + NA * 16384, mb, bar, 64 * NA, h, x2, x3, x4);
}

template <int NA, int RB>
__global__ void __launch_bounds__(256, 1)
    fmha_bf16_tc_kernel(const __grid_constant__ CUtensorMap tq_a, const __grid_constant__ CUtensorMap tq_b,
                        const __grid_constant__ CUtensorMap tk_a, const __grid_constant__ CUtensorMap tk_b,
                        const __grid_constant__ CUtensorMap tv_a, const __grid_constant__ CUtensorMap tv_b,
                        const FmhaParams p) {
  using Cfg = FmhaCfg<NA, RB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::TILE;          // 2 stages
  uint8_t* sV = sK + 2 * Cfg::TILE;      // 2 stages
  uint8_t* sP = sV + 2 * Cfg::TILE;      // 2 x [128 rows x 128 B] SW128
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + Cfg::P_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* v_full = bars + 3;   // [2]
  uint64_t* kv_empty = bars + 5; // [2]
  uint64_t* s_full = bars + 7;   // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = warp_id();
  const int item = blockIdx.x;
  const int n = p.n_kv;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tq_a); tma_prefetch(&tk_a); tma_prefetch(&tv_a);
    if (RB) { tma_prefetch(&tq_b); tma_prefetch(&tk_b); tma_prefetch(&tv_b); }
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
    }
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t tS = tmem;          // 2 x 128 columns
  const uint32_t tO = tmem + 256;    // DP columns

  if (warp == 0) {
    if (elect_one()) {
      int h, x2, x3, x4;
      tile_coords(p, item, -1, h, x2, x3, x4);
      mbar_arrive_expect_tx(q_full, Cfg::TX);
      load_tile<NA, RB>(sQ, &tq_a, &tq_b, q_full, h, x2, x3, x4);
      for (int j = 0; j < n; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        tile_coords(p, item, j, h, x2, x3, x4);
        mbar_arrive_expect_tx(&k_full[st], Cfg::TX);
        load_tile<NA, RB>(sK + st * Cfg::TILE, &tk_a, &tk_b, &k_full[st], h, x2, x3, x4);
        mbar_arrive_expect_tx(&v_full[st], Cfg::TX);
        load_tile<NA, RB>(sV + st * Cfg::TILE, &tv_a, &tv_b, &v_full[st], h, x2, x3, x4);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idS = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idPVa = make_idesc_bf16(128, 64, 0, 1);
    constexpr uint32_t idPVb = make_idesc_bf16(128, RB == 0 ? 16 : RB, 0, 1);
    const uint32_t q0 = smem_u32(sQ);
    auto issue_s = [&](int j) {
      const int st = j & 1;
      mbar_wait(&k_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t k0 = smem_u32(sK + st * Cfg::TILE);
        const uint32_t d = tS + st * 128;
        int step = 0;
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k, ++step)
            umma_bf16_ss(d, make_sdesc(q0 + i * 16384 + k * 32, 16, 1024, SW_128B),
                         make_sdesc(k0 + i * 16384 + k * 32, 16, 1024, SW_128B), idS, step != 0);
        if (RB) {
#pragma unroll
          for (int k = 0; k < RB / 16; ++k, ++step)
            umma_bf16_ss(d, make_sdesc(q0 + NA * 16384 + k * 32, 16, 8 * Cfg::RB_ROW, Cfg::RB_SW),
                         make_sdesc(k0 + NA * 16384 + k * 32, 16, 8 * Cfg::RB_ROW, Cfg::RB_SW), idS, step != 0);
        }
        umma_commit(&s_full[st]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    issue_s(0);
    for (int j = 0; j < n; ++j) {
      if (j + 1 < n) issue_s(j + 1);
      const int st = j & 1;
      mbar_wait(p_full, j & 1);
      mbar_wait(&v_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t p0 = smem_u32(sP);
        const uint32_t v0 = smem_u32(sV + st * Cfg::TILE);
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 128 keys in steps of 16
          const uint64_t ad = make_sdesc(p0 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SW_128B);
#pragma unroll
          for (int i = 0; i < NA; ++i)
            umma_bf16_ss(tO + 64 * i, ad, make_sdesc(v0 + i * 16384 + k * 2048, 16384, 1024, SW_128B), idPVa,
                         (j | k) != 0);
          if (RB)
            umma_bf16_ss(tO + 64 * NA, ad,
                         make_sdesc(v0 + NA * 16384 + k * 16 * Cfg::RB_ROW, 16384, 8 * Cfg::RB_ROW, Cfg::RB_SW),
                         idPVb, (j | k) != 0);
        }
        umma_commit(o_done);
        umma_commit(&kv_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int row = q * 32 + lane_id();
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float sl2 = p.scale_log2;
    // sequence id of key column i and of this row (block-diagonal packing)
    auto seq_of = [&](int i) { return p.mode == SPG ? i / p.L : (p.mode == TPG ? i % p.G : 0); };
    const int my_seq = seq_of(row);
    const bool masked = (p.mode == SPG || p.mode == TPG);
    float m = -INFINITY, l = 0.f;
    uint8_t* prow = sP + row * 128;
    for (int j = 0; j < n; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tS + lane_off + st * 128 + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]);
      }
      if (masked) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (seq_of(i) != my_seq) s[i] = -INFINITY;
      }
      float mx = s[0];
#pragma unroll
      for (int i = 1; i < 128; ++i) mx = fmaxf(mx, s[i]);
      const float mx2 = mx * sl2;
      // lazy rescale: keep the stale max unless the new one exceeds it by > 8 (log2)
      const bool bump = (j == 0) || (mx2 > m + 8.f);
      const float m_new = bump ? mx2 : m;
      const float alpha = (j == 0) ? 0.f : fast_exp2(m - m_new);
      float rs = 0.f;
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        s[i] = fast_exp2(fmaf(s[i], sl2, -m_new));
        rs += s[i];
      }
      l = l * alpha + rs;
      m = m_new;
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);   // PV_{j-1} done: O stable, P buffer free
        tc_fence_after();
        if (__any_sync(0xffffffffu, bump)) {
          const float a = bump ? alpha : 1.f;
#pragma unroll
          for (int c = 0; c < Cfg::DP / 16; ++c) {
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
      // P (bf16) -> smem, SW128 K-major: 16-B chunk c of row r at chunk position c ^ (r & 7)
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int kb = c >> 3, cc = c & 7;
        uint4 w = make_uint4(pack_bf16x2(s[8 * c + 0], s[8 * c + 1]), pack_bf16x2(s[8 * c + 2], s[8 * c + 3]),
                             pack_bf16x2(s[8 * c + 4], s[8 * c + 5]), pack_bf16x2(s[8 * c + 6], s[8 * c + 7]));
        *reinterpret_cast<uint4*>(prow + kb * 16384 + ((cc ^ (row & 7)) << 4)) = w;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 -> o[tok, h*Dh + d]
    mbar_wait(o_done, (n - 1) & 1);
    tc_fence_after();
    int hh, x2, x3, x4;
    tile_coords(p, item, -1, hh, x2, x3, x4);
    long tok = -1;
    switch (p.mode) {
      case SP1: tok = (long)x3 * p.S_loc + x2 + row; break;
      case SPG: {
        const int f = x3 + row / p.L;
        if (f < p.B * p.T_loc) tok = (long)f * p.S_loc + row % p.L;
        break;
      }
      case TP1: tok = ((long)x4 * p.T_loc + x3 + row) * p.S_loc + x2; break;
      default: {
        const int s = x2 + row % p.G;
        if (s < p.S_loc) tok = ((long)x4 * p.T_loc + row / p.G) * p.S_loc + s;
      }
    }
    const float inv_l = 1.f / l;
    __nv_bfloat16* orow = p.o + tok * p.C + hh * p.Dh;
#pragma unroll
    for (int c = 0; c < Cfg::DP / 16; ++c) {
      uint32_t v[16];
      tmem_ld16(tO + lane_off + c * 16, v);
      tmem_ld_wait();
      if (tok >= 0) {
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8) {
          const int d = c * 16 + h8 * 8;
          if (d < p.Dh) {
            uint4 w = make_uint4(pack_bf16x2(__uint_as_float(v[h8 * 8 + 0]) * inv_l, __uint_as_float(v[h8 * 8 + 1]) * inv_l),
                                 pack_bf16x2(__uint_as_float(v[h8 * 8 + 2]) * inv_l, __uint_as_float(v[h8 * 8 + 3]) * inv_l),
                                 pack_bf16x2(__uint_as_float(v[h8 * 8 + 4]) * inv_l, __uint_as_float(v[h8 * 8 + 5]) * inv_l),
                                 pack_bf16x2(__uint_as_float(v[h8 * 8 + 6]) * inv_l, __uint_as_float(v[h8 * 8 + 7]) * inv_l));
            *reinterpret_cast<uint4*>(orow + d) = w;
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int NA, int RB>
cudaError_t run_fmha(const void* qkv, const FmhaParams& p, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box_rows, cudaStream_t st, std::string* why) {
  using Cfg = FmhaCfg<NA, RB>;
  CUtensorMap m[6];
  const auto* base = static_cast<const __nv_bfloat16*>(qkv);
  for (int part = 0; part < 3; ++part) {
    const void* b = base + part * p.C;
    uint32_t boxa[5] = {64, 1, box_rows[0], box_rows[1], 1};
    uint32_t boxb[5] = {(uint32_t)(RB ? RB : 16), 1, box_rows[0], box_rows[1], 1};
    if (!make_tmap_bf16(&m[2 * part], b, 5, dims, strides, boxa, CU_TENSOR_MAP_SWIZZLE_128B, why)) return cudaErrorInvalidValue;
    if (RB) {
      if (!make_tmap_bf16(&m[2 * part + 1], b, 5, dims, strides, boxb,
                          RB == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B, why))
        return cudaErrorInvalidValue;
    } else {
      m[2 * part + 1] = m[2 * part];
    }
  }
  auto kern = fmha_bf16_tc_kernel<NA, RB>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  kern<<<p.items, 256, Cfg::SMEM, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fmha_bf16(const void* qkv, void* o, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C, int NH,
                             int dim, cudaStream_t st, std::string* why) {
  FmhaParams p{};
  p.NH = NH;
  p.Dh = (int)(C / NH);
  p.C = (int)C;
  p.S_loc = (int)S_loc;
  p.T_loc = (int)T_loc;
  p.B = (int)B;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)p.Dh));
  const uint64_t e = 2, rowb = 3 * (uint64_t)C * e;
  uint64_t dims[5], strides[4];
  uint32_t box_rows[2];
  const bool spatial = (dim == DSP_DIM_S);
  p.L = (int)(spatial ? S_loc : T_loc);
  if (p.L % 128 == 0) {
    p.G = 1;
    p.n_kv = p.L / 128;
    p.n_qt = p.L / 128;
  } else if (128 % p.L == 0) {
    p.G = 128 / p.L;
    p.n_kv = 1;
    p.n_qt = 1;
  } else {
    if (why) *why = "bf16 attention needs the sequence length to divide 128 or be a multiple of 128";
    return cudaErrorNotSupported;
  }
  if (spatial) {
    dims[0] = p.Dh; dims[1] = NH; dims[2] = S_loc; dims[3] = B * T_loc; dims[4] = 1;
    strides[0] = p.Dh * e; strides[1] = rowb; strides[2] = S_loc * rowb; strides[3] = B * T_loc * S_loc * rowb;
    if (p.G == 1) {
      p.mode = SP1; box_rows[0] = 128; box_rows[1] = 1;
      p.items = (int)(B * T_loc * NH * p.n_qt);
    } else {
      p.mode = SPG; box_rows[0] = p.L; box_rows[1] = p.G;
      p.items = (int)(((B * T_loc + p.G - 1) / p.G) * NH);
    }
  } else {
    dims[0] = p.Dh; dims[1] = NH; dims[2] = S_loc; dims[3] = T_loc; dims[4] = B;
    strides[0] = p.Dh * e; strides[1] = rowb; strides[2] = S_loc * rowb; strides[3] = T_loc * S_loc * rowb;
    if (p.G == 1) {
      p.mode = TP1; box_rows[0] = 1; box_rows[1] = 128;
      p.items = (int)(B * S_loc * NH * p.n_qt);
    } else {
      p.mode = TPG; box_rows[0] = p.G; box_rows[1] = p.L;
      p.items = (int)(B * ((S_loc + p.G - 1) / p.G) * NH);
    }
  }
  if (p.items == 0) return cudaSuccess;
  const int dp = ((p.Dh + 15) / 16) * 16;
  int na = dp / 64, rb = dp % 64;
  if (rb == 48) { na += 1; rb = 0; }
  if (na == 1 && rb == 16) return run_fmha<1, 16>(qkv, p, dims, strides, box_rows, st, why);   // Dh 72, 80
  if (na == 0 && rb == 16) return run_fmha<0, 16>(qkv, p, dims, strides, box_rows, st, why);   // Dh 8, 16
  if (na == 0 && rb == 32) return run_fmha<0, 32>(qkv, p, dims, strides, box_rows, st, why);   // Dh 24, 32
  if (na == 1 && rb == 0) return run_fmha<1, 0>(qkv, p, dims, strides, box_rows, st, why);     // Dh 40..64
  if (na == 1 && rb == 32) return run_fmha<1, 32>(qkv, p, dims, strides, box_rows, st, why);   // Dh 88, 96
  if (na == 2 && rb == 0) return run_fmha<2, 0>(qkv, p, dims, strides, box_rows, st, why);     // Dh 104..128
  if (why) *why = "bf16 attention supports head dims up to 128";
  return cudaErrorNotSupported;
}

}  // namespace dsp
