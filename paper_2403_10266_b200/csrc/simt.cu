// simt.cu — fp32 check path: plain SIMT CUDA kernels for the
// 1e-4 gate at the tiny config.  tcgen05 kind::tf32 is not used here (10-bit
// mantissa would not meet 1e-4).  Same semantics as the bf16 tensor-core path.
#include <cuda_bf16.h>
#include <cmath>
#include <type_traits>

#include "dsp_internal.h"
#include "sm100.cuh"

namespace dsp {
namespace {

// D[M,N] = epi(A[M,K] W[N,K]^T), 64x64 tile, 16x16 threads, 4x4 outputs per thread.
template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, const float* __restrict__ W,
                                                       const float* R, float* D, int M, int N, int K) {
  __shared__ float As[16][65];
  __shared__ float Ws[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i / 16, kk = i % 16;
      As[kk][r] = (m0 + r < M && k0 + kk < K) ? A[(size_t)(m0 + r) * K + k0 + kk] : 0.f;
      Ws[kk][r] = (n0 + r < N && k0 + kk < K) ? W[(size_t)(n0 + r) * K + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[kk][ty * 4 + i], Ws[kk][tx * 4 + j], acc[i][j]);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, nn = n0 + tx * 4 + j;
      if (m < M && nn < N) {
        float v = acc[i][j];
        if (EPI == DSP_EPI_RESIDUAL) v += R[(size_t)m * N + nn];
        if (EPI == DSP_EPI_GELU) v = 0.5f * v * (1.f + tanhf(0.7978845608028654f * (v + 0.044715f * v * v * v)));
        D[(size_t)m * N + nn] = v;
      }
    }
}

// One warp per (sequence, head, query row); exact softmax in two passes over keys.
// qkv [tok, 3C]; token of position `pos` in sequence `seq`:
//   tok = (seq / n_in) * stride_out + (seq % n_in) * stride_in + pos * pos_stride
__global__ void attn_f32_kernel(const float* __restrict__ qkv, float* __restrict__ o, int nseq, int L, int NH, int Dh,
                                int C, int n_in, long stride_out, long stride_in, long pos_stride) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long total = (long)nseq * NH * L;
  if (gw >= total) return;
  const int i = gw % L;
  const int h = (gw / L) % NH;
  const int seq = gw / (L * NH);
  const long base = (seq / n_in) * stride_out + (long)(seq % n_in) * stride_in;
  const float scale = 1.f / sqrtf((float)Dh);
  const float* qrow = qkv + (base + i * pos_stride) * 3 * C + h * Dh;
  float mx = -INFINITY;
  for (int j = 0; j < L; ++j) {
    const float* krow = qkv + (base + j * pos_stride) * 3 * C + C + h * Dh;
    float d = 0.f;
    for (int t = lane; t < Dh; t += 32) d = fmaf(qrow[t], krow[t], d);
    for (int off = 16; off; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
    mx = fmaxf(mx, d * scale);
  }
  float accv[4] = {0.f, 0.f, 0.f, 0.f};  // Dh <= 128
  float sum = 0.f;
  for (int j = 0; j < L; ++j) {
    const float* krow = qkv + (base + j * pos_stride) * 3 * C + C + h * Dh;
    const float* vrow = krow + C;
    float d = 0.f;
    for (int t = lane; t < Dh; t += 32) d = fmaf(qrow[t], krow[t], d);
    for (int off = 16; off; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
    const float pj = expf(d * scale - mx);
    sum += pj;
    for (int t = lane, u = 0; t < Dh; t += 32, ++u) accv[u] = fmaf(pj, vrow[t], accv[u]);
  }
  float* orow = o + (base + i * pos_stride) * C + h * Dh;
  for (int t = lane, u = 0; t < Dh; t += 32, ++u) orow[t] = accv[u] / sum;
}

// LayerNorm: one warp per row, fp32 math, two-pass (mean, then centred variance).
template <typename T>
__device__ __forceinline__ float ldf(const T* p, long i);
template <>
__device__ __forceinline__ float ldf<float>(const float* p, long i) { return p[i]; }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p, long i) { return __bfloat162float(p[i]); }

template <typename T>
__global__ void layer_norm_kernel(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b, float eps,
                                  T* y, long rows, int C) {
  griddep_wait();
  griddep_launch_dependents();
  const long r = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const T* xr = x + r * C;
  constexpr int kMax = 48;  // up to C = 1536 held in registers for bf16
  float v[kMax];
  float s = 0.f;
  int n = 0;
  for (int c = lane; c < C; c += 32, ++n) {
    const float f = ldf(xr, c);
    if (n < kMax) v[n] = f;
    s += f;
  }
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  const float mean = s / C;
  float q = 0.f;
  n = 0;
  for (int c = lane; c < C; c += 32, ++n) {
    const float d = (n < kMax ? v[n] : ldf(xr, c)) - mean;
    q += d * d;
  }
  for (int off = 16; off; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
  const float rstd = rsqrtf(q / C + eps);
  T* yr = y + r * C;
  n = 0;
  for (int c = lane; c < C; c += 32, ++n) {
    const float f = (n < kMax ? v[n] : ldf(xr, c));
    const float o = (f - mean) * rstd * ldf(g, c) + ldf(b, c);
    if constexpr (std::is_same<T, float>::value) yr[c] = o;
    else yr[c] = __float2bfloat16_rn(o);
  }
}

// bf16 LayerNorm for C % 8 == 0: 16-B vector accesses and the whole row in registers (C <= 256
// kMaxV), the arithmetic on bf16 pairs with packed f32x2 adds / multiplies / FMAs (ncu of the scalar
// version: issue-active 75 %, i.e. bound by its instruction count, not by HBM).
__device__ __forceinline__ float2 bf16x2_f2(uint32_t v) { return make_float2(bf16lo(v), bf16hi(v)); }
template <int kMaxV>
__global__ void __launch_bounds__(256) layer_norm_bf16_vec_kernel(const __nv_bfloat16* __restrict__ x,
                                                                  const __nv_bfloat16* __restrict__ g,
                                                                  const __nv_bfloat16* __restrict__ b, float eps,
                                                                  __nv_bfloat16* y, long rows, int C) {
  griddep_wait();
  griddep_launch_dependents();
  const long r = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int nv = C / 8;  // 16-B vectors per row
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * C);
  uint4 buf[kMaxV];
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
    if (lane + 32 * k < nv) buf[k] = xr[lane + 32 * k];
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
    if (lane + 32 * k < nv) {
      s2 = fadd2(s2, fadd2(bf16x2_f2(buf[k].x), bf16x2_f2(buf[k].y)));
      s2 = fadd2(s2, fadd2(bf16x2_f2(buf[k].z), bf16x2_f2(buf[k].w)));
    }
  float s = s2.x + s2.y;
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  const float mean = s / C;
  const float2 nm = make_float2(-mean, -mean);
  float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
    if (lane + 32 * k < nv) {
      const uint32_t w[4] = {buf[k].x, buf[k].y, buf[k].z, buf[k].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 d = fadd2(bf16x2_f2(w[t]), nm);
        q2 = ffma2(d, d, q2);
      }
    }
  float q = q2.x + q2.y;
  for (int off = 16; off; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
  const float rstd = rsqrtf(q / C + eps);
  const float2 rs = make_float2(rstd, rstd);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
  uint4* yr = reinterpret_cast<uint4*>(y + r * C);
#pragma unroll
  for (int k = 0; k < kMaxV; ++k) {
    const int vi = lane + 32 * k;
    if (vi < nv) {
      const uint4 gg = gv[vi], bb = bv[vi];
      const uint32_t w[4] = {buf[k].x, buf[k].y, buf[k].z, buf[k].w};
      const uint32_t gw[4] = {gg.x, gg.y, gg.z, gg.w};
      const uint32_t bw[4] = {bb.x, bb.y, bb.z, bb.w};
      uint32_t o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 xh = fmul2(fadd2(bf16x2_f2(w[t]), nm), rs);
        const float2 v = ffma2(xh, bf16x2_f2(gw[t]), bf16x2_f2(bw[t]));
        o[t] = pack_bf16x2(v.x, v.y);
      }
      yr[vi] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

#ifndef DSP_ROWSTATS_R
#define DSP_ROWSTATS_R 1  // measured: 1 row per warp 14.2 us, 2: 16.2, 4: 28.5 (LN1 stage, blk N=1)
#endif
// Per-row LayerNorm statistics (mean, rstd) of a bf16 [rows, C] activation, two-pass in
// registers like the LayerNorm kernel; 8 bytes out per row.  Used to fold LN into the GEMM
// that consumes it (LN(x) W^T = rstd (x (W o gamma)^T - mean u) + W beta).
template <int kMaxV>  // 16-B vectors per lane: C <= 256 * kMaxV
__global__ void __launch_bounds__(256, kMaxV <= 5 ? 4 : 2) row_stats_bf16_kernel(const __nv_bfloat16* __restrict__ x, float eps,
                                                                float2* __restrict__ stats, long rows, int C,
                                                                unsigned long long* clk) {
  griddep_wait();
  griddep_launch_dependents();
  clk_start(clk);
  // DSP_ROWSTATS_R rows per warp (32 warps resident per SM), all loads issued before any reduction
  constexpr int R = DSP_ROWSTATS_R;
  const long r0 = (((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * R;
  const int lane = threadIdx.x & 31;
  const int nv = C / 8;
  uint4 buf[R][kMaxV];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + (r0 + q) * C);
#pragma unroll
    for (int k = 0; k < kMaxV; ++k) {
      const int vi = lane + 32 * k;
      buf[q][k] = (r0 + q < rows && vi < nv) ? xr[vi] : make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxV; ++k) {
      const uint32_t w[4] = {buf[q][k].x, buf[q][k].y, buf[q][k].z, buf[q][k].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) s += __uint_as_float(w[t] << 16) + __uint_as_float(w[t] & 0xFFFF0000u);
    }
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const float mean = s / C;
    float qq = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxV; ++k) {
      if (lane + 32 * k < nv) {
        const uint32_t w[4] = {buf[q][k].x, buf[q][k].y, buf[q][k].z, buf[q][k].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float a = __uint_as_float(w[t] << 16) - mean, c = __uint_as_float(w[t] & 0xFFFF0000u) - mean;
          qq += a * a + c * c;
        }
      }
    }
    for (int off = 16; off; off >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, off);
    if (lane == 0 && r0 + q < rows) stats[r0 + q] = make_float2(mean, rsqrtf(qq / C + eps));
  }
  if (clk) {
    __syncthreads();
    clk_end(clk);
  }
}

// Per-row LayerNorm partials (mean_p, M2_p) of a bf16 [rows, C] activation over column segments
// of `seg` values, BITWISE identical to the partials the residual GEMM epilogue writes for the
// rows it stores (gemm_tc.cu, kStats; R30): per segment, values shifted by the segment's first
// value, even / odd columns summed in two lanes in column order (s1, s2 = sum d, sum d*d),
// a = s1e + s1o, mp = a * (1/seg), partial = (mp + x0, max(s2e + s2o - a*mp, 0)), every step
// with explicit round-to-nearest intrinsics (no contraction differences).  Used after a switch
// (N > 1), where the rows arrive without the partials their producer computed, so the LN
// statistics the consuming GEMM combines are the same bits at every N.
// One thread per (row, segment).
__device__ __forceinline__ void wait_peer_rows(const PeerWait& pw, uint64_t epoch, long row) {
  const int src = pw.mode == 2 ? (int)(row % pw.S) / pw.Sn : (int)((row / pw.S_loc) % pw.T) / pw.Tn;
  const uint64_t* slot = pw.pad + src;
  uint64_t v = 0, t0 = 0;
  if (pw.timeout_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
    if (v >= epoch) return;
    if (pw.timeout_ns) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > pw.timeout_ns) {
        atomicCAS(reinterpret_cast<unsigned long long*>(const_cast<uint64_t*>(pw.pad) + kPadError), 0ull,
                  (unsigned long long)((epoch << 16) | (2u << 8) | (unsigned)src));
        return;
      }
    }
    __nanosleep(64);
  }
}

__global__ void __launch_bounds__(256) row_partials_bf16_kernel(const __nv_bfloat16* __restrict__ x, long rows, int C,
                                                                int seg, float2* __restrict__ parts,
                                                                unsigned long long* clk, PeerWait pw) {
  griddep_wait();
  // a waiting launch lets its dependent (the next, SM-filling GEMM) launch only once its rows are
  // in: early-resident dependents would hold the SMs the peers' producers need when virtual ranks
  // share one GPU
  if (!pw.pad) griddep_launch_dependents();
  clk_start(clk);
  const int nseg = C / seg;
  const uint64_t epoch = pw.pad ? *reinterpret_cast<const volatile uint64_t*>(pw.pad + kPadEpoch) : 0;
  // grid-stride (a waiting launch is capped at one CTA per SM, so it never crowds out the peers'
  // producers when virtual ranks share one GPU)
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < rows * nseg;
       idx += (long)gridDim.x * blockDim.x) {
    const long row = idx / nseg;
    const int sg = (int)(idx % nseg);
    if (pw.pad) wait_peer_rows(pw, epoch, row);
    const uint4* p = reinterpret_cast<const uint4*>(x + row * C + (long)sg * seg);
    float x0 = 0.f, s1e = 0.f, s1o = 0.f, s2e = 0.f, s2o = 0.f;
    for (int j = 0; j < seg / 8; ++j) {
      const uint4 v = p[j];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float lo = __uint_as_float(w[t] << 16), hi = __uint_as_float(w[t] & 0xFFFF0000u);
        if (j == 0 && t == 0) x0 = lo;
        const float de = __fadd_rn(lo, -x0), dd = __fadd_rn(hi, -x0);
        s1e = __fadd_rn(s1e, de);
        s1o = __fadd_rn(s1o, dd);
        s2e = __fmaf_rn(de, de, s2e);
        s2o = __fmaf_rn(dd, dd, s2o);
      }
    }
    const float a = __fadd_rn(s1e, s1o), mp = __fmul_rn(a, __frcp_rn((float)seg));
    parts[idx] = make_float2(__fadd_rn(mp, x0), fmaxf(__fmaf_rn(-a, mp, __fadd_rn(s2e, s2o)), 0.f));
  }
  if (pw.pad) griddep_launch_dependents();
  if (clk) clk_end(clk);  // thread 0 (partial of CTA-wide span; the CTA's other rows finish alongside)
}

// Fold a LayerNorm's affine parameters into the weight of the following linear layer:
//   W'[n, c] = bf16(W[n, c] * gamma[c]),  u[n] = sum_c W'[n, c],  v[n] = sum_c W[n, c] * beta[c]
// One warp per output row n; up to 3 matrices per launch (blockIdx.y).
struct FoldJob {
  const __nv_bfloat16* W;
  const __nv_bfloat16* gamma;
  const __nv_bfloat16* beta;
  __nv_bfloat16* Wf;
  float* u;
  float* v;
  int N;
};
struct FoldJobs {
  FoldJob j[4];
};
__global__ void fold_ln_weights_kernel(FoldJobs jobs, int K) {
  griddep_wait();
  griddep_launch_dependents();
  const FoldJob& J = jobs.j[blockIdx.y];
  const long n = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (n >= J.N) return;
  const uint4* wr = reinterpret_cast<const uint4*>(J.W + n * K);
  const uint4* g4 = reinterpret_cast<const uint4*>(J.gamma);
  const uint4* b4 = reinterpret_cast<const uint4*>(J.beta);
  uint4* wf = reinterpret_cast<uint4*>(J.Wf + n * K);
  float su = 0.f, sv = 0.f;
  for (int vi = lane; vi < K / 8; vi += 32) {
    const uint4 w = wr[vi], g = g4[vi], b = b4[vi];
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w}, gg[4] = {g.x, g.y, g.z, g.w}, bb[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float w0 = __uint_as_float(ww[t] << 16), w1 = __uint_as_float(ww[t] & 0xFFFF0000u);
      const float p0 = w0 * __uint_as_float(gg[t] << 16), p1 = w1 * __uint_as_float(gg[t] & 0xFFFF0000u);
      __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);
      o[t] = *reinterpret_cast<uint32_t*>(&pb);
      su += __low2float(pb) + __high2float(pb);
      sv += w0 * __uint_as_float(bb[t] << 16) + w1 * __uint_as_float(bb[t] & 0xFFFF0000u);
    }
    wf[vi] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  for (int off = 16; off; off >>= 1) {
    su += __shfl_xor_sync(0xffffffffu, su, off);
    sv += __shfl_xor_sync(0xffffffffu, sv, off);
  }
  if (lane == 0) {
    J.u[n] = su;
    J.v[n] = sv;
  }
}
}  // namespace

cudaError_t launch_gemm_f32(const float* A, const float* W, const float* R, float* D, int64_t M, int64_t N, int64_t K,
                            int epi, cudaStream_t st) {
  if (M == 0 || N == 0) return cudaSuccess;
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
  switch (epi) {
    case DSP_EPI_NONE: gemm_f32_kernel<DSP_EPI_NONE><<<grid, 256, 0, st>>>(A, W, R, D, (int)M, (int)N, (int)K); break;
    case DSP_EPI_RESIDUAL: gemm_f32_kernel<DSP_EPI_RESIDUAL><<<grid, 256, 0, st>>>(A, W, R, D, (int)M, (int)N, (int)K); break;
    case DSP_EPI_GELU: gemm_f32_kernel<DSP_EPI_GELU><<<grid, 256, 0, st>>>(A, W, R, D, (int)M, (int)N, (int)K); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_attn_f32(const float* qkv, float* o, int64_t B, int64_t T_loc, int64_t S_loc, int64_t C, int NH,
                            int dim, cudaStream_t st) {
  int nseq, L, n_in;
  long so, si, ps;
  if (dim == DSP_DIM_S) {  // sequences over S per frame
    nseq = (int)(B * T_loc); L = (int)S_loc; n_in = 1; so = S_loc; si = 0; ps = 1;
  } else {                 // sequences over T per (b, s)
    nseq = (int)(B * S_loc); L = (int)T_loc; n_in = (int)S_loc; so = T_loc * S_loc; si = 1; ps = S_loc;
  }
  const long warps = (long)nseq * NH * L;
  if (warps == 0) return cudaSuccess;
  const int threads = 256;
  const long blocks = (warps * 32 + threads - 1) / threads;
  attn_f32_kernel<<<(unsigned)blocks, threads, 0, st>>>(qkv, o, nseq, L, NH, (int)(C / NH), (int)C, n_in, so, si, ps);
  return cudaGetLastError();
}

cudaError_t launch_layer_norm(int dtype, int64_t rows, int64_t C, const void* x, const void* g, const void* b, float eps,
                              void* y, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const int threads = 256;
  const unsigned blocks = (unsigned)((rows * 32 + threads - 1) / threads);
  if (dtype == DSP_F32) {
    return launch_k(layer_norm_kernel<float>, dim3(blocks), dim3(threads), 0, st, 1, (const float*)x, (const float*)g,
                    (const float*)b, eps, (float*)y, rows, (int)C);
  } else if (C % 8 == 0 && C <= 2048) {
    auto kern = C <= 256 * 5 ? layer_norm_bf16_vec_kernel<5> : layer_norm_bf16_vec_kernel<8>;
    return launch_k(kern, dim3(blocks), dim3(threads), 0, st, 1, (const __nv_bfloat16*)x, (const __nv_bfloat16*)g,
                    (const __nv_bfloat16*)b, eps, (__nv_bfloat16*)y, rows, (int)C);
  } else {
    return launch_k(layer_norm_kernel<__nv_bfloat16>, dim3(blocks), dim3(threads), 0, st, 1, (const __nv_bfloat16*)x,
                    (const __nv_bfloat16*)g, (const __nv_bfloat16*)b, eps, (__nv_bfloat16*)y, rows, (int)C);
  }
  return cudaGetLastError();
}

}  // namespace dsp

namespace dsp {

cudaError_t launch_row_stats(int64_t rows, int64_t C, const void* x, float eps, void* stats, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const int threads = 256;
  const long warps = (rows + DSP_ROWSTATS_R - 1) / DSP_ROWSTATS_R;
  const unsigned blocks = (unsigned)((warps * 32 + threads - 1) / threads);
  if (C % 8 || C > 256 * kRowStatsMaxV) return cudaErrorNotSupported;
  if (C <= 1280)  // the model widths of the paper (1152): 5 vectors per lane
    return launch_k(row_stats_bf16_kernel<5>, dim3(blocks), dim3(threads), 0, st, 1, (const __nv_bfloat16*)x, eps,
                    (float2*)stats, rows, (int)C, t_clk);
  return launch_k(row_stats_bf16_kernel<kRowStatsMaxV>, dim3(blocks), dim3(threads), 0, st, 1,
                  (const __nv_bfloat16*)x, eps, (float2*)stats, rows, (int)C, t_clk);
}

// Temporal positional embedding (R37): x[b, t, s, :] += pe[t, :] on an S-sharded activation
// [B, T, S_loc, C] (bf16, in place; fp32 add, one rounding).  One thread per 8 channels.
__global__ void __launch_bounds__(256) add_temporal_pe_kernel(__nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ pe, long rows,
                                                              int T, int S_loc, int C, unsigned long long* clk) {
  griddep_wait();
  griddep_launch_dependents();
  clk_start(clk);
  const int cv = C / 8;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < rows * cv) {
    const long row = idx / cv;
    const int c8 = (int)(idx % cv);
    const int t = (int)((row / S_loc) % T);
    uint4* px = reinterpret_cast<uint4*>(x + row * C) + c8;
    const uint4 a = *px, b = reinterpret_cast<const uint4*>(pe + (long)t * C)[c8];
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      o[i] = pack_bf16x2(bf16lo(aw[i]) + bf16lo(bw[i]), bf16hi(aw[i]) + bf16hi(bw[i]));
    *px = make_uint4(o[0], o[1], o[2], o[3]);
  }
  if (clk) clk_end(clk);
}

cudaError_t launch_add_temporal_pe(void* x, const void* pe, int64_t B, int64_t T, int64_t S_loc, int64_t C,
                                   cudaStream_t st) {
  const long rows = (long)(B * T * S_loc);
  if (C % 8) return cudaErrorNotSupported;
  const long n = rows * (C / 8);
  if (n == 0) return cudaSuccess;
  return launch_k(add_temporal_pe_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, 1,
                  (__nv_bfloat16*)x, (const __nv_bfloat16*)pe, rows, (int)T, (int)S_loc, (int)C, t_clk);
}

// adaLN-Zero fold for one sample (R36): per sublayer k, LN affine (1 + scale_k) and shift_k, and
// the output projection's rows scaled by gate_k.  blockIdx.y = job; grid-stride over elements.
struct AdaJob {
  const __nv_bfloat16 *g, *b, *W;  // LN gamma / beta [C], output weight [C, K] (rows = C outputs)
  __nv_bfloat16 *g_out, *b_out, *W_out;
  const float* mod;                // [3][C]: shift, scale, gate
  int K;
};
struct AdaJobs {
  AdaJob j[4];
};
__global__ void __launch_bounds__(256) adaln_fold_kernel(AdaJobs jobs, int C) {
  griddep_wait();
  griddep_launch_dependents();
  const AdaJob& J = jobs.j[blockIdx.y];
  const float* shift = J.mod;
  const float* scale = J.mod + C;
  const float* gate = J.mod + 2 * C;
  const long nW = (long)C * J.K;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nW + C; i += (long)gridDim.x * blockDim.x) {
    if (i < nW) {
      const int n = (int)(i / J.K);
      J.W_out[i] = __float2bfloat16_rn(__bfloat162float(J.W[i]) * gate[n]);
    } else {
      const int c = (int)(i - nW);
      const float sc = 1.f + scale[c];
      J.g_out[c] = __float2bfloat16_rn(__bfloat162float(J.g[c]) * sc);
      J.b_out[c] = __float2bfloat16_rn(__fmaf_rn(__bfloat162float(J.b[c]), sc, shift[c]));
    }
  }
}

cudaError_t launch_adaln_fold(int njobs, const AdaFold* jobs, int64_t C, cudaStream_t st) {
  AdaJobs aj{};
  for (int i = 0; i < njobs; ++i)
    aj.j[i] = AdaJob{(const __nv_bfloat16*)jobs[i].gamma, (const __nv_bfloat16*)jobs[i].beta,
                     (const __nv_bfloat16*)jobs[i].W, (__nv_bfloat16*)jobs[i].gamma_out,
                     (__nv_bfloat16*)jobs[i].beta_out, (__nv_bfloat16*)jobs[i].W_out, jobs[i].mod, (int)jobs[i].K};
  if (njobs == 0) return cudaSuccess;
  return launch_k(adaln_fold_kernel, dim3(148 * 4, njobs), dim3(256), 0, st, 1, aj, (int)C);
}

cudaError_t launch_row_partials(int64_t rows, int64_t C, int seg, const void* x, float2* parts, cudaStream_t st,
                                const PeerWait& pw, int num_sms) {
  if (rows == 0) return cudaSuccess;
  if (seg % 8 || C % seg) return cudaErrorNotSupported;
  const long n = rows * (C / seg);
  long blocks = (n + 255) / 256;
  if (pw.pad && blocks > num_sms) blocks = num_sms;
  return launch_k(row_partials_bf16_kernel, dim3((unsigned)blocks), dim3(256), 0, st, 1, (const __nv_bfloat16*)x,
                  (long)rows, (int)C, seg, parts, t_clk, pw);
}

cudaError_t launch_fold_ln_weights(int njobs, const LnFold* jobs, int64_t K, cudaStream_t st) {
  FoldJobs fj{};
  int maxN = 0;
  for (int i = 0; i < njobs; ++i) {
    fj.j[i] = FoldJob{(const __nv_bfloat16*)jobs[i].W, (const __nv_bfloat16*)jobs[i].gamma,
                      (const __nv_bfloat16*)jobs[i].beta, (__nv_bfloat16*)jobs[i].Wf, jobs[i].u, jobs[i].v,
                      (int)jobs[i].N};
    if (jobs[i].N > maxN) maxN = (int)jobs[i].N;
  }
  const int threads = 256;
  dim3 grid((unsigned)((maxN * 32 + threads - 1) / threads), (unsigned)njobs);
  return launch_k(fold_ln_weights_kernel, grid, dim3(threads), 0, st, 1, fj, (int)K);
}

}  // namespace dsp
