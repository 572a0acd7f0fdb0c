// bwd.cu — memory-bound helpers of the ST block's backward pass.
//
//   ln_bwd_bf16_kernel     LayerNorm backward fused with the residual-gradient add (P:40 pre-LN
//                          residual block): dx = dres + rstd (g - mean(g) - xhat mean(g xhat)),
//                          g = dh * gamma; mean / rstd recomputed from x in registers (the row is
//                          read once); per-CTA column partials of dgamma = sum dh xhat and
//                          dbeta = sum dh, summed in CTA order by wgrad_reduce_kernel.
//   wgrad_reduce_kernel    out (+)= sum_s part[s] in slice order (split-K weight gradients and the
//                          LayerNorm parameter partials: deterministic, no atomics).
//   attn_bwd_dvec_kernel   D[tok, h] = sum_d dO * O (the softmax-backward row term
//                          rowsum(dP * P) = dO . O, oracle/backward.py attention_core_bwd).
//   dq_convert_kernel      dQ accumulated in fp32 by the FMHA backward -> bf16 into dqkv[:, 0:C].
// All bound by HBM bytes: one 16-B vector per lane access, rows across warps.
#include <cuda_bf16.h>

#include "dsp_internal.h"
#include "sm100.cuh"

namespace dsp {
namespace {

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    f[2 * t] = bf16lo(w[t]);
    f[2 * t + 1] = bf16hi(w[t]);
  }
}

// elements [0, h4) go to out0, [h4, n4) to out1 (float4 units; LayerNorm: dgamma | dbeta)
__global__ void __launch_bounds__(256) wgrad_reduce_kernel(const float4* __restrict__ part, int nparts, long n4,
                                                           long h4, float4* out0, float4* out1, int accumulate) {
  griddep_wait();
  griddep_launch_dependents();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4* o = i < h4 ? out0 + i : out1 + (i - h4);
    float4 a = accumulate ? *o : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nparts; ++s) {
      const float4 b = part[(long)s * n4 + i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    *o = a;
  }
}

// One warp per row (rows strided over the grid's warps), kMaxV 16-B vectors per lane (C <= 256 kMaxV).
// Dynamic smem: [warps][2][C] f32 column partials, summed over the warps in warp order at the end.
template <int kMaxV>
__global__ void __launch_bounds__(256) ln_bwd_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const __nv_bfloat16* __restrict__ dh,
                                                          const __nv_bfloat16* __restrict__ dres,
                                                          __nv_bfloat16* __restrict__ dx, float* __restrict__ part,
                                                          long rows, int C, float eps) {
  extern __shared__ float red[];
  griddep_wait();
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nv = C / 8;
  float ag[kMaxV][8], ab[kMaxV][8];  // this lane's dgamma / dbeta column accumulators
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) ag[k][i] = ab[k][i] = 0.f;
  const uint4* gvec = reinterpret_cast<const uint4*>(gamma);
  for (long r = (long)blockIdx.x * nw + wib; r < rows; r += (long)gridDim.x * nw) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + r * C);
    const uint4* hr = reinterpret_cast<const uint4*>(dh + r * C);
    float xv[kMaxV][8], hv[kMaxV][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxV; ++k) {
      const int vi = lane + 32 * k;
      if (vi < nv) {
        unpack8(xr[vi], xv[k]);
        unpack8(hr[vi], hv[k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += xv[k][i];
      }
    }
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const float mean = s / C;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxV; ++k)
      if (lane + 32 * k < nv) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float d = xv[k][i] - mean;
          q += d * d;
        }
      }
    for (int off = 16; off; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
    const float rstd = rsqrtf(q / C + eps);
    // xhat in place of x, g = dh * gamma in place of dh; sums of g and of g * xhat
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxV; ++k)
      if (lane + 32 * k < nv) {
        float gm[8];
        unpack8(gvec[lane + 32 * k], gm);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float xh = (xv[k][i] - mean) * rstd;
          xv[k][i] = xh;
          ag[k][i] += hv[k][i] * xh;
          ab[k][i] += hv[k][i];
          const float g = hv[k][i] * gm[i];
          hv[k][i] = g;
          s1 += g;
          s2 += g * xh;
        }
      }
    for (int off = 16; off; off >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    const float m1 = s1 / C, m2 = s2 / C;
    uint4* dxr = reinterpret_cast<uint4*>(dx + r * C);
    const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + r * C) : nullptr;
#pragma unroll
    for (int k = 0; k < kMaxV; ++k) {
      const int vi = lane + 32 * k;
      if (vi < nv) {
        float rv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (rr) unpack8(rr[vi], rv);
        uint32_t o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float a = rv[2 * t] + rstd * (hv[k][2 * t] - m1 - xv[k][2 * t] * m2);
          const float b = rv[2 * t + 1] + rstd * (hv[k][2 * t + 1] - m1 - xv[k][2 * t + 1] * m2);
          o[t] = pack_bf16x2(a, b);
        }
        dxr[vi] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
  // column partials: warps -> smem -> summed in warp order by the CTA's threads
#pragma unroll
  for (int k = 0; k < kMaxV; ++k) {
    const int vi = lane + 32 * k;
    if (vi < nv) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        red[(size_t)wib * 2 * C + vi * 8 + i] = ag[k][i];
        red[(size_t)wib * 2 * C + C + vi * 8 + i] = ab[k][i];
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * C; c += blockDim.x) {
    float a = 0.f;
    for (int w = 0; w < nw; ++w) a += red[(size_t)w * 2 * C + c];
    part[(size_t)blockIdx.x * 2 * C + c] = a;
  }
}

// one thread per (token, head): Dh / 8 vectors of dO and O
__global__ void __launch_bounds__(256) attn_bwd_dvec_kernel(const __nv_bfloat16* __restrict__ o,
                                                            const __nv_bfloat16* __restrict__ dout,
                                                            float* __restrict__ dvec, long n, int NH, int Dh) {
  griddep_wait();
  griddep_launch_dependents();
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long tok = i / NH;
  const int h = (int)(i % NH);
  const size_t base = (size_t)tok * NH * Dh + (size_t)h * Dh;
  const uint4* ov = reinterpret_cast<const uint4*>(o + base);
  const uint4* dv = reinterpret_cast<const uint4*>(dout + base);
  float acc = 0.f;
  for (int j = 0; j < Dh / 8; ++j) {
    float a[8], b[8];
    unpack8(ov[j], a);
    unpack8(dv[j], b);
#pragma unroll
    for (int t = 0; t < 8; ++t) acc = fmaf(a[t], b[t], acc);
  }
  dvec[i] = acc;
}

__global__ void __launch_bounds__(256) dq_convert_kernel(const float4* __restrict__ dq, uint2* __restrict__ dqkv,
                                                         long tok, int C4) {
  griddep_wait();
  griddep_launch_dependents();
  const long n = tok * C4;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long r = i / C4;
    const int c = (int)(i % C4);
    const float4 v = dq[i];
    dqkv[r * 3 * C4 + c] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
}

}  // namespace

cudaError_t launch_wgrad_reduce(const float* part, int nparts, int64_t n, float* out, int accumulate, cudaStream_t st,
                                int64_t split_at, float* out1) {
  if (n == 0) return cudaSuccess;
  if (n % 4 != 0 || (out1 && split_at % 4 != 0)) return cudaErrorInvalidValue;
  const long n4 = n / 4, h4 = out1 ? split_at / 4 : n4;
  const unsigned blocks = (unsigned)std::min<long>((n4 + 255) / 256, 148 * 8);
  return launch_k(wgrad_reduce_kernel, dim3(blocks), dim3(256), 0, st, 1, reinterpret_cast<const float4*>(part),
                  nparts, n4, h4, reinterpret_cast<float4*>(out), reinterpret_cast<float4*>(out1), accumulate);
}

int ln_bwd_blocks(int64_t rows, int num_sms) {
  const int64_t need = (rows + 7) / 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, 2 * num_sms));
}

template <int kMaxV>
static cudaError_t run_ln_bwd(int blocks, size_t smem, cudaStream_t st, const void* x, const void* gamma,
                              const void* dh, const void* dres, void* dx, float* part, int64_t rows, int64_t C,
                              float eps) {
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ln_bwd_bf16_kernel<kMaxV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         8 * 2 * 256 * kMaxV * 4);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_k(ln_bwd_bf16_kernel<kMaxV>, dim3(blocks), dim3(256), smem, st, 1, (const __nv_bfloat16*)x,
                  (const __nv_bfloat16*)gamma, (const __nv_bfloat16*)dh, (const __nv_bfloat16*)dres,
                  (__nv_bfloat16*)dx, part, (long)rows, (int)C, eps);
}

cudaError_t launch_ln_bwd(int64_t rows, int64_t C, const void* x, const void* gamma, const void* dh, const void* dres,
                          void* dx, float* part, float eps, int num_sms, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  if (C % 8 != 0 || C > 2048) return cudaErrorNotSupported;
  const int blocks = ln_bwd_blocks(rows, num_sms);
  const size_t smem = (size_t)8 * 2 * C * sizeof(float);
  if (C <= 256 * 5) return run_ln_bwd<5>(blocks, smem, st, x, gamma, dh, dres, dx, part, rows, C, eps);
  return run_ln_bwd<8>(blocks, smem, st, x, gamma, dh, dres, dx, part, rows, C, eps);
}

cudaError_t launch_attn_bwd_dvec(int64_t tok, int NH, int Dh, const void* o, const void* dout, float* dvec,
                                 cudaStream_t st) {
  const long n = tok * NH;
  if (n == 0) return cudaSuccess;
  if (Dh % 8 != 0) return cudaErrorNotSupported;
  return launch_k(attn_bwd_dvec_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, 1,
                  (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, dvec, n, NH, Dh);
}

cudaError_t launch_dq_convert(int64_t tok, int64_t C, const float* dq_acc, void* dqkv, cudaStream_t st) {
  if (tok == 0) return cudaSuccess;
  if (C % 4 != 0) return cudaErrorNotSupported;
  const long n = tok * (C / 4);
  const unsigned blocks = (unsigned)std::min<long>((n + 255) / 256, 148 * 8);
  return launch_k(dq_convert_kernel, dim3(blocks), dim3(256), 0, st, 1, reinterpret_cast<const float4*>(dq_acc),
                  reinterpret_cast<uint2*>(dqkv), (long)tok, (int)(C / 4));
}

}  // namespace dsp
