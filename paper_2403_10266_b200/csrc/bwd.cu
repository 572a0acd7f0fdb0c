// bwd.cu — memory-bound helpers of the ST block's backward pass.
//
//   ln_bwd_bf16_kernel     LayerNorm backward fused with the residual-gradient add (P:40 pre-LN
//                          residual block): dx = dres + rstd (g - mean(g) - xhat mean(g xhat)),
//                          g = dh * gamma; mean / rstd recomputed from x in registers (the row is
//                          read once); per-CTA column partials of dgamma = sum dh xhat and
//                          dbeta = sum dh, summed in CTA order by wgrad_reduce_kernel.
//   wgrad_reduce_kernel    out (+)= sum_s part[s] in slice order (split-K weight gradients and the
//                          LayerNorm parameter partials: deterministic, no atomics).
//   attn_bwd_dvec_kernel   D[tok, h] = sum_d dO * O / sqrt(Dh) (the softmax-backward row term
//                          rowsum(dP * P) = dO . O, oracle/backward.py attention_core_bwd, pre-scaled).
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
#pragma unroll 4
    for (int s = 0; s < nparts; ++s) {
      const float4 b = part[(long)s * n4 + i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    *o = a;
  }
}

// LayerNorm backward, pass 1: one warp per row, kMaxV 16-B vectors per lane (C <= 256 kMaxV); the
// row's (mean, rstd) is recomputed from x and written to `stats` for pass 2.  No column accumulators
// here, so the kernel stays small enough for several CTAs per SM (rows in flight hide HBM latency).
template <int kMaxV>
__global__ void __launch_bounds__(256) ln_bwd_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const __nv_bfloat16* __restrict__ dh,
                                                          const __nv_bfloat16* __restrict__ dres,
                                                          __nv_bfloat16* __restrict__ dx, float2* __restrict__ stats,
                                                          long rows, int C, float eps) {
  griddep_wait();
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31;
  const long r = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= rows) return;
  const int nv = C / 8;
  const uint4* gvec = reinterpret_cast<const uint4*>(gamma);
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * C);
  const uint4* hr = reinterpret_cast<const uint4*>(dh + r * C);
  const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + r * C) : nullptr;
  // the row stays packed (bf16) in registers and is unpacked per pass: ~half the registers of fp32
  // copies, so three CTAs fit per SM and more rows are in flight
  uint4 xp[kMaxV], hp[kMaxV], rp[kMaxV];
#pragma unroll
  for (int k = 0; k < kMaxV; ++k) {
    const int vi = lane + 32 * k;
    if (vi < nv) {
      xp[k] = xr[vi];
      hp[k] = hr[vi];
      if (rr) rp[k] = rr[vi];
    }
  }
  // arithmetic on bf16 pairs with packed f32x2 operations (the kernel is issue-bound, not HBM-bound)
  auto f2 = [](uint32_t v) { return make_float2(bf16lo(v), bf16hi(v)); };
  auto w4 = [](const uint4& u, int t) { return t == 0 ? u.x : t == 1 ? u.y : t == 2 ? u.z : u.w; };
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
    if (lane + 32 * k < nv) {
#pragma unroll
      for (int t = 0; t < 4; ++t) s2 = fadd2(s2, f2(w4(xp[k], t)));
    }
  float s = s2.x + s2.y;
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  const float mean = s / C;
  const float2 nm = make_float2(-mean, -mean);
  float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
    if (lane + 32 * k < nv) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 d = fadd2(f2(w4(xp[k], t)), nm);
        q2 = ffma2(d, d, q2);
      }
    }
  float q = q2.x + q2.y;
  for (int off = 16; off; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
  const float rstd = rsqrtf(q / C + eps);
  const float2 rs = make_float2(rstd, rstd);
  // sums of g = dh * gamma and of g * xhat
  float2 a1 = make_float2(0.f, 0.f), a2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kMaxV; ++k)
    if (lane + 32 * k < nv) {
      const uint4 gm = gvec[lane + 32 * k];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 g = fmul2(f2(w4(hp[k], t)), f2(w4(gm, t)));
        a1 = fadd2(a1, g);
        a2 = ffma2(g, fmul2(fadd2(f2(w4(xp[k], t)), nm), rs), a2);
      }
    }
  float s1 = a1.x + a1.y, s2s = a2.x + a2.y;
  for (int off = 16; off; off >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2s += __shfl_xor_sync(0xffffffffu, s2s, off);
  }
  const float m1 = s1 / C, m2 = s2s / C;
  const float2 nm1 = make_float2(-m1, -m1), nm2 = make_float2(-m2, -m2);
  uint4* dxr = reinterpret_cast<uint4*>(dx + r * C);
#pragma unroll
  for (int k = 0; k < kMaxV; ++k) {
    const int vi = lane + 32 * k;
    if (vi < nv) {
      const uint4 gm = gvec[vi];
      uint32_t o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        // dx = dres + rstd (g - m1 - xhat m2)
        const float2 g = fmul2(f2(w4(hp[k], t)), f2(w4(gm, t)));
        const float2 xh = fmul2(fadd2(f2(w4(xp[k], t)), nm), rs);
        const float2 u = ffma2(xh, nm2, fadd2(g, nm1));
        const float2 v = rr ? ffma2(u, rs, f2(w4(rp[k], t))) : fmul2(u, rs);
        o[t] = pack_bf16x2(v.x, v.y);
      }
      dxr[vi] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
  if (lane == 0) stats[r] = make_float2(mean, rstd);
}

// LayerNorm backward, pass 2: column partials of dgamma = sum dh xhat and dbeta = sum dh over a chunk
// of kLnRows rows per CTA.  Thread (x, y) = 8 columns (one 16-B vector of each row: a row group reads
// whole rows, coalesced) of rows r0 + y, r0 + y + kLnRG, ...; the kLnRG row groups are then added in
// y order.  part[chunk][0:C] = dgamma, part[chunk][C:2C] = dbeta, summed in chunk order after.
// kLnRG = 3: 480 threads at C = 1152, two CTAs per SM (the 256 chunks in one wave); measured per
// dsp_layer_norm_bwd call (scripts/ln_bwd_ab.py): 6 groups 55.9 us, 4 59.5, 3 52.8, 2 58.1, 1 78.8
constexpr int kLnRows = 64, kLnRG = 3;
__global__ void __launch_bounds__(1024) ln_bwd_param_kernel(const __nv_bfloat16* __restrict__ x,
                                                            const __nv_bfloat16* __restrict__ dh,
                                                            const float2* __restrict__ stats,
                                                            float* __restrict__ part, long rows, int C) {
  extern __shared__ float red[];  // [blockDim.y row groups][2][C]
  griddep_wait();
  griddep_launch_dependents();
  const int nv = C / 8;
  const int v = threadIdx.x, y = threadIdx.y;
  const long r0 = (long)blockIdx.x * kLnRows, r1 = r0 + kLnRows < rows ? r0 + kLnRows : rows;
  float ag[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, ab[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (v < nv) {
#pragma unroll 4
    for (long r = r0 + y; r < r1; r += blockDim.y) {
      const float2 st = stats[r];
      float xv[8], hv[8];
      unpack8(reinterpret_cast<const uint4*>(x + r * C)[v], xv);
      unpack8(reinterpret_cast<const uint4*>(dh + r * C)[v], hv);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        ag[i] = fmaf(hv[i], (xv[i] - st.x) * st.y, ag[i]);
        ab[i] += hv[i];
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      red[(size_t)y * 2 * C + 8 * v + i] = ag[i];
      red[(size_t)y * 2 * C + C + 8 * v + i] = ab[i];
    }
  }
  __syncthreads();
  const int nt = blockDim.x * blockDim.y, t = y * blockDim.x + v;
  for (int c = t; c < 2 * C; c += nt) {
    float a = 0.f;
    for (int k = 0; k < (int)blockDim.y; ++k) a += red[(size_t)k * 2 * C + c];
    part[(size_t)blockIdx.x * 2 * C + c] = a;
  }
}

// out[c] (+)= sum_b part[b][c] for few, long columns (nparts large, n small): warp w of the CTA sums
// parts b = w, w + 8, ... for 32 consecutive columns (lanes), then the 8 warp sums are added in warp
// order (deterministic).  out1 / split_at as wgrad_reduce_kernel.
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ part, int nparts, long n, long split_at,
                                                     float* out0, float* out1, int accumulate) {
  __shared__ float red[8][32];
  griddep_wait();
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long c = (long)blockIdx.x * 32 + lane;
  float a = 0.f;
  if (c < n)
    for (int b = w; b < nparts; b += 8) a += part[(long)b * n + c];
  red[w][lane] = a;
  __syncthreads();
  if (w == 0 && c < n) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][lane];
    float* o = (out1 && c >= split_at) ? out1 + (c - split_at) : out0 + c;
    *o = accumulate ? *o + t : t;
  }
}

// one warp per token row: lane l reads the row's 16-B vectors l, l + 32, ... of O and dO (each
// warp load instruction covers 512 contiguous bytes), the per-vector dot products go to shared memory
// and lane h adds its head's Dh / 8 of them in column order.  C <= 8 * 32 * kDvecV.
constexpr int kDvecV = 8;
__global__ void __launch_bounds__(256) attn_bwd_dvec_kernel(const __nv_bfloat16* __restrict__ o,
                                                            const __nv_bfloat16* __restrict__ dout,
                                                            float* __restrict__ dvec, long tok, int NH, int Dh) {
  __shared__ float part[8][32 * kDvecV];
  griddep_wait();
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long r = (long)blockIdx.x * 8 + w;
  if (r >= tok) return;
  const int nv = NH * Dh / 8;
  const uint4* ov = reinterpret_cast<const uint4*>(o + r * NH * Dh);
  const uint4* dv = reinterpret_cast<const uint4*>(dout + r * NH * Dh);
  uint4 a[kDvecV], b[kDvecV];
#pragma unroll
  for (int k = 0; k < kDvecV; ++k)
    if (lane + 32 * k < nv) {
      a[k] = ov[lane + 32 * k];
      b[k] = dv[lane + 32 * k];
    }
#pragma unroll
  for (int k = 0; k < kDvecV; ++k)
    if (lane + 32 * k < nv) {
      float fa[8], fb[8];
      unpack8(a[k], fa);
      unpack8(b[k], fb);
      float acc = 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t) acc = fmaf(fa[t], fb[t], acc);
      part[w][lane + 32 * k] = acc;
    }
  __syncwarp();
  const int vh = Dh / 8;
  const float sc = rsqrtf((float)Dh);  // pre-scaled: dS = P (dP - D) / sqrt(Dh) in the FMHA backward
  for (int h = lane; h < NH; h += 32) {
    float acc = 0.f;
    for (int j = 0; j < vh; ++j) acc += part[w][h * vh + j];
    dvec[r * NH + h] = acc * sc;
  }
}

// out[c][r] = in[r][c] (bf16), 64 x 64 tiles through padded smem: 16-B row-segment loads, 4-B stores
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const __nv_bfloat16* __restrict__ in,
                                                             __nv_bfloat16* __restrict__ out, int R, int Cc) {
  __shared__ __nv_bfloat16 t[64][66];
  griddep_wait();
  griddep_launch_dependents();
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {  // 64 rows x 8 vectors of 8
    const int r = i >> 3, v = i & 7;
    if (r0 + r < R && c0 + 8 * v < Cc) {
      const uint4 w = *reinterpret_cast<const uint4*>(in + (size_t)(r0 + r) * Cc + c0 + 8 * v);
      const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&w);
#pragma unroll
      for (int k = 0; k < 8; ++k) t[r][8 * v + k] = e[k];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) {  // 64 output rows (columns of in) x 32 pairs
    const int c = i >> 5, rp = i & 31;
    if (c0 + c < Cc && r0 + 2 * rp + 1 < R + 1) {
      __nv_bfloat162 v2;
      v2.x = t[2 * rp][c];
      v2.y = t[2 * rp + 1][c];
      if (r0 + 2 * rp + 1 < R) *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(c0 + c) * R + r0 + 2 * rp) = v2;
      else if (r0 + 2 * rp < R) out[(size_t)(c0 + c) * R + r0 + 2 * rp] = v2.x;
    }
  }
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
  (void)num_sms;
  return (int)std::max<int64_t>(1, (rows + kLnRows - 1) / kLnRows);  // pass-2 row chunks = partials
}

int64_t ln_bwd_scratch_bytes(int64_t rows, int64_t C) {
  return ((rows * 8 + 255) / 256) * 256 + (int64_t)ln_bwd_blocks(rows, 0) * 2 * C * 4;
}

cudaError_t launch_ln_bwd(int64_t rows, int64_t C, const void* x, const void* gamma, const void* dh, const void* dres,
                          void* dx, float* scratch, float* dgamma, float* dbeta, int accumulate, float eps,
                          int num_sms, cudaStream_t st) {
  (void)num_sms;
  if (rows == 0) return cudaSuccess;
  if (C % 8 != 0 || C > 2048) return cudaErrorNotSupported;
  float2* stats = reinterpret_cast<float2*>(scratch);
  float* part = scratch + ((rows * 8 + 255) / 256) * 256 / 4;
  const unsigned blocks = (unsigned)((rows * 32 + 255) / 256);
  cudaError_t e;
  if (C <= 256 * 5)
    e = launch_k(ln_bwd_bf16_kernel<5>, dim3(blocks), dim3(256), 0, st, 1, (const __nv_bfloat16*)x,
                 (const __nv_bfloat16*)gamma, (const __nv_bfloat16*)dh, (const __nv_bfloat16*)dres, (__nv_bfloat16*)dx,
                 stats, (long)rows, (int)C, eps);
  else
    e = launch_k(ln_bwd_bf16_kernel<8>, dim3(blocks), dim3(256), 0, st, 1, (const __nv_bfloat16*)x,
                 (const __nv_bfloat16*)gamma, (const __nv_bfloat16*)dh, (const __nv_bfloat16*)dres, (__nv_bfloat16*)dx,
                 stats, (long)rows, (int)C, eps);
  if (e != cudaSuccess) return e;
  const int chunks = ln_bwd_blocks(rows, num_sms), nv = (int)(C / 8);
  const int bx = ((nv + 31) / 32) * 32, rg = std::min(kLnRG, 1024 / bx);  // row groups per CTA
  const size_t smem = (size_t)rg * 2 * C * sizeof(float);
  static bool attr = false;
  if (!attr) {
    if ((e = cudaFuncSetAttribute(ln_bwd_param_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kLnRG * 2 * 2048 * 4)) != cudaSuccess)
      return e;
    attr = true;
  }
  e = launch_k(ln_bwd_param_kernel, dim3((unsigned)chunks), dim3((unsigned)bx, (unsigned)rg), smem, st, 1,
               (const __nv_bfloat16*)x, (const __nv_bfloat16*)dh, (const float2*)stats, part, (long)rows, (int)C);
  if (e != cudaSuccess) return e;
  return launch_k(colsum_kernel, dim3((unsigned)((2 * C + 31) / 32)), dim3(256), 0, st, 1, (const float*)part, chunks,
                  (long)(2 * C), (long)C, dgamma, dbeta, accumulate);
}

cudaError_t launch_attn_bwd_dvec(int64_t tok, int NH, int Dh, const void* o, const void* dout, float* dvec,
                                 cudaStream_t st) {
  if (tok == 0 || NH == 0) return cudaSuccess;
  if (Dh % 8 != 0 || (int64_t)NH * Dh > 8 * 32 * kDvecV) return cudaErrorNotSupported;
  return launch_k(attn_bwd_dvec_kernel, dim3((unsigned)((tok + 7) / 8)), dim3(256), 0, st, 1,
                  (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, dvec, (long)tok, NH, Dh);
}

cudaError_t launch_transpose_bf16(const void* in, void* out, int64_t R, int64_t Cc, cudaStream_t st) {
  if (R == 0 || Cc == 0) return cudaSuccess;
  if (Cc % 8 != 0 || R % 2 != 0) return cudaErrorNotSupported;
  return launch_k(transpose_bf16_kernel, dim3((unsigned)((Cc + 63) / 64), (unsigned)((R + 63) / 64)), dim3(256), 0, st, 1,
                  (const __nv_bfloat16*)in, (__nv_bfloat16*)out, (int)R, (int)Cc);
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
