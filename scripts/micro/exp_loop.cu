// Microbenchmark: the softmax exponential loop of the FMHA (x = s*c - m on pairs, 2^x on the
// MUFU or the FMA-pipe polynomial, bf16 pack) in isolation: clk per 64-element row chunk for
// 1, 2, 4 warps per SMSP and poly fractions 0..8/16.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace dsp;

template <int PN, int MODE>
__global__ void k(uint32_t* out, int iters, long long* cyc, float c, float m) {
  uint32_t v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __float_as_uint(-0.01f * (i + threadIdx.x % 7));
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pk[32];
    const float2 cc = make_float2(c, c), mm = make_float2(-m, -m);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), cc, mm);
      float2 e;
      if ((i % 16) < PN) {
        e = poly_exp2_x2(x);
      } else {
        e.x = fast_exp2(x.x);
        e.y = fast_exp2(x.y);
      }
      pk[i] = MODE == 0 ? pack_bf16x2(e.x, e.y) : (__float_as_uint(e.x) ^ __float_as_uint(e.y));
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) { acc ^= pk[i]; v[2 * i] ^= (acc & 1); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int PN, int MODE>
void run(int sms, uint32_t* out, long long* cyc) {
  for (int warps : {4, 8, 16}) {
    const int iters = 2000;
    k<PN, MODE><<<sms, warps * 32>>>(out, iters, cyc, 0.17f, 0.5f);
    cudaDeviceSynchronize();
    k<PN, MODE><<<sms, warps * 32>>>(out, iters, cyc, 0.17f, 0.5f);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    // per SMSP: warps/4 warps each doing 64 elements per iteration
    printf("poly %2d/16 %s warps/SMSP %d : %6.1f clk per 64-elt chunk per warp-slot  (%.2f elt/clk/SMSP)\n", PN,
           MODE == 0 ? "pack" : "nopack", warps / 4, double(c) / iters / (warps / 4),
           64.0 * 32 * (warps / 4) * iters / double(c));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, sms * 1024 * sizeof(uint32_t));
  long long* cyc; cudaMalloc(&cyc, sms * sizeof(long long));
  run<0, 0>(sms, out, cyc);
  run<4, 0>(sms, out, cyc);
  run<6, 0>(sms, out, cyc);
  run<8, 0>(sms, out, cyc);
  run<6, 1>(sms, out, cyc);
  run<16, 0>(sms, out, cyc);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
