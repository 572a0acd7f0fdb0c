// Microbenchmark: MUFU.EX2 and FFMA throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (MODE == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A000000;" : "+f"(a[i]));
      else { float t; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(a[i])); asm volatile("fma.rn.f32 %0, %1, 0f3F7FFFFF, %0;" : "+f"(a[i]) : "f"(t)); }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms * 8 * 1024 * sizeof(float));
  const int iters = 4096;
  const char* names[3] = {"MUFU.EX2", "FFMA", "EX2+FFMA"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16, 32}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto launch = [&] {
        if (mode == 0) k<0><<<sms, warps * 32>>>(out, iters);
        else if (mode == 1) k<1><<<sms, warps * 32>>>(out, iters);
        else k<2><<<sms, warps * 32>>>(out, iters);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = double(sms) * warps * 32 * iters * 16;
      // cycles at the clock actually used are unknown here; report ops / ns and per-SM per-ns
      printf("%-9s warps/SM %2d : %8.1f Gop/s  = %6.2f op/ns/SM\n", names[mode], warps, ops / ms / 1e6, ops / ms / 1e6 / sms);
    }
  }
  printf("SMs %d, nominal max clock %.0f MHz\n", sms, clk / 1e3);
  return 0;
}
