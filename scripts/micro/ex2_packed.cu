// Microbenchmark: exp2 throughput per SM for fp32 (MUFU.EX2), packed f16x2 and bf16x2
// ex2.approx variants, plus the conversions a packed-softmax path would need.
// Results in "exponentials / ns / SM" (a packed op counts 2).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  uint32_t a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a[i]));
      else if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      else if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
      else if (MODE == 3) {  // f32 pair -> f16x2 pack (the conversion in front of a packed exp)
        asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i + 1) & 15]));
      } else if (MODE == 4) {  // fma.rn.f16x2 (HFMA2) as the row-sum accumulate
        asm volatile("fma.rn.f16x2 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(a[(i + 3) & 15]));
      } else if (MODE == 5) {  // mix: 1 cvt f16x2 + 1 ex2 f16x2 + 1 hadd2 (a packed softmax element pair)
        uint32_t t;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(t) : "r"(a[i]), "r"(a[(i + 1) & 15]));
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(t));
        asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(t));
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sms * 8 * 1024 * sizeof(float));
  const int iters = 4096;
  const char* names[6] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2", "cvt.f16x2.f32", "fma.f16x2", "cvt+ex2+add f16x2"};
  const double per[6] = {1, 2, 2, 1, 1, 2};  // results per instruction (exps for 0-2, 5)
  for (int mode = 0; mode < 6; ++mode) {
    for (int warps : {8, 16, 32}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto launch = [&] {
        switch (mode) {
          case 0: k<0><<<sms, warps * 32>>>(out, iters); break;
          case 1: k<1><<<sms, warps * 32>>>(out, iters); break;
          case 2: k<2><<<sms, warps * 32>>>(out, iters); break;
          case 3: k<3><<<sms, warps * 32>>>(out, iters); break;
          case 4: k<4><<<sms, warps * 32>>>(out, iters); break;
          default: k<5><<<sms, warps * 32>>>(out, iters); break;
        }
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ins = double(sms) * warps * 32 * iters * 16;
      printf("%-18s warps/SM %2d : %7.2f thread-instr/ns/SM  %7.2f results/ns/SM\n", names[mode], warps,
             ins / ms / 1e6 / sms, ins * per[mode] / ms / 1e6 / sms);
    }
  }
  return 0;
}
