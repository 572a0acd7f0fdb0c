// Microbenchmark: which pipe F2FP (cvt.rn.bf16x2.f32) issues to, relative to MUFU.EX2.
// Throughput per SM per ns for EX2 alone, CVT alone, EX2 + CVT mixed 2:1 (the softmax mix),
// and FMNMX / FFMA2 for scale.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
      } else if (MODE == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        a[i] = __uint_as_float(r);
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i + 1]), "f"(a[i]));
        a[i + 1] = __uint_as_float(r);
      } else if (MODE == 2) {  // 2 EX2 : 1 CVT
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        a[(i + 2) & 15] += __uint_as_float(r);
      } else if (MODE == 3) {
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[i + 1]));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i + 1]) : "f"(a[i]));
      } else if (MODE == 4) {
        asm volatile("{.reg .b64 x; mov.b64 x, {%0, %1}; fma.rn.f32x2 x, x, x, x; mov.b64 {%0, %1}, x;}"
                     : "+f"(a[i]), "+f"(a[i + 1]));
      } else if (MODE == 5) {  // 2 EX2 : 1 FFMA2 : 1 FADD (no CVT) control
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        a[(i + 2) & 15] += a[i];
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sms * 8 * 1024 * sizeof(float));
  const int iters = 4096;
  const char* names[6] = {"EX2", "CVT.bf16x2", "2EX2+1CVT", "FMNMX", "FFMA2", "2EX2+1FADD"};
  const double per_iter[6] = {16, 16, 24, 16, 8, 24};  // instructions per thread per iteration
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
      double ins = double(sms) * warps * 32 * iters * per_iter[mode];
      printf("%-11s warps/SM %2d : %7.2f instr(thread)/ns/SM  (%.1f us)\n", names[mode], warps, ins / ms / 1e6 / sms, ms * 1e3);
    }
  }
  return 0;
}
