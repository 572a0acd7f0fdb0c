// Microbenchmark: tcgen05.ld throughput per SM (TMEM -> registers), 32x32b.x32 shape, with 4
// and 8 warps (1 or 2 per TMEM lane quadrant) and 1 / 2 / 4 loads in flight per wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace dsp;

template <int INFLIGHT>
__global__ void k(float* out, int iters, long long* cyc) {
  __shared__ uint32_t holder;
  if (warp_id() == 0) { tmem_alloc(&holder, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = holder + (((warp_id() & 3) * 32) << 16) + (warp_id() >> 2) * 128;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[4][32];
#pragma unroll
    for (int i = 0; i < INFLIGHT; ++i) tmem_ld32(tm + i * 32, v[i]);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < INFLIGHT; ++i)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= v[i][j];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(acc);
  tc_fence_before(); __syncthreads();
  if (warp_id() == 0) { tc_fence_after(); tmem_dealloc(holder, 512); }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sms * 1024 * sizeof(float));
  long long* cyc; cudaMalloc(&cyc, sms * sizeof(long long));
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int inflight : {1, 2, 4}) {
      auto launch = [&] {
        if (inflight == 1) k<1><<<sms, warps * 32>>>(out, iters, cyc);
        else if (inflight == 2) k<2><<<sms, warps * 32>>>(out, iters, cyc);
        else k<4><<<sms, warps * 32>>>(out, iters, cyc);
      };
      launch(); cudaDeviceSynchronize();
      launch(); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      double bytes = double(warps) * 32 * 32 * 4 * inflight * iters;  // per SM
      printf("warps %2d inflight %d : %7.1f B/clk/SM  (%lld clk)\n", warps, inflight, bytes / c, c);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
