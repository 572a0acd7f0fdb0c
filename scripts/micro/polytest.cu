#include <cstdio>
#include <cmath>
#include "sm100.cuh"
using namespace dsp;
__global__ void k(const float* in, float* out, int n) {
  int i = threadIdx.x;
  if (i < n) {
    float2 x = make_float2(in[i], in[i]);
    float2 e = poly_exp2_x2(x);
    out[2 * i] = e.x;
    out[2 * i + 1] = fast_exp2(in[i]);
  }
}
int main() {
  float h[6] = {-INFINITY, -1e30f, -200.f, -127.f, -126.f, -3.5f};
  float *d, *o; cudaMalloc(&d, 64); cudaMalloc(&o, 128);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, o, 6);
  float r[12]; cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 6; ++i) printf("x=%g poly=%g mufu=%g\n", h[i], r[2 * i], r[2 * i + 1]);
}
