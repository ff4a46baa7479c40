#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* clk, int iters) {
  double v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += __shfl_sync(0xffffffffu, v[i], (it + i) & 31);
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[0] = (t1 - t0) / iters;
}
__global__ void k2(double* out, long long* clk, int iters) {
  double v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
  double acc[16] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(__shfl_sync(0xffffffffu, v[i], (it + i) & 31), 1.0001, acc[i]);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) clk[0] = (t1 - t0) / iters;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 8 * 32); cudaMalloc(&c, 8);
  long long h;
  k<<<1, 32>>>(d, c, 100); cudaDeviceSynchronize(); k<<<1, 32>>>(d, c, 1000); cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("16 shfl(double) + dependent adds: %lld cycles/iter\n", h);
  k2<<<1, 32>>>(d, c, 100); cudaDeviceSynchronize(); k2<<<1, 32>>>(d, c, 1000); cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("16 shfl(double) + independent fma: %lld cycles/iter\n", h);
}
