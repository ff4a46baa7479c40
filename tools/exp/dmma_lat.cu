// latency of dependent FP64 mma.sync (m16n8k4 / m16n8k16) on one warp
#include <cstdio>
#include "../../paper_2209_13049_b200/csrc/ptx.cuh"
using namespace cmpc;
__global__ void k(double* out, long long* cyc, int reps) {
  double acc[4] = {0, 0, 0, 0};
  double a[2] = {1e-3 * threadIdx.x, 2e-3}, b = 3e-3;
  double a8[8], b4[4];
  for (int i = 0; i < 8; ++i) a8[i] = 1e-3 * i;
  for (int i = 0; i < 4; ++i) b4[i] = 1e-3 * i;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) dmma1684(acc, a, b);
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) dmma16816(acc, a8, b4);
  long long t2 = clock64();
  double acc2[4][4] = {};
  for (int r = 0; r < reps; ++r)
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma1684(acc2[u], a, b);
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; cyc[1] = (t2 - t1) / reps; cyc[2] = (t3 - t2) / reps; }
  out[threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3] + acc2[0][0] + acc2[3][3];
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 1000); k<<<1, 32>>>(o, c, 1000);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("dependent m16n8k4: %lld cyc; dependent m16n8k16: %lld cyc; 4 independent m16n8k4 chains: %lld cyc/step\n", h[0], h[1], h[2]);
  return 0;
}
