// dependent-chain latencies on B200: DFMA, DMUL, DADD, FFMA, SHFL, double div/sqrt, rsqrtf
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void chain(double* out, float* outf, int iters, double seed) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  float xf = (float)seed, yf = 1.0001f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = fma(x, y, 1e-12);
    if (OP == 1) x = x * y;
    if (OP == 2) x = x + 1e-9;
    if (OP == 3) xf = fmaf(xf, yf, 1e-6f);
    if (OP == 4) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    if (OP == 5) x = 1.0 / (x + 1.5);
    if (OP == 6) x = sqrt(x + 1.5);
    if (OP == 7) xf = rsqrtf(xf + 1.5f);
    if (OP == 8) x = (double)rsqrtf((float)(x + 1.5));
    if (OP == 9) { x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31); x = fma(x, y, 1e-12); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; outf[0] = xf; out[1] = (double)(t1 - t0) / iters; }
}
template <int OP>
void run(const char* name) {
  double* d; float* f; cudaMalloc(&d, 16); cudaMalloc(&f, 8);
  chain<OP><<<1, 32>>>(d, f, 1000, 0.5); cudaDeviceSynchronize();
  chain<OP><<<1, 32>>>(d, f, 10000, 0.5); cudaDeviceSynchronize();
  double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-22s %7.1f cycles/op\n", name, h[1]);
}
int main() {
  run<0>("DFMA chain"); run<1>("DMUL chain"); run<2>("DADD chain"); run<3>("FFMA chain");
  run<4>("SHFL chain"); run<5>("double 1/x chain"); run<6>("double sqrt chain");
  run<7>("rsqrtf chain"); run<8>("f2f+rsqrtf+f2f"); run<9>("shfl+dfma chain");
}
