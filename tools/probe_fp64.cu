// FP64 throughput probe for B200 (sm_100a): DMMA (mma.sync .f64 shapes) and DFMA.
// Also checks the m16n8k16 / m16n8k4 / m8n8k4 f64 fragment layouts against a host product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_fp64 probe_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void mma_m8n8k4(double* d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k4(double* d, const double* a, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k8(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma_m16n8k16(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE, int NACC>
__global__ void peak_mma(double* out, int iters, double seed) {
  double acc[NACC][4];
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = seed * (threadIdx.x - i);
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) acc[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      if (SHAPE == 0) mma_m8n8k4(acc[j], a[0], b[0]);
      if (SHAPE == 1) mma_m16n8k4(acc[j], a, b[0]);
      if (SHAPE == 2) mma_m16n8k8(acc[j], a, b);
      if (SHAPE == 3) mma_m16n8k16(acc[j], a, b);
    }
  }
  double s = 0;
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void peak_dfma(double* out, int iters, double seed) {
  double acc[NACC];
  for (int j = 0; j < NACC; ++j) acc[j] = seed * (threadIdx.x + j);
  const double m = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j] = fma(acc[j], m, c);
  }
  double s = 0;
  for (int j = 0; j < NACC; ++j) s += acc[j];
  if (s == 12345.678) out[0] = s;
}

// layout check for m16n8k16: A 16x16 row-major, B 16x8 (k x n), C 16x8
__global__ void layout_k16(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4], d[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i % 2)) * 16 + t + 4 * (i / 2)];
  for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  mma_m16n8k16(d, a, b);
  C[g * 8 + 2 * t] = d[0]; C[g * 8 + 2 * t + 1] = d[1];
  C[(g + 8) * 8 + 2 * t] = d[2]; C[(g + 8) * 8 + 2 * t + 1] = d[3];
}
__global__ void layout_k8(const double* A, const double* B, double* C) {  // A 16x8, B 8x8
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[4], b[2], d[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; ++i) a[i] = A[(g + 8 * (i % 2)) * 8 + t + 4 * (i / 2)];
  for (int i = 0; i < 2; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  mma_m16n8k8(d, a, b);
  C[g * 8 + 2 * t] = d[0]; C[g * 8 + 2 * t + 1] = d[1];
  C[(g + 8) * 8 + 2 * t] = d[2]; C[(g + 8) * 8 + 2 * t + 1] = d[3];
}

template <typename K>
double time_kernel(K kern, int blocks, int threads, int iters, double flops_per_thread_iter) {
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters / 10, 1e-3); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters, 1e-3);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return flops_per_thread_iter * (double)blocks * threads * iters / (ms * 1e-3) / 1e12;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d, clock %d kHz\n", sms, clk);
  // flops per thread per iter: mma flops = 2*M*N*K per warp per mma, / 32 threads, * NACC
  const int it = 20000;
  for (int wpb : {4, 8, 16}) {
    int th = 32 * wpb;
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      printf("warps/blk %2d blk/SM %d: ", wpb, bps);
      printf("m8n8k4 %.2f  ", time_kernel(peak_mma<0, 8>, blocks, th, it, 8.0 * 2 * 8 * 8 * 4 / 32));
      printf("m16n8k4 %.2f  ", time_kernel(peak_mma<1, 8>, blocks, th, it, 8.0 * 2 * 16 * 8 * 4 / 32));
      printf("m16n8k8 %.2f  ", time_kernel(peak_mma<2, 8>, blocks, th, it / 2, 8.0 * 2 * 16 * 8 * 8 / 32));
      printf("m16n8k16 %.2f  ", time_kernel(peak_mma<3, 8>, blocks, th, it / 4, 8.0 * 2 * 16 * 8 * 16 / 32));
      printf("dfma %.2f TF/s\n", time_kernel(peak_dfma<8>, blocks, th, it, 8.0 * 2));
    }
  }
  // sustained: long run of m16n8k16
  printf("sustained m16n8k16 (long): %.2f TF/s\n", time_kernel(peak_mma<3, 8>, sms * 2, 256, 400000, 8.0 * 2 * 16 * 8 * 16 / 32));
  printf("sustained dfma (long): %.2f TF/s\n", time_kernel(peak_dfma<8>, sms * 2, 256, 1600000, 16.0));

  // layout checks
  std::vector<double> A(256), B(128), C(128), R(128);
  for (int i = 0; i < 256; ++i) A[i] = (i * 7 % 13) - 6 + 0.5 * (i % 3);
  for (int i = 0; i < 128; ++i) B[i] = (i * 5 % 11) - 5 + 0.25 * (i % 4);
  double *dA, *dB, *dC;
  CK(cudaMalloc(&dA, 256 * 8)); CK(cudaMalloc(&dB, 128 * 8)); CK(cudaMalloc(&dC, 128 * 8));
  CK(cudaMemcpy(dA, A.data(), 256 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), 128 * 8, cudaMemcpyHostToDevice));
  layout_k16<<<1, 32>>>(dA, dB, dC); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(C.data(), dC, 128 * 8, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 8; ++j) {
    double s = 0; for (int k = 0; k < 16; ++k) s += A[i * 16 + k] * B[k * 8 + j];
    err = fmax(err, fabs(s - C[i * 8 + j]));
  }
  printf("layout m16n8k16 max err %g\n", err);
  layout_k8<<<1, 32>>>(dA, dB, dC); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(C.data(), dC, 128 * 8, cudaMemcpyDeviceToHost));
  err = 0;
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 8; ++j) {
    double s = 0; for (int k = 0; k < 8; ++k) s += A[i * 8 + k] * B[k * 8 + j];
    err = fmax(err, fabs(s - C[i * 8 + j]));
  }
  printf("layout m16n8k8 max err %g\n", err);
  return 0;
}
