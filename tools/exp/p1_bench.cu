// Cycles of the 8 x 8 pivot-block factor (+ inverse, + stores) on one warp, in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 p1_bench.cu -o p1_bench
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

__device__ __forceinline__ double rsqrt_fast(double x) {
  if (x > 1e-30 && x < 1e30) {
    double y = (double)rsqrtf((float)x);
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y;
  }
  return 1.0 / sqrt(x);
}
// branch-free: float seed from the exponent-halved value
__device__ __forceinline__ double rsqrt_nb(double x) {
  double y = (double)rsqrtf((float)x);
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rsqrt_mufu(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double rcp_mufu(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = fma(y, fma(-x, y, 1.0), y);
  y = fma(y, fma(-x, y, 1.0), y);
  return y;
}

// LDL-style chain: eliminate with unscaled columns (pivot reciprocal on the chain), scale
// by rsqrt off the chain
template <bool INV, bool STORE>
__global__ void kl(double* g, long long* out, int reps) {
  __shared__ double a[8 * 8 + 128];
  __shared__ double st[128];
  const int lane = threadIdx.x;
  for (int e = lane; e < 64; e += 32) a[e] = g[e];
  __syncwarp();
  long long t0 = clock64();
  double acc = 0.0;
#pragma unroll 1
  for (int it = 0; it < reps; ++it) {
    double u[8][8], l[8][8], wi[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) u[i][j] = a[i * 8 + j] + acc;
    int fail = -1;
    double rl[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double d = u[j][j];
      if (fail < 0 && (!(d > 0.0) || !isfinite(d))) fail = j;
      const double r = rcp_mufu(d);
#pragma unroll
      for (int k = j + 1; k < 8; ++k) {
        const double f = u[k][j] * r;
#pragma unroll
        for (int i = k; i < 8; ++i) u[i][k] = fma(-u[i][j], f, u[i][k]);
      }
      const double y = rsqrt_mufu(d);
      rl[j] = y;
      l[j][j] = d * y;
#pragma unroll
      for (int i = j + 1; i < 8; ++i) l[i][j] = u[i][j] * y;
    }
    if (INV) {
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        wi[p][p] = rl[p];
#pragma unroll
        for (int kk = 0; kk < p; ++kk) {
          double s = 0.0;
#pragma unroll
          for (int q = kk; q < p; ++q) s = fma(l[p][q], wi[q][kk], s);
          wi[p][kk] = -rl[p] * s;
        }
      }
    }
    if (STORE) {
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) {
            st[i * 8 + j] = l[i][j];
            if (INV) st[64 + i * 8 + j] = wi[i][j];
          }
      }
      __syncwarp();
      acc = st[lane] * 1e-300;
    } else {
      acc = (l[7][7] + (INV ? wi[7][0] : 0.0) + fail) * 1e-300;
    }
    if (it == 0 && lane == 0) {
      for (int i = 0; i < 8; ++i) for (int j = 0; j <= i; ++j) g[200 + i * 8 + j] = l[i][j];
    }
  }
  long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / reps;
  g[64 + lane] = acc;
}

template <int RSQ, bool INV, bool STORE>
__global__ void k(double* g, long long* out, int reps) {
  __shared__ double a[8 * 8 + 128];
  __shared__ double st[128];
  const int lane = threadIdx.x;
  for (int e = lane; e < 64; e += 32) a[e] = g[e];
  __syncwarp();
  long long t0 = clock64();
  double acc = 0.0;
#pragma unroll 1
  for (int it = 0; it < reps; ++it) {
    double l[8][8], wi[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) l[i][j] = a[i * 8 + j] + acc;
    int fail = -1;
    double rl[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double d = l[j][j];
      if (fail < 0 && (!(d > 0.0) || !isfinite(d))) fail = j;
      const double y = RSQ == 0 ? rsqrt_fast(d) : RSQ == 1 ? rsqrt_nb(d) : rsqrt_mufu(d);
      rl[j] = y;
      l[j][j] = d * y;
#pragma unroll
      for (int i = j + 1; i < 8; ++i) l[i][j] *= y;
#pragma unroll
      for (int kk = j + 1; kk < 8; ++kk)
#pragma unroll
        for (int i = kk; i < 8; ++i) l[i][kk] = fma(-l[i][j], l[kk][j], l[i][kk]);
    }
    if (INV) {
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        wi[p][p] = rl[p];
#pragma unroll
        for (int kk = 0; kk < p; ++kk) {
          double s = 0.0;
#pragma unroll
          for (int q = kk; q < p; ++q) s = fma(l[p][q], wi[q][kk], s);
          wi[p][kk] = -rl[p] * s;
        }
      }
    }
    if (STORE) {
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) {
            st[i * 8 + j] = l[i][j];
            if (INV) st[64 + i * 8 + j] = wi[i][j];
          }
      }
      __syncwarp();
      acc = st[lane] * 1e-300;
    } else {
      acc = (l[7][7] + (INV ? wi[7][0] : 0.0) + fail) * 1e-300;
    }
  }
  long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / reps;
  g[64 + lane] = acc;
}

int main() {
  double h[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) h[i * 8 + j] = (i == j) ? 10.0 : 1.0 / (1 + i + j);
  double* g;
  long long* o;
  cudaMalloc(&g, 8 * 300);
  cudaMalloc(&o, 8);
  cudaMemcpy(g, h, 8 * 64, cudaMemcpyHostToDevice);
  long long c;
#define RUN(R, I, S)                                                         \
  k<R, I, S><<<1, 32>>>(g, o, 1000);                                         \
  k<R, I, S><<<1, 32>>>(g, o, 1000);                                         \
  cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);                              \
  printf("rsq=%d inv=%d store=%d: %lld cycles/factor\n", R, (int)I, (int)S, c);
  RUN(0, false, false)
  RUN(0, true, false)
  RUN(0, true, true)
  RUN(1, true, true)
  RUN(2, true, true)
  RUN(1, false, false)
  RUN(2, false, false)
#define RUNL(I, S)                                                        \
  kl<I, S><<<1, 32>>>(g, o, 1000);                                        \
  kl<I, S><<<1, 32>>>(g, o, 1000);                                        \
  cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);                           \
  printf("LDL-chain inv=%d store=%d: %lld cycles/factor\n", (int)I, (int)S, c);
  RUNL(false, false)
  RUNL(true, true)
  {
    double L[64];
    cudaMemcpy(L, g + 200, 8 * 64, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j <= i; ++j) {
        double s2 = 0;
        for (int k = 0; k <= j; ++k) s2 += L[i * 8 + k] * L[j * 8 + k];
        err = fmax(err, fabs(s2 - h[i * 8 + j]));
      }
    printf("LDL-chain reconstruction error %.3e\n", err);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
