// Experiment: where does the 64x64 register-blocked potf2 spend its time?
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
constexpr int kNB = 64;
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
template <int V>
__global__ void __launch_bounds__(256) kpotf2(double* L, int n, double* Wout, long long* clk) {
  __shared__ double col[kNB], wrow[kNB], piv[kNB + 1];
  const int t = threadIdx.x, bi = t & 15, bk = t >> 4;
  const int r0 = 4 * bi, c0 = 4 * bk;
  double a[4][4], w[4][4];
  long long t0 = clock64();
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = r0 + r, k = c0 + c;
      a[r][c] = (i >= k) ? L[i + k * n] : 0.0;
      w[r][c] = (i == k) ? 1.0 : 0.0;
    }
  if (t == 0) piv[0] = a[0][0];
  __syncthreads();
  long long t1 = clock64();
  for (int j = 0; j < kNB; ++j) {
    const double d = piv[j];
    double l;
    if (V & 1) l = 1.5; else l = sqrt(d);
    const int jb = j >> 2, jc = j & 3;
    if (bk == jb) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = r0 + r;
        double x = jc == 0 ? a[r][0] : jc == 1 ? a[r][1] : jc == 2 ? a[r][2] : a[r][3];
        if (i > j) {
          const double v = (V & 2) ? x * 0.7 : dv(x, l);
          if (jc == 0) a[r][0] = v; if (jc == 1) a[r][1] = v; if (jc == 2) a[r][2] = v; if (jc == 3) a[r][3] = v;
          col[i] = v;
        }
      }
    }
    if (!(V & 4) && bi == jb) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double x = jc == 0 ? w[0][c] : jc == 1 ? w[1][c] : jc == 2 ? w[2][c] : w[3][c];
        const double v = (V & 2) ? x * 0.7 : dv(x, l);
        if (jc == 0) w[0][c] = v; if (jc == 1) w[1][c] = v; if (jc == 2) w[2][c] = v; if (jc == 3) w[3][c] = v;
        wrow[c0 + c] = v;
      }
    }
    __syncthreads();
    const bool a_act = bk <= bi && c0 + 3 > j;
    const bool w_act = !(V & 4) && r0 + 3 > j && c0 <= j;
    if (a_act || w_act) {
      double ci[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) ci[r] = (r0 + r > j) ? col[r0 + r] : 0.0;
      if (a_act) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int k = c0 + c;
          if (k > j) {
            const double ck = col[k];
#pragma unroll
            for (int r = 0; r < 4; ++r) if (r0 + r >= k) a[r][c] = fma(-ci[r], ck, a[r][c]);
          }
        }
      }
      if (w_act) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c0 + c <= j) {
            const double wq = wrow[c0 + c];
#pragma unroll
            for (int r = 0; r < 4; ++r) w[r][c] = fma(-ci[r], wq, w[r][c]);
          }
        }
      }
    }
    if (j + 1 < kNB && bi == bk && bi == ((j + 1) >> 2)) {
      const int q = (j + 1) & 3;
      piv[j + 1] = q == 0 ? a[0][0] : q == 1 ? a[1][1] : q == 2 ? a[2][2] : a[3][3];
    }
    __syncthreads();
  }
  long long t2 = clock64();
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = r0 + r, k = c0 + c;
      L[i + k * n] = a[r][c];
      Wout[i + k * kNB] = w[r][c];
    }
  long long t3 = clock64();
  if (t == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; }
}

template <int V>
void run(double* dL, double* dW, long long* dc, const std::vector<double>& M, int n, const char* name) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(dL, M.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    kpotf2<V><<<1, 256>>>(dL, n, dW, dc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c[3]; cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("%-28s %8.2f us  cycles load %lld loop %lld store %lld  (%s)\n", name, ms * 1e3, c[0], c[1], c[2], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int n = 64;
  std::vector<double> M(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) M[i + j * n] = (i == j) ? n + 1.0 : 1.0 / (1 + i + j);
  double *dL, *dW; long long* dc;
  cudaMalloc(&dL, 8 * n * n); cudaMalloc(&dW, 8 * n * n); cudaMalloc(&dc, 64);
  run<0>(dL, dW, dc, M, n, "full");
  run<1>(dL, dW, dc, M, n, "no sqrt");
  run<2>(dL, dW, dc, M, n, "no div");
  run<3>(dL, dW, dc, M, n, "no sqrt no div");
  run<4>(dL, dW, dc, M, n, "no W");
  run<7>(dL, dW, dc, M, n, "no W no sqrt/div");
  return 0;
}
