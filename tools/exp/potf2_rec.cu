#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
constexpr int kNB = 64; constexpr int kLD = 65;
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
// load the b x b diagonal block at (k0, k0); identity padding beyond b
__device__ void load_diag(const double* L, int64_t n, int64_t k0, int b, double* a) {
  for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
    const int i = e & 63, j = e >> 6;
    double v = 0.0;
    if (i < b && j < b) {
      if (i >= j) v = L[(k0 + i) + (k0 + j) * n];
    } else if (i == j) {
      v = 1.0;
    }
    a[i + j * kLD] = v;
  }
}

// write the lower b x b part of a to L and the full (zero-upper) 64 x 64 W
__device__ void store_diag(double* L, int64_t n, int64_t k0, int b, const double* a, const double* w,
                           double* Wout, bool write_l) {
  for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
    const int i = e & 63, j = e >> 6;
    if (write_l && i < b && j < b && i >= j) L[(k0 + i) + (k0 + j) * n] = a[i + j * kLD];
    Wout[e] = (i >= j) ? w[i + j * kLD] : 0.0;
  }
}

// 1/sqrt(x) from a float seed and two Newton steps in FP64 (the FP64 sqrt and divide
// sequences cost several hundred cycles each on the pivot's critical path); exact
// fallback outside the float range
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

constexpr unsigned kFull = 0xffffffffu;

// One warp factors the 16 x 16 lower block of a at (o, o) in registers (lane & 15 = row;
// lanes 16..31 mirror 0..15 so every shuffle is warp-uniform) and writes L and L^{-1}
// (into w) back to shared memory. Returns the first failing local pivot or -1.
// The step loops are deliberately not unrolled (the register row is rotated instead of
// indexed): a fully unrolled body is ~30 KB of straight-line SASS whose instruction fetch,
// not the arithmetic, set the pace (27k cycles measured vs ~4k for this form).
__device__ int warp_potf2_inv16(double* a, double* w, int o, int bvalid) {
  const int lane = threadIdx.x & 31, row = lane & 15;
  double r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = (k <= row) ? a[(o + row) + (o + k) * kLD] : 0.0;
  int fail = -1;
  double myrl = 1.0;
#pragma unroll 1
  for (int j = 0; j < 16; ++j) {
    // r[0] holds column j of this row (rotated)
    const double pj = __shfl_sync(kFull, r[0], j);
    if (fail < 0 && j < bvalid && (!(pj > 0.0) || !isfinite(pj))) fail = j;
    const double y = rsqrt_fast(pj);
    double lij = r[0];
    if (row == j) {
      lij = pj * y;
      myrl = y;
    } else if (row > j) {
      lij = r[0] * y;
    }
    if (lane < 16 && row >= j) a[(o + row) + (o + j) * kLD] = lij;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      const double lkj = __shfl_sync(kFull, lij, (j + k) & 15);
      if (row >= j + k) r[k] = fma(-lij, lkj, r[k]);
    }
#pragma unroll
    for (int k = 0; k < 15; ++k) r[k] = r[k + 1];
    r[15] = 0.0;
  }
  if (fail >= 0) return fail;
  __syncwarp();
  // inverse by substitution on L W = I, one row of W per lane
  double wr[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) wr[k] = (k == row) ? 1.0 : 0.0;
#pragma unroll 1
  for (int p = 0; p < 16; ++p) {
    if (row == p) {
#pragma unroll
      for (int k = 0; k < 16; ++k) wr[k] *= myrl;
    }
    const double lip = a[(o + row) + (o + p) * kLD];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double wpk = __shfl_sync(kFull, wr[k], p);
      if (row > p) wr[k] = fma(-lip, wpk, wr[k]);
    }
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) w[(o + row) + (o + k) * kLD] = (k <= row) ? wr[k] : 0.0;
  }
  return -1;
}

// Factor the b x b diagonal block at (k0, k0) and build W = L_kk^{-1}: four 16-wide
// column blocks, each factored (with its inverse) inside one warp's registers, then the
// panel below (A_ik <- A_ik W16^T) and the trailing update by all 8 warps; W's off-diagonal
// blocks follow from W_ij = -W_ii sum_{k=j}^{i-1} L_ik W_kj (three dependent stages).
__global__ void __launch_bounds__(256) k_potf2_inv(double* __restrict__ L, int64_t n, int64_t k0,
                                                   int b, long long* info, double* __restrict__ Wout, long long* clk) {
  long long c0 = clock64(); int ci = 0;
  extern __shared__ double sm[];
  double* a = sm;              // kNB x kLD
  double* w = sm + kNB * kLD;  // kNB x kLD
  double* tt = w + kNB * kLD;  // 64 x 17 scratch (panel / W stages)
  __shared__ int fail;
  if (*info != 0) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  load_diag(L, n, k0, b, a);
  for (int e = tid; e < kNB * kNB; e += blockDim.x) w[(e & 63) + (e >> 6) * kLD] = 0.0;
  if (tid == 0) fail = -1;
  __syncthreads();
  if (threadIdx.x == 0) clk[ci++] = clock64() - c0;
  for (int kb = 0; kb < 4; ++kb) {
    const int o = 16 * kb;
    if (warp == 0) {
      const int bv = b - o < 0 ? 0 : (b - o > 16 ? 16 : b - o);
      const int f = warp_potf2_inv16(a, w, o, bv);
      if (f >= 0 && tid == 0) fail = o + f;
    }
    __syncthreads();
    if (threadIdx.x == 0) clk[ci++] = clock64() - c0;
    if (fail >= 0) {
      if (tid == 0) *info = (long long)(k0 + fail + 1);
      return;
    }
    const int rows = kNB - o - 16;  // panel rows below the block
    if (rows > 0) {
      // panel: X(i, c) = sum_{p <= c} A(i, o+p) W16(c, p), rows i = o+16.., 16 columns
      for (int e = tid; e < rows * 16; e += blockDim.x) {
        const int i = o + 16 + e % rows, c = e / rows;
        double s = 0.0;
#pragma unroll 4
        for (int q = 0; q <= c; ++q) s = fma(a[i + (o + q) * kLD], w[(o + c) + (o + q) * kLD], s);
        tt[(i - o - 16) + c * 65] = s;
      }
      __syncthreads();
      for (int e = tid; e < rows * 16; e += blockDim.x) {
        const int i = e % rows, c = e / rows;
        a[(o + 16 + i) + (o + c) * kLD] = tt[i + c * 65];
      }
      __syncthreads();
      // trailing: A(i, j) -= sum_p X(i, p) X(j, p) for o+16 <= j <= i < 64
      const int cnt = rows * rows;
      for (int e = tid; e < cnt; e += blockDim.x) {
        const int ii = e % rows, jj = e / rows;
        if (ii < jj) continue;
        const int i = o + 16 + ii, j = o + 16 + jj;
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < 16; ++p) s = fma(a[i + (o + p) * kLD], a[j + (o + p) * kLD], s);
        a[i + j * kLD] -= s;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) clk[ci++] = clock64() - c0;
  // off-diagonal blocks of W, by block distance d = i - j
  for (int d = 1; d < 4; ++d) {
    const int nblk = 4 - d;  // blocks (j + d, j), j = 0 .. nblk-1
    // T(j) = sum_{k=j}^{j+d-1} L(j+d, k) W(k, j)   (16 x 16 each)
    for (int e = tid; e < nblk * 256; e += blockDim.x) {
      const int jb = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const int ib = jb + d;
      double s = 0.0;
      for (int kb2 = jb; kb2 < ib; ++kb2)
#pragma unroll 4
        for (int q = 0; q < 16; ++q)
          s = fma(a[(16 * ib + r) + (16 * kb2 + q) * kLD], w[(16 * kb2 + q) + (16 * jb + c) * kLD], s);
      tt[(e & 255) + jb * 256] = s;
    }
    __syncthreads();
    // W(j+d, j) = -W(j+d, j+d) T(j)
    for (int e = tid; e < nblk * 256; e += blockDim.x) {
      const int jb = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const int ib = jb + d;
      double s = 0.0;
#pragma unroll 4
      for (int q = 0; q <= r; ++q) s = fma(w[(16 * ib + r) + (16 * ib + q) * kLD], tt[(q << 4 | c) + jb * 256], s);
      w[(16 * ib + r) + (16 * jb + c) * kLD] = -s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) clk[ci++] = clock64() - c0;
  store_diag(L, n, k0, b, a, w, Wout, true);
  if (threadIdx.x == 0) clk[ci++] = clock64() - c0;
}


int main() {
  const int n = 500;
  std::vector<double> M(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) M[i + j * n] = (i == j) ? n + 1.0 : 1.0 / (1 + i + j);
  double *dL, *dW; long long *dc, *info;
  cudaMalloc(&dL, 8 * n * n); cudaMalloc(&dW, 8 * 64 * 64); cudaMalloc(&dc, 8 * 32); cudaMalloc(&info, 8);
  const int smem = (2 * 64 * 65 + 16 * 65) * 8;
  cudaFuncSetAttribute(k_potf2_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(dL, M.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaMemset(info, 0, 8);
    cudaEventRecord(e0);
    k_potf2_inv<<<1, 256, smem>>>(dL, n, 0, 64, info, dW, dc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[8]; cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%.2f us  stamps:", ms * 1e3); for (int k = 0; k < 7; ++k) printf(" %lld", c[k]); printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
  }
}
