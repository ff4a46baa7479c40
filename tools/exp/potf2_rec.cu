#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
constexpr int kNB = 64; constexpr int kLD = 65; __device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
// load the b x b diagonal block at (k0, k0); identity padding beyond b. All 16 loads of a
// thread are issued before any shared store (generic pointers would otherwise serialise them).
__device__ void load_diag(const double* L, int64_t n, int64_t k0, int b, double* a) {
  double v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = threadIdx.x + 256 * u, i = e & 63, j = e >> 6;
    double x = 0.0;
    if (i < b && j < b) {
      if (i >= j) x = L[(k0 + i) + (k0 + j) * n];
    } else if (i == j) {
      x = 1.0;
    }
    v[u] = x;
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = threadIdx.x + 256 * u;
    a[(e & 63) + (e >> 6) * kLD] = v[u];
  }
}

// write the lower b x b part of a to L and the full (zero-upper) 64 x 64 W
__device__ void store_diag(double* L, int64_t n, int64_t k0, int b, const double* a, const double* w,
                           double* Wout, bool write_l) {
  double va[16], vw[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = threadIdx.x + 256 * u, i = e & 63, j = e >> 6;
    va[u] = a[i + j * kLD];
    vw[u] = (i >= j) ? w[i + j * kLD] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = threadIdx.x + 256 * u, i = e & 63, j = e >> 6;
    if (write_l && i < b && j < b && i >= j) L[(k0 + i) + (k0 + j) * n] = va[u];
    Wout[e] = vw[u];
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

// 1/x for x > 0 from a float seed and two Newton steps (exact fallback outside float range)
__device__ __forceinline__ double rcp_fast(double x) {
  if (x > 1e-30 && x < 1e30) {
    double y = (double)__frcp_rn((float)x);
    y = y * fma(-x, y, 2.0);
    y = y * fma(-x, y, 2.0);
    return y;
  }
  return 1.0 / x;
}

// One warp factors the 16 x 16 lower block of a at (o, o) in registers (lane & 15 = row;
// lanes 16..31 mirror 0..15 so every shuffle is warp-uniform), writes L back and the
// pivot reciprocals to rl[o..o+16). Returns the first failing local pivot or -1.
// The step loop is not unrolled (the register row is rotated instead of indexed): a fully
// unrolled body is ~30 KB of straight-line SASS whose instruction fetch set the pace.
__device__ int warp_potf2_16(double* a, int o, int bvalid, double* bc, double* rl) {
  const int lane = threadIdx.x & 31, row = lane & 15;
  double r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = (k <= row) ? a[(o + row) + (o + k) * kLD] : 0.0;
  int fail = -1;
#pragma unroll 1
  for (int j = 0; j < 16; ++j) {
    double* cb = bc + 16 * (j & 1);
    const double pj = __shfl_sync(kFull, r[0], j);  // r[0] holds column j (rotated)
    if (fail < 0 && j < bvalid && (!(pj > 0.0) || !isfinite(pj))) fail = j;
    const double y = rsqrt_fast(pj);
    double lij = r[0];
    if (row == j) lij = pj * y;
    else if (row > j) lij = r[0] * y;
    if (lane < 16) {
      cb[row] = lij;
      if (row >= j) a[(o + row) + (o + j) * kLD] = lij;
      if (row == j) rl[o + j] = y;
    }
    __syncwarp();
    if (row > j) {
#pragma unroll
      for (int k = 1; k < 16; ++k)
        if (row >= j + k) r[k] = fma(-lij, cb[(j + k) & 15], r[k]);
    }
#pragma unroll
    for (int k = 0; k < 15; ++k) r[k] = r[k + 1];
    r[15] = 0.0;
  }
  return fail;
}

// One warp: w(o.., o..) = inverse of the factored 16 x 16 block of a at (o, o); rl holds the
// reciprocals of its diagonal. Substitution on L W = I, one row of W per lane.
__device__ void warp_inv16(const double* a, double* w, int o, const double* rl, double* bc) {
  const int lane = threadIdx.x & 31, row = lane & 15;
  double wr[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) wr[k] = (k == row) ? 1.0 : 0.0;
#pragma unroll 1
  for (int p = 0; p < 16; ++p) {
    double* cb = bc + 16 * (p & 1);
    if (row == p) {
      const double y = rl[o + p];
#pragma unroll
      for (int k = 0; k < 16; ++k) wr[k] *= y;
      if (lane == p) {
#pragma unroll
        for (int k = 0; k < 16; ++k) cb[k] = wr[k];
      }
    }
    __syncwarp();
    if (row > p) {
      const double lip = a[(o + row) + (o + p) * kLD];
#pragma unroll
      for (int k = 0; k < 16; ++k) wr[k] = fma(-lip, cb[k], wr[k]);
    }
    __syncwarp();
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) w[(o + row) + (o + k) * kLD] = (k <= row) ? wr[k] : 0.0;
  }
}

// Factor the b x b diagonal block at (k0, k0) and build W = L_kk^{-1}. Four 16-wide column
// blocks: the 16 x 16 diagonal block is factored inside one warp's registers (the sequential
// pivot chain), the rows below are solved against it by substitution (one thread per row),
// then all 8 warps apply the trailing update. The four 16 x 16 inverses are built afterwards
// in parallel (one warp each), and W's off-diagonal blocks follow from
// W_ij = -W_ii sum_{k=j}^{i-1} L_ik W_kj (three dependent stages).
__global__ void __launch_bounds__(256) k_potf2_inv(double* __restrict__ L, int64_t n, int64_t k0,
                                                   int b, long long* info, double* __restrict__ Wout, long long* clk) {
  long long c0 = clock64(); int ci = 0;
#define STAMP() if (threadIdx.x == 0) clk[ci++] = clock64() - c0;
  extern __shared__ double sm[];
  double* a = sm;               // kNB x kLD
  double* w = sm + kNB * kLD;   // kNB x kLD
  double* tt = w + kNB * kLD;   // 16 x 65 scratch (W stages)
  double* rl = tt + 16 * 65;    // 64 pivot reciprocals
  double* bc = rl + kNB;        // 4 warps x 32 broadcast scratch
  __shared__ int fail;
  if (*info != 0) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  load_diag(L, n, k0, b, a);
  if (tid == 0) fail = -1;
  __syncthreads();
  STAMP()
  for (int kb = 0; kb < 4; ++kb) {
    const int o = 16 * kb;
    if (warp == 0) {
      const int bv = b - o < 0 ? 0 : (b - o > 16 ? 16 : b - o);
      const int f = warp_potf2_16(a, o, bv, bc, rl);
      if (f >= 0 && tid == 0) fail = o + f;
    }
    __syncthreads();
    STAMP()
    if (fail >= 0) {
      if (tid == 0) *info = (long long)(k0 + fail + 1);
      return;
    }
    const int rows = kNB - o - 16;  // panel rows below the block
    if (rows > 0) {
      // panel: X(i, c) = (A(i, o+c) - sum_{p<c} X(i, p) L(o+c, o+p)) / L(o+c, o+c)
      if (tid < rows) {
        const int i = o + 16 + tid;
        double x[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) x[c] = a[i + (o + c) * kLD];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          double sacc = x[c];
#pragma unroll
          for (int p = 0; p < c; ++p) sacc = fma(-x[p], a[(o + c) + (o + p) * kLD], sacc);
          x[c] = sacc * rl[o + c];
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) a[i + (o + c) * kLD] = x[c];
      }
      __syncthreads();
      STAMP()
      // trailing: A(i, j) -= sum_p X(i, p) X(j, p) for o+16 <= j <= i < 64
      const int cnt = rows * rows;
      for (int e = tid; e < cnt; e += blockDim.x) {
        const int ii = e % rows, jj = e / rows;
        if (ii < jj) continue;
        const int i = o + 16 + ii, j = o + 16 + jj;
        double sacc = 0.0;
#pragma unroll
        for (int p = 0; p < 16; ++p) sacc = fma(a[i + (o + p) * kLD], a[j + (o + p) * kLD], sacc);
        a[i + j * kLD] -= sacc;
      }
      __syncthreads();
    }
  }
  STAMP()
  // W: the four diagonal 16 x 16 inverses in parallel, then the off-diagonal blocks
  if (warp < 4) warp_inv16(a, w, 16 * warp, rl, bc + 32 * warp);
  for (int e = tid; e < kNB * kNB; e += blockDim.x) {
    const int i = e & 63, j = e >> 6;
    if ((i >> 4) != (j >> 4)) w[i + j * kLD] = 0.0;
  }
  __syncthreads();
  STAMP()
  for (int d = 1; d < 4; ++d) {
    const int nblk = 4 - d;  // blocks (j + d, j), j = 0 .. nblk-1
    // T(j) = sum_{k=j}^{j+d-1} L(j+d, k) W(k, j)   (16 x 16 each)
    for (int e = tid; e < nblk * 256; e += blockDim.x) {
      const int jb = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const int ib = jb + d;
      double sacc = 0.0;
      for (int kb2 = jb; kb2 < ib; ++kb2)
#pragma unroll 4
        for (int q = 0; q < 16; ++q)
          sacc = fma(a[(16 * ib + r) + (16 * kb2 + q) * kLD], w[(16 * kb2 + q) + (16 * jb + c) * kLD], sacc);
      tt[(e & 255) + jb * 256] = sacc;
    }
    __syncthreads();
    // W(j+d, j) = -W(j+d, j+d) T(j)
    for (int e = tid; e < nblk * 256; e += blockDim.x) {
      const int jb = e >> 8, r = (e >> 4) & 15, c = e & 15;
      const int ib = jb + d;
      double sacc = 0.0;
#pragma unroll 4
      for (int q = 0; q <= r; ++q) sacc = fma(w[(16 * ib + r) + (16 * ib + q) * kLD], tt[(q << 4 | c) + jb * 256], sacc);
      w[(16 * ib + r) + (16 * jb + c) * kLD] = -sacc;
    }
    __syncthreads();
  }
  STAMP()
  store_diag(L, n, k0, b, a, w, Wout, true);
  STAMP()
}


int main() {
  const int n = 500;
  std::vector<double> M(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) M[i + j * n] = (i == j) ? n + 1.0 : 1.0 / (1 + i + j);
  double *dL, *dW; long long *dc, *info;
  cudaMalloc(&dL, 8 * n * n); cudaMalloc(&dW, 8 * 64 * 64); cudaMalloc(&dc, 8 * 64); cudaMalloc(&info, 8);
  const int smem = (2 * 64 * 65 + 16 * 65 + 64 + 128) * 8;
  cudaFuncSetAttribute(k_potf2_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(dL, M.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaMemset(info, 0, 8); cudaMemset(dc, 0, 8 * 64);
    cudaEventRecord(e0);
    k_potf2_inv<<<1, 256, smem>>>(dL, n, 0, 64, info, dW, dc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[16]; cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%.2f us  stamps:", ms * 1e3); long long prev = 0; for (int k = 0; k < 16 && c[k]; ++k) { printf(" %lld", c[k] - prev); prev = c[k]; } printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
  }
}
