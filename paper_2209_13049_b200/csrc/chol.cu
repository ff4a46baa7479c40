// K2/K3/K4: Cholesky of the condensed matrix with the reference's failure rule, and
// the two triangular solves.
//
// Reference: ReferenceBackend::factorize (proj/src/dense_linalg.cpp:59-77, block 64:
// potf2 :24-40, trsm :43-51, trailing rankUpdate), failure "!(diag > 0) || !isfinite"
// at the first pivot; Factor::solve (:102-110). The shift ladder (proj/src/ipm.cpp:
// 205-221) re-factors M + delta I; here M is kept intact and L written separately, so a
// retry never repeats the SYRK. info = failing pivot + 1 (0 = success).
//
// Blocked right-looking, 64-wide panels: potf2 of the diagonal block in shared memory
// (1 CTA), panel TRSM (1 CTA per 64-row block), trailing lower SYRK on DMMA tensor
// cores (1 CTA per 64x64 tile). Every kernel returns immediately once info != 0.
#include "internal.cuh"
#include "ptx.cuh"

namespace cmpc {

namespace {

constexpr int kNB = 64;
constexpr int kLD = kNB + 1;
constexpr int kTrsmSmem = 2 * kNB * kLD * 8;
constexpr int kTrailSmem = 2 * kNB * 68 * 8;

__global__ void k_chol_copy(const double* __restrict__ M, double* __restrict__ L, int64_t n,
                            double delta, long long* info) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) *info = 0;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (i >= n) return;
  double v = 0.0;
  if (i > j) v = M[i + j * n];
  else if (i == j) v = delta == 0.0 ? M[i + j * n] : add(M[i + j * n], delta);
  L[i + j * n] = v;
}

// factor the b x b diagonal block at (k0, k0)
__global__ void k_potf2(double* __restrict__ L, int64_t n, int64_t k0, int b, long long* info) {
  __shared__ double a[kNB * kLD];
  __shared__ int fail;
  if (*info != 0) return;
  const int tid = threadIdx.x;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int i = e % b, j = e / b;
    if (i >= j) a[i + j * kLD] = L[(k0 + i) + (k0 + j) * n];
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (tid == 0) {
      const double d = a[j + j * kLD];
      if (!(d > 0.0) || !isfinite(d)) {
        fail = 1;
        *info = (long long)(k0 + j + 1);
      } else {
        a[j + j * kLD] = sqrt(d);
      }
    }
    __syncthreads();
    if (fail) return;
    const double djj = a[j + j * kLD];
    for (int i = j + 1 + tid; i < b; i += blockDim.x) a[i + j * kLD] = dv(a[i + j * kLD], djj);
    __syncthreads();
    const int w = b - j - 1;
    for (int e = tid; e < w * w; e += blockDim.x) {
      const int i = j + 1 + e % w, k = j + 1 + e / w;
      if (i >= k) a[i + k * kLD] -= a[i + j * kLD] * a[k + j * kLD];
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int i = e % b, j = e / b;
    if (i >= j) L[(k0 + i) + (k0 + j) * n] = a[i + j * kLD];
  }
}

// X <- X L11^{-T} for the 64-row block below the diagonal block (4 threads per row)
__global__ void k_trsm(double* __restrict__ L, int64_t n, int64_t k0, int b, long long* info) {
  extern __shared__ double sm_trsm[];
  double* l11 = sm_trsm;
  double* x = sm_trsm + kNB * kLD;  // x[r + j*kLD]
  if (*info != 0) return;
  const int tid = threadIdx.x;
  const int64_t r0 = k0 + b + (int64_t)blockIdx.x * kNB;
  const int rows = (int)(n - r0 < kNB ? n - r0 : kNB);
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int i = e % b, j = e / b;
    l11[i + j * kLD] = (i >= j) ? L[(k0 + i) + (k0 + j) * n] : 0.0;
  }
  for (int e = tid; e < kNB * b; e += blockDim.x) {
    const int i = e % kNB, j = e / kNB;
    x[i + j * kLD] = (i < rows) ? L[(r0 + i) + (k0 + j) * n] : 0.0;
  }
  __syncthreads();
  const int r = tid >> 2, q = tid & 3;
  for (int j = 0; j < b; ++j) {
    double s = 0.0;
    for (int p = q; p < j; p += 4) s += x[r + p * kLD] * l11[j + p * kLD];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q == 0) x[r + j * kLD] = dv(x[r + j * kLD] - s, l11[j + j * kLD]);
    __syncwarp();
  }
  __syncthreads();
  for (int e = tid; e < rows * b; e += blockDim.x) {
    const int i = e % rows, j = e / rows;
    L[(r0 + i) + (k0 + j) * n] = x[i + j * kLD];
  }
}

// trailing update A22(I,J) -= X_I X_J^T, lower tiles only, DMMA m16n8k4
__global__ void __launch_bounds__(128) k_trail(double* __restrict__ L, int64_t n, int64_t k0, int b,
                                               long long* info) {
  extern __shared__ double sm_trail[];
  double* xi = sm_trail;  // xi[k*68 + i]
  double* xj = sm_trail + kNB * 68;
  if (*info != 0) return;
  const int ti = blockIdx.x, tj = blockIdx.y;
  if (ti < tj) return;
  const int64_t base = k0 + b;
  const int64_t i0 = base + (int64_t)ti * kNB, j0 = base + (int64_t)tj * kNB;
  const int tid = threadIdx.x;
  for (int e = tid; e < kNB * kNB; e += blockDim.x) {
    const int i = e % kNB, k = e / kNB;
    xi[k * 68 + i] = (k < b && i0 + i < n) ? L[(i0 + i) + (k0 + k) * n] : 0.0;
    xj[k * 68 + i] = (k < b && j0 + i < n) ? L[(j0 + i) + (k0 + k) * n] : 0.0;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  double acc[2][4][4] = {};
  for (int ks = 0; ks < b; ks += 4) {
    double af[2][2], bf[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r = 32 * wm + 16 * mi + g;
      af[mi][0] = xi[(ks + t) * 68 + r];
      af[mi][1] = xi[(ks + t) * 68 + r + 8];
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bf[ni] = xj[(ks + t) * 68 + 32 * wn + 8 * ni + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma1684(acc[mi][ni], af[mi], bf[ni]);
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t r = i0 + 32 * wm + 16 * mi + g + 8 * (e >> 1);
        const int64_t c = j0 + 32 * wn + 8 * ni + 2 * t + (e & 1);
        if (r < n && c < n && r >= c) L[r + c * n] -= acc[mi][ni][e];
      }
}

// x = L^{-T} L^{-1} b, one CTA; x may alias b
__global__ void __launch_bounds__(512) k_trsv(const double* __restrict__ L, const double* b,
                                              double* x, int64_t n) {
  extern __shared__ double xs[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = blockDim.x >> 5;
  for (int64_t i = tid; i < n; i += blockDim.x) xs[i] = b[i];
  __syncthreads();
  // forward: L y = b (blocks of 32; right-looking)
  for (int64_t blk = 0; blk < n; blk += 32) {
    const int bs = (int)(n - blk < 32 ? n - blk : 32);
    if (warp == 0) {
      double xv = lane < bs ? xs[blk + lane] : 0.0;
      for (int jj = 0; jj < bs; ++jj) {
        if (lane == jj) xv = dv(xv, L[(blk + jj) + (blk + jj) * n]);
        const double xj = __shfl_sync(0xffffffffu, xv, jj);
        if (lane > jj && lane < bs) xv -= L[(blk + lane) + (blk + jj) * n] * xj;
      }
      if (lane < bs) xs[blk + lane] = xv;
    }
    __syncthreads();
    for (int64_t i = blk + bs + tid; i < n; i += blockDim.x) {
      double s = 0.0;
      for (int p = 0; p < bs; ++p) s += L[i + (blk + p) * n] * xs[blk + p];
      xs[i] -= s;
    }
    __syncthreads();
  }
  // backward: L^T x = y (blocks of 32 from the bottom; left-looking column dots)
  const int64_t nblk = (n + 31) / 32;
  for (int64_t bi = nblk - 1; bi >= 0; --bi) {
    const int64_t blk = bi * 32;
    const int bs = (int)(n - blk < 32 ? n - blk : 32);
    const int64_t tail = blk + bs;
    for (int r = warp; r < bs; r += nw) {
      const int64_t i = blk + r;
      double s = 0.0;
      for (int64_t p = tail + lane; p < n; p += 32) s += L[p + i * n] * xs[p];
      s = warp_sum(s);
      if (lane == 0) xs[i] -= s;
    }
    __syncthreads();
    if (warp == 0) {
      double xv = lane < bs ? xs[blk + lane] : 0.0;
      for (int jj = bs - 1; jj >= 0; --jj) {
        if (lane == jj) xv = dv(xv, L[(blk + jj) + (blk + jj) * n]);
        const double xj = __shfl_sync(0xffffffffu, xv, jj);
        if (lane < jj) xv -= L[(blk + jj) + (blk + lane) * n] * xj;
      }
      if (lane < bs) xs[blk + lane] = xv;
    }
    __syncthreads();
  }
  for (int64_t i = tid; i < n; i += blockDim.x) x[i] = xs[i];
}

}  // namespace

void launch_cholesky(Ctx& c, const double* M, double* L, double delta) {
  const int64_t n = c.n;
  long long* info = &c.pk->info;
  if (n == 0) {
    CMPC_CUDA(cudaMemsetAsync(info, 0, sizeof(long long), c.stream));
    return;
  }
  static bool attr = false;
  if (!attr) {
    CMPC_CUDA(cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmSmem));
    CMPC_CUDA(cudaFuncSetAttribute(k_trail, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrailSmem));
    attr = true;
  }
  dim3 g0((unsigned)ceil_div(n, 256), (unsigned)n);
  k_chol_copy<<<g0, 256, 0, c.stream>>>(M, L, n, delta, info);
  CMPC_LAUNCHED();
  for (int64_t k0 = 0; k0 < n; k0 += kNB) {
    const int b = (int)std::min<int64_t>(kNB, n - k0);
    k_potf2<<<1, 256, 0, c.stream>>>(L, n, k0, b, info);
    CMPC_LAUNCHED();
    const int64_t rest = n - k0 - b;
    if (rest > 0) {
      const unsigned nb = (unsigned)ceil_div(rest, kNB);
      k_trsm<<<nb, 256, kTrsmSmem, c.stream>>>(L, n, k0, b, info);
      CMPC_LAUNCHED();
      k_trail<<<dim3(nb, nb), 128, kTrailSmem, c.stream>>>(L, n, k0, b, info);
      CMPC_LAUNCHED();
    }
  }
}

void launch_chol_solve(Ctx& c, const double* L, const double* b, double* x) {
  if (c.n == 0) return;
  const size_t sm = sizeof(double) * (size_t)c.n;
  static bool attr = false;
  if (!attr) {
    CMPC_CUDA(cudaFuncSetAttribute(k_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  if (sm > 200 * 1024) throw CudaError("chol_solve: n too large for the single-CTA TRSV");
  k_trsv<<<1, 512, sm, c.stream>>>(L, b, x, c.n);
  CMPC_LAUNCHED();
}

}  // namespace cmpc
