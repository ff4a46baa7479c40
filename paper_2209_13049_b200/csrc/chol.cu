// K2/K3/K4: Cholesky of the condensed matrix with the reference's failure rule, and
// the two triangular solves.
//
// Reference: ReferenceBackend::factorize (proj/src/dense_linalg.cpp:59-77, block 64:
// potf2 :24-40, trsm :43-51, trailing rankUpdate), failure "!(diag > 0) || !isfinite"
// at the first pivot; Factor::solve (:102-110). The shift ladder (proj/src/ipm.cpp:
// 205-221) re-factors M + delta I; here M is kept intact and L written separately, so a
// retry never repeats the SYRK. info = failing pivot + 1 (0 = success).
//
// Blocked right-looking with 64-wide panels, three kernels per panel:
//   k_potf2_inv  1 CTA: right-looking potf2 of the diagonal block in shared memory with
//                the inverse W = L_kk^{-1} built in the same column sweep;
//   k_panel      L_ik = A_ik W^T for every 64-row block below (DMMA GEMM, no sequential
//                triangular solve on the critical path);
//   k_trail      A_ij -= L_ik L_jk^T on the trailing lower tiles (DMMA).
// The W blocks are kept, so the triangular solves (k_trsv) are block GEMVs.
// Every kernel returns immediately once info != 0.
#include <algorithm>

#include "internal.cuh"
#include "ptx.cuh"

namespace cmpc {

namespace {

constexpr int kNB = 64;
constexpr int kLD = kNB + 1;
constexpr int kGemmLD = 68;
constexpr int kGemmSmem = 2 * kNB * kGemmLD * 8;
constexpr int kPotfSmem = (2 * kNB * kLD + 8 * 64) * 8;

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

// W = L^{-1} for the factored 64 x 64 lower block in a (identity padding beyond b),
// right-looking substitution on L W = I: step p scales row p of W, then rows i > p
// subtract l_ip W_p. 256 threads, 2 barriers per step.
__device__ void inv64(const double* a, double* w) {
  const int tid = threadIdx.x;
  for (int e = tid; e < kNB * kNB; e += blockDim.x) w[(e & 63) + (e >> 6) * kLD] = ((e & 63) == (e >> 6)) ? 1.0 : 0.0;
  __syncthreads();
  const int i = tid & 63, kg = tid >> 6;
  for (int p = 0; p < kNB; ++p) {
    const double l = a[p + p * kLD];
    if (tid >= 64 && tid - 64 <= p) w[p + (tid - 64) * kLD] = dv(w[p + (tid - 64) * kLD], l);
    __syncthreads();
    if (i > p) {
      const double lip = a[i + p * kLD];
      for (int k = kg; k <= p; k += 4) w[i + k * kLD] = fma(-lip, w[p + k * kLD], w[i + k * kLD]);
    }
    __syncthreads();
  }
}

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

// Every thread factors the same 8 x 8 diagonal block in its own registers (redundantly:
// no shuffles, no barriers on the pivot chain) and forms its inverse. Returns the first
// failing local pivot (< bvalid) or -1. l, wi: lower triangles, row-major packed by hand.
__device__ __forceinline__ int potf2_inv8(const double* a, int o, int bvalid, double (&l)[8][8],
                                          double (&wi)[8][8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) l[i][j] = a[(o + i) + (o + j) * kLD];
  int fail = -1;
  double rl[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double d = l[j][j];
    if (fail < 0 && j < bvalid && (!(d > 0.0) || !isfinite(d))) fail = j;
    const double y = rsqrt_fast(d);
    rl[j] = y;
    l[j][j] = d * y;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) l[i][j] *= y;
#pragma unroll
    for (int k = j + 1; k < 8; ++k)
#pragma unroll
      for (int i = k; i < 8; ++i) l[i][k] = fma(-l[i][j], l[k][j], l[i][k]);
  }
  // W = L^{-1}: W_pp = 1/l_pp, W_pk = -(1/l_pp) sum_{q=k}^{p-1} l_pq W_qk
#pragma unroll
  for (int p2 = 0; p2 < 8; ++p2) {
    wi[p2][p2] = rl[p2];
#pragma unroll
    for (int k = 0; k < p2; ++k) {
      double sacc = 0.0;
#pragma unroll
      for (int q = k; q < p2; ++q) sacc = fma(l[p2][q], wi[q][k], sacc);
      wi[p2][k] = -rl[p2] * sacc;
    }
  }
  return fail;
}

// Factor the b x b diagonal block at (k0, k0) and build W = L_kk^{-1}. Eight 8-wide column
// blocks: each 8 x 8 diagonal block is factored (with its inverse) redundantly in every
// thread's registers, so the sequential pivot chain runs without any communication; the rows
// below become X = A W8^T (each thread its row, W8 in registers) and all threads apply the
// rank-8 trailing update. W's off-diagonal 8 x 8 blocks follow from
// W_ij = -W_ii sum_{k=j}^{i-1} L_ik W_kj (seven dependent stages).
__global__ void __launch_bounds__(256) k_potf2_inv(double* __restrict__ L, int64_t n, int64_t k0,
                                                   int b, long long* info, double* __restrict__ Wout) {
  extern __shared__ double sm[];
  double* a = sm;               // kNB x kLD
  double* w = sm + kNB * kLD;   // kNB x kLD
  double* tt = w + kNB * kLD;   // 8 x 64 scratch (W stages)
  __shared__ int fail;
  if (*info != 0) return;
  const int tid = threadIdx.x;
  load_diag(L, n, k0, b, a);
  for (int e = tid; e < kNB * kNB; e += blockDim.x) w[(e & 63) + (e >> 6) * kLD] = 0.0;
  if (tid == 0) fail = -1;
  __syncthreads();
  for (int kb = 0; kb < 8; ++kb) {
    const int o = 8 * kb;
    const int bv = b - o < 0 ? 0 : (b - o > 8 ? 8 : b - o);
    double l[8][8], wi[8][8];
    const int f = potf2_inv8(a, o, bv, l, wi);
    if (f >= 0) {
      if (tid == 0) *info = (long long)(k0 + o + f + 1);
      return;  // uniform: every thread computed the same block
    }
    __syncthreads();  // all threads have read the block before it is overwritten
    if (tid < 64) {
      const int i = tid & 7, j = tid >> 3;
      if (j <= i) {
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
          for (int jj = 0; jj <= ii; ++jj)
            if (ii == i && jj == j) {
              a[(o + i) + (o + j) * kLD] = l[ii][jj];
              w[(o + i) + (o + j) * kLD] = wi[ii][jj];
            }
      }
    }
    const int rows = kNB - o - 8;
    if (rows > 0) {
      // panel: X(i, :) = A(i, o:o+8) W8^T, one thread per row
      if (tid < rows) {
        const int i = o + 8 + tid;
        double x[8], y[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = a[i + (o + c) * kLD];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double sacc = 0.0;
#pragma unroll
          for (int q = 0; q <= c; ++q) sacc = fma(x[q], wi[c][q], sacc);
          y[c] = sacc;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) a[i + (o + c) * kLD] = y[c];
      }
      __syncthreads();
      // trailing: A(i, j) -= sum_p X(i, p) X(j, p) for o+8 <= j <= i < 64
      const int cnt = rows * (rows + 1) / 2;
      for (int e = tid; e < cnt; e += blockDim.x) {
        // e -> (ii, jj) with jj <= ii, row-major over the lower triangle
        int ii = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
        while ((ii + 1) * (ii + 2) / 2 <= e) ++ii;
        while (ii * (ii + 1) / 2 > e) --ii;
        const int jj = e - ii * (ii + 1) / 2;
        const int i = o + 8 + ii, j = o + 8 + jj;
        double sacc = 0.0;
#pragma unroll
        for (int p2 = 0; p2 < 8; ++p2) sacc = fma(a[i + (o + p2) * kLD], a[j + (o + p2) * kLD], sacc);
        a[i + j * kLD] -= sacc;
      }
    }
    __syncthreads();
  }
  // off-diagonal 8 x 8 blocks of W by block distance d = i - j
  for (int d = 1; d < 8; ++d) {
    const int nblk = 8 - d;  // blocks (j + d, j)
    for (int e = tid; e < nblk * 64; e += blockDim.x) {
      const int jb = e >> 6, r = (e >> 3) & 7, c = e & 7;
      const int ib = jb + d;
      double sacc = 0.0;
      for (int kb2 = jb; kb2 < ib; ++kb2)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          sacc = fma(a[(8 * ib + r) + (8 * kb2 + q) * kLD], w[(8 * kb2 + q) + (8 * jb + c) * kLD], sacc);
      tt[e] = sacc;
    }
    __syncthreads();
    for (int e = tid; e < nblk * 64; e += blockDim.x) {
      const int jb = e >> 6, r = (e >> 3) & 7, c = e & 7;
      const int ib = jb + d;
      double sacc = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q <= r) sacc = fma(w[(8 * ib + r) + (8 * ib + q) * kLD], tt[(jb << 6) | (q << 3) | c], sacc);
      w[(8 * ib + r) + (8 * jb + c) * kLD] = -sacc;
    }
    __syncthreads();
  }
  store_diag(L, n, k0, b, a, w, Wout, true);
}

// inverse of every 64 x 64 diagonal block of an existing factor (one CTA per block)
__global__ void __launch_bounds__(256) k_diag_inv(const double* __restrict__ L, int64_t n,
                                                  double* __restrict__ Winv) {
  extern __shared__ double sm[];
  double* a = sm;
  double* w = sm + kNB * kLD;
  const int64_t k0 = (int64_t)blockIdx.x * kNB;
  const int b = (int)(n - k0 < kNB ? n - k0 : kNB);
  load_diag(L, n, k0, b, a);
  __syncthreads();
  inv64(a, w);
  store_diag(nullptr, n, k0, b, a, w, Winv + (size_t)blockIdx.x * kNB * kNB, false);
}

// acc(i, j) += sum_k X[i][k] Y[j][k] for 64x64 smem tiles stored x[k*kGemmLD + i];
// 4 warps, 32 x 32 per warp, DMMA m16n8k4
__device__ __forceinline__ void tile_xyt(const double* x, const double* y, int kmax,
                                         double (&acc)[2][4][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  for (int ks = 0; ks < kmax; ks += 4) {
    double af[2][2], bf[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r = 32 * wm + 16 * mi + g;
      af[mi][0] = x[(ks + t) * kGemmLD + r];
      af[mi][1] = x[(ks + t) * kGemmLD + r + 8];
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bf[ni] = y[(ks + t) * kGemmLD + 32 * wn + 8 * ni + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma1684(acc[mi][ni], af[mi], bf[ni]);
  }
}

// L_ik = A_ik W^T for the 64-row block i below the diagonal block
__global__ void __launch_bounds__(128) k_panel(double* __restrict__ L, int64_t n, int64_t k0, int b,
                                               long long* info, const double* __restrict__ W) {
  extern __shared__ double sm[];
  double* xa = sm;                  // A_ik: xa[k*LD + i]
  double* xw = sm + kNB * kGemmLD;  // W:    xw[k*LD + j] = W[j][k]
  if (*info != 0) return;
  const int64_t r0 = k0 + b + (int64_t)blockIdx.x * kNB;
  {
    double ra[32], rw[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int e = threadIdx.x + u * 128, i = e & 63, k = e >> 6;
      ra[u] = (k < b && r0 + i < n) ? L[(r0 + i) + (k0 + k) * n] : 0.0;
      rw[u] = W[i + k * kNB];  // W col-major: W[i][k] at i + k*64
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int e = threadIdx.x + u * 128, i = e & 63, k = e >> 6;
      xa[k * kGemmLD + i] = ra[u];
      xw[k * kGemmLD + i] = rw[u];
    }
  }
  __syncthreads();
  double acc[2][4][4] = {};
  tile_xyt(xa, xw, b, acc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t r = r0 + 32 * wm + 16 * mi + g + 8 * (e >> 1);
        const int c = 32 * wn + 8 * ni + 2 * t + (e & 1);
        if (r < n && c < b) L[r + (k0 + c) * n] = acc[mi][ni][e];
      }
}

// trailing update A22(I,J) -= L_Ik L_Jk^T, lower tiles only
__global__ void __launch_bounds__(128) k_trail(double* __restrict__ L, int64_t n, int64_t k0, int b,
                                               long long* info) {
  extern __shared__ double sm[];
  double* xi = sm;
  double* xj = sm + kNB * kGemmLD;
  if (*info != 0) return;
  // blockIdx.x enumerates the lower tiles (ti >= tj) of the trailing matrix
  int ti = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= (int)blockIdx.x) ++ti;
  while (ti * (ti + 1) / 2 > (int)blockIdx.x) --ti;
  const int tj = (int)blockIdx.x - ti * (ti + 1) / 2;
  const int64_t base = k0 + b;
  const int64_t i0 = base + (int64_t)ti * kNB, j0 = base + (int64_t)tj * kNB;
  {
    double ra[32], rb[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int e = threadIdx.x + u * 128, i = e & 63, k = e >> 6;
      ra[u] = (k < b && i0 + i < n) ? L[(i0 + i) + (k0 + k) * n] : 0.0;
      rb[u] = (k < b && j0 + i < n) ? L[(j0 + i) + (k0 + k) * n] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int e = threadIdx.x + u * 128, i = e & 63, k = e >> 6;
      xi[k * kGemmLD + i] = ra[u];
      xj[k * kGemmLD + i] = rb[u];
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  // prefetch the tile being updated (all loads in flight before the MMA loop)
  double old[2][4][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t r = i0 + 32 * wm + 16 * mi + g + 8 * (e >> 1);
        const int64_t c = j0 + 32 * wn + 8 * ni + 2 * t + (e & 1);
        old[mi][ni][e] = (r < n && c < n && r >= c) ? L[r + c * n] : 0.0;
      }
  double acc[2][4][4] = {};
  tile_xyt(xi, xj, b, acc);
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t r = i0 + 32 * wm + 16 * mi + g + 8 * (e >> 1);
        const int64_t c = j0 + 32 * wn + 8 * ni + 2 * t + (e & 1);
        if (r < n && c < n && r >= c) L[r + c * n] = old[mi][ni][e] - acc[mi][ni][e];
      }
}

// x = L^{-T} L^{-1} b with the 64 x 64 diagonal-block inverses W; one CTA of 512
// threads; x may alias b. Forward: y_k = W_k (b_k - sum_{j<k} L_kj y_j); backward:
// x_k = W_k^T (y_k - sum_{i>k} L_ik^T x_i).
__global__ void __launch_bounds__(512) k_trsv(const double* __restrict__ L,
                                              const double* __restrict__ W, const double* b,
                                              double* x, int64_t n) {
  extern __shared__ double xs[];
  double* t = xs + n;  // 64 scratch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int64_t i = tid; i < n; i += blockDim.x) xs[i] = b[i];
  __syncthreads();
  const int64_t nb = (n + kNB - 1) / kNB;
  const int row = tid >> 3, part = tid & 7;  // 64 rows x 8 parts
  for (int64_t kb = 0; kb < nb; ++kb) {
    const int64_t r0 = kb * kNB;
    const int bs = (int)(n - r0 < kNB ? n - r0 : kNB);
    const double* Wk = W + kb * kNB * kNB;
    // y_k = W_k b'_k (W lower: row i uses columns j <= i)
    double s = 0.0;
    if (row < bs)
      for (int j = part; j <= row; j += 8) s += Wk[row + j * kNB] * xs[r0 + j];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    __syncthreads();
    if (part == 0 && row < bs) xs[r0 + row] = s;
    __syncthreads();
    for (int64_t i = r0 + bs + tid; i < n; i += blockDim.x) {
      double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0;
      int p = 0;
      for (; p + 3 < bs; p += 4) {
        u0 += L[i + (r0 + p) * n] * xs[r0 + p];
        u1 += L[i + (r0 + p + 1) * n] * xs[r0 + p + 1];
        u2 += L[i + (r0 + p + 2) * n] * xs[r0 + p + 2];
        u3 += L[i + (r0 + p + 3) * n] * xs[r0 + p + 3];
      }
      for (; p < bs; ++p) u0 += L[i + (r0 + p) * n] * xs[r0 + p];
      xs[i] -= (u0 + u1) + (u2 + u3);
    }
    __syncthreads();
  }
  for (int64_t kb = nb - 1; kb >= 0; --kb) {
    const int64_t r0 = kb * kNB;
    const int bs = (int)(n - r0 < kNB ? n - r0 : kNB);
    const int64_t tail = r0 + bs;
    const double* Wk = W + kb * kNB * kNB;
    // t_i = y_i - sum_{p >= tail} L[p, i] x_p (column dots, one warp per column)
    for (int i = warp; i < bs; i += 16) {
      double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0;
      const double* Lc = L + (r0 + i) * n;
      int64_t p = tail + lane;
      for (; p + 96 < n; p += 128) {
        u0 += Lc[p] * xs[p];
        u1 += Lc[p + 32] * xs[p + 32];
        u2 += Lc[p + 64] * xs[p + 64];
        u3 += Lc[p + 96] * xs[p + 96];
      }
      for (; p < n; p += 32) u0 += Lc[p] * xs[p];
      const double u = warp_sum((u0 + u1) + (u2 + u3));
      if (lane == 0) t[i] = xs[r0 + i] - u;
    }
    __syncthreads();
    // x_k = W_k^T t: x_i = sum_{j >= i} W[j][i] t_j
    double s = 0.0;
    if (row < bs)
      for (int j = row + part; j < bs; j += 8) s += Wk[j + row * kNB] * t[j];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (part == 0 && row < bs) xs[r0 + row] = s;
    __syncthreads();
  }
  for (int64_t i = tid; i < n; i += blockDim.x) x[i] = xs[i];
}

void set_attrs() {
  static bool done = false;
  if (done) return;
  CMPC_CUDA(cudaFuncSetAttribute(k_potf2_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotfSmem));
  CMPC_CUDA(cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotfSmem));
  CMPC_CUDA(cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem));
  CMPC_CUDA(cudaFuncSetAttribute(k_trail, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem));
  CMPC_CUDA(cudaFuncSetAttribute(k_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  done = true;
}

}  // namespace

void chol_alloc(Ctx& c) {
  const int64_t nb = ceil_div(std::max<int64_t>(c.n, 1), kNB);
  c.Winv = dev_zeros<double>((size_t)nb * kNB * kNB, c.stream);
}

void chol_free(Ctx& c) {
  dev_free(c.Winv, c.stream);
  c.Winv = nullptr;
}

void launch_cholesky(Ctx& c, const double* M, double* L, double delta) {
  const int64_t n = c.n;
  long long* info = &c.pk->info;
  if (n == 0) {
    CMPC_CUDA(cudaMemsetAsync(info, 0, sizeof(long long), c.stream));
    return;
  }
  set_attrs();
  dim3 g0((unsigned)ceil_div(n, 256), (unsigned)n);
  k_chol_copy<<<g0, 256, 0, c.stream>>>(M, L, n, delta, info);
  CMPC_LAUNCHED();
  for (int64_t k0 = 0; k0 < n; k0 += kNB) {
    const int b = (int)std::min<int64_t>(kNB, n - k0);
    double* Wk = c.Winv + (k0 / kNB) * kNB * kNB;
    k_potf2_inv<<<1, 256, kPotfSmem, c.stream>>>(L, n, k0, b, info, Wk);
    CMPC_LAUNCHED();
    const int64_t rest = n - k0 - b;
    if (rest > 0) {
      const unsigned nb = (unsigned)ceil_div(rest, kNB);
      k_panel<<<nb, 128, kGemmSmem, c.stream>>>(L, n, k0, b, info, Wk);
      CMPC_LAUNCHED();
      k_trail<<<nb * (nb + 1) / 2, 128, kGemmSmem, c.stream>>>(L, n, k0, b, info);
      CMPC_LAUNCHED();
    }
  }
}

void launch_factor_inverses(Ctx& c, const double* L) {
  if (c.n == 0) return;
  set_attrs();
  k_diag_inv<<<(unsigned)ceil_div(c.n, kNB), 256, kPotfSmem, c.stream>>>(L, c.n, c.Winv);
  CMPC_LAUNCHED();
}

void launch_chol_solve(Ctx& c, const double* L, const double* b, double* x) {
  if (c.n == 0) return;
  set_attrs();
  const size_t sm = sizeof(double) * ((size_t)c.n + kNB);
  if (sm > 200 * 1024) throw CudaError("chol_solve: n too large for the single-CTA TRSV");
  k_trsv<<<1, 512, sm, c.stream>>>(L, c.Winv, b, x, c.n);
  CMPC_LAUNCHED();
}

}  // namespace cmpc
