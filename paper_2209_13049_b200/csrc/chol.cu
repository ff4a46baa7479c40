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
constexpr int kPotfSmem = (2 * kNB * kLD + kNB) * 8;

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

// factor the b x b diagonal block at (k0, k0) (right-looking, 2 barriers per column) and
// build W = L_kk^{-1} in the same sweep: once column j of L is final, step j of the
// substitution L W = I runs alongside the rank-1 trailing update. 256 threads.
__global__ void __launch_bounds__(256) k_potf2_inv(double* __restrict__ L, int64_t n, int64_t k0,
                                                   int b, long long* info, double* __restrict__ Wout) {
  extern __shared__ double sm[];
  double* a = sm;              // kNB x kLD
  double* w = sm + kNB * kLD;  // kNB x kLD
  double* dj = w + kNB * kLD;  // pivots
  if (*info != 0) return;
  const int tid = threadIdx.x;
  load_diag(L, n, k0, b, a);
  for (int e = tid; e < kNB * kNB; e += blockDim.x) w[(e & 63) + (e >> 6) * kLD] = ((e & 63) == (e >> 6)) ? 1.0 : 0.0;
  __syncthreads();
  const int i = tid & 63, kg = tid >> 6;
  for (int j = 0; j < kNB; ++j) {
    const double d = a[j + j * kLD];
    if (j < b && (!(d > 0.0) || !isfinite(d))) {
      if (tid == 0) *info = (long long)(k0 + j + 1);
      return;
    }
    const double l = sqrt(d);
    if (tid < 64) {
      if (i > j) a[i + j * kLD] = dv(a[i + j * kLD], l);
    } else if (tid - 64 <= j) {
      w[j + (tid - 64) * kLD] = dv(w[j + (tid - 64) * kLD], l);
    }
    if (tid == 0) dj[j] = l;
    __syncthreads();
    if (i > j) {
      // batch every load of this step before any store (the smem updates are independent)
      const double lij = a[i + j * kLD];
      double av[16], cv[16], wv[16], rv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = j + 1 + kg + 4 * u;
        if (k <= i) {
          av[u] = a[i + k * kLD];
          cv[u] = a[k + j * kLD];
        }
        const int q = kg + 4 * u;
        if (q <= j) {
          wv[u] = w[i + q * kLD];
          rv[u] = w[j + q * kLD];
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = j + 1 + kg + 4 * u;
        if (k <= i) a[i + k * kLD] = fma(-lij, cv[u], av[u]);
        const int q = kg + 4 * u;
        if (q <= j) w[i + q * kLD] = fma(-lij, rv[u], wv[u]);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < kNB; e += blockDim.x) a[e + e * kLD] = dj[e];
  __syncthreads();
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
      double u = 0.0;
      for (int64_t p = tail + lane; p < n; p += 32) u += L[p + (r0 + i) * n] * xs[p];
      u = warp_sum(u);
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
  CMPC_CUDA(cudaMalloc(&c.Winv, sizeof(double) * nb * kNB * kNB));
  CMPC_CUDA(cudaMemset(c.Winv, 0, sizeof(double) * nb * kNB * kNB));
}

void chol_free(Ctx& c) {
  if (c.Winv) cudaFree(c.Winv);
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
