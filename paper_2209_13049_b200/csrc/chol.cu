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
constexpr int kPotfSmem = (2 * kNB * kLD + 16 * 65 + 64) * 8;

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
__device__ int warp_potf2_inv16(double* a, double* w, int o, int bvalid, double* bc) {
  // bc: 2 x 32 doubles of shared scratch, double-buffered by step parity:
  // [0,16) column j of L, [16,32) row j of W
  const int lane = threadIdx.x & 31, row = lane & 15;
  double r[16], wr[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    r[k] = (k <= row) ? a[(o + row) + (o + k) * kLD] : 0.0;
    wr[k] = (k == row) ? 1.0 : 0.0;
  }
  int fail = -1;
  // step j: factor column j of L and, interleaved, step j of the substitution L W = I
  // (row j of W is final once scaled by 1/l_jj; rows below subtract l_ij W_j). The column
  // and the row are broadcast through shared memory: a 64-bit shuffle costs ~10 issue
  // cycles per lane-pair on one warp, a broadcast LDS far less.
#pragma unroll 1
  for (int j = 0; j < 16; ++j) {
    double* cb = bc + 32 * (j & 1);
    // r[0] holds column j of this row (rotated)
    const double pj = __shfl_sync(kFull, r[0], j);
    if (fail < 0 && j < bvalid && (!(pj > 0.0) || !isfinite(pj))) fail = j;
    const double y = rsqrt_fast(pj);
    double lij = r[0];
    if (row == j) {
      lij = pj * y;
#pragma unroll
      for (int k = 0; k < 16; ++k) wr[k] *= y;
      if (lane == j) {
#pragma unroll
        for (int k = 0; k < 16; ++k) cb[16 + k] = wr[k];
      }
    } else if (row > j) {
      lij = r[0] * y;
    }
    if (lane < 16) {
      cb[row] = lij;
      if (row >= j) a[(o + row) + (o + j) * kLD] = lij;
    }
    __syncwarp();
    if (row > j) {
#pragma unroll
      for (int k = 1; k < 16; ++k) {
        if (row >= j + k) r[k] = fma(-lij, cb[(j + k) & 15], r[k]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) wr[k] = fma(-lij, cb[16 + k], wr[k]);
    }
#pragma unroll
    for (int k = 0; k < 15; ++k) r[k] = r[k + 1];
    r[15] = 0.0;
  }
  if (fail >= 0) return fail;
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
                                                   int b, long long* info, double* __restrict__ Wout) {
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
  for (int kb = 0; kb < 4; ++kb) {
    const int o = 16 * kb;
    if (warp == 0) {
      const int bv = b - o < 0 ? 0 : (b - o > 16 ? 16 : b - o);
      const int f = warp_potf2_inv16(a, w, o, bv, tt + 16 * 65);
      if (f >= 0 && tid == 0) fail = o + f;
    }
    __syncthreads();
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
