// K2/K3/K4: Cholesky of the condensed matrix with the reference's failure rule, and
// the two triangular solves.
//
// Reference: ReferenceBackend::factorize (proj/src/dense_linalg.cpp:59-77, block 64:
// potf2 :24-40, trsm :43-51, trailing rankUpdate), failure "!(diag > 0) || !isfinite"
// at the first pivot; Factor::solve (:102-110). The shift ladder (proj/src/ipm.cpp:
// 205-221) re-factors M + delta I; here M is kept intact and L written separately, so a
// retry never repeats the SYRK. info = failing pivot + 1 (0 = success).
//
// One persistent dataflow kernel (k_chol_df) factors the whole matrix, tile by tile
// (64 x 64, lower tiles only), left-looking:
//   tile (i, j):  A_ij <- M_ij - sum_{k<j} L_ik L_jk^T        (DMMA, accumulator in registers)
//                 i == j: L_jj = potf2(A_jj) and W_j = L_jj^{-1} (register-blocked, in smem)
//                 i >  j: L_ij = A_ij W_j^T                   (DMMA, no sequential TRSM)
// Every finished tile publishes a per-tile flag (release/acquire at GPU scope) stamped with
// the launch's generation number, so flags never need resetting. CTAs grab tiles from an
// atomic counter in column-major (topological) order, and a tile only waits for tiles
// earlier in that order, which were grabbed by CTAs that are already running: the kernel
// cannot deadlock whatever the residency. The last CTA out publishes info and advances the
// generation. The W blocks are kept, so the triangular solves (k_trsv) are block GEMVs.
#include <algorithm>

#include "internal.cuh"
#include "ptx.cuh"

namespace cmpc {

namespace {

#ifdef CMPC_TRACE
__device__ unsigned long long g_trace[256];
#define TRACE(i)                                                   \
  do {                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_trace[(i)] = clock64(); \
  } while (0)
#define TRACEW(i)                                                   \
  do {                                                              \
    if (blockIdx.x == 0 && threadIdx.x == 32) g_trace[(i)] = clock64(); \
  } while (0)
#else
#define TRACE(i) \
  do {           \
  } while (0)
#define TRACEW(i) \
  do {            \
  } while (0)
#endif

constexpr int kNB = 64;
constexpr int kLD = kNB + 1;
constexpr int kGemmLD = 68;
constexpr int kPotfSmem = (2 * kNB * kLD + 8 * 64) * 8;
constexpr int kDfThreads = 256;

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

__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 1/sqrt(x): MUFU.RSQ64H seed + two Newton steps (~1/3 the latency of the float-seed
// path with its range branch, measured in tools/exp/p1_bench.cu); flushes subnormals, so
// the caller re-factors exactly when a pivot leaves [1e-300, 1e300]
__device__ __forceinline__ double rsqrt_mufu(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// 8 x 8 Cholesky + inverse in registers (every lane redundantly) from the lower block at
// a + o * (kLD + 1). Returns the first failing pivot (< bv) or -1; *odd flags a pivot out of
// the fast reciprocal square root's range.
template <bool EXACT>
__device__ __forceinline__ int factor8(const double* a, int o, int bv, double (&l)[8][8], double (&wi)[8][8],
                                       bool* odd) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) l[i][j] = a[(o + i) + (o + j) * kLD];
  int fail = -1;
  bool bad = false;
  double rl[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double d = l[j][j];
    if (fail < 0 && j < bv && (!(d > 0.0) || !isfinite(d))) fail = j;
    bad |= !(d >= 1e-300 && d <= 1e300);
    const double y = EXACT ? 1.0 / sqrt(d) : rsqrt_mufu(d);
    rl[j] = y;
    l[j][j] = d * y;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) l[i][j] *= y;
#pragma unroll
    for (int k = j + 1; k < 8; ++k)
#pragma unroll
      for (int i = k; i < 8; ++i) l[i][k] = fma(-l[i][j], l[k][j], l[i][k]);
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    wi[p][p] = rl[p];
#pragma unroll
    for (int k = 0; k < p; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = k; q < p; ++q) s = fma(l[p][q], wi[q][k], s);
      wi[p][k] = -rl[p] * s;
    }
  }
  *odd = bad;
  return fail;
}



// Factor the 64 x 64 block a (LD kLD; lower, zero upper part, identity padding beyond b)
// in place and build W = L^{-1} in w (LD kLD, lower). Right-looking over eight 8-wide
// column blocks with one block of lookahead:
//   warp 0 (pivot warp)  P1 factor the 8 x 8 diagonal block kb and its inverse W8 in
//                        registers (the pivot chain), then, once the workers have finished
//                        step kb-1, P3 the panel rows X of block kb+1 (W8 from registers)
//                        and P4 the update of diagonal block kb+1, so P1(kb+1) starts
//                        without waiting for the rest of step kb;
//   warps 1-3, 5-7       every other product of the step, as DMMA m16n8k4 fragments
//   (workers)            (K = 8) spread warp-uniformly over the six warps: W2 the W rows of
//                        block kb, W(o+i, :o) = -W8(i,:) B(o:o+8, :o) (B = sum L W
//                        accumulates in w), the panel rows X(r,:) = A(r, o:o+8) W8' below
//                        block kb+1, then S3 A(r, c) -= X(r,:) X(c,:)' below block kb+1 and
//                        B(r, c) += X(r,:) W(o:o+8, c);
//   warp 4               parked, so the pivot warp owns its scheduler's instruction cache.
// X and the block's W rows are stored p-major with stride kXLD (conflict-free fragments).
// Named barriers: 1 = step published (pivot -> workers), 3 = workers done with a step
// (workers -> pivot), 4 = worker-only. The loops stay rolled: a fully unrolled body
// overflows the instruction cache. Returns the first failing pivot (uniform) or -1.
constexpr int kXLD = 68;
__device__ int diag_factor(double* __restrict__ a, double* __restrict__ w, double* __restrict__ sc, int b) {
  constexpr int kW = 192, kWarps = 6;  // worker threads / warps
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  double* xs = sc;                  // 2 x [8 x kXLD]: X(r, p) at xs[buf][p * kXLD + r]
  double* wsb = xs + 2 * 8 * kXLD;  // [8 x kXLD]: W(o + p, c) at wsb[p * kXLD + c]
  double* l8s = wsb + 8 * kXLD;     // 2 x [8 x 8] factor (row-major)
  double* w8s = l8s + 128;          // 2 x [8 x 8] inverse
  volatile int* fls = reinterpret_cast<volatile int*>(w8s + 128);
  for (int e = tid; e < kNB * kLD; e += kDfThreads) w[e] = 0.0;
  l8s[tid] = 0.0;  // l8s and w8s (256 doubles): strictly upper parts stay zero
  if (tid == 0) *fls = -1;
  __syncthreads();
  if (warp == 0) {
#pragma unroll 1
    for (int kb = 0; kb < 8; ++kb) {
      const int o = 8 * kb, buf = kb & 1;
      TRACE(10 + 4 * kb);
      const int bv = b - o < 0 ? 0 : (b - o > 8 ? 8 : b - o);
      double l[8][8], wi[8][8];
      bool odd;
      int fail = factor8<false>(a, o, bv, l, wi, &odd);
      if (odd) fail = factor8<true>(a, o, bv, l, wi, &odd);
      double* l8 = l8s + 64 * buf;
      double* w8 = w8s + 64 * buf;
      if (lane == 0) {  // straight-line stores (a lane-indexed store compiles to a jump table)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) {
            l8[i * 8 + j] = l[i][j];
            w8[i * 8 + j] = wi[i][j];
          }
        if (fail >= 0) *fls = o + fail;
      }
      TRACE(11 + 4 * kb);
      if (kb < 7) {
        bar_sync_n(3, 224);  // workers are done with step kb-1
#ifdef CMPC_TRACE
        if (*fls > 1000) break;  // never: a shared read that waits for the barrier (trace)
#endif
        TRACE(12 + 4 * kb);
        if (fail < 0) {
          double* x = xs + 8 * kXLD * buf;
          // P3: X rows of block kb+1, lane i < 8 takes row o+8+i: X(r, p) = sum_{q<=p} A(r, o+q) W8(p, q)
          if (lane < 8) {
            const int r = o + 8 + lane;
            double ar[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) ar[q] = a[r + (o + q) * kLD];
#pragma unroll
            for (int p = 0; p < 8; ++p) {
              double s = 0.0;
#pragma unroll
              for (int q = 0; q <= p; ++q) s = fma(ar[q], wi[p][q], s);
              x[p * kXLD + r] = s;
              a[r + (o + p) * kLD] = s;
            }
          }
          __syncwarp();
          TRACE(60 + kb);
          // P4: diagonal block kb+1 -= X X', lane (i, j0) takes entries (i, j0) and (i, j0 + 4)
          {
            const int ri = o + 8 + g, r0 = o + 8 + t, r1 = r0 + 4;
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int p = 0; p < 8; ++p) {
              const double xi = x[p * kXLD + ri];
              s0 = fma(xi, x[p * kXLD + r0], s0);
              s1 = fma(xi, x[p * kXLD + r1], s1);
            }
            if (t <= g) a[ri + r0 * kLD] -= s0;
            if (t + 4 <= g) a[ri + r1 * kLD] -= s1;
          }
          __syncwarp();
        }
      }
      TRACE(13 + 4 * kb);
      bar_arrive_n(1, 224);  // step kb published
      if (fail >= 0) break;
    }
  } else if (warp != 4) {
    const int wid = warp < 4 ? warp - 1 : warp - 2;  // 0..5
    const int wt = wid * 32 + lane;                   // 0..191
    bar_arrive_n(3, 224);
#pragma unroll 1
    for (int kb = 0; kb < 8; ++kb) {
      const int o = 8 * kb, buf = kb & 1;
      bar_sync_n(1, 224);
      if (*fls >= 0) break;
      TRACEW(100 + 4 * kb);
      const double* l8 = l8s + 64 * buf;
      const double* w8 = w8s + 64 * buf;
      double* x = xs + 8 * kXLD * buf;
      // the block's L entries and its diagonal W entries
      if (wt < 64) {
        const int i = wt >> 3, j = wt & 7;
        wsb[i * kXLD + o + j] = w8[i * 8 + j];
        a[(o + i) + (o + j) * kLD] = l8[i * 8 + j];
      }
      // W2: D(c, i) = sum_p B(o+p, c) W8(i, p), c < o; W(o+i, c) = -D
      for (int f = wid; f < (o + 15) / 16; f += kWarps) {
        const int m0 = 16 * f;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k0 = 0; k0 < 8; k0 += 4) {
          const int p = k0 + t;
          double af[2];
          af[0] = m0 + g < o ? w[(o + p) + (m0 + g) * kLD] : 0.0;
          af[1] = m0 + g + 8 < o ? w[(o + p) + (m0 + g + 8) * kLD] : 0.0;
          dmma1684(acc, af, w8[g * 8 + p]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = m0 + g + 8 * (e >> 1), i = 2 * t + (e & 1);
          if (c < o) wsb[i * kXLD + c] = -acc[e];
        }
      }
      // X rows below block kb+1: D(r, p) = sum_q A(r, o+q) W8(p, q), r >= o+16
      for (int f = wid; f < (kNB - 1 - o) / 16; f += kWarps) {
        const int m0 = o + 16 + 16 * f;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k0 = 0; k0 < 8; k0 += 4) {
          const int q = k0 + t;
          double af[2];
          af[0] = m0 + g < kNB ? a[(m0 + g) + (o + q) * kLD] : 0.0;
          af[1] = m0 + g + 8 < kNB ? a[(m0 + g + 8) + (o + q) * kLD] : 0.0;
          dmma1684(acc, af, w8[g * 8 + q]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = m0 + g + 8 * (e >> 1), p = 2 * t + (e & 1);
          if (r < kNB) x[p * kXLD + r] = acc[e];
        }
      }
      TRACEW(101 + 4 * kb);
      bar_sync_n(4, kW);
#ifdef CMPC_TRACE
      if (*fls > 1000) break;  // never: waits for the barrier (trace)
#endif
      TRACEW(102 + 4 * kb);
      // S3a: A(r, c) -= X(r,:) X(c,:)' for r >= o+16, o+8 <= c <= r, in 16 x 8 fragments
      // (row group rg holds min(2 rg + 3, ncg) of them); two fragments in flight per warp
      {
        const int nrg = (kNB - 1 - o) / 16, ncg = (kNB - 8 - o) / 8;
        int total = 0;
        for (int rg = 0; rg < nrg; ++rg) total += min(2 * rg + 3, ncg);
        for (int f = wid; f < total; f += 2 * kWarps) {
          const bool two = f + kWarps < total;
          int m0[2], n0[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            int ff = (u == 0 || !two) ? f : f + kWarps, rg = 0, cnt = min(3, ncg);
            while (ff >= cnt) {
              ff -= cnt;
              ++rg;
              cnt = min(2 * rg + 3, ncg);
            }
            m0[u] = o + 16 + 16 * rg;
            n0[u] = o + 8 + 8 * ff;
          }
          double acc[2][4], af[2][2][2], bf[2][2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
              const int r = m0[u] + g + 8 * (e2 >> 1), c = n0[u] + 2 * t + (e2 & 1);
              acc[u][e2] = (r < kNB && c <= r) ? a[r + c * kLD] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int p = 4 * k + t;
              af[u][k][0] = m0[u] + g < kNB ? -x[p * kXLD + m0[u] + g] : 0.0;
              af[u][k][1] = m0[u] + g + 8 < kNB ? -x[p * kXLD + m0[u] + g + 8] : 0.0;
              bf[u][k] = x[p * kXLD + n0[u] + g];
            }
          }
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int u = 0; u < 2; ++u) dmma1684(acc[u], af[u][k], bf[u][k]);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) break;
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
              const int r = m0[u] + g + 8 * (e2 >> 1), c = n0[u] + 2 * t + (e2 & 1);
              if (r < kNB && c <= r) a[r + c * kLD] = acc[u][e2];
            }
          }
        }
      }
      TRACEW(140 + 2 * kb);
      // S3b: B(r, c) += X(r,:) W(o:o+8, c) for r >= o+8, c < o+8; two fragments in flight
      {
        const int nrg = (kNB - 8 - o + 15) / 16, ncg = kb + 1, total = nrg * ncg;
        for (int f = wid; f < total; f += 2 * kWarps) {
          const bool two = f + kWarps < total;
          int m0[2], n0[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int ff = (u == 0 || !two) ? f : f + kWarps;
            const int rg = ff / ncg;
            m0[u] = o + 8 + 16 * rg;
            n0[u] = 8 * (ff - rg * ncg);
          }
          double acc[2][4], af[2][2][2], bf[2][2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
              const int r = m0[u] + g + 8 * (e2 >> 1), c = n0[u] + 2 * t + (e2 & 1);
              acc[u][e2] = r < kNB ? w[r + c * kLD] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int p = 4 * k + t;
              af[u][k][0] = m0[u] + g < kNB ? x[p * kXLD + m0[u] + g] : 0.0;
              af[u][k][1] = m0[u] + g + 8 < kNB ? x[p * kXLD + m0[u] + g + 8] : 0.0;
              bf[u][k] = wsb[p * kXLD + n0[u] + g];
            }
          }
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int u = 0; u < 2; ++u) dmma1684(acc[u], af[u][k], bf[u][k]);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) break;
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
              const int r = m0[u] + g + 8 * (e2 >> 1), c = n0[u] + 2 * t + (e2 & 1);
              if (r < kNB) w[r + c * kLD] = acc[u][e2];
            }
          }
        }
      }
      TRACEW(141 + 2 * kb);
      // finished W rows of block kb; the panel L(r, o:o+8) = X below block kb+1
      for (int e = wt; e < 8 * (o + 8); e += kW) {
        const int i = e & 7, c = e >> 3;
        w[(o + i) + c * kLD] = wsb[i * kXLD + c];
      }
      for (int e = wt; e < 8 * (kNB - 16 - o); e += kW) {
        const int r = o + 16 + (e >> 3), p = e & 7;
        a[r + (o + p) * kLD] = x[p * kXLD + r];
      }
      TRACEW(103 + 4 * kb);
      if (kb < 6) bar_arrive_n(3, 224);
    }
  }
  __syncthreads();
  return *fls;
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

constexpr int kTB = kNB * kGemmLD;    // doubles per staged 64 x 64 tile
constexpr int kDfExt = 512;           // solve scratch after the staging buffers (doubles)
constexpr int kDfSmem = (4 * kTB + kDfExt) * 8;  // two stages of (X, Y); the potf2 scratch aliases stage 0

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// stage a packed 64 x 64 tile (column-major, 64 contiguous doubles per column) into
// x[k * kGemmLD + i] with 16-byte cp.async (L2 only: tiles written by other CTAs)
__device__ __forceinline__ void stage_tile(double* x, const double* src) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int ch = threadIdx.x + kDfThreads * u;
    const int k = ch >> 5, i2 = (ch & 31) * 2;
    cp_async16(x + k * kGemmLD + i2, src + k * kNB + i2);
  }
}

// acc += X Y^T (k = 0..63) for this warp's 32 x 16 block; 8 warps cover the 64 x 64 tile.
// acc[mi][ni][e] holds element (32 wm + 16 mi + g + 8 (e >> 1), 16 wn + 8 ni + 2 t + (e & 1)).
__device__ __forceinline__ void gemm_xyt(const double* x, const double* y, double (&acc)[2][2][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double* xa = x + t * kGemmLD + 32 * (warp & 1) + g;
  const double* yb = y + t * kGemmLD + 16 * (warp >> 1) + g;
#pragma unroll 4
  for (int ks = 0; ks < kNB; ks += 4) {
    const int o = ks * kGemmLD;
    double af[2][2], bf[2];
    af[0][0] = xa[o];
    af[0][1] = xa[o + 8];
    af[1][0] = xa[o + 16];
    af[1][1] = xa[o + 24];
    bf[0] = yb[o];
    bf[1] = yb[o + 8];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma1684(acc[mi][ni], af[mi], bf[ni]);
  }
}

struct DfArgs {
  const double* M;  // n x n, lower part read
  double* L;        // n x n column-major factor (lower tiles and diagonal tiles written)
  double* Lt;       // nt x nt packed 64 x 64 tiles of L (off-diagonal tiles), read by other CTAs
  double* W;        // nt packed 64 x 64 inverses of the diagonal tiles
  int64_t n;
  double delta;
  int nt, ntiles;
  unsigned* flags;  // nt x nt per-tile done flags (== generation when done)
  unsigned* ctl;    // [0] generation, [1] exit count, [2] failure generation, [3] pivot + 1, [4] tile counter
  long long* info;
  // fused triangular solves (rhs == nullptr: factor only). The diagonal tile i also forms
  // y_i = W_i (b_i - sum_k L_ik y_k) while it streams L_ik; nt backward tasks follow the
  // tiles: x_i = W_i' (y_i - sum_{j>i} L_ji' x_j), published through xflags.
  const double* rhs;  // n
  double* x;          // n (may alias rhs only if rhs is not read after the forward pass: it is not)
  double* ybuf;       // nt * 64
  double* xbuf;       // nt * 64
  unsigned* xflags;   // nt
  int nback;          // nt when solving, else 0
};

// thread 0: spin until both tile flags carry the generation; false on a published failure
__device__ __forceinline__ bool wait_flags(const unsigned* f1, const unsigned* f2, const unsigned* fail,
                                           unsigned target) {
  while (true) {
    if (ld_acquire(f1) == target && ld_acquire(f2) == target) return true;
    if (ld_acquire(fail) == target) return false;
  }
}

// one lower tile (i, j): left-looking updates, then potf2 + inverse (i == j) or the panel
// product with W_j (i > j). Returns false when the factorization failed somewhere.
__device__ bool df_tile(const DfArgs& A, int i, int j, unsigned target, double* sm, volatile unsigned* s_flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int nt = A.nt;
  const int64_t n = A.n, r0 = (int64_t)kNB * i, c0 = (int64_t)kNB * j;
  const bool diag = i == j;
  const bool idle = diag && wm == 0 && wn >= 2;  // strictly upper 32 x 16 blocks of a diagonal tile
  const unsigned* fl = A.flags;
  const unsigned* failw = A.ctl + 2;
  const bool fwd = diag && A.rhs != nullptr;
  double* ext = sm + 4 * kTB;  // [0,128) y_k stages, [128,192) t_i, [192,448) quarter partials
  const int fr = tid & 63, qd = tid >> 6;
  double fpart = 0.0;

  // acc = -(M_ij) (+ -delta on the diagonal), so the updates accumulate with DMMA's "+"
  double acc[2][2][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = 32 * wm + 16 * mi + g + 8 * (e >> 1), cl = 16 * wn + 8 * ni + 2 * t + (e & 1);
        double v = 0.0;
        if (r0 + r < n && c0 + cl < n && (!diag || r >= cl)) {
          v = A.M[(r0 + r) + (c0 + cl) * n];
          if (diag && r == cl && A.delta != 0.0) v = add(v, A.delta);
        }
        acc[mi][ni][e] = -v;
      }

  // A_ij -= sum_k L_ik L_jk^T, double-buffered: tile k+1 is prefetched when already published
  if (j > 0) {
    if (tid == 0) *s_flag = wait_flags(fl + i * nt, fl + j * nt, failw, target) ? 1u : 2u;
    __syncthreads();
    if (*s_flag == 2u) return false;
    stage_tile(sm, A.Lt + ((size_t)i * nt) * (kNB * kNB));
    if (!diag) stage_tile(sm + kTB, A.Lt + ((size_t)j * nt) * (kNB * kNB));
    if (fwd && tid < 32) cp_async16(ext + 2 * tid, A.ybuf + 2 * tid);
    cp_commit();
    for (int k = 0; k < j; ++k) {
      const int s = k & 1;
      double* xs = sm + 2 * s * kTB;
      double* xo = sm + 2 * (s ^ 1) * kTB;
      const bool more = k + 1 < j;
      if (tid == 0)
        *s_flag = (more && ld_acquire(fl + i * nt + k + 1) == target && ld_acquire(fl + j * nt + k + 1) == target)
                      ? 1u : 0u;
      __syncthreads();  // buffer s^1 is free (gemm k-1 done); s_flag visible
      const bool pre = *s_flag == 1u;
      if (pre) {
        stage_tile(xo, A.Lt + ((size_t)i * nt + k + 1) * (kNB * kNB));
        if (!diag) stage_tile(xo + kTB, A.Lt + ((size_t)j * nt + k + 1) * (kNB * kNB));
        if (fwd && tid < 32) cp_async16(ext + 64 * (s ^ 1) + 2 * tid, A.ybuf + 64 * (k + 1) + 2 * tid);
      }
      cp_commit();
      cp_wait1();
      __syncthreads();  // tile k visible to every warp
      if (!idle) gemm_xyt(xs, diag ? xs : xs + kTB, acc);
      if (fwd) {  // forward substitution partial: sum_k L_ik y_k, quarter qd of the columns
        const double* yk = ext + 64 * s;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) fpart = fma(xs[(16 * qd + kk) * kGemmLD + fr], yk[16 * qd + kk], fpart);
      }
      if (more && !pre) {
        if (tid == 0) *s_flag = wait_flags(fl + i * nt + k + 1, fl + j * nt + k + 1, failw, target) ? 1u : 2u;
        __syncthreads();
        if (*s_flag == 2u) return false;
        stage_tile(xo, A.Lt + ((size_t)i * nt + k + 1) * (kNB * kNB));
        if (!diag) stage_tile(xo + kTB, A.Lt + ((size_t)j * nt + k + 1) * (kNB * kNB));
        if (fwd && tid < 32) cp_async16(ext + 64 * (s ^ 1) + 2 * tid, A.ybuf + 64 * (k + 1) + 2 * tid);
        cp_commit();
      }
    }
  }
  __syncthreads();  // staging buffers free
  if (fwd) {  // t_i = b_i - sum_k L_ik y_k (fixed-order quarter sums)
    double* red = ext + 192;
    red[qd * 64 + fr] = fpart;
    __syncthreads();
    if (tid < 64) {
      const double bi = c0 + tid < n ? A.rhs[c0 + tid] : 0.0;
      ext[128 + tid] = bi - ((red[tid] + red[64 + tid]) + (red[128 + tid] + red[192 + tid]));
    }
  }

  if (diag) {
    double* a = sm;
    const int b = (int)(n - c0 < kNB ? n - c0 : kNB);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 32 * wm + 16 * mi + g + 8 * (e >> 1), cl = 16 * wn + 8 * ni + 2 * t + (e & 1);
          double v;
          if (r >= b || cl >= b) v = (r == cl) ? 1.0 : 0.0;
          else v = (r >= cl) ? -acc[mi][ni][e] : 0.0;
          a[r + cl * kLD] = v;
        }
    __syncthreads();
    TRACE(2);
    double* w = sm + kNB * kLD;
    const int f = diag_factor(a, w, w + kNB * kLD, b);
    if (f >= 0) {
      if (tid == 0) {
        A.ctl[3] = (unsigned)(c0 + f + 1);
        __threadfence();
        st_release(A.ctl + 2, target);
      }
      return false;
    }
    double* Wj = A.W + (size_t)j * (kNB * kNB);
    for (int e = tid; e < kNB * kNB; e += kDfThreads) {
      const int r = e & 63, cl = e >> 6;
      if (r < b && cl < b) A.L[(c0 + r) + (c0 + cl) * n] = (r >= cl) ? a[r + cl * kLD] : 0.0;
      Wj[e] = (r >= cl) ? w[r + cl * kLD] : 0.0;
    }
    if (fwd) {  // y_i = W_i t_i (W lower), published with the tile flag
      double* red = ext + 192;
      const double* tv = ext + 128;
      double s = 0.0;
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int c = 16 * qd + cc;
        if (c <= fr) s = fma(w[fr + c * kLD], tv[c], s);
      }
      red[qd * 64 + fr] = s;
      __syncthreads();
      if (tid < 64) A.ybuf[c0 + tid] = (red[tid] + red[64 + tid]) + (red[128 + tid] + red[192 + tid]);
    }
  } else {
    double* x = sm;
    double* y = sm + kTB;
    if (tid == 0) *s_flag = wait_flags(fl + j * nt + j, fl + j * nt + j, failw, target) ? 1u : 2u;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 32 * wm + 16 * mi + g + 8 * (e >> 1), cl = 16 * wn + 8 * ni + 2 * t + (e & 1);
          x[cl * kGemmLD + r] = -acc[mi][ni][e];
        }
    __syncthreads();
    if (*s_flag == 2u) return false;
    stage_tile(y, A.W + (size_t)j * (kNB * kNB));
    cp_commit();
    cp_wait0();
    __syncthreads();
    double out[2][2][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) out[mi][ni][e] = 0.0;
    gemm_xyt(x, y, out);  // L_ij = A_ij W_j^T
    __syncthreads();
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 32 * wm + 16 * mi + g + 8 * (e >> 1), cl = 16 * wn + 8 * ni + 2 * t + (e & 1);
          x[cl * kGemmLD + r] = out[mi][ni][e];
        }
    __syncthreads();
    double* Lt = A.Lt + ((size_t)i * nt + j) * (kNB * kNB);
    for (int e = tid; e < kNB * kNB; e += kDfThreads) {
      const int r = e & 63, cl = e >> 6;
      const double v = x[cl * kGemmLD + r];
      Lt[e] = v;
      if (r0 + r < n) A.L[(r0 + r) + (c0 + cl) * n] = v;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(A.flags + i * nt + j, target);
  }
  return true;
}

// backward block i: x_i = W_i' (y_i - sum_{j>i} L_ji' x_j), j from the last block down (the
// tile L_ji is staged before x_j is awaited). Warp w owns columns 8w..8w+7; lanes split the
// 64 rows, fixed-order warp sums.
__device__ bool df_back(const DfArgs& A, int i, unsigned target, double* sm, volatile unsigned* s_flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = A.nt;
  const unsigned* fl = A.flags;
  const unsigned* failw = A.ctl + 2;
  // W_i and y_i are final once the diagonal tile is
  if (tid == 0) *s_flag = wait_flags(fl + i * nt + i, fl + i * nt + i, failw, target) ? 1u : 2u;
  __syncthreads();
  if (*s_flag == 2u) return false;
  const double* Wi = A.W + (size_t)i * (kNB * kNB);
  double wv0[8], wv1[8];
#pragma unroll
  for (int cl = 0; cl < 8; ++cl) {
    wv0[cl] = __ldcg(Wi + (8 * warp + cl) * kNB + lane);
    wv1[cl] = __ldcg(Wi + (8 * warp + cl) * kNB + lane + 32);
  }
  double part[8];
#pragma unroll
  for (int cl = 0; cl < 8; ++cl) part[cl] = 0.0;
  for (int j = nt - 1; j > i; --j) {
    if (tid == 0) *s_flag = wait_flags(fl + j * nt + i, fl + j * nt + i, failw, target) ? 1u : 2u;
    __syncthreads();
    if (*s_flag == 2u) return false;
    stage_tile(sm, A.Lt + ((size_t)j * nt + i) * (kNB * kNB));
    cp_commit();
    if (tid == 0) *s_flag = wait_flags(A.xflags + j, A.xflags + j, failw, target) ? 1u : 2u;
    cp_wait0();
    __syncthreads();
    if (*s_flag == 2u) return false;
    const double x0 = __ldcg(A.xbuf + 64 * j + lane), x1 = __ldcg(A.xbuf + 64 * j + lane + 32);
#pragma unroll
    for (int cl = 0; cl < 8; ++cl) {
      const int c = 8 * warp + cl;
      part[cl] = fma(sm[c * kGemmLD + lane], x0, part[cl]);
      part[cl] = fma(sm[c * kGemmLD + lane + 32], x1, part[cl]);
    }
    __syncthreads();  // staging buffer reused by the next j
  }
  double* accv = sm + 4 * kTB;  // 64
  const double* yi = A.ybuf + 64 * i;
#pragma unroll
  for (int cl = 0; cl < 8; ++cl) {
    const double s = warp_sum(part[cl]);
    if (lane == 0) accv[8 * warp + cl] = __ldcg(yi + 8 * warp + cl) - s;
  }
  __syncthreads();
  const double a0 = accv[lane], a1 = accv[lane + 32];
  const int64_t r0 = (int64_t)kNB * i;
#pragma unroll
  for (int cl = 0; cl < 8; ++cl) {
    const int c = 8 * warp + cl;  // x(c) = sum_{r >= c} W(r, c) acc(r)
    const double s = warp_sum(fma(wv0[cl], a0, wv1[cl] * a1));
    if (lane == 0) {
      A.xbuf[64 * i + c] = s;
      if (r0 + c < A.n) A.x[r0 + c] = s;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(A.xflags + i, target);
  }
  return true;
}

__global__ void __launch_bounds__(kDfThreads, 1) k_chol_df(const DfArgs A) {
  extern __shared__ __align__(16) double sm_df[];
  __shared__ unsigned s_target, s_q, s_flag;
  const int tid = threadIdx.x;
  if (tid == 0) s_target = *reinterpret_cast<volatile unsigned*>(A.ctl) + 1u;
  __syncthreads();
  const unsigned target = s_target;
  TRACE(0);
  while (true) {
    if (tid == 0) s_q = atomicAdd(A.ctl + 4, 1u);
    __syncthreads();
    const int q = (int)s_q;
    if (q >= A.ntiles + A.nback) break;
    if (q >= A.ntiles) {  // backward solve tasks, last block first
      if (!df_back(A, A.nt - 1 - (q - A.ntiles), target, sm_df, &s_flag)) break;
      continue;
    }
    int j = 0, rem = q;  // column-major enumeration of the lower tiles
    while (rem >= A.nt - j) {
      rem -= A.nt - j;
      ++j;
    }
    if (!df_tile(A, j + rem, j, target, sm_df, &s_flag)) break;
  }
  TRACE(3);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(A.ctl + 1, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      const bool failed = ld_acquire(A.ctl + 2) == target;
      *A.info = failed ? (long long)*reinterpret_cast<volatile unsigned*>(A.ctl + 3) : 0;
      A.ctl[1] = 0;
      A.ctl[4] = 0;
      __threadfence();
      st_release(A.ctl, target);
    }
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

// the > 48 KB dynamic shared memory opt-ins, once per device (the context's device)
void set_attrs(int device) {
  static std::once_flag flags[kMaxDevices];
  once_per_device(flags, device, [] {
    CMPC_CUDA(cudaFuncSetAttribute(k_chol_df, cudaFuncAttributeMaxDynamicSharedMemorySize, kDfSmem));
    CMPC_CUDA(cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotfSmem));
    CMPC_CUDA(cudaFuncSetAttribute(k_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
}

}  // namespace

void chol_alloc(Ctx& c) {
  const int64_t nb = ceil_div(std::max<int64_t>(c.n, 1), kNB);
  c.Winv = dev_zeros<double>((size_t)nb * kNB * kNB, c.stream);
  c.Lt = dev_zeros<double>((size_t)nb * nb * kNB * kNB, c.stream);
  c.df_flags = dev_zeros<unsigned>((size_t)nb * nb, c.stream);
  c.df_ctl = dev_zeros<unsigned>(8, c.stream);
  c.df_y = dev_zeros<double>((size_t)nb * kNB, c.stream);
  c.df_x = dev_zeros<double>((size_t)nb * kNB, c.stream);
  c.df_xflags = dev_zeros<unsigned>((size_t)nb, c.stream);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  c.df_grid = sms;
}

void chol_free(Ctx& c) {
  for (void* p : {(void*)c.Winv, (void*)c.Lt, (void*)c.df_flags, (void*)c.df_ctl, (void*)c.df_y,
                  (void*)c.df_x, (void*)c.df_xflags})
    dev_free(p, c.stream);
  c.Winv = c.Lt = c.df_y = c.df_x = nullptr;
  c.df_flags = c.df_ctl = c.df_xflags = nullptr;
}

void launch_cholesky(Ctx& c, const double* M, double* L, double delta, const double* rhs, double* x) {
  const int64_t n = c.n;
  long long* info = &c.pk->info;
  if (n == 0) {
    CMPC_CUDA(cudaMemsetAsync(info, 0, sizeof(long long), c.stream));
    return;
  }
  set_attrs(c.device);
  const int nt = (int)ceil_div(n, kNB);
  DfArgs a;
  a.M = M;
  a.L = L;
  a.Lt = c.Lt;
  a.W = c.Winv;
  a.n = n;
  a.delta = delta;
  a.nt = nt;
  a.ntiles = nt * (nt + 1) / 2;
  a.flags = c.df_flags;
  a.ctl = c.df_ctl;
  a.info = info;
  a.rhs = rhs;
  a.x = x;
  a.ybuf = c.df_y;
  a.xbuf = c.df_x;
  a.xflags = c.df_xflags;
  a.nback = rhs ? nt : 0;
  const int grid = std::min(a.ntiles + a.nback, c.df_grid);
  k_chol_df<<<grid, kDfThreads, kDfSmem, c.stream>>>(a);
  CMPC_LAUNCHED();
}

void launch_factor_inverses(Ctx& c, const double* L) {
  if (c.n == 0) return;
  set_attrs(c.device);
  k_diag_inv<<<(unsigned)ceil_div(c.n, kNB), 256, kPotfSmem, c.stream>>>(L, c.n, c.Winv);
  CMPC_LAUNCHED();
}

void launch_chol_solve(Ctx& c, const double* L, const double* b, double* x) {
  if (c.n == 0) return;
  set_attrs(c.device);
  const size_t sm = sizeof(double) * ((size_t)c.n + kNB);
  if (sm > 200 * 1024) throw CudaError("chol_solve: n too large for the single-CTA TRSV");
  k_trsv<<<1, 512, sm, c.stream>>>(L, c.Winv, b, x, c.n);
  CMPC_LAUNCHED();
}

}  // namespace cmpc
