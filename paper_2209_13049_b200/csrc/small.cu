// Small QPs (n <= 32 and J within shared memory: BASELINE config 1, n = 20, m = 240): the whole
// of condmpc::ipm::solve (proj/src/ipm.cpp:160-268) in ONE CTA, the QP and the iterate in
// shared memory, every decision taken on the device. The general path pays two host
// round trips and ~15 kernel launches per iteration, which at this size are the whole cost
// (the general path is slower than one CPU core here). Used by cmpc_solve when
// no inspect hook is set; the log hook is replayed from a per-iteration record buffer.
//
// The arithmetic follows the reference's formulas with separate multiply and add (its SSE2
// build has no FMA): J v and H v per output in ascending column order; the sums over the rows (J'x, the gram entries of W = sqrt(sigma) J,
// the log-barrier and l1 merit terms, sum ps/s) are fixed-order warp / CTA trees, and the
// Cholesky and the triangular solves run right-looking in one warp (deterministic; parity at
// the north-star tolerance, not bitwise).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace cmpc {

namespace {

constexpr int kSmT = 256;
constexpr int kSmMaxN = 32;  // one warp holds the factor's rows

struct SmallArgs {
  int n, m;
  const double *H, *h, *J, *d;  // H n x n, J m x n column-major (ld m)
  double h0;
  double tol, mu_init, kappa_mu, tau, eta;
  int max_iter;
  double *v, *s, *lam, *z;  // outputs (device)
  double* res;              // status, iter, kkt, objective, trials
  double* log;              // max_iter x 8: iter, mu, alpha, alpha_z, kkt, objective, delta, trial
  long long* prof;          // debug (CMPC_SMALL_PROF): clock cycles per phase, 8 phases
};

// fixed-order CTA max (every thread gets the result)
__device__ double cta_max(double x, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  x = warp_max(x);
  __syncthreads();
  if (lane == 0) red[w] = x;
  __syncthreads();
  double t = red[0];
  for (int i = 1; i < kSmT / 32; ++i) t = fmax(t, red[i]);
  return t;
}

// K values at once (one barrier pair): sums (MAX = false) or maxima in x[0..K)
template <int K, bool MAX>
__device__ void cta_reduce(double (&x)[K], double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = MAX ? warp_max(x[k]) : warp_sum(x[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[k * 8 + w] = x[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = red[k * 8];
    for (int i = 1; i < kSmT / 32; ++i) t = MAX ? fmax(t, red[k * 8 + i]) : add(t, red[k * 8 + i]);
    x[k] = t;
  }
}

__global__ void __launch_bounds__(kSmT, 1) k_small_ipm(const SmallArgs a) {
  extern __shared__ double sm[];
  const int n = a.n, m = a.m, tid = threadIdx.x;
  // J's leading dimension odd: the per-column loops (J'x, the gram entries) read one row of
  // several columns at once, which an even stride would put in one bank
  const int lj = m | 1;
  double* J = sm;              // m x n, leading dimension lj
  double* W = J + lj * n;      // sqrt(sigma) J, the same layout
  double* H = W + lj * n;      // n x n
  const int ll = n | 1;        // L's leading dimension (odd: the backward solve reads rows)
  double* L = H + n * n;       // n x n, leading dimension ll
  double* mt = L + ll * n;     // n x n: M + delta I (lower)
  double* rd = mt + n * n;     // 1 / l_pp
  double* v = rd + n;          // n-vectors
  double* pv = v + n;
  double* vt = pv + n;
  double* r1 = vt + n;
  double* hv = r1 + n;         // H v
  double* rhs = hv + n;
  double* hh = rhs + n;
  double* s = hh + n;          // m-vectors
  double* lam = s + m;
  double* z = lam + m;
  double* dd = z + m;
  double* r2 = dd + m;
  double* r3 = r2 + m;
  double* sg = r3 + m;
  double* ps = sg + m;
  double* pl = ps + m;
  double* pz = pl + m;
  double* jv = pz + m;         // J v of the current point
  double* jp = jv + m;         // J pv
  double* st = jp + m;         // trial slack
  double* red = st + m;        // 6 x 8 partials

  for (int i = tid; i < m * n; i += kSmT) J[(i % m) + (i / m) * lj] = a.J[i];
  for (int i = tid; i < n * n; i += kSmT) H[i] = a.H[i];
  for (int i = tid; i < n; i += kSmT) {
    hh[i] = a.h[i];
    v[i] = 0.0;
  }
  double mu = a.mu_init;
  for (int r = tid; r < m; r += kSmT) {  // init (ipm.cpp:170-177)
    dd[r] = a.d[r];
    s[r] = fmax(1.0, a.d[r]);
    z[r] = mul(mu, dv(1.0, s[r]));
    lam[r] = z[r];
  }
  __syncthreads();
  const double hmax = [&] {
    double x = 0.0;
    for (int i = tid; i < n; i += kSmT) x = fmax(x, fabs(hh[i]));
    return cta_max(x, red);
  }();

  // y = A x for a column-major rows x cols block with leading dimension ld (per output in
  // ascending column order)
  auto gemv_rows = [&](const double* A, int rows, int cols, int ld, const double* x, double* y) {
    for (int r = tid; r < rows; r += kSmT) {
      double acc = 0.0;
      for (int c = 0; c < cols; ++c) acc = add(acc, mul(A[r + c * ld], x[c]));
      y[r] = acc;
    }
  };
  const int warp = tid >> 5, lane = tid & 31;
  // y = J'x: a warp per column, lanes over the rows, fixed-order warp sum (every thread must
  // call it; y is complete after the caller's next barrier)
  // (a warp's columns c, c + 8, c + 16, c + 24 side by side: four independent chains and warp
  // sums instead of one after the other; each column's own order is unchanged)
  auto gemv_jt = [&](const double* x, double* y) {
    constexpr int kW = kSmT / 32;
    for (int c0 = warp; c0 < n; c0 += 4 * kW) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int r = lane; r < m; r += 32) {
        const double xr = x[r];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (c0 + kW * k < n) acc[k] = add(acc[k], mul(J[r + (c0 + kW * k) * lj], xr));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (c0 + kW * k < n) {
          const double t = warp_sum(acc[k]);
          if (lane == 0) y[c0 + kW * k] = t;
        }
      }
    }
  };
  // compute_residuals (ipm.cpp:46-70): r1, r2, r3, jv, hv; returns kkt
  // kkt from the residual maxima {|r1|, |lambda|, |s|, |z|, |r3|} and the complementarity max
  double kmax[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  auto kkt_of = [&](double mc) -> double {
    const double ds = fmax(1.0, fmax(hmax, kmax[1]) / (double)(n + m));
    double kkt = kmax[0] / ds;
    if (m > 0) {
      const double cs = fmax(1.0, fmax(kmax[2], kmax[3]) / (double)(2 * m));
      kkt = fmax(kkt, kmax[4]);
      kkt = fmax(kkt, mc / cs);
    }
    return kkt;
  };
  auto residuals = [&]() -> double {
    gemv_rows(H, n, n, n, v, hv);
    gemv_rows(J, m, n, lj, v, jv);
    gemv_jt(lam, rhs);  // rhs: scratch J'lambda
    __syncthreads();
    double mr1 = 0.0;
    for (int i = tid; i < n; i += kSmT) {
      double t = add(hv[i], hh[i]);
      if (m > 0) t = add(t, rhs[i]);
      r1[i] = t;
      mr1 = fmax(mr1, fabs(t));
    }
    double ml = 0.0, ms = 0.0, mz = 0.0, mc = 0.0, mr3 = 0.0;
    for (int r = tid; r < m; r += kSmT) {
      r2[r] = sub(lam[r], mul(mu, dv(1.0, s[r])));
      const double t3 = add(sub(jv[r], dd[r]), s[r]);
      r3[r] = t3;
      ml = fmax(ml, fabs(lam[r]));
      ms = fmax(ms, fabs(s[r]));
      mz = fmax(mz, fabs(z[r]));
      mr3 = fmax(mr3, fabs(t3));
      mc = fmax(mc, fabs(sub(mul(s[r], z[r]), mu)));
    }
    double mx[6] = {mr1, ml, ms, mz, mr3, mc};
    cta_reduce<6, true>(mx, red);
    for (int k = 0; k < 5; ++k) kmax[k] = mx[k];  // (kept for a barrier update)
    return kkt_of(mx[5]);
  };
  // the same after a barrier update: only r2 and the complementarity change with mu (v, s,
  // lambda, z do not), so r1, r3 and the other maxima stay those of the last full pass
  auto residuals_mu = [&]() -> double {
    double mc = 0.0;
    for (int r = tid; r < m; r += kSmT) {
      r2[r] = sub(lam[r], mul(mu, dv(1.0, s[r])));
      mc = fmax(mc, fabs(sub(mul(s[r], z[r]), mu)));
    }
    return kkt_of(cta_max(mc, red));
  };
  // 0.5 v'Hv + h'v for x (hx = H x given), per ascending index
  auto quad = [&](const double* x, const double* hx) {
    double a1 = 0.0, a2 = 0.0;
    for (int i = 0; i < n; ++i) {
      a1 = add(a1, mul(x[i], hx[i]));
      a2 = add(a2, mul(hh[i], x[i]));
    }
    return add(mul(0.5, a1), a2);
  };

  // debug phase clock (thread 0; CMPC_SMALL_PROF)
  long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_t = clock64();
  auto mark = [&](int ph) {
    if (a.prof && tid == 0) {
      const long long t = clock64();
      ph_acc[ph] += t - ph_t;
      ph_t = t;
    }
  };
  double kkt = residuals();
  int iter = 0, status = -1, trials = 0;
  constexpr double kShifts[7] = {0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1.0, 1e2};
  while (true) {
    if (kkt <= a.tol && mu <= a.tol) {  // check_termination (ipm.cpp:153-158)
      status = 0;
      break;
    }
    if (iter >= a.max_iter) {
      status = 1;
      break;
    }
    const double mu_next = kkt <= mul(10.0, mu) ? fmax(a.tol / 10.0, mul(a.kappa_mu, mu)) : mu;  // :146-151
    if (mu_next != mu) {
      mu = mu_next;
      __syncthreads();
      kkt = residuals_mu();
    }
    // sigma = z / s; M = H + W'W, W = sqrt(sigma) J (assemble_condensed + gram_weighted)
    // W = sqrt(sigma) J, formed once per iteration (the square root once per row, kept in jp:
    // J pv is formed after the factorization)
    for (int r = tid; r < m; r += kSmT) {
      sg[r] = dv(z[r], s[r]);
      jp[r] = sqrt(sg[r]);
    }
    __syncthreads();
    for (int r = tid; r < m; r += kSmT) {
      const double q = jp[r];
      for (int c = 0; c < n; ++c) W[r + c * lj] = mul(q, J[r + c * lj]);
    }
    __syncthreads();
    mark(0);
    double delta = 0.0;
    bool factored = false;
#pragma unroll 1
    for (int sh = 0; sh < 7 && !factored; ++sh) {
      delta = kShifts[sh];
      // lower triangle of M (+ delta I) = H + W'W, W = sqrt(sigma) J: entry (i, j) over the rows
      // in four interleaved partial sums; a thread takes a 2 x 2 block of entries, so each W
      // element it loads serves two products (the gram is bound by shared-memory loads)
      {
        const int nb = (n + 1) / 2;
        for (int e = tid; e < nb * nb; e += kSmT) {
          const int bi = e % nb, bj = e / nb;
          if (bi < bj) continue;
          const int i0 = 2 * bi, j0 = 2 * bj;
          const int i1 = min(i0 + 1, n - 1), j1 = min(j0 + 1, n - 1);  // (odd n: a duplicate)
          double g[2][2][4];
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v2 = 0; v2 < 2; ++v2)
#pragma unroll
              for (int q = 0; q < 4; ++q) g[u][v2][q] = 0.0;
          int r = 0;
          for (; r + 4 <= m; r += 4)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double a0 = W[r + q + i0 * lj], a1 = W[r + q + i1 * lj];
              const double b0 = W[r + q + j0 * lj], b1 = W[r + q + j1 * lj];
              g[0][0][q] = add(g[0][0][q], mul(a0, b0));
              g[0][1][q] = add(g[0][1][q], mul(a0, b1));
              g[1][0][q] = add(g[1][0][q], mul(a1, b0));
              g[1][1][q] = add(g[1][1][q], mul(a1, b1));
            }
          for (; r < m; ++r) {
            const double a0 = W[r + i0 * lj], a1 = W[r + i1 * lj];
            const double b0 = W[r + j0 * lj], b1 = W[r + j1 * lj];
            g[0][0][0] = add(g[0][0][0], mul(a0, b0));
            g[0][1][0] = add(g[0][1][0], mul(a0, b1));
            g[1][0][0] = add(g[1][0][0], mul(a1, b0));
            g[1][1][0] = add(g[1][1][0], mul(a1, b1));
          }
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v2 = 0; v2 < 2; ++v2) {
              const int i = i0 + u, j = j0 + v2;
              if (i >= n || j >= n || i < j) continue;
              const int e2 = i + j * n;
              double x = add(H[e2], add(add(g[u][v2][0], g[u][v2][1]), add(g[u][v2][2], g[u][v2][3])));
              if (i == j && delta != 0.0) x = add(x, delta);
              mt[e2] = x;
            }
        }
      }
      __syncthreads();
      mark(1);
      // Cholesky of M + delta I, right-looking over the whole CTA (pivot rule of potf2_lower,
      // dense_linalg.cpp:24-40: !(d > 0) || !isfinite(d)); the pivot's 1 / sqrt by the MUFU seed
      // and two Newton steps (the IEEE sqrt and division are long subroutines on the chain)
      // one barrier per pivot: every thread forms the pivot's reciprocal square root itself (the
      // same operations on the same value), L[i, p] and L[c, p] on the fly from column p (which
      // the trailing update of this pivot does not touch). (Two pivots per barrier measured no
      // faster: the per-thread work doubles what the saved barriers give back.)
      int bad = 0;
      for (int p = 0; p < n; ++p) {
        const double dp = mt[p + p * n];
        if (!(dp > 0.0) || !isfinite(dp)) {  // (uniform)
          bad = 1;
          break;
        }
        double rp;
        if (dp >= 1e-300 && dp <= 1e300) {
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rp) : "d"(dp));
          const double hx = 0.5 * dp;
          rp = rp * fma(-hx * rp, rp, 1.5);
          rp = rp * fma(-hx * rp, rp, 1.5);
        } else {
          rp = 1.0 / sqrt(dp);
        }
        if (tid == 0) {
          L[p + p * ll] = mul(dp, rp);
          rd[p] = rp;
        }
        // trailing update: thread (row i = tid % 32, columns c = tid / 32 + 8 k) of the lower
        // part (n <= 32); warp 0 also stores the column
        const int i = tid & 31;
        if (i > p && i < n) {
          const double lip = mul(mt[i + p * n], rp);
          if (warp == 0) L[i + p * ll] = lip;
          for (int c = p + 1 + (tid >> 5); c <= i; c += kSmT / 32)
            mt[i + c * n] = sub(mt[i + c * n], mul(lip, mul(mt[c + p * n], rp)));
        }
        __syncthreads();
      }
      factored = !bad;  // (uniform)
      __syncthreads();
      mark(2);
    }
    if (!factored) {
      status = 2;
      break;
    }
    // step_directions (ipm.cpp:79-103): rhs = -r1 + J'(r2 - sigma r3), pv = L^-T L^-1 rhs
    for (int r = tid; r < m; r += kSmT) st[r] = sub(r2[r], mul(sg[r], r3[r]));  // st: scratch y
    __syncthreads();
    gemv_jt(st, vt);  // vt: scratch J'y
    __syncthreads();
    for (int i = tid; i < n; i += kSmT) pv[i] = m > 0 ? add(-r1[i], vt[i]) : -r1[i];
    __syncthreads();
    if (warp == 0) {  // factor_solve (dense_linalg.cpp:102-110), right-looking in one warp:
      // pv[i] in lane i's register (n <= 32), each x_j broadcast by a shuffle
      const int i = lane;
      double pvi = i < n ? pv[i] : 0.0;
      for (int j = 0; j < n; ++j) {
        const double xj = __shfl_sync(0xffffffffu, mul(pvi, rd[j]), j);
        if (i > j && i < n) pvi = sub(pvi, mul(L[i + j * ll], xj));
        if (i == j) pvi = xj;
      }
      for (int j = n - 1; j >= 0; --j) {
        const double xj = __shfl_sync(0xffffffffu, mul(pvi, rd[j]), j);
        if (i < j) pvi = sub(pvi, mul(L[j + i * ll], xj));
        if (i == j) pvi = xj;
      }
      if (i < n) pv[i] = pvi;
    }
    __syncthreads();
    mark(3);
    gemv_rows(J, m, n, lj, pv, jp);
    __syncthreads();
    double as = 1.0, az = 1.0;  // fraction_to_boundary (ipm.cpp:105-116)
    for (int r = tid; r < m; r += kSmT) {
      const double p_s = sub(-r3[r], jp[r]);
      ps[r] = p_s;
      pl[r] = add(-r2[r], mul(sg[r], add(r3[r], jp[r])));
      const double p_z = sub(sub(mul(mu, dv(1.0, s[r])), z[r]), mul(sg[r], p_s));
      pz[r] = p_z;
      if (p_s < 0.0) as = fmin(as, mul(a.tau, dv(-s[r], p_s)));
      if (p_z < 0.0) az = fmin(az, mul(a.tau, dv(-z[r], p_z)));
    }
    // line_search + merit (ipm.cpp:118-144, :25-32): the step-length minima (min as the
    // negated max, exact; 1.0 when no blocking entry) and max |lambda| in one reduction, the
    // merit sums in another
    double ml = 0.0;
    for (int r = tid; r < m; r += kSmT) ml = fmax(ml, fabs(lam[r]));
    double mx3[3] = {-as, -az, ml};
    cta_reduce<3, true>(mx3, red);
    const double alpha_max = -mx3[0], alpha_z = -mx3[1];
    ml = mx3[2];
    const double rho = add(mul(10.0, ml), 1.0);
    double slog = 0.0, sl1 = 0.0, sq = 0.0;
    for (int r = tid; r < m; r += kSmT) {
      slog += log(s[r]);
      sl1 += fabs(add(sub(jv[r], dd[r]), s[r]));
      sq += dv(ps[r], s[r]);
    }
    __syncthreads();  // (red is reused)
    double su3[3] = {slog, sl1, sq};
    cta_reduce<3, false>(su3, red);
    slog = su3[0];
    sl1 = su3[1];
    sq = su3[2];
    double phi0 = quad(v, hv), deriv = 0.0;
    {
      double gpv = 0.0;
      for (int i = 0; i < n; ++i) gpv = add(gpv, mul(add(hv[i], hh[i]), pv[i]));
      deriv = gpv;
    }
    if (m > 0) {
      phi0 = add(sub(phi0, mul(mu, slog)), mul(rho, sl1));
      deriv = sub(sub(deriv, mul(mu, sq)), mul(rho, sl1));
    }
    constexpr double band = 10.0 * 2.220446049250313e-16;
    mark(4);
    double alpha = alpha_max;
    int jacc = -1;
    for (int j = 0; j <= 30; ++j, alpha *= 0.5) {
      ++trials;
      for (int i = tid; i < n; i += kSmT) vt[i] = add(v[i], mul(alpha, pv[i]));
      int bad = 0;
      for (int r = tid; r < m; r += kSmT) {
        const double t = add(s[r], mul(alpha, ps[r]));
        st[r] = t;
        bad |= t <= 0.0;
      }
      bad = __syncthreads_or(bad);
      if (m > 0 && bad) continue;
      gemv_rows(H, n, n, n, vt, rhs);  // scratch: H v_t (rhs is spent)
      gemv_rows(J, m, n, lj, vt, sg);   // scratch: J v_t (sigma is spent: the directions are formed)
      __syncthreads();
      double tl = 0.0, t1 = 0.0;
      for (int r = tid; r < m; r += kSmT) {
        tl += log(st[r]);
        t1 += fabs(add(sub(sg[r], dd[r]), st[r]));
      }
      double su2[2] = {tl, t1};
      cta_reduce<2, false>(su2, red);
      tl = su2[0];
      t1 = su2[1];
      double phi = quad(vt, rhs);
      if (m > 0) phi = add(sub(phi, mul(mu, tl)), mul(rho, t1));
      if (deriv <= 0.0 && phi <= add(phi0, mul(mul(a.eta, alpha), deriv))) {
        jacc = j;
        break;
      }
      if (fabs(sub(phi, phi0)) <= mul(band, add(1.0, fabs(phi0)))) {
        jacc = j;
        break;
      }
    }
    if (jacc < 0) {
      status = 3;
      break;
    }
    __syncthreads();
    mark(5);
    const double mu_used = mu;
    for (int i = tid; i < n; i += kSmT) v[i] = add(v[i], mul(alpha, pv[i]));
    for (int r = tid; r < m; r += kSmT) {
      s[r] = add(s[r], mul(alpha, ps[r]));
      lam[r] = add(lam[r], mul(alpha, pl[r]));
      z[r] = add(z[r], mul(alpha_z, pz[r]));
    }
    __syncthreads();
    ++iter;
    kkt = residuals();
    __syncthreads();
    if (tid == 0) {
      double* rec = a.log + (size_t)(iter - 1) * 8;
      rec[0] = iter;
      rec[1] = mu_used;
      rec[2] = alpha;
      rec[3] = alpha_z;
      rec[4] = kkt;
      rec[5] = add(quad(v, hv), a.h0);
      rec[6] = delta;
      rec[7] = jacc;
    }
    mark(6);
  }
  __syncthreads();
  if (a.prof && tid == 0)
    for (int i = 0; i < 8; ++i) a.prof[i] = ph_acc[i];
  for (int i = tid; i < n; i += kSmT) a.v[i] = v[i];
  for (int r = tid; r < m; r += kSmT) {
    a.s[r] = s[r];
    a.lam[r] = lam[r];
    a.z[r] = z[r];
  }
  if (tid == 0) {
    a.res[0] = status;
    a.res[1] = iter;
    a.res[2] = kkt;
    a.res[3] = add(quad(v, hv), a.h0);
    a.res[4] = trials;
  }
}

}  // namespace

size_t small_smem_bytes(int64_t n, int64_t m) {
  return sizeof(double) * (size_t)(2 * (m | 1) * n + 2 * n * n + (n | 1) * n + 8 * n + 14 * m + 64);
}
bool small_fits(int64_t n, int64_t m) {
  return n >= 1 && n <= kSmMaxN && small_smem_bytes(n, m) <= 200 * 1024;
}

int small_solve(Ctx& c, const double* opts, int64_t max_iter, double* v_out, double* s_out, double* lam_out,
                double* z_out, double* out, cmpc_log_fn log, void* user) {
  NvtxRange nv("cmpc_solve: one-CTA solver");
  const int64_t n = c.n, m = c.m;
  const double t0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  if (c.small_log_cap < max_iter) {
    dev_free(c.small_log, c.stream);
    c.small_log = dev_alloc<double>((size_t)max_iter * 8, c.stream);
    c.small_log_cap = max_iter;
  }
  if (!c.small_res) c.small_res = dev_alloc<double>(8, c.stream);
  static std::once_flag flags[kMaxDevices];
  once_per_device(flags, c.device, [] {
    CMPC_CUDA(cudaFuncSetAttribute(k_small_ipm, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  SmallArgs a;
  a.n = (int)n;
  a.m = (int)m;
  a.H = c.H;
  a.h = c.h;
  a.J = c.Jsmall;
  a.d = c.d;
  a.h0 = c.h0;
  a.tol = opts[0];
  a.mu_init = opts[1];
  a.kappa_mu = opts[2];
  a.tau = opts[3];
  a.eta = opts[4];
  a.max_iter = (int)max_iter;
  a.v = c.v;
  a.s = c.s;
  a.lam = c.lam;
  a.z = c.z;
  a.res = c.small_res;
  a.log = c.small_log;
  static const bool sprof = getenv("CMPC_SMALL_PROF") != nullptr;
  a.prof = nullptr;
  if (sprof) a.prof = dev_zeros<long long>(8, c.stream);
  cudaEvent_t e0, e1;
  CMPC_CUDA(cudaEventCreate(&e0));
  CMPC_CUDA(cudaEventCreate(&e1));
  CMPC_CUDA(cudaEventRecord(e0, c.stream));
  k_small_ipm<<<1, kSmT, small_smem_bytes(n, m), c.stream>>>(a);
  CMPC_LAUNCHED();
  CMPC_CUDA(cudaEventRecord(e1, c.stream));
  double res[8] = {0};
  CMPC_CUDA(cudaMemcpyAsync(res, c.small_res, sizeof(double) * 5, cudaMemcpyDeviceToHost, c.stream));
  CMPC_CUDA(cudaStreamSynchronize(c.stream));
  if (a.prof) {  // debug: cycles per phase over the solve
    long long ph[8];
    CMPC_CUDA(cudaMemcpy(ph, a.prof, sizeof(ph), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[small prof] sigma+W %lld gram %lld chol %lld solves %lld dirs+ls-setup %lld trials %lld update+res %lld (cycles, %d iterations)\n",
            ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6], (int)res[1]);
    dev_free(a.prof, c.stream);
  }
  const int64_t iters = (int64_t)res[1];
  std::vector<double> lg;
  if (log && iters > 0) {
    lg.resize(size_t(iters) * 8);
    CMPC_CUDA(cudaMemcpy(lg.data(), c.small_log, sizeof(double) * lg.size(), cudaMemcpyDeviceToHost));
  }
  if (v_out) CMPC_CUDA(cudaMemcpy(v_out, c.v, sizeof(double) * n, cudaMemcpyDeviceToHost));
  if (s_out) CMPC_CUDA(cudaMemcpy(s_out, c.s, sizeof(double) * m, cudaMemcpyDeviceToHost));
  if (lam_out) CMPC_CUDA(cudaMemcpy(lam_out, c.lam, sizeof(double) * m, cudaMemcpyDeviceToHost));
  if (z_out) CMPC_CUDA(cudaMemcpy(z_out, c.z, sizeof(double) * m, cudaMemcpyDeviceToHost));
  float ms = 0.f;
  CMPC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (int64_t k = 0; k < iters && log; ++k) log(user, lg.data() + k * 8);
  if (out) {
    out[0] = res[0];
    out[1] = res[1];
    out[2] = res[2];
    out[3] = res[3];
    out[4] = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - t0;
    out[5] = 0.0;
    out[6] = ms * 1e-3;
    out[7] = 1;   // launches
    out[8] = 1;   // host syncs
    out[9] = res[4];
    for (int k = 10; k < 14; ++k) out[k] = 0.0;
  }
  return (int)res[0];
}

}  // namespace cmpc
