// the dense QP built on the device from the structured MPC data,
// the receding-horizon refresh of the initial state, and the trajectory recovery.
//
// Reference: build_dense_qp (proj/src/reduction.cpp:255-268) with the Hessian :88-117, the
// affine terms :119-180 and the inequality rows :182-251; refresh_initial_state :270-280;
// recover_trajectory :282-314. The reference materialises bigA / bigAtilde / bigB
// (bigAtilde alone is 127 GB at config 3); like the host restatement (problem.py) this keeps
// only the first block column of bigB, G_k = A_K^k B (k < T), and the free response
// x0_{t+1} = A_K x0_t + w_t. On the device:
//   Gall = [G_0 .. G_{T-1}] (n_x x T n_u)    C  = Gall' Q_K Gall,  Cf = Gall' Qf Gall
//   H_jk = 2 (sum_{s < T-1-max(j,k)} C[a0+s, b0+s] + Cf[T-1-j, T-1-k] + R_jk + cross)
//          (a0, b0) = (max - j, max - k): the block-Toeplitz sums of bigB' Q bigB
//   h_j  = 2 sum_{t > j} (Gall' Q_t x0_t)[block t-1-j] + 2 S_K' x0_j,   h0 = sum x0' Q_t x0
//   J, d: one row per finite bound in the reference's row order, filled from Gall (state
//         rows), K Gall (input rows) and (E + F K) Gall (mixed rows).
// The built H, h, h0, J, d are then loaded like a host QP (structure analysis, plan); Gall,
// x0 and the row table stay resident for refresh_initial_state and recover_trajectory, so a
// receding-horizon step uploads n_x numbers and never re-analyses J.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace cmpc {

namespace {

// ---------------------------------------------------------------- plain tiled DGEMM
// C(M x N) = alpha op(A) op(B) + beta C, column-major; 64 x 64 tiles, 256 threads, 4 x 4
// outputs per thread. Setup-time GEMMs only (the solve's products are the tuned kernels).
constexpr int kGT = 64, kGK = 16;
__global__ void __launch_bounds__(256) k_gemm(int M, int N, int K, double alpha, const double* __restrict__ A,
                                              int64_t lda, int ta, const double* __restrict__ B, int64_t ldb,
                                              int tb, double beta, double* __restrict__ C, int64_t ldc) {
  __shared__ double As[kGK][kGT + 1], Bs[kGK][kGT + 1];
  const int tid = threadIdx.x, tr = tid & 15, tc = tid >> 4;
  const int i0 = blockIdx.x * kGT, j0 = blockIdx.y * kGT;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kGK) {
    for (int e = tid; e < kGK * kGT; e += 256) {
      const int kk = e / kGT, ii = e % kGT;  // consecutive threads: consecutive rows
      const int gi = i0 + ii, gk = k0 + kk;
      double av = 0.0;
      if (gi < M && gk < K) av = ta ? A[gk + (int64_t)gi * lda] : A[gi + (int64_t)gk * lda];
      As[kk][ii] = av;
      const int gj = j0 + ii;
      double bv = 0.0;
      if (gj < N && gk < K) bv = tb ? B[gj + (int64_t)gk * ldb] : B[gk + (int64_t)gj * ldb];
      Bs[kk][ii] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][tr + 16 * u];
        b[u] = Bs[kk][tc + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int gi = i0 + tr + 16 * u, gj = j0 + tc + 16 * v;
      if (gi < M && gj < N) {
        double* p = C + gi + (int64_t)gj * ldc;
        *p = alpha * acc[u][v] + (beta == 0.0 ? 0.0 : beta * *p);
      }
    }
}

void gemm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
          int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  dim3 g((unsigned)ceil_div(M, kGT), (unsigned)ceil_div(N, kGT));
  k_gemm<<<g, 256, 0, st>>>((int)M, (int)N, (int)K, alpha, A, lda, ta ? 1 : 0, B, ldb, tb ? 1 : 0, beta, C, ldc);
  CMPC_LAUNCHED();
}

// one row of J: kind 0 mixed (E + F K), 1 state, 2 input; upper bound or lower; stage t; index i
struct RowDesc {
  int kind, upper, t, i;
};

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i] + (b == 0.0 ? 0.0 : b * y[i]);
}

// H(p, q), both triangles: 2 (block-Toeplitz sums of C + Cf + R + cross), symmetrised
__global__ void k_hess(int64_t n, int nu, int T, const double* __restrict__ C, const double* __restrict__ Cf,
                       const double* __restrict__ R, const double* __restrict__ CS, double* __restrict__ H) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int p = (int)(e % n), q = (int)(e / n);
  auto raw = [&](int pr, int qc) {
    const int j = pr / nu, k = qc / nu, pp = pr % nu, qq = qc % nu;
    const int mx = j > k ? j : k, L = T - 1 - mx, a0 = mx - j, b0 = mx - k;
    double s = 0.0;
    for (int t = 0; t < L; ++t) s += C[((a0 + t) * nu + pp) + (int64_t)((b0 + t) * nu + qq) * n];
    s += Cf[((T - 1 - j) * nu + pp) + (int64_t)((T - 1 - k) * nu + qq) * n];
    if (j == k) s += R[pp + qq * nu];
    // cross terms bigB_t' S_K at column block t = k (rows j < k) and their transpose
    if (CS) {
      if (j < k) s += CS[((k - 1 - j) * nu + pp) + (int64_t)qq * n];
      if (k < j) s += CS[((j - 1 - k) * nu + qq) + (int64_t)pp * n];
    }
    return 2.0 * s;
  };
  H[e] = 0.5 * (raw(p, q) + raw(q, p));
}

// h_j = 2 sum_{t=j+1}^{T} D[(t-1-j) nu + pp, t] + 2 SX[pp, j];  D = Gall' QX (T nu x (T+1))
__global__ void k_lin(int64_t n, int nu, int T, const double* __restrict__ D, const double* __restrict__ SX,
                      double* __restrict__ h) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int j = (int)(e / nu), pp = (int)(e % nu);
  double s = 0.0;
  for (int t = j + 1; t <= T; ++t) s += D[((t - 1 - j) * nu + pp) + (int64_t)t * n];
  s *= 2.0;
  if (SX) s += 2.0 * SX[pp + (int64_t)j * nu];
  h[e] = s;
}

// h0 = sum_t x0_t . QX_t (fixed-order block sum, one block)
__global__ void __launch_bounds__(1024) k_h0(int64_t len, const double* __restrict__ X0,
                                             const double* __restrict__ QX, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) s = fma(X0[i], QX[i], s);
  s = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) *out = s;
}

// d[r] from the row table: state rows x0_t, input rows (K x0_t), mixed rows (EFK x0_t)
__global__ void k_rows_d(int64_t m, const RowDesc* __restrict__ rd, const double* __restrict__ bound,
                         const double* __restrict__ X0, const double* __restrict__ KX,
                         const double* __restrict__ EX, int nx, int nu, int nc, double* __restrict__ d) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const RowDesc q = rd[r];
  double off;
  if (q.kind == 1) off = X0[q.i + (int64_t)q.t * nx];
  else if (q.kind == 2) off = KX[q.i + (int64_t)q.t * nu];
  else off = EX[q.i + (int64_t)q.t * nc];
  d[r] = q.upper ? bound[r] - off : off - bound[r];
}

// J (m x n, column-major), row-fastest so the writes coalesce
__global__ void k_rows_J(int64_t m, int64_t n, const RowDesc* __restrict__ rd, const double* __restrict__ G,
                         const double* __restrict__ KG, const double* __restrict__ EG,
                         const double* __restrict__ F, int nx, int nu, int nc, double* __restrict__ J) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % m, col = e / m;
    const RowDesc q = rd[r];
    const int j = (int)(col / nu), cc = (int)(col % nu);
    const double sg = q.upper ? 1.0 : -1.0;
    double v = 0.0;
    if (j < q.t) {
      const int64_t gc = (int64_t)(q.t - 1 - j) * nu + cc;  // column of G_{t-1-j}
      if (q.kind == 1) v = G[q.i + gc * nx];
      else if (q.kind == 2) v = KG ? KG[q.i + gc * nu] : 0.0;
      else v = EG[q.i + gc * nc];
      v *= sg;
    }
    if (q.kind == 2 && col == (int64_t)q.t * nu + q.i) v += sg;
    if (q.kind == 0 && j == q.t) v += sg * F[q.i + (int64_t)cc * nc];
    J[e] = v;
  }
}

// x_t = x0_t + sum_{j<t} G_{t-1-j} v_j (X: n_x x (T+1))
__global__ void k_traj(int nx, int nu, int T, const double* __restrict__ X0, const double* __restrict__ G,
                       const double* __restrict__ v, double* __restrict__ X) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * (T + 1)) return;
  const int i = (int)(e % nx), t = (int)(e / nx);
  double s = X0[e];
  for (int j = 0; j < t; ++j)
    for (int c = 0; c < nu; ++c) s = fma(G[i + ((int64_t)(t - 1 - j) * nu + c) * nx], v[j * nu + c], s);
  X[e] = s;
}

// per stage t: x_t' Q x_t (+ 2 x_t' S u_t + u_t' R u_t for t < T), Qf at t = T; QX, SU, RU
// are the products; fixed-order block sum
__global__ void __launch_bounds__(1024) k_traj_obj(int nx, int nu, int T, const double* __restrict__ X,
                                                   const double* __restrict__ QX, const double* __restrict__ U,
                                                   const double* __restrict__ SU, const double* __restrict__ RU,
                                                   double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)nx * (T + 1); e += blockDim.x) s = fma(X[e], QX[e], s);
  for (int64_t e = threadIdx.x; e < (int64_t)nx * T; e += blockDim.x) s = fma(2.0 * X[e], SU[e], s);
  for (int64_t e = threadIdx.x; e < (int64_t)nu * T; e += blockDim.x) s = fma(U[e], RU[e], s);
  s = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) *out = s;
}

}  // namespace

struct ProblemDev {
  int64_t nx = 0, nu = 0, nc = 0, T = 0, n = 0, m = 0;
  bool has_K = false, has_S = false;
  double *AK = nullptr, *G = nullptr, *QK = nullptr, *Qf = nullptr, *R = nullptr, *SK = nullptr,
         *S = nullptr, *K = nullptr, *EFK = nullptr, *F = nullptr, *W = nullptr, *X0 = nullptr,
         *bound = nullptr, *Q = nullptr;
  RowDesc* rows = nullptr;
};

void prob_free(Ctx& c) {
  auto* p = static_cast<ProblemDev*>(c.prob);
  if (!p) return;
  for (void* q : {(void*)p->AK, (void*)p->G, (void*)p->QK, (void*)p->Qf, (void*)p->R, (void*)p->SK,
                  (void*)p->S, (void*)p->K, (void*)p->EFK, (void*)p->F, (void*)p->W, (void*)p->X0,
                  (void*)p->bound, (void*)p->Q, (void*)p->rows})
    dev_free(q, c.stream);
  delete p;
  c.prob = nullptr;
}

namespace {

// free response X0 (n_x x (T+1)) from x_bar (device) and W
void free_response(Ctx& c, ProblemDev& p) {
  const int64_t nx = p.nx;
  for (int64_t t = 0; t < p.T; ++t) {
    double* next = p.X0 + (t + 1) * nx;
    CMPC_CUDA(cudaMemcpyAsync(next, p.W + t * nx, sizeof(double) * nx, cudaMemcpyDeviceToDevice, c.stream));
    gemm(c.stream, false, false, nx, 1, nx, 1.0, p.AK, nx, p.X0 + t * nx, nx, 1.0, next, nx);
  }
}

// h, h0, d of the current X0 into the given device buffers
void affine(Ctx& c, ProblemDev& p, double* h, double* h0_dev, double* d) {
  const int64_t nx = p.nx, nu = p.nu, nc = p.nc, T = p.T, n = p.n;
  cudaStream_t st = c.stream;
  double* QX = dev_alloc<double>(size_t(nx * (T + 1)), st);
  gemm(st, false, false, nx, T, nx, 1.0, p.QK, nx, p.X0, nx, 0.0, QX, nx);
  gemm(st, false, false, nx, 1, nx, 1.0, p.Qf, nx, p.X0 + T * nx, nx, 0.0, QX + T * nx, nx);
  double* D = dev_alloc<double>(size_t(n * (T + 1)), st);
  gemm(st, true, false, n, T + 1, nx, 1.0, p.G, nx, QX, nx, 0.0, D, n);
  double* SX = nullptr;
  if (p.has_S || p.has_K) {  // S_K' x0_t for t < T
    SX = dev_alloc<double>(size_t(nu * T), st);
    gemm(st, true, false, nu, T, nx, 1.0, p.SK, nx, p.X0, nx, 0.0, SX, nu);
  }
  k_lin<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, (int)nu, (int)T, D, SX, h);
  CMPC_LAUNCHED();
  k_h0<<<1, 1024, 0, st>>>(nx * (T + 1), p.X0, QX, h0_dev);
  CMPC_LAUNCHED();
  double *KX = nullptr, *EX = nullptr;
  if (p.has_K) {
    KX = dev_alloc<double>(size_t(nu * (T + 1)), st);
    gemm(st, false, false, nu, T + 1, nx, 1.0, p.K, nu, p.X0, nx, 0.0, KX, nu);
  } else {
    KX = dev_zeros<double>(size_t(nu * (T + 1)), st);
  }
  if (nc > 0) {
    EX = dev_alloc<double>(size_t(nc * (T + 1)), st);
    gemm(st, false, false, nc, T + 1, nx, 1.0, p.EFK, nc, p.X0, nx, 0.0, EX, nc);
  }
  if (p.m > 0) {
    k_rows_d<<<(unsigned)ceil_div(p.m, 256), 256, 0, st>>>(p.m, p.rows, p.bound, p.X0, KX, EX, (int)nx,
                                                           (int)nu, (int)nc, d);
    CMPC_LAUNCHED();
  }
  for (void* q : {(void*)QX, (void*)D, (void*)SX, (void*)KX, (void*)EX}) dev_free(q, st);
}

}  // namespace

void prob_build(Ctx& c, const cmpc_lq_problem& in, double** H_out, double** h_out, double* h0_out,
                double** J_out, double** d_out, int64_t* m_out) {
  prob_free(c);
  auto* pp = new ProblemDev;
  c.prob = pp;
  ProblemDev& p = *pp;
  const int64_t nx = in.nx, nu = in.nu, nc = in.nc, T = in.T;
  if (nx < 1 || nu < 1 || nc < 0 || T < 1) throw DimError("build_dense_qp: bad dimensions");
  p.nx = nx;
  p.nu = nu;
  p.nc = nc;
  p.T = T;
  p.n = T * nu;
  const int64_t n = p.n;
  cudaStream_t st = c.stream;
  auto up = [&](const double* src, int64_t count) {
    double* dst = dev_alloc<double>(size_t(std::max<int64_t>(count, 1)), st);
    if (count > 0) CMPC_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyHostToDevice, st));
    return dst;
  };
  auto any_nz = [](const double* a, int64_t k) {
    for (int64_t i = 0; i < k; ++i)
      if (a[i] != 0.0) return true;
    return false;
  };
  p.has_K = in.K && any_nz(in.K, nu * nx);
  p.has_S = in.S && any_nz(in.S, nx * nu);
  double* A = up(in.A, nx * nx);
  double* B = up(in.B, nx * nu);
  p.Q = up(in.Q, nx * nx);
  p.Qf = up(in.Qf, nx * nx);
  p.R = up(in.R, nu * nu);
  p.S = p.has_S ? up(in.S, nx * nu) : dev_zeros<double>(size_t(nx * nu), st);
  p.K = p.has_K ? up(in.K, nu * nx) : dev_zeros<double>(size_t(nu * nx), st);
  p.F = up(in.F, nc * nu);
  p.W = dev_zeros<double>(size_t(nx * T), st);
  if (in.w) CMPC_CUDA(cudaMemcpyAsync(p.W, in.w, sizeof(double) * nx * T, cudaMemcpyHostToDevice, st));
  // A_K = A + B K; S_K = S + K' R; Q_K = Q + S K + (S K)' + K' R K
  p.AK = A;
  p.SK = dev_alloc<double>(size_t(nx * nu), st);
  CMPC_CUDA(cudaMemcpyAsync(p.SK, p.S, sizeof(double) * nx * nu, cudaMemcpyDeviceToDevice, st));
  p.QK = dev_alloc<double>(size_t(nx * nx), st);
  CMPC_CUDA(cudaMemcpyAsync(p.QK, p.Q, sizeof(double) * nx * nx, cudaMemcpyDeviceToDevice, st));
  if (p.has_K) {
    gemm(st, false, false, nx, nx, nu, 1.0, B, nx, p.K, nu, 1.0, p.AK, nx);
    gemm(st, true, false, nx, nu, nu, 1.0, p.K, nu, p.R, nu, 1.0, p.SK, nx);
    double* RK = dev_alloc<double>(size_t(nu * nx), st);
    gemm(st, false, false, nu, nx, nu, 1.0, p.R, nu, p.K, nu, 0.0, RK, nu);
    gemm(st, true, false, nx, nx, nu, 1.0, p.K, nu, RK, nu, 1.0, p.QK, nx);      // K' R K
    gemm(st, false, false, nx, nx, nu, 1.0, p.S, nx, p.K, nu, 1.0, p.QK, nx);    // S K
    gemm(st, true, true, nx, nx, nu, 1.0, p.K, nu, p.S, nx, 1.0, p.QK, nx);      // (S K)'
    dev_free(RK, st);
  }
  // Gall = [G_0 .. G_{T-1}], G_0 = B, G_k = A_K G_{k-1}
  p.G = dev_alloc<double>(size_t(nx * n), st);
  CMPC_CUDA(cudaMemcpyAsync(p.G, B, sizeof(double) * nx * nu, cudaMemcpyDeviceToDevice, st));
  for (int64_t k = 1; k < T; ++k)
    gemm(st, false, false, nx, nu, nx, 1.0, p.AK, nx, p.G + (k - 1) * nu * nx, nx, 0.0, p.G + k * nu * nx, nx);
  dev_free(B, st);
  // Hessian
  double* QG = dev_alloc<double>(size_t(nx * n), st);
  double* Cm = dev_alloc<double>(size_t(n * n), st);
  double* Cf = dev_alloc<double>(size_t(n * n), st);
  gemm(st, false, false, nx, n, nx, 1.0, p.QK, nx, p.G, nx, 0.0, QG, nx);
  gemm(st, true, false, n, n, nx, 1.0, p.G, nx, QG, nx, 0.0, Cm, n);
  gemm(st, false, false, nx, n, nx, 1.0, p.Qf, nx, p.G, nx, 0.0, QG, nx);
  gemm(st, true, false, n, n, nx, 1.0, p.G, nx, QG, nx, 0.0, Cf, n);
  double* CS = nullptr;
  if (p.has_S || p.has_K) {
    CS = dev_alloc<double>(size_t(n * nu), st);
    gemm(st, true, false, n, nu, nx, 1.0, p.G, nx, p.SK, nx, 0.0, CS, n);
  }
  double* H = dev_alloc<double>(size_t(n * n), st);
  k_hess<<<(unsigned)ceil_div(n * n, 256), 256, 0, st>>>(n, (int)nu, (int)T, Cm, Cf, p.R, CS, H);
  CMPC_LAUNCHED();
  for (void* q : {(void*)QG, (void*)Cm, (void*)Cf, (void*)CS}) dev_free(q, st);
  // rows of J in the reference's order, one per finite bound
  std::vector<RowDesc> rows;
  std::vector<double> bnd;
  auto fin = [](const double* b, int64_t i) { return b && std::isfinite(b[i]); };
  for (int upper = 1; upper >= 0; --upper) {
    const double* b = upper ? in.gu : in.gl;
    for (int64_t t = 0; t < (nc > 0 ? T : 0); ++t)
      for (int64_t i = 0; i < nc; ++i)
        if (fin(b, i)) {
          rows.push_back({0, upper, (int)t, (int)i});
          bnd.push_back(b[i]);
        }
  }
  for (int upper = 1; upper >= 0; --upper) {
    const double* b = upper ? in.xu : in.xl;
    for (int64_t t = 1; t <= T; ++t)
      for (int64_t i = 0; i < nx; ++i)
        if (fin(b, i)) {
          rows.push_back({1, upper, (int)t, (int)i});
          bnd.push_back(b[i]);
        }
  }
  for (int upper = 1; upper >= 0; --upper) {
    const double* b = upper ? in.uu : in.ul;
    for (int64_t t = 0; t < T; ++t)
      for (int64_t i = 0; i < nu; ++i)
        if (fin(b, i)) {
          rows.push_back({2, upper, (int)t, (int)i});
          bnd.push_back(b[i]);
        }
  }
  const int64_t m = (int64_t)rows.size();
  p.m = m;
  p.rows = dev_alloc<RowDesc>(size_t(std::max<int64_t>(m, 1)), st);
  p.bound = dev_alloc<double>(size_t(std::max<int64_t>(m, 1)), st);
  if (m > 0) {
    CMPC_CUDA(cudaMemcpyAsync(p.rows, rows.data(), sizeof(RowDesc) * m, cudaMemcpyHostToDevice, st));
    CMPC_CUDA(cudaMemcpyAsync(p.bound, bnd.data(), sizeof(double) * m, cudaMemcpyHostToDevice, st));
  }
  double *KG = nullptr, *EG = nullptr;
  if (p.has_K) {
    KG = dev_alloc<double>(size_t(nu * n), st);
    gemm(st, false, false, nu, n, nx, 1.0, p.K, nu, p.G, nx, 0.0, KG, nu);
  }
  if (nc > 0) {  // E + F K
    p.EFK = up(in.E, nc * nx);
    if (p.has_K) gemm(st, false, false, nc, nx, nu, 1.0, p.F, nc, p.K, nu, 1.0, p.EFK, nc);
    EG = dev_alloc<double>(size_t(nc * n), st);
    gemm(st, false, false, nc, n, nx, 1.0, p.EFK, nc, p.G, nx, 0.0, EG, nc);
  }
  double* J = dev_alloc<double>(size_t(std::max<int64_t>(m * n, 1)), st);
  if (m > 0) {
    k_rows_J<<<4096, 256, 0, st>>>(m, n, p.rows, p.G, KG, EG, p.F, (int)nx, (int)nu, (int)nc, J);
    CMPC_LAUNCHED();
  }
  dev_free(KG, st);
  dev_free(EG, st);
  // affine terms from the free response
  p.X0 = dev_alloc<double>(size_t(nx * (T + 1)), st);
  CMPC_CUDA(cudaMemcpyAsync(p.X0, in.x_bar, sizeof(double) * nx, cudaMemcpyHostToDevice, st));
  free_response(c, p);
  double* h = dev_alloc<double>(size_t(n), st);
  double* d = dev_alloc<double>(size_t(std::max<int64_t>(m, 1)), st);
  double* h0d = dev_alloc<double>(1, st);
  affine(c, p, h, h0d, d);
  CMPC_CUDA(cudaMemcpyAsync(h0_out, h0d, sizeof(double), cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaStreamSynchronize(st));
  dev_free(h0d, st);
  *H_out = H;
  *h_out = h;
  *J_out = J;
  *d_out = d;
  *m_out = m;
}

void prob_refresh(Ctx& c, const double* x_bar) {
  auto* p = static_cast<ProblemDev*>(c.prob);
  if (!p) throw DimError("refresh_initial_state: the QP was not built from problem data on this context");
  CMPC_CUDA(cudaMemcpyAsync(p->X0, x_bar, sizeof(double) * p->nx, cudaMemcpyHostToDevice, c.stream));
  free_response(c, *p);
  double* h0d = dev_alloc<double>(1, c.stream);
  affine(c, *p, c.h, h0d, c.d);
  CMPC_CUDA(cudaMemcpyAsync(&c.h0, h0d, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  CMPC_CUDA(cudaStreamSynchronize(c.stream));
  dev_free(h0d, c.stream);
}

void prob_recover(Ctx& c, const double* v_dev, double* x_out, double* u_out, double* obj_out) {
  auto* p = static_cast<ProblemDev*>(c.prob);
  if (!p) throw DimError("recover_trajectory: the QP was not built from problem data on this context");
  const int64_t nx = p->nx, nu = p->nu, T = p->T;
  cudaStream_t st = c.stream;
  double* X = dev_alloc<double>(size_t(nx * (T + 1)), st);
  k_traj<<<(unsigned)ceil_div(nx * (T + 1), 256), 256, 0, st>>>((int)nx, (int)nu, (int)T, p->X0, p->G, v_dev, X);
  CMPC_LAUNCHED();
  // u_t = K x_t + v_t (U: n_u x T)
  double* U = dev_alloc<double>(size_t(nu * T), st);
  CMPC_CUDA(cudaMemcpyAsync(U, v_dev, sizeof(double) * nu * T, cudaMemcpyDeviceToDevice, st));
  if (p->has_K) gemm(st, false, false, nu, T, nx, 1.0, p->K, nu, X, nx, 1.0, U, nu);
  // objective (reduction.cpp:300-313): sum_t x'Qx + 2 x'S u + u'R u, x_T' Qf x_T
  double* QX = dev_alloc<double>(size_t(nx * (T + 1)), st);
  gemm(st, false, false, nx, T, nx, 1.0, p->Q, nx, X, nx, 0.0, QX, nx);
  gemm(st, false, false, nx, 1, nx, 1.0, p->Qf, nx, X + T * nx, nx, 0.0, QX + T * nx, nx);
  double* SU = dev_zeros<double>(size_t(nx * T), st);
  if (p->has_S) gemm(st, false, false, nx, T, nu, 1.0, p->S, nx, U, nu, 0.0, SU, nx);
  double* RU = dev_alloc<double>(size_t(nu * T), st);
  gemm(st, false, false, nu, T, nu, 1.0, p->R, nu, U, nu, 0.0, RU, nu);
  double* od = dev_alloc<double>(1, st);
  k_traj_obj<<<1, 1024, 0, st>>>((int)nx, (int)nu, (int)T, X, QX, U, SU, RU, od);
  CMPC_LAUNCHED();
  if (x_out) CMPC_CUDA(cudaMemcpyAsync(x_out, X, sizeof(double) * nx * (T + 1), cudaMemcpyDeviceToHost, st));
  if (u_out) CMPC_CUDA(cudaMemcpyAsync(u_out, U, sizeof(double) * nu * T, cudaMemcpyDeviceToHost, st));
  if (obj_out) CMPC_CUDA(cudaMemcpyAsync(obj_out, od, sizeof(double), cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaStreamSynchronize(st));
  for (void* q : {(void*)X, (void*)U, (void*)QX, (void*)SU, (void*)RU, (void*)od}) dev_free(q, st);
}

}  // namespace cmpc
