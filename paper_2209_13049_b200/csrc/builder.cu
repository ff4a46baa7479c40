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
//   J, d: one row per finite bound in the reference's row order, from Gall (state rows),
//         K Gall (input rows) and (E + F K) Gall (mixed rows). J is never stored (SURVEY
//         §8(f) row 2): the structure analysis reads it row by row (jrows.cuh, BuiltJ) and
//         keeps only the distinct rows P.
// The built H, h, h0, d are then loaded like a host QP (structure analysis, plan); Gall, x0 and
// the row table stay resident for refresh_initial_state and recover_trajectory, so a
// receding-horizon step uploads n_x numbers and never re-analyses J.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "internal.cuh"
#include "jrows.cuh"

namespace cmpc {

namespace {

// ---------------------------------------------------------------- plain tiled DGEMM
// C(M x N) = alpha op(A) op(B) + beta C, column-major; 64 x 64 tiles, 256 threads, 4 x 4
// outputs per thread. Setup-time GEMMs only (the solve's products are the tuned kernels).
constexpr int kGK = 16;
// 256 threads as 16 x 16, each RU x RV outputs: tile (16 RU) x (16 RV); <4,4> for square
// products, <16,1> for skinny ones (N <= 16). blockIdx.z = split of K (kc columns each); a
// split's raw product goes to C + z * zs.
template <int RU, int RV>
__global__ void __launch_bounds__(256) k_gemm(int M, int N, int K, int kc, double alpha,
                                              const double* __restrict__ A, int64_t lda, int ta,
                                              const double* __restrict__ B, int64_t ldb, int tb, double beta,
                                              double* __restrict__ C, int64_t ldc, int64_t zs) {
  constexpr int TM = 16 * RU, TN = 16 * RV;
  __shared__ double As[kGK][TM + 1], Bs[kGK][TN + 1];
  const int tid = threadIdx.x, tr = tid & 15, tc = tid >> 4;
  const int i0 = blockIdx.x * TM, j0 = blockIdx.y * TN;
  const int kb = blockIdx.z * kc, ke = min(K, kb + kc);
  C += blockIdx.z * zs;
  double acc[RU][RV] = {};
  for (int k0 = kb; k0 < ke; k0 += kGK) {
    for (int e = tid; e < kGK * TM; e += 256) {
      const int kk = e / TM, ii = e % TM;  // consecutive threads: consecutive rows
      const int gi = i0 + ii, gk = k0 + kk;
      double av = 0.0;
      if (gi < M && gk < ke) av = ta ? A[gk + (int64_t)gi * lda] : A[gi + (int64_t)gk * lda];
      As[kk][ii] = av;
    }
    for (int e = tid; e < kGK * TN; e += 256) {
      const int kk = e / TN, jj = e % TN;
      const int gj = j0 + jj, gk = k0 + kk;
      double bv = 0.0;
      if (gj < N && gk < ke) bv = tb ? B[gj + (int64_t)gk * ldb] : B[gk + (int64_t)gj * ldb];
      Bs[kk][jj] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      double a[RU], b[RV];
#pragma unroll
      for (int u = 0; u < RU; ++u) a[u] = As[kk][tr + 16 * u];
#pragma unroll
      for (int v = 0; v < RV; ++v) b[v] = Bs[kk][tc + 16 * v];
#pragma unroll
      for (int u = 0; u < RU; ++u)
#pragma unroll
        for (int v = 0; v < RV; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < RU; ++u)
#pragma unroll
    for (int v = 0; v < RV; ++v) {
      const int gi = i0 + tr + 16 * u, gj = j0 + tc + 16 * v;
      if (gi < M && gj < N) {
        double* p = C + gi + (int64_t)gj * ldc;
        *p = alpha * acc[u][v] + (beta == 0.0 ? 0.0 : beta * *p);
      }
    }
}

// C = alpha sum_z W[z] + beta C, splits summed in order (deterministic)
__global__ void k_gemm_splits(int M, int N, int S, const double* __restrict__ W, double alpha, double beta,
                              double* __restrict__ C, int64_t ldc) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t MN = (int64_t)M * N;
  if (e >= MN) return;
  double s = 0.0;
  for (int z = 0; z < S; ++z) s += W[z * MN + e];
  double* p = C + e % M + (e / M) * ldc;
  *p = alpha * s + (beta == 0.0 ? 0.0 : beta * *p);
}

// Y = A X for a skinny X (N <= NC columns, A not transposed): a thread owns one row of A and
// streams its K-chunk (eight loads in flight), the chunk of X staged in shared memory and read
// as broadcasts. blockIdx.y = split of K; the split's partial goes to W + y * M * N.
constexpr int kSkRows = 128, kSkK = 128;
template <int NC>
__global__ void __launch_bounds__(kSkRows) k_skinny(int M, int N, int K, const double* __restrict__ A, int64_t lda,
                                                    const double* __restrict__ X, int64_t ldx, int tb,
                                                    double* __restrict__ W) {
  __shared__ __align__(16) double Xs[kSkK][NC];
  const int kb = blockIdx.y * kSkK, ke = min(K, kb + kSkK);
  for (int e = threadIdx.x; e < kSkK * NC; e += kSkRows) {
    const int kk = e / NC, j = e % NC, gk = kb + kk;
    Xs[kk][j] = (gk < ke && j < N) ? (tb ? X[j + (int64_t)gk * ldx] : X[gk + (int64_t)j * ldx]) : 0.0;
  }
  __syncthreads();
  const int i = blockIdx.x * kSkRows + threadIdx.x;
  if (i >= M) return;
  double acc[NC] = {};
  const double* a = A + i;
  int k = kb;
  for (; k + 8 <= ke; k += 8) {
    double av[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) av[u] = __ldg(a + (int64_t)(k + u) * lda);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[j] = fma(av[u], Xs[k - kb + u][j], acc[j]);
  }
  for (; k < ke; ++k) {
    const double av = __ldg(a + (int64_t)k * lda);
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = fma(av, Xs[k - kb][j], acc[j]);
  }
  W += (int64_t)blockIdx.y * M * N;
#pragma unroll
  for (int j = 0; j < NC; ++j)
    if (j < N) W[i + (int64_t)j * M] = acc[j];
}

// Setup products. Skinny ones (G_k = A_K G_{k-1}: 2500 x 10 x 2500; the free response's
// 2500 x 1 x 2500) go to k_skinny; the rest to the tiled kernel, K split until about four CTAs
// per SM are busy. Splits are summed in a fixed order.
void gemm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
          int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  if (!ta && N <= 16 && K >= kSkK) {
    const int64_t S = ceil_div(K, kSkK);
    double* W = dev_alloc<double>(size_t(S * M * N), st);
    dim3 g((unsigned)ceil_div(M, kSkRows), (unsigned)S);
    if (N == 1)
      k_skinny<1><<<g, kSkRows, 0, st>>>((int)M, (int)N, (int)K, A, lda, B, ldb, tb ? 1 : 0, W);
    else
      k_skinny<16><<<g, kSkRows, 0, st>>>((int)M, (int)N, (int)K, A, lda, B, ldb, tb ? 1 : 0, W);
    CMPC_LAUNCHED();
    k_gemm_splits<<<(unsigned)ceil_div(M * N, 256), 256, 0, st>>>((int)M, (int)N, (int)S, W, alpha, beta, C, ldc);
    CMPC_LAUNCHED();
    dev_free(W, st);
    return;
  }
  const int64_t tiles = ceil_div(M, 64) * ceil_div(N, 64);
  int64_t S = std::min<int64_t>(std::max<int64_t>(1, ceil_div(592, tiles)), std::max<int64_t>(1, K / 128));
  const int64_t kc = ceil_div(ceil_div(std::max<int64_t>(K, 1), S), kGK) * kGK;
  S = std::max<int64_t>(1, ceil_div(K, kc));
  dim3 g((unsigned)ceil_div(M, 64), (unsigned)ceil_div(N, 64), (unsigned)S);
  if (S == 1) {
    k_gemm<4, 4><<<g, 256, 0, st>>>((int)M, (int)N, (int)K, (int)std::max<int64_t>(K, 1), alpha, A, lda, ta ? 1 : 0,
                                    B, ldb, tb ? 1 : 0, beta, C, ldc, 0);
    CMPC_LAUNCHED();
    return;
  }
  double* W = dev_alloc<double>(size_t(S * M * N), st);
  k_gemm<4, 4><<<g, 256, 0, st>>>((int)M, (int)N, (int)K, (int)kc, 1.0, A, lda, ta ? 1 : 0, B, ldb, tb ? 1 : 0, 0.0,
                                  W, M, M * N);
  CMPC_LAUNCHED();
  k_gemm_splits<<<(unsigned)ceil_div(M * N, 256), 256, 0, st>>>((int)M, (int)N, (int)S, W, alpha, beta, C, ldc);
  CMPC_LAUNCHED();
  dev_free(W, st);
}

// dst (r x c, column-major) from src holding it row-major (= the c x r column-major transpose)
__global__ void k_transpose(int64_t r, int64_t c, const double* __restrict__ src, double* __restrict__ dst) {
  __shared__ double t[32][33];
  const int64_t i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {  // read rows i of src along j (contiguous)
    const int64_t i = i0 + y, j = j0 + threadIdx.x;
    if (i < r && j < c) t[y][threadIdx.x] = src[i * c + j];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {  // write columns j of dst along i (contiguous)
    const int64_t j = j0 + y, i = i0 + threadIdx.x;
    if (i < r && j < c) dst[i + j * r] = t[threadIdx.x][y];
  }
}


// the six (kind, side) groups of rows in the reference's order: group g holds rows
// first .. first + nt * len - 1, stage t0 + r / len, index list[r % len]
struct RowGroup {
  int kind, upper, t0, list, len;
  int64_t first;
};
struct RowGroups {
  RowGroup g[6];
  int count;
  int64_t m;
};

__global__ void k_row_table(RowGroups gr, const int32_t* __restrict__ idx, const double* __restrict__ bvals,
                            RowDesc* __restrict__ rows, double* __restrict__ bound) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= gr.m) return;
  int k = 0;
  while (k + 1 < gr.count && r >= gr.g[k + 1].first) ++k;
  const RowGroup g = gr.g[k];
  const int64_t loc = r - g.first;
  const int64_t tt = loc / g.len;
  const int j = (int)(loc - tt * g.len);
  rows[r] = RowDesc{g.kind, g.upper, g.t0 + (int)tt, idx[g.list + j]};
  bound[r] = bvals[g.list + j];
}

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
  double *KG = nullptr, *EG = nullptr;  // K Gall, (E + F K) Gall: the input and mixed rows
  BuiltJ J{};                           // J, row by row, for the structure analysis
};

void prob_free(Ctx& c) {
  auto* p = static_cast<ProblemDev*>(c.prob);
  if (!p) return;
  for (void* q : {(void*)p->AK, (void*)p->G, (void*)p->QK, (void*)p->Qf, (void*)p->R, (void*)p->SK,
                  (void*)p->S, (void*)p->K, (void*)p->EFK, (void*)p->F, (void*)p->W, (void*)p->X0,
                  (void*)p->bound, (void*)p->Q, (void*)p->rows, (void*)p->KG, (void*)p->EG})
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
  const bool verbose = getenv("CMPC_VERBOSE") != nullptr;
  auto wall = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double last = wall();
  auto tick = [&](const char* what) {
    if (!verbose) return;
    CMPC_CUDA(cudaStreamSynchronize(st));
    const double now = wall();
    fprintf(stderr, "[cmpc build] %-10s %8.2f ms\n", what, (now - last) * 1e3);
    last = now;
  };
  auto up = [&](const double* src, int64_t count) {
    double* dst = dev_alloc<double>(size_t(std::max<int64_t>(count, 1)), st);
    if (count > 0) upload_h2d(dst, src, sizeof(double) * count, st);
    return dst;
  };
  // a matrix argument: column-major as given, or row-major (layout 1) transposed on the device
  auto upm = [&](const double* src, int64_t r, int64_t cc) {
    if (!in.layout || r * cc == 0) return up(src, r * cc);
    double* tmp = up(src, r * cc);
    double* dst = dev_alloc<double>(size_t(r * cc), st);
    k_transpose<<<dim3((unsigned)ceil_div(cc, 32), (unsigned)ceil_div(r, 32)), dim3(32, 8), 0, st>>>(r, cc, tmp, dst);
    CMPC_LAUNCHED();
    dev_free(tmp, st);
    return dst;
  };
  auto any_nz = [](const double* a, int64_t k) {
    for (int64_t i = 0; i < k; ++i)
      if (a[i] != 0.0) return true;
    return false;
  };
  p.has_K = in.K && any_nz(in.K, nu * nx);
  p.has_S = in.S && any_nz(in.S, nx * nu);
  double* A = upm(in.A, nx, nx);
  double* B = upm(in.B, nx, nu);
  p.Q = upm(in.Q, nx, nx);
  p.Qf = upm(in.Qf, nx, nx);
  p.R = upm(in.R, nu, nu);
  p.S = p.has_S ? upm(in.S, nx, nu) : dev_zeros<double>(size_t(nx * nu), st);
  p.K = p.has_K ? upm(in.K, nu, nx) : dev_zeros<double>(size_t(nu * nx), st);
  p.F = upm(in.F, nc, nu);
  p.W = dev_zeros<double>(size_t(nx * T), st);
  if (in.w) CMPC_CUDA(cudaMemcpyAsync(p.W, in.w, sizeof(double) * nx * T, cudaMemcpyHostToDevice, st));
  tick("h2d");
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
  tick("G");
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
  tick("H");
  // rows of J in the reference's order, one per finite bound. A bound vector is the same at
  // every stage, so each (kind, side) group is T copies of its list of finite indices: the
  // lists go to the device and k_row_table expands them.
  RowGroups gr{};
  std::vector<int32_t> idx;
  std::vector<double> bvals;
  int64_t m = 0;
  auto group = [&](int kind, int upper, int t0, int64_t nt, const double* b, int64_t len) {
    RowGroup& g = gr.g[gr.count++];
    g.kind = kind;
    g.upper = upper;
    g.t0 = t0;
    g.list = (int)idx.size();
    for (int64_t i = 0; i < len; ++i)
      if (b && std::isfinite(b[i])) {
        idx.push_back((int32_t)i);
        bvals.push_back(b[i]);
      }
    g.len = (int)idx.size() - g.list;
    g.first = m;
    m += (g.len > 0 ? nt : 0) * g.len;
  };
  for (int upper = 1; upper >= 0; --upper) group(0, upper, 0, nc > 0 ? T : 0, upper ? in.gu : in.gl, nc);
  for (int upper = 1; upper >= 0; --upper) group(1, upper, 1, T, upper ? in.xu : in.xl, nx);
  for (int upper = 1; upper >= 0; --upper) group(2, upper, 0, T, upper ? in.uu : in.ul, nu);
  gr.m = m;
  p.m = m;
  p.rows = dev_alloc<RowDesc>(size_t(std::max<int64_t>(m, 1)), st);
  p.bound = dev_alloc<double>(size_t(std::max<int64_t>(m, 1)), st);
  if (m > 0) {
    int32_t* di = dev_alloc<int32_t>(idx.size(), st);
    double* db = dev_alloc<double>(bvals.size(), st);
    CMPC_CUDA(cudaMemcpyAsync(di, idx.data(), sizeof(int32_t) * idx.size(), cudaMemcpyHostToDevice, st));
    CMPC_CUDA(cudaMemcpyAsync(db, bvals.data(), sizeof(double) * bvals.size(), cudaMemcpyHostToDevice, st));
    k_row_table<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(gr, di, db, p.rows, p.bound);
    CMPC_LAUNCHED();
    dev_free(di, st);
    dev_free(db, st);
  }
  tick("rows");
  double *KG = nullptr, *EG = nullptr;
  if (p.has_K) {
    KG = dev_alloc<double>(size_t(nu * n), st);
    gemm(st, false, false, nu, n, nx, 1.0, p.K, nu, p.G, nx, 0.0, KG, nu);
  }
  if (nc > 0) {  // E + F K
    p.EFK = upm(in.E, nc, nx);
    if (p.has_K) gemm(st, false, false, nc, nx, nu, 1.0, p.F, nc, p.K, nu, 1.0, p.EFK, nc);
    EG = dev_alloc<double>(size_t(nc * n), st);
    gemm(st, false, false, nc, n, nx, 1.0, p.EFK, nc, p.G, nx, 0.0, EG, nc);
  }
  // J itself is never stored: the structure analysis reads it row by row through BuiltJ
  p.KG = KG;
  p.EG = EG;
  p.J = BuiltJ{p.rows, p.G, KG, EG, p.F, (int)nx, (int)nu, (int)nc};
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
  tick("affine");
  dev_free(h0d, st);
  *H_out = H;
  *h_out = h;
  *J_out = nullptr;
  *d_out = d;
  *m_out = m;
}

const BuiltJ* prob_rows(Ctx& c) {
  auto* p = static_cast<ProblemDev*>(c.prob);
  return p ? &p->J : nullptr;
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
