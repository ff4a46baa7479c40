// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle_core.hpp header).
// Each function cites the reference file:line it restates.
#include "oracle_core.hpp"

#include <algorithm>
#include <array>
#include <bit>
#include <chrono>
#include <complex>
#include <optional>
#include <sstream>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

namespace {
int g_threads = 1;
bool g_skip_zeros = false;
// Structural-zero map of the J being solved (set_skip_zeros mode, test speed only): one bit
// per (column, 512-row chunk) saying whether the chunk holds a nonzero of that column. A
// skipped chunk contributes only products with an exact zero factor (+-0), so every sum keeps
// its value and its order: results are bitwise those of the dense loops (finite data).
struct ZeroMap {
  const double* data = nullptr;
  Index m = 0, n = 0, nchunk = 0;
  std::vector<unsigned char> nz;  // [j * nchunk + c]
  bool has(Index j, Index c) const { return nz[size_t(j * nchunk + c)] != 0; }
};
constexpr Index kZChunk = 512;
const ZeroMap* g_zmap = nullptr;
const ZeroMap* zmap_for(const Mat& A) {
  return (g_zmap && A.r == g_zmap->m && A.c == g_zmap->n && A.a.data() == g_zmap->data) ? g_zmap : nullptr;
}
ZeroMap make_zmap(const Mat& J) {
  ZeroMap z;
  z.data = J.a.data();
  z.m = J.r;
  z.n = J.c;
  z.nchunk = (J.r + kZChunk - 1) / kZChunk;
  z.nz.assign(size_t(z.n * z.nchunk), 0);
#pragma omp parallel for schedule(static) num_threads(g_threads)
  for (Index j = 0; j < J.c; ++j) {
    const double* c = J.col(j);
    for (Index k = 0; k < z.nchunk; ++k) {
      const Index i1 = std::min(J.r, (k + 1) * kZChunk);
      for (Index i = k * kZChunk; i < i1; ++i)
        if (c[i] != 0.0) {
          z.nz[size_t(j * z.nchunk + k)] = 1;
          break;
        }
    }
  }
  return z;
}
double now_seconds() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

void set_threads(int n) { g_threads = std::max(1, n); }
void set_skip_zeros(bool on) { g_skip_zeros = on; }
bool get_skip_zeros() { return g_skip_zeros; }
int get_threads() { return g_threads; }

// ------------------------------------------------------------------ helpers
double inf_norm(const Vec& v) {  // types.hpp:21
  double m = 0.0;
  for (double x : v) m = std::max(m, std::abs(x));
  return m;
}
double max_abs(const Mat& m) {  // types.hpp:23
  double r = 0.0;
  for (double x : m.a) r = std::max(r, std::abs(x));
  return r;
}

Vec gemv(const Mat& A, const Vec& x) {
  const Index m = A.r, n = A.c;
  Vec y(size_t(m), 0.0);
  const Index chunk = 4096;
  const Index nchunks = (m + chunk - 1) / chunk;
  const ZeroMap* z = zmap_for(A);
#pragma omp parallel for schedule(static) num_threads(g_threads) if (m * n > 200000)
  for (Index b = 0; b < nchunks; ++b) {
    const Index i0 = b * chunk, i1 = std::min(m, i0 + chunk);
    for (Index j = 0; j < n; ++j) {
      const double xj = x[size_t(j)];
      const double* c = A.col(j);
      if (z) {  // the same per-element order over j, zero chunks left out
        for (Index k0 = i0; k0 < i1; k0 += kZChunk) {
          if (!z->has(j, k0 / kZChunk)) continue;
          const Index k1 = std::min(i1, k0 + kZChunk);
          for (Index i = k0; i < k1; ++i) y[size_t(i)] += c[i] * xj;
        }
        continue;
      }
      for (Index i = i0; i < i1; ++i) y[size_t(i)] += c[i] * xj;
    }
  }
  return y;
}

Vec gemv_t(const Mat& A, const Vec& x) {
  const Index m = A.r, n = A.c;
  Vec y(size_t(n), 0.0);
  const ZeroMap* z = zmap_for(A);
#pragma omp parallel for schedule(static) num_threads(g_threads) if (m * n > 200000)
  for (Index j = 0; j < n; ++j) {
    const double* c = A.col(j);
    double s = 0.0;
    if (z) {
      for (Index k = 0; k < z->nchunk; ++k) {
        if (!z->has(j, k)) continue;
        const Index i1 = std::min(m, (k + 1) * kZChunk);
        for (Index i = k * kZChunk; i < i1; ++i) s += c[i] * x[size_t(i)];
      }
    } else {
      for (Index i = 0; i < m; ++i) s += c[i] * x[size_t(i)];
    }
    y[size_t(j)] = s;
  }
  return y;
}

double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
#pragma omp parallel for schedule(static) num_threads(g_threads) if (A.r * A.c * B.c > 1000000)
  for (Index j = 0; j < B.c; ++j) {
    double* cj = C.col(j);
    for (Index p = 0; p < A.c; ++p) {
      const double b = B(p, j);
      const double* ap = A.col(p);
      for (Index i = 0; i < A.r; ++i) cj[i] += ap[i] * b;
    }
  }
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (Index j = 0; j < A.c; ++j)
    for (Index i = 0; i < A.r; ++i) T(j, i) = A(i, j);
  return T;
}

// ------------------------------------------------------------------ dense_linalg
namespace {
[[noreturn]] void throw_not_pd(Index pivot) {
  std::ostringstream msg;
  msg << "cholesky failed: matrix not positive definite at pivot " << pivot;
  throw NotPositiveDefinite(pivot, msg.str());
}

// potf2_lower on the b x b block at (k0,k0) of a (dense_linalg.cpp:24-40)
void potf2_lower(Mat& a, Index k0, Index b, Index pivot_offset) {
  auto A = [&](Index i, Index j) -> double& { return a(k0 + i, k0 + j); };
  std::vector<double> tmp(static_cast<size_t>(b));
  for (Index j = 0; j < b; ++j) {
    double diag = A(j, j);
    if (j > 0) {
      double sq = 0.0;
      for (Index p = 0; p < j; ++p) sq += A(j, p) * A(j, p);
      diag -= sq;
    }
    if (!(diag > 0.0) || !std::isfinite(diag)) throw_not_pd(pivot_offset + j);
    diag = std::sqrt(diag);
    A(j, j) = diag;
    if (j + 1 < b) {
      if (j > 0) {
        for (Index i = j + 1; i < b; ++i) tmp[size_t(i)] = 0.0;
        for (Index p = 0; p < j; ++p) {
          const double ajp = A(j, p);
          for (Index i = j + 1; i < b; ++i) tmp[size_t(i)] += A(i, p) * ajp;
        }
        for (Index i = j + 1; i < b; ++i) A(i, j) -= tmp[size_t(i)];
      }
      for (Index i = j + 1; i < b; ++i) A(i, j) /= diag;
    }
  }
}

// X <- X L^{-T}; X = a[r0:r0+rows, k0:k0+b], L = a[k0:k0+b, k0:k0+b] (dense_linalg.cpp:43-51)
void trsm_right_lower_transposed(Mat& a, Index r0, Index rows, Index k0, Index b) {
#pragma omp parallel num_threads(g_threads) if (rows * b * b > 200000)
  {
    std::vector<double> tmp;
#pragma omp for schedule(static)
    for (Index ib = 0; ib < (rows + 255) / 256; ++ib) {
      const Index i0 = r0 + ib * 256, i1 = std::min(r0 + rows, i0 + 256);
      tmp.assign(size_t(i1 - i0), 0.0);
      for (Index j = 0; j < b; ++j) {
        if (j > 0) {
          std::fill(tmp.begin(), tmp.end(), 0.0);
          for (Index p = 0; p < j; ++p) {
            const double l = a(k0 + j, k0 + p);
            const double* xp = a.col(k0 + p);
            for (Index i = i0; i < i1; ++i) tmp[size_t(i - i0)] += xp[i] * l;
          }
          double* xj = a.col(k0 + j);
          for (Index i = i0; i < i1; ++i) xj[i] -= tmp[size_t(i - i0)];
        }
        const double d = a(k0 + j, k0 + j);
        double* xj = a.col(k0 + j);
        for (Index i = i0; i < i1; ++i) xj[i] /= d;
      }
    }
  }
}
}  // namespace

Mat factorize_reference(const Mat& sym) {  // dense_linalg.cpp:59-77
  const Index n = sym.r;
  Mat a = sym;
  constexpr Index block = 64;
  for (Index k = 0; k < n; k += block) {
    const Index b = std::min(block, n - k);
    potf2_lower(a, k, b, k);
    const Index rest = n - k - b;
    if (rest > 0) {
      trsm_right_lower_transposed(a, k + b, rest, k, b);
      // trailing lower rankUpdate(X, -1): a(i,j) -= sum_p X(i,p) X(j,p), i >= j
      const Index r0 = k + b;
#pragma omp parallel for schedule(dynamic, 4) num_threads(g_threads) if (rest * rest * b > 400000)
      for (Index j = r0; j < n; ++j) {
        double* cj = a.col(j);
        std::vector<double> tmp(size_t(n - j), 0.0);
        for (Index p = 0; p < b; ++p) {
          const double xjp = a(j, k + p);
          const double* xp = a.col(k + p);
          for (Index i = j; i < n; ++i) tmp[size_t(i - j)] += xp[i] * xjp;
        }
        for (Index i = j; i < n; ++i) cj[i] -= tmp[size_t(i - j)];
      }
    }
  }
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < j; ++i) a(i, j) = 0.0;
  return a;
}

Mat factorize_llt(const Mat& sym) {  // dense_linalg.cpp:86-97 (unblocked restatement)
  const Index n = sym.r;
  Mat a = sym;
  potf2_lower(a, 0, n, 0);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < j; ++i) a(i, j) = 0.0;
  return a;
}

Mat factorize(const std::string& backend, const Mat& sym) {  // make_backend :112-116
  if (backend == "reference") return factorize_reference(sym);
  if (backend == "eigen") return factorize_llt(sym);
  throw std::invalid_argument("unknown factorization backend: " + backend);
}

Vec factor_solve(const Mat& L, const Vec& rhs) {  // dense_linalg.cpp:102-110
  require(Index(rhs.size()) == L.r, "cholesky_solve: rhs length " + std::to_string(rhs.size()) +
                                        " does not match factor dimension " + std::to_string(L.r));
  const Index n = L.r;
  Vec x = rhs;
  for (Index i = 0; i < n; ++i) {
    double s = 0.0;
    for (Index j = 0; j < i; ++j) s += L(i, j) * x[size_t(j)];
    x[size_t(i)] = (x[size_t(i)] - s) / L(i, i);
  }
  for (Index i = n - 1; i >= 0; --i) {
    double s = 0.0;
    for (Index j = i + 1; j < n; ++j) s += L(j, i) * x[size_t(j)];
    x[size_t(i)] = (x[size_t(i)] - s) / L(i, i);
  }
  return x;
}

Mat gram_weighted(const Mat& J, const Vec& sigma) {  // dense_linalg.cpp:128-137
  require(J.r == Index(sigma.size()), "gram_weighted: sigma length must equal row count of J");
  const Index n = J.c, m = J.r;
  Mat g(n, n);
  if (m == 0) return g;
  Vec rs(static_cast<size_t>(m));
  for (Index i = 0; i < m; ++i) rs[size_t(i)] = std::sqrt(sigma[size_t(i)]);
  // W = diag(sqrt(sigma)) J, formed chunk by chunk (512 rows) in panels of 8 columns
  // (panel-major, then row, then column: a row of a panel is 8 contiguous doubles); lower
  // triangle of W'W by 4x8 entry blocks, each entry summed over the rows in ascending order
  // (separate multiply and add: the vector lanes compute exactly the scalar recurrence)
  const Index RB = kZChunk;
  constexpr Index PW = 8;
  const Index np = (n + PW - 1) / PW;
  const ZeroMap* z = zmap_for(J);
  std::vector<std::pair<Index, Index>> blocks;  // (4-row block of entries, panel of columns)
  for (Index pj = 0; pj < np; ++pj)
    for (Index bi = pj * 2; bi < (n + 3) / 4; ++bi) blocks.push_back({bi, pj});
  std::vector<double> W(static_cast<size_t>(RB * np * PW), 0.0);
  std::vector<unsigned char> live(static_cast<size_t>(np));
#ifdef __AVX2__
  typedef double v4 __attribute__((vector_size(32)));
#else
  typedef double v4 __attribute__((vector_size(16)));
#endif
  constexpr int VW = int(sizeof(v4) / sizeof(double)), NV = int(PW) / VW;
  for (Index i0 = 0; i0 < m; i0 += RB) {
    const Index rb = std::min(RB, m - i0);
    for (Index p = 0; p < np; ++p) {
      bool any = !z;
      for (Index c = p * PW; c < std::min(n, p * PW + PW) && !any; ++c) any = z->has(c, i0 / RB);
      live[size_t(p)] = any;
    }
#pragma omp parallel num_threads(g_threads) if (m * n * n > 2000000)
    {
#pragma omp for schedule(static)
      for (Index p = 0; p < np; ++p) {
        if (!live[size_t(p)]) continue;  // all-zero panel: its blocks are skipped below
        double* dst = W.data() + p * RB * PW;
        for (Index c = 0; c < PW; ++c) {
          const Index j = p * PW + c;
          if (j >= n || (z && !z->has(j, i0 / RB))) {
            for (Index i = 0; i < rb; ++i) dst[i * PW + c] = 0.0;
            continue;
          }
          const double* src = J.col(j) + i0;
          for (Index i = 0; i < rb; ++i) dst[i * PW + c] = rs[size_t(i0 + i)] * src[i];
        }
      }
#pragma omp for schedule(dynamic, 4)
      for (size_t b = 0; b < blocks.size(); ++b) {
        const Index bi = blocks[b].first, pj = blocks[b].second;
        const Index pa = bi / 2, ca = (bi % 2) * 4;  // the 4 rows' columns inside their panel
        if (!live[size_t(pa)] || !live[size_t(pj)]) continue;  // every product is an exact zero
        v4 acc[4][NV];
        for (int x = 0; x < 4; ++x)
          for (int y = 0; y < 8; ++y) {
            const Index l = bi * 4 + x, k = pj * PW + y;
            acc[x][y / VW][y % VW] = (l < n && k < n && l >= k) ? g(l, k) : 0.0;
          }
        const double* A = W.data() + pa * RB * PW + ca;
        const double* B = W.data() + pj * RB * PW;
        for (Index i = 0; i < rb; ++i) {
          v4 bv[NV];
          __builtin_memcpy(bv, B + i * PW, sizeof(bv));
          for (int x = 0; x < 4; ++x) {
            const double a = A[i * PW + x];
            for (int q = 0; q < NV; ++q) {
              const v4 t = bv[q] * a;
              acc[x][q] += t;
            }
          }
        }
        for (int x = 0; x < 4; ++x)
          for (int y = 0; y < 8; ++y) {
            const Index l = bi * 4 + x, k = pj * PW + y;
            if (l < n && k < n && l >= k) g(l, k) = acc[x][y / VW][y % VW];
          }
      }
    }
  }
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < j; ++i) g(i, j) = g(j, i);
  return g;
}

// ------------------------------------------------------------------ problem
LqProblemData LqProblemData::basic(Mat A, Mat B, Mat Q, Mat R, Mat Qf, Vec x_bar, Index T) {
  // problem.cpp:10-34
  const Index n_x = A.r, n_u = B.c;
  LqProblemData d;
  d.A = std::move(A);
  d.B = std::move(B);
  d.Q = std::move(Q);
  d.R = std::move(R);
  d.Qf = std::move(Qf);
  d.S = Mat(n_x, n_u);
  d.E = Mat(0, n_x);
  d.F = Mat(0, n_u);
  d.xl = Vec(size_t(n_x), -kInf);
  d.xu = Vec(size_t(n_x), kInf);
  d.ul = Vec(size_t(n_u), -kInf);
  d.uu = Vec(size_t(n_u), kInf);
  d.w.assign(size_t(T), Vec(size_t(n_x), 0.0));
  d.x_bar = std::move(x_bar);
  d.K = Mat(n_u, n_x);
  d.T = T;
  return d;
}

Dims dims(const LqProblemData& d) {  // problem.cpp:42-69
  const Index n_x = d.A.r, n_u = d.B.c, n_c = d.E.r, T = Index(d.w.size());
  auto bad = [](const std::string& m) { throw DimensionError("dimension mismatch: " + m); };
  if (d.A.c != n_x) bad("A is not square");
  if (d.B.r != n_x) bad("B rows do not match A");
  if (d.Q.r != n_x || d.Q.c != n_x) bad("Q does not match A");
  if (d.Qf.r != n_x || d.Qf.c != n_x) bad("Qf does not match A");
  if (d.R.r != n_u || d.R.c != n_u) bad("R does not match B");
  if (d.S.r != n_x || d.S.c != n_u) bad("S does not match A and B");
  if (n_c > 0 && d.E.c != n_x) bad("E cols do not match A");
  if (d.F.r != n_c || (n_c > 0 && d.F.c != n_u)) bad("F does not match E and B");
  if (Index(d.gl.size()) != n_c || Index(d.gu.size()) != n_c) bad("gl/gu do not match E");
  if (Index(d.xl.size()) != n_x || Index(d.xu.size()) != n_x) bad("xl/xu do not match A");
  if (Index(d.ul.size()) != n_u || Index(d.uu.size()) != n_u) bad("ul/uu do not match B");
  if (Index(d.x_bar.size()) != n_x) bad("x_bar does not match A");
  if (d.K.r != n_u || d.K.c != n_x) bad("K does not match B and A");
  if (d.T != T) bad("T field does not match w");
  if (T < 1) bad("horizon T must be positive");
  for (const auto& wt : d.w)
    if (Index(wt.size()) != n_x) bad("w entry does not match A");
  return Dims{n_x, n_u, n_c, T};
}

// ------------------------------------------------------------------ reduction
namespace {
Mat block(const Mat& M, Index r0, Index c0, Index rows, Index cols) {
  Mat b(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) b(i, j) = M(r0 + i, c0 + j);
  return b;
}
void set_block(Mat& M, Index r0, Index c0, const Mat& b) {
  for (Index j = 0; j < b.c; ++j)
    for (Index i = 0; i < b.r; ++i) M(r0 + i, c0 + j) = b(i, j);
}
Mat add(const Mat& a, const Mat& b) {
  Mat c = a;
  for (size_t i = 0; i < c.a.size(); ++i) c.a[i] += b.a[i];
  return c;
}

Vec stacked_free_response(const BlockMatrices& bl, const LqProblemData& data) {  // :10-18
  const Index n_x = bl.A_K.r, T = Index(data.w.size());
  Vec ws(static_cast<size_t>(T * n_x));
  for (Index t = 0; t < T; ++t)
    for (Index i = 0; i < n_x; ++i) ws[size_t(t * n_x + i)] = data.w[size_t(t)][size_t(i)];
  Vec x0 = gemv(bl.bigA, data.x_bar);
  Vec x1 = gemv(bl.bigAtilde, ws);
  for (size_t i = 0; i < x0.size(); ++i) x0[i] += x1[i];
  return x0;
}

struct SubstitutedCost {
  Mat Q_K, S_K;
};
SubstitutedCost substituted_cost(const LqProblemData& d) {  // :78-84
  SubstitutedCost c;
  Mat SK = matmul(d.S, d.K);
  c.Q_K = add(add(add(d.Q, SK), transpose(SK)), matmul(matmul(transpose(d.K), d.R), d.K));
  c.S_K = add(d.S, matmul(transpose(d.K), d.R));
  return c;
}

Mat assemble_hessian(const LqProblemData& data, const BlockMatrices& bl,
                     const SubstitutedCost& cost) {  // :88-117
  const Dims dm = dims(data);
  const Index n_x = dm.n_x, n_u = dm.n_u, T = dm.T;
  Mat H(T * n_u, T * n_u);
  for (Index t = 0; t < T; ++t) set_block(H, t * n_u, t * n_u, data.R);
  for (Index t = 1; t <= T; ++t) {
    const Mat& Qt = (t == T) ? data.Qf : cost.Q_K;
    const Index width = t * n_u;
    const Mat Bt = block(bl.bigB, t * n_x, 0, n_x, width);
    const Mat QtBt = matmul(Qt, Bt);
    const Mat P = matmul(transpose(Bt), QtBt);
    for (Index j = 0; j < width; ++j)
      for (Index i = 0; i < width; ++i) H(i, j) += P(i, j);
  }
  for (Index t = 1; t < T; ++t) {
    const Index width = t * n_u;
    const Mat Bt = block(bl.bigB, t * n_x, 0, n_x, width);
    const Mat cross = matmul(transpose(Bt), cost.S_K);
    for (Index j = 0; j < n_u; ++j)
      for (Index i = 0; i < width; ++i) {
        H(i, t * n_u + j) += cross(i, j);
        H(t * n_u + j, i) += cross(i, j);
      }
  }
  for (double& x : H.a) x *= 2.0;
  Mat Hs = H;
  for (Index j = 0; j < H.c; ++j)
    for (Index i = 0; i < H.r; ++i) Hs(i, j) = 0.5 * (H(i, j) + H(j, i));
  return Hs;
}

struct AffineParts {
  Vec h;
  double h0 = 0.0;
  Vec d;
};

AffineParts assemble_affine(const LqProblemData& data, const BlockMatrices& bl,
                            const SubstitutedCost& cost, const Vec& x0) {  // :119-180
  const Dims dm = dims(data);
  const Index n_x = dm.n_x, n_u = dm.n_u, n_c = dm.n_c, T = dm.T;
  AffineParts parts;
  parts.h.assign(size_t(T * n_u), 0.0);
  parts.h0 = 0.0;
  auto seg = [&](Index t) { return Vec(x0.begin() + t * n_x, x0.begin() + (t + 1) * n_x); };
  for (Index t = 0; t <= T; ++t) {
    const Mat& Qt = (t == T) ? data.Qf : cost.Q_K;
    const Vec x0t = seg(t);
    const Vec Qx = gemv(Qt, x0t);
    parts.h0 += dot(x0t, Qx);
    if (t > 0) {
      const Index width = std::min(t, T) * n_u;
      const Mat Bt = block(bl.bigB, t * n_x, 0, n_x, width);
      const Vec p = gemv_t(Bt, Qx);
      for (Index i = 0; i < width; ++i) parts.h[size_t(i)] += 2.0 * p[size_t(i)];
    }
    if (t < T) {
      const Vec p = gemv_t(cost.S_K, x0t);
      for (Index i = 0; i < n_u; ++i) parts.h[size_t(t * n_u + i)] += 2.0 * p[size_t(i)];
    }
  }
  std::vector<double> dv;
  Mat EFK = (n_c > 0) ? add(data.E, matmul(data.F, data.K)) : Mat(0, n_x);
  auto emit = [&](const Vec& bound, const Vec& off, bool upper) {
    for (size_t i = 0; i < bound.size(); ++i) {
      if (!std::isfinite(bound[i])) continue;
      dv.push_back(upper ? bound[i] - off[i] : off[i] - bound[i]);
    }
  };
  for (int upper = 1; upper >= 0; --upper)
    for (Index t = 0; t < T; ++t) {
      if (n_c == 0) break;
      emit(upper ? data.gu : data.gl, gemv(EFK, seg(t)), upper != 0);
    }
  for (int upper = 1; upper >= 0; --upper)
    for (Index t = 1; t <= T; ++t) emit(upper ? data.xu : data.xl, seg(t), upper != 0);
  for (int upper = 1; upper >= 0; --upper)
    for (Index t = 0; t < T; ++t) emit(upper ? data.uu : data.ul, gemv(data.K, seg(t)), upper != 0);
  parts.d = dv;
  return parts;
}

Mat assemble_inequality_rows(const LqProblemData& data, const BlockMatrices& bl) {  // :182-251
  const Dims dm = dims(data);
  const Index n_x = dm.n_x, n_u = dm.n_u, n_c = dm.n_c, T = dm.T;
  Mat EFK = (n_c > 0) ? add(data.E, matmul(data.F, data.K)) : Mat(0, n_x);
  Index rows = 0;
  auto count = [&](const Vec& lo, const Vec& hi, Index rep) {
    for (size_t i = 0; i < lo.size(); ++i) {
      if (std::isfinite(hi[i])) rows += rep;
      if (std::isfinite(lo[i])) rows += rep;
    }
  };
  count(data.gl, data.gu, T);
  count(data.xl, data.xu, T);
  count(data.ul, data.uu, T);
  Mat J(rows, T * n_u);
  Index next = 0;
  for (int upper = 1; upper >= 0; --upper)
    for (Index t = 0; t < T && n_c > 0; ++t) {
      const Vec& bound = upper ? data.gu : data.gl;
      const double sign = upper ? 1.0 : -1.0;
      const Index width = t * n_u;
      for (Index i = 0; i < n_c; ++i) {
        if (!std::isfinite(bound[size_t(i)])) continue;
        const Index r = next++;
        if (t > 0) {
          for (Index c = 0; c < width; ++c) {
            double s = 0.0;
            for (Index p = 0; p < n_x; ++p) s += EFK(i, p) * bl.bigB(t * n_x + p, c);
            J(r, c) = sign * s;
          }
        }
        for (Index c = 0; c < n_u; ++c) J(r, t * n_u + c) += sign * data.F(i, c);
      }
    }
  for (int upper = 1; upper >= 0; --upper)
    for (Index t = 1; t <= T; ++t) {
      const Vec& bound = upper ? data.xu : data.xl;
      const double sign = upper ? 1.0 : -1.0;
      const Index width = t * n_u;
      for (Index i = 0; i < n_x; ++i) {
        if (!std::isfinite(bound[size_t(i)])) continue;
        const Index r = next++;
        for (Index c = 0; c < width; ++c) J(r, c) = sign * bl.bigB(t * n_x + i, c);
      }
    }
  for (int upper = 1; upper >= 0; --upper)
    for (Index t = 0; t < T; ++t) {
      const Vec& bound = upper ? data.uu : data.ul;
      const double sign = upper ? 1.0 : -1.0;
      const Index width = t * n_u;
      for (Index i = 0; i < n_u; ++i) {
        if (!std::isfinite(bound[size_t(i)])) continue;
        const Index r = next++;
        if (t > 0) {
          for (Index c = 0; c < width; ++c) {
            double s = 0.0;
            for (Index p = 0; p < n_x; ++p) s += data.K(i, p) * bl.bigB(t * n_x + p, c);
            J(r, c) = sign * s;
          }
        }
        J(r, t * n_u + i) += sign;
      }
    }
  require(next == rows, "inequality assembly row count mismatch");
  return J;
}
}  // namespace

BlockMatrices build_block_matrices(const LqProblemData& data) {  // reduction.cpp:22-62
  const Dims d = dims(data);
  const Index n_x = d.n_x, n_u = d.n_u, T = d.T;
  BlockMatrices b;
  b.A_K = add(data.A, matmul(data.B, data.K));
  b.bigA = Mat((T + 1) * n_x, n_x);
  b.bigB = Mat((T + 1) * n_x, T * n_u);
  b.bigAtilde = Mat((T + 1) * n_x, T * n_x);
  set_block(b.bigA, 0, 0, Mat::identity(n_x));
  for (Index i = 1; i <= T; ++i)
    set_block(b.bigA, i * n_x, 0, matmul(b.A_K, block(b.bigA, (i - 1) * n_x, 0, n_x, n_x)));
  for (Index i = 1; i <= T; ++i) {
    if (i == 1) {
      set_block(b.bigB, n_x, 0, data.B);
      set_block(b.bigAtilde, n_x, 0, Mat::identity(n_x));
    } else {
      set_block(b.bigB, i * n_x, 0, matmul(b.A_K, block(b.bigB, (i - 1) * n_x, 0, n_x, n_u)));
      set_block(b.bigAtilde, i * n_x, 0,
                matmul(b.A_K, block(b.bigAtilde, (i - 1) * n_x, 0, n_x, n_x)));
    }
  }
  for (Index j = 1; j < T; ++j) {
    const Index height = (T - j) * n_x;
    set_block(b.bigB, (j + 1) * n_x, j * n_u, block(b.bigB, n_x, 0, height, n_u));
    set_block(b.bigAtilde, (j + 1) * n_x, j * n_x, block(b.bigAtilde, n_x, 0, height, n_x));
  }
  return b;
}

DenseQp build_dense_qp(const LqProblemData& data) {  // reduction.cpp:255-268
  DenseQp qp;
  qp.source = data;
  qp.has_source = true;
  qp.blocks = build_block_matrices(data);
  const SubstitutedCost cost = substituted_cost(data);
  qp.H = assemble_hessian(data, qp.blocks, cost);
  qp.J = assemble_inequality_rows(data, qp.blocks);
  const Vec x0 = stacked_free_response(qp.blocks, data);
  AffineParts p = assemble_affine(data, qp.blocks, cost, x0);
  qp.h = p.h;
  qp.h0 = p.h0;
  qp.d = p.d;
  return qp;
}

void refresh_initial_state(DenseQp& qp, const Vec& x_bar) {  // reduction.cpp:270-280
  require(x_bar.size() == qp.source.x_bar.size(), "refresh_initial_state: x_bar length mismatch");
  qp.source.x_bar = x_bar;
  const SubstitutedCost cost = substituted_cost(qp.source);
  const Vec x0 = stacked_free_response(qp.blocks, qp.source);
  AffineParts p = assemble_affine(qp.source, qp.blocks, cost, x0);
  qp.h = p.h;
  qp.h0 = p.h0;
  qp.d = p.d;
}

Trajectory recover_trajectory(const DenseQp& qp, const Vec& v) {  // reduction.cpp:282-314
  const Dims dm = dims(qp.source);
  const Index n_x = dm.n_x, n_u = dm.n_u, T = dm.T;
  require(Index(v.size()) == T * n_u, "recover_trajectory: v has length " +
                                           std::to_string(v.size()) + ", expected " +
                                           std::to_string(T * n_u));
  Vec xs = stacked_free_response(qp.blocks, qp.source);
  const Vec bv = gemv(qp.blocks.bigB, v);
  for (size_t i = 0; i < xs.size(); ++i) xs[i] += bv[i];
  Trajectory tr;
  for (Index t = 0; t <= T; ++t) tr.x.emplace_back(xs.begin() + t * n_x, xs.begin() + (t + 1) * n_x);
  for (Index t = 0; t < T; ++t) {
    Vec vt(v.begin() + t * n_u, v.begin() + (t + 1) * n_u);
    Vec u = gemv(qp.source.K, tr.x[size_t(t)]);
    for (Index i = 0; i < n_u; ++i) u[size_t(i)] += vt[size_t(i)];
    tr.u.push_back(u);
    tr.v.push_back(vt);
  }
  double obj = dot(tr.x.back(), gemv(qp.source.Qf, tr.x.back()));
  for (Index t = 0; t < T; ++t) {
    const Vec& xt = tr.x[size_t(t)];
    const Vec& ut = tr.u[size_t(t)];
    obj += dot(xt, gemv(qp.source.Q, xt)) + 2.0 * dot(xt, gemv(qp.source.S, ut)) +
           dot(ut, gemv(qp.source.R, ut));
  }
  tr.objective = obj;
  return tr;
}

double dense_objective(const DenseQp& qp, const Vec& v) {  // reduction.cpp:316-321
  require(Index(v.size()) == qp.H.r, "dense_objective: v has length " + std::to_string(v.size()) +
                                         ", expected " + std::to_string(qp.H.r));
  return 0.5 * dot(v, gemv(qp.H, v)) + dot(qp.h, v) + qp.h0;
}

// ------------------------------------------------------------------ heat3d
void laplacian_system(Index N, const HeatParams& params, Mat& A, Mat& B) {  // heat3d.cpp:7-37
  require(N >= 1, "grid must have at least one interior point per dimension");
  const double c = params.stability_factor();
  if (!(c < 1.0 / 6.0)) throw std::runtime_error("explicit Euler unstable");
  const Index n_x = N * N * N;
  A = Mat(n_x, n_x);
  B = Mat(n_x, 6);
  auto cell = [N](Index i, Index j, Index k) { return i + N * j + N * N * k; };
  for (Index k = 0; k < N; ++k)
    for (Index j = 0; j < N; ++j)
      for (Index i = 0; i < N; ++i) {
        const Index row = cell(i, j, k);
        A(row, row) = 1.0 - 6.0 * c;
        if (i > 0) A(row, cell(i - 1, j, k)) = c; else B(row, 0) += c;
        if (i < N - 1) A(row, cell(i + 1, j, k)) = c; else B(row, 1) += c;
        if (j > 0) A(row, cell(i, j - 1, k)) = c; else B(row, 2) += c;
        if (j < N - 1) A(row, cell(i, j + 1, k)) = c; else B(row, 3) += c;
        if (k > 0) A(row, cell(i, j, k - 1)) = c; else B(row, 4) += c;
        if (k < N - 1) A(row, cell(i, j, k + 1)) = c; else B(row, 5) += c;
      }
}

LqProblemData build_heat_problem(const HeatParams& p) {  // heat3d.cpp:39-60
  require(p.T >= 1, "horizon must be at least 1");
  Mat A, B;
  laplacian_system(p.N, p, A, B);
  const Index n_x = A.r;
  Mat Q = Mat::identity(n_x), Qf = Mat::identity(n_x), R = Mat::identity(6);
  for (double& x : Q.a) x *= p.q_weight;
  for (double& x : Qf.a) x *= p.q_weight;
  for (double& x : R.a) x *= p.r_weight;
  LqProblemData d =
      LqProblemData::basic(A, B, Q, R, Qf, Vec(size_t(n_x), p.x_init - p.setpoint), p.T);
  Vec defect(static_cast<size_t>(n_x));
  for (Index i = 0; i < n_x; ++i) {
    double ra = 0.0, rb = 0.0;
    for (Index j = 0; j < n_x; ++j) ra += A(i, j);
    for (Index j = 0; j < 6; ++j) rb += B(i, j);
    defect[size_t(i)] = (ra + rb - 1.0) * p.setpoint;
  }
  for (auto& wt : d.w) wt = defect;
  d.xl = Vec(size_t(n_x), p.x_min - p.setpoint);
  d.xu = Vec(size_t(n_x), p.x_max - p.setpoint);
  d.ul = Vec(6, p.u_min - p.setpoint);
  d.uu = Vec(6, p.u_max - p.setpoint);
  return d;
}

// ------------------------------------------------------------------ random problems
namespace {
Mat uniform_matrix(std::mt19937_64& rng, Index rows, Index cols, double lo, double hi) {
  // random_problems.cpp:10-17
  std::uniform_real_distribution<double> dist(lo, hi);
  Mat m(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) m(i, j) = dist(rng);
  return m;
}
Mat random_spd(std::mt19937_64& rng, Index n) {  // :19-22
  const Mat m = uniform_matrix(rng, n, n, -1.0, 1.0);
  Mat s = matmul(transpose(m), m);
  for (Index i = 0; i < n; ++i) s(i, i) += 0.1;
  return s;
}
Vec col0(const Mat& m) { return Vec(m.a.begin(), m.a.begin() + m.r); }

// eigenvalues of a small general real matrix: complex shifted QR (restates the
// role of Eigen::EigenSolver in spectral_radius, random_problems.cpp:24-29)
double spectral_radius(const Mat& a) {
  using C = std::complex<double>;
  const Index n = a.r;
  if (n == 1) return std::abs(a(0, 0));
  std::vector<C> H(static_cast<size_t>(n * n));
  auto h = [&](Index i, Index j) -> C& { return H[size_t(i * n + j)]; };
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) h(i, j) = a(i, j);
  // Hessenberg reduction by Householder
  for (Index k = 0; k + 2 < n; ++k) {
    double alpha = 0;
    for (Index i = k + 1; i < n; ++i) alpha += std::norm(h(i, k));
    alpha = std::sqrt(alpha);
    if (alpha == 0.0) continue;
    std::vector<C> v(size_t(n), 0.0);
    const C x0 = h(k + 1, k);
    const C ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : C(1.0);
    v[size_t(k + 1)] = x0 + ph * alpha;
    for (Index i = k + 2; i < n; ++i) v[size_t(i)] = h(i, k);
    double vn = 0;
    for (auto& z : v) vn += std::norm(z);
    if (vn == 0) continue;
    for (Index j = 0; j < n; ++j) {  // H = (I - 2vv*/v*v) H
      C s = 0;
      for (Index i = k + 1; i < n; ++i) s += std::conj(v[size_t(i)]) * h(i, j);
      s *= 2.0 / vn;
      for (Index i = k + 1; i < n; ++i) h(i, j) -= v[size_t(i)] * s;
    }
    for (Index i = 0; i < n; ++i) {  // H = H (I - 2vv*/v*v)
      C s = 0;
      for (Index j = k + 1; j < n; ++j) s += h(i, j) * v[size_t(j)];
      s *= 2.0 / vn;
      for (Index j = k + 1; j < n; ++j) h(i, j) -= s * std::conj(v[size_t(j)]);
    }
  }
  std::vector<C> eig;
  Index hi = n - 1;
  int iter = 0;
  const double eps = std::numeric_limits<double>::epsilon();
  while (hi >= 0) {
    if (hi == 0) {
      eig.push_back(h(0, 0));
      break;
    }
    Index l = hi;
    while (l > 0 && std::abs(h(l, l - 1)) > eps * (std::abs(h(l, l)) + std::abs(h(l - 1, l - 1)))) --l;
    if (l == hi) {
      eig.push_back(h(hi, hi));
      --hi;
      iter = 0;
      continue;
    }
    if (l > 0) h(l, l - 1) = 0.0;
    // Wilkinson shift from the trailing 2x2 of the active block
    const C a11 = h(hi - 1, hi - 1), a12 = h(hi - 1, hi), a21 = h(hi, hi - 1), a22 = h(hi, hi);
    const C tr = a11 + a22, det = a11 * a22 - a12 * a21;
    const C disc = std::sqrt(tr * tr - 4.0 * det);
    const C e1 = (tr + disc) / 2.0, e2 = (tr - disc) / 2.0;
    C mu = std::abs(e1 - a22) < std::abs(e2 - a22) ? e1 : e2;
    if (++iter % 11 == 10) mu += C(std::abs(h(hi, hi - 1)), 0.0) * 0.75;  // exceptional shift
    if (iter > 3000) break;
    // QR step on rows/cols l..hi via Givens rotations
    for (Index i = l; i <= hi; ++i) h(i, i) -= mu;
    std::vector<std::pair<C, C>> rot;
    for (Index k = l; k < hi; ++k) {
      const C x = h(k, k), y = h(k + 1, k);
      const double r = std::sqrt(std::norm(x) + std::norm(y));
      C c = 1.0, s = 0.0;
      if (r > 0) {
        c = x / r;
        s = y / r;
      }
      for (Index j = k; j < n; ++j) {
        const C t1 = h(k, j), t2 = h(k + 1, j);
        h(k, j) = std::conj(c) * t1 + std::conj(s) * t2;
        h(k + 1, j) = -s * t1 + c * t2;
      }
      rot.push_back({c, s});
    }
    for (Index k = l; k < hi; ++k) {
      const C c = rot[size_t(k - l)].first, s = rot[size_t(k - l)].second;
      for (Index i = 0; i <= hi; ++i) {
        const C t1 = h(i, k), t2 = h(i, k + 1);
        h(i, k) = t1 * c + t2 * s;
        h(i, k + 1) = -t1 * std::conj(s) + t2 * std::conj(c);
      }
    }
    for (Index i = l; i <= hi; ++i) h(i, i) += mu;
  }
  double r = 0;
  for (auto& e : eig) r = std::max(r, std::abs(e));
  return r;
}

// smallest eigenvalue of a symmetric matrix (cyclic Jacobi), restating the role of
// Eigen::SelfAdjointEigenSolver at random_problems.cpp:74-77
double sym_min_eig(Mat a) {
  const Index n = a.r;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (Index i = 0; i < n; ++i)
      for (Index j = i + 1; j < n; ++j) off += a(i, j) * a(i, j);
    if (off < 1e-30) break;
    for (Index p = 0; p < n; ++p)
      for (Index q = p + 1; q < n; ++q) {
        if (a(p, q) == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2 * a(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1));
        const double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (Index k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (Index k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
      }
  }
  double mn = kInf;
  for (Index i = 0; i < n; ++i) mn = std::min(mn, a(i, i));
  return mn;
}
}  // namespace

std::mt19937_64 instance_rng(std::uint64_t seed, std::uint64_t index) {  // :33-37
  std::seed_seq seq{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32),
                    static_cast<std::uint32_t>(index), static_cast<std::uint32_t>(index >> 32)};
  return std::mt19937_64(seq);
}

LqProblemData random_problem(std::mt19937_64& rng, const RandomProblemOptions& o) {  // :39-126
  require(o.max_n_x >= 1 && o.max_n_u >= 1 && o.max_T >= 1, "ensemble dimensions must be at least 1");
  auto draw = [&rng](Index lo, Index hi) {
    std::uniform_int_distribution<long> dist(lo, hi);
    return Index(dist(rng));
  };
  Index T, n_x, n_u, n_c;
  if (o.fixed_dims) {
    T = o.T;
    n_x = o.n_x;
    n_u = o.n_u;
    n_c = o.n_c;
  } else {
    do {
      T = draw(1, o.max_T);
      n_x = draw(1, o.max_n_x);
      n_u = draw(1, o.max_n_u);
      n_c = o.max_n_c > 0 ? draw(0, o.max_n_c) : 0;
    } while (o.cap_rows_for_oracle && 2 * T * (n_c + n_x + n_u) > 22);
  }
  Mat A = uniform_matrix(rng, n_x, n_x, -1.0, 1.0);
  const double radius = spectral_radius(A);
  if (radius > o.spectral_radius_cap)
    for (double& x : A.a) x *= o.spectral_radius_cap / radius;
  LqProblemData data = LqProblemData::basic(
      A, uniform_matrix(rng, n_x, n_u, -1.0, 1.0), random_spd(rng, n_x), random_spd(rng, n_u),
      random_spd(rng, n_x), col0(uniform_matrix(rng, n_x, 1, -1.0, 1.0)), T);
  data.S = uniform_matrix(rng, n_x, n_u, -1.0, 1.0);
  Mat stage(n_x + n_u, n_x + n_u);
  set_block(stage, 0, 0, data.Q);
  set_block(stage, n_x, n_x, data.R);
  for (;;) {
    set_block(stage, 0, n_x, data.S);
    set_block(stage, n_x, 0, transpose(data.S));
    if (sym_min_eig(stage) >= 0.05) break;
    for (double& x : data.S.a) x *= 0.5;
  }
  for (auto& wt : data.w) wt = col0(uniform_matrix(rng, n_x, 1, -0.1, 0.1));
  if (n_c > 0) {
    data.E = uniform_matrix(rng, n_c, n_x, -1.0, 1.0);
    data.F = uniform_matrix(rng, n_c, n_u, -1.0, 1.0);
  }
  std::vector<Vec> xs(size_t(T) + 1), us(static_cast<size_t>(T));
  xs[0] = data.x_bar;
  for (Index t = 0; t < T; ++t) {
    us[size_t(t)] = col0(uniform_matrix(rng, n_u, 1, -0.5, 0.5));
    Vec ax = gemv(data.A, xs[size_t(t)]);
    Vec bu = gemv(data.B, us[size_t(t)]);
    Vec nx(static_cast<size_t>(n_x));
    for (Index i = 0; i < n_x; ++i) nx[size_t(i)] = ax[size_t(i)] + bu[size_t(i)] + data.w[size_t(t)][size_t(i)];
    xs[size_t(t) + 1] = nx;
  }
  const double margin = o.bound_margin;
  data.xl = xs[0];
  data.xu = xs[0];
  for (const Vec& x : xs)
    for (Index i = 0; i < n_x; ++i) {
      data.xl[size_t(i)] = std::min(data.xl[size_t(i)], x[size_t(i)]);
      data.xu[size_t(i)] = std::max(data.xu[size_t(i)], x[size_t(i)]);
    }
  for (auto& x : data.xl) x -= margin;
  for (auto& x : data.xu) x += margin;
  data.ul = Vec(size_t(n_u), -0.5 - margin);
  data.uu = Vec(size_t(n_u), 0.5 + margin);
  if (n_c > 0) {
    auto efx = [&](Index t) {
      Vec a = gemv(data.E, xs[size_t(t)]), b = gemv(data.F, us[size_t(t)]);
      for (size_t i = 0; i < a.size(); ++i) a[i] += b[i];
      return a;
    };
    Vec lo = efx(0), hi = lo;
    for (Index t = 0; t < T; ++t) {
      const Vec y = efx(t);
      for (size_t i = 0; i < y.size(); ++i) {
        lo[i] = std::min(lo[i], y[i]);
        hi[i] = std::max(hi[i], y[i]);
      }
    }
    for (auto& x : lo) x -= margin;
    for (auto& x : hi) x += margin;
    data.gl = lo;
    data.gu = hi;
  }
  return data;
}

// ------------------------------------------------------------------ enumeration oracle
namespace {
// full-pivot LU with Eigen's relative threshold semantics (rank counts pivots with
// |p| > threshold * |max pivot|)
struct FullPivLU {
  Index n = 0, rank = 0;
  Mat lu;
  std::vector<Index> rp, cp;
  FullPivLU(const Mat& a, double thr) {
    const Index r = a.r, c = a.c;
    n = std::min(r, c);
    lu = a;
    rp.resize(static_cast<size_t>(r));
    cp.resize(static_cast<size_t>(c));
    for (Index i = 0; i < r; ++i) rp[size_t(i)] = i;
    for (Index i = 0; i < c; ++i) cp[size_t(i)] = i;
    double maxpivot = 0.0;
    Index nonzero = 0;
    for (Index k = 0; k < n; ++k) {
      Index bi = k, bj = k;
      double best = -1;
      for (Index j = k; j < c; ++j)
        for (Index i = k; i < r; ++i)
          if (std::abs(lu(i, j)) > best) {
            best = std::abs(lu(i, j));
            bi = i;
            bj = j;
          }
      if (k == 0) maxpivot = best;
      if (best == 0.0) break;
      if (bi != k) {
        for (Index j = 0; j < c; ++j) std::swap(lu(k, j), lu(bi, j));
        std::swap(rp[size_t(k)], rp[size_t(bi)]);
      }
      if (bj != k) {
        for (Index i = 0; i < r; ++i) std::swap(lu(i, k), lu(i, bj));
        std::swap(cp[size_t(k)], cp[size_t(bj)]);
      }
      ++nonzero;
      for (Index i = k + 1; i < r; ++i) {
        lu(i, k) /= lu(k, k);
        for (Index j = k + 1; j < c; ++j) lu(i, j) -= lu(i, k) * lu(k, j);
      }
    }
    rank = 0;
    for (Index k = 0; k < nonzero; ++k)
      if (std::abs(lu(k, k)) > thr * maxpivot) ++rank;
  }
  Vec solve(const Vec& b) const {  // square invertible only
    Vec y(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) y[size_t(i)] = b[size_t(rp[size_t(i)])];
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < i; ++j) y[size_t(i)] -= lu(i, j) * y[size_t(j)];
    for (Index i = n - 1; i >= 0; --i) {
      for (Index j = i + 1; j < n; ++j) y[size_t(i)] -= lu(i, j) * y[size_t(j)];
      y[size_t(i)] /= lu(i, i);
    }
    Vec x(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) x[size_t(cp[size_t(i)])] = y[size_t(i)];
    return x;
  }
};
}  // namespace

EnumResult solve_enumeration(const Mat& H, const Vec& h, double h0, const Mat& J, const Vec& d) {
  // oracle.cpp:34-112
  const Index n = H.r, m = J.r;
  if (m > 22) throw std::runtime_error("oracle: row cap exceeded");
  const double kFeas = 1e-9, kRank = 1e-10;
  EnumResult best;
  bool any = false, have = false;
  const std::uint32_t end = std::uint32_t(1) << m;
  for (std::uint32_t mask = 0; mask < end; ++mask) {
    const int active = std::popcount(mask);
    if (active > n) continue;
    std::vector<Index> rows;
    for (Index i = 0, mm = mask; mm != 0; ++i, mm >>= 1)
      if (mm & 1) rows.push_back(i);
    Mat Jw(active, n);
    Vec dw(static_cast<size_t>(active));
    for (int k = 0; k < active; ++k) {
      for (Index j = 0; j < n; ++j) Jw(k, j) = J(rows[size_t(k)], j);
      dw[size_t(k)] = d[size_t(rows[size_t(k)])];
    }
    if (active > 0) {
      FullPivLU rc(Jw, kRank);
      if (rc.rank < active) continue;
    }
    Mat kkt(n + active, n + active);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) kkt(i, j) = H(i, j);
    for (int k = 0; k < active; ++k)
      for (Index j = 0; j < n; ++j) {
        kkt(j, n + k) = Jw(k, j);
        kkt(n + k, j) = Jw(k, j);
      }
    Vec rhs(static_cast<size_t>(n + active));
    for (Index i = 0; i < n; ++i) rhs[size_t(i)] = -h[size_t(i)];
    for (int k = 0; k < active; ++k) rhs[size_t(n + k)] = dw[size_t(k)];
    FullPivLU lu(kkt, kRank);
    if (lu.rank < n + active) continue;
    any = true;
    const Vec sol = lu.solve(rhs);
    Vec v(sol.begin(), sol.begin() + n), lam(sol.begin() + n, sol.end());
    if (m > 0) {
      const Vec jv = gemv(J, v);
      bool bad = false;
      for (Index i = 0; i < m; ++i)
        if (jv[size_t(i)] - d[size_t(i)] > kFeas) bad = true;
      if (bad) continue;
    }
    bool neg = false;
    for (double l : lam)
      if (l < -kFeas) neg = true;
    if (active > 0 && neg) continue;
    const double obj = 0.5 * dot(v, gemv(H, v)) + dot(h, v) + h0;
    const double scale = 1.0 + std::abs(have ? best.objective : obj);
    bool take = false;
    if (!have || obj < best.objective - kFeas * scale) take = true;
    else if (obj <= best.objective + kFeas * scale)
      take = std::lexicographical_compare(rows.begin(), rows.end(), best.active_set.begin(),
                                          best.active_set.end());
    if (take) {
      best.status = 0;
      best.v = v;
      best.objective = obj;
      best.active_set = rows;
      best.multipliers = lam;
      have = true;
    }
  }
  if (!have) {
    best.status = any ? 1 : 2;
    best.v.assign(size_t(n), 0.0);
    best.objective = std::numeric_limits<double>::quiet_NaN();
  }
  return best;
}

// ------------------------------------------------------------------ ipm
double merit(const DenseQp& qp, const Vec& v, const Vec& s, double mu, double rho) {  // ipm.cpp:25-32
  double phi = 0.5 * dot(v, gemv(qp.H, v)) + dot(qp.h, v);
  if (!s.empty()) {
    double ls = 0.0;
    for (double x : s) ls += std::log(x);
    phi -= mu * ls;
    const Vec jv = gemv(qp.J, v);
    double l1 = 0.0;
    for (size_t i = 0; i < s.size(); ++i) l1 += std::abs(jv[i] - qp.d[i] + s[i]);
    phi += rho * l1;
  }
  return phi;
}

Residuals compute_residuals(const DenseQp& qp, const IpmState& st) {  // ipm.cpp:46-70
  const Index m = qp.J.r, n = qp.H.r;
  require(Index(st.v.size()) == n, "state.v does not match the QP");
  require(Index(st.s.size()) == m && Index(st.lambda.size()) == m && Index(st.z.size()) == m,
          "state slack/dual lengths do not match the QP row count");
  Residuals res;
  res.r1 = gemv(qp.H, st.v);
  for (Index i = 0; i < n; ++i) res.r1[size_t(i)] += qp.h[size_t(i)];
  if (m > 0) {
    const Vec jl = gemv_t(qp.J, st.lambda);
    for (Index i = 0; i < n; ++i) res.r1[size_t(i)] += jl[size_t(i)];
  }
  res.r2.resize(static_cast<size_t>(m));
  for (Index i = 0; i < m; ++i) res.r2[size_t(i)] = st.lambda[size_t(i)] - st.mu * (1.0 / st.s[size_t(i)]);
  const Vec jv = m > 0 ? gemv(qp.J, st.v) : Vec();
  res.r3.resize(static_cast<size_t>(m));
  for (Index i = 0; i < m; ++i) res.r3[size_t(i)] = jv[size_t(i)] - qp.d[size_t(i)] + st.s[size_t(i)];
  double mh = 0.0, ml = 0.0;
  for (double x : qp.h) mh = std::max(mh, std::abs(x));
  for (double x : st.lambda) ml = std::max(ml, std::abs(x));
  const double dual_scale = std::max(1.0, std::max(mh, ml) / double(n + m));
  res.kkt_error = inf_norm(res.r1) / dual_scale;
  if (m > 0) {
    double ms = 0.0, mz = 0.0, mc = 0.0;
    for (double x : st.s) ms = std::max(ms, std::abs(x));
    for (double x : st.z) mz = std::max(mz, std::abs(x));
    const double comp_scale = std::max(1.0, std::max(ms, mz) / double(2 * m));
    for (Index i = 0; i < m; ++i) mc = std::max(mc, std::abs(st.s[size_t(i)] * st.z[size_t(i)] - st.mu));
    res.kkt_error = std::max(res.kkt_error, inf_norm(res.r3));
    res.kkt_error = std::max(res.kkt_error, mc / comp_scale);
  }
  return res;
}

Mat assemble_condensed(const DenseQp& qp, const Vec& sigma) {  // ipm.cpp:72-77
  require(Index(sigma.size()) == qp.J.r, "sigma length does not match the QP row count");
  Mat M = qp.H;
  if (!sigma.empty()) {
    const Mat G = gram_weighted(qp.J, sigma);
    for (size_t i = 0; i < M.a.size(); ++i) M.a[i] += G.a[i];
  }
  return M;
}

StepDirections step_directions(const DenseQp& qp, const IpmState& st, const Residuals& res,
                               const Mat& L) {  // ipm.cpp:79-103
  const Index m = qp.J.r, n = qp.H.r;
  StepDirections dirs;
  Vec rhs(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) rhs[size_t(i)] = -res.r1[size_t(i)];
  Vec sigma;
  if (m > 0) {
    sigma.resize(static_cast<size_t>(m));
    for (Index i = 0; i < m; ++i) sigma[size_t(i)] = st.z[size_t(i)] / st.s[size_t(i)];
    Vec y(static_cast<size_t>(m));
    for (Index i = 0; i < m; ++i) y[size_t(i)] = res.r2[size_t(i)] - sigma[size_t(i)] * res.r3[size_t(i)];
    const Vec jy = gemv_t(qp.J, y);
    for (Index i = 0; i < n; ++i) rhs[size_t(i)] += jy[size_t(i)];
  }
  dirs.pv = factor_solve(L, rhs);
  if (m > 0) {
    const Vec jpv = gemv(qp.J, dirs.pv);
    dirs.ps.resize(static_cast<size_t>(m));
    dirs.plambda.resize(static_cast<size_t>(m));
    dirs.pz.resize(static_cast<size_t>(m));
    for (Index i = 0; i < m; ++i) {
      const size_t k = size_t(i);
      dirs.ps[k] = -res.r3[k] - jpv[k];
      dirs.plambda[k] = -res.r2[k] + sigma[k] * (res.r3[k] + jpv[k]);
      dirs.pz[k] = st.mu * (1.0 / st.s[k]) - st.z[k] - sigma[k] * dirs.ps[k];
    }
  }
  return dirs;
}

void fraction_to_boundary(const Vec& s, const Vec& ps, const Vec& z, const Vec& pz, double tau,
                          double* alpha, double* alpha_z) {  // ipm.cpp:105-116
  require(tau > 0.0 && tau < 1.0, "tau must lie in (0,1)");
  auto largest = [tau](const Vec& x, const Vec& px) {
    double a = 1.0;
    for (size_t i = 0; i < x.size(); ++i)
      if (px[i] < 0.0) a = std::min(a, tau * (-x[i] / px[i]));
    return a;
  };
  *alpha = largest(s, ps);
  *alpha_z = largest(z, pz);
}

int line_search(const DenseQp& qp, const IpmState& st, const StepDirections& dirs, double alpha_max,
                const IpmOptions& opts, double* alpha_out) {  // ipm.cpp:118-144
  require(alpha_max > 0.0 && alpha_max <= 1.0, "alpha_max must lie in (0,1]");
  const Index m = qp.J.r, n = qp.H.r;
  double ml = 0.0;
  for (double x : st.lambda) ml = std::max(ml, std::abs(x));
  const double rho = 10.0 * ml + 1.0;
  const double phi0 = merit(qp, st.v, st.s, st.mu, rho);
  Vec g = gemv(qp.H, st.v);
  for (Index i = 0; i < n; ++i) g[size_t(i)] += qp.h[size_t(i)];
  double derivative = dot(g, dirs.pv);
  if (m > 0) {
    double q = 0.0;
    for (Index i = 0; i < m; ++i) q += dirs.ps[size_t(i)] / st.s[size_t(i)];
    derivative -= st.mu * q;
    const Vec jv = gemv(qp.J, st.v);
    double l1 = 0.0;
    for (Index i = 0; i < m; ++i) l1 += std::abs(jv[size_t(i)] - qp.d[size_t(i)] + st.s[size_t(i)]);
    derivative -= rho * l1;
  }
  constexpr double band = 10.0 * std::numeric_limits<double>::epsilon();
  double alpha = alpha_max;
  Vec vt(static_cast<size_t>(n)), stt(static_cast<size_t>(m));
  for (int j = 0; j <= 30; ++j, alpha *= 0.5) {
    for (Index i = 0; i < n; ++i) vt[size_t(i)] = st.v[size_t(i)] + alpha * dirs.pv[size_t(i)];
    bool nonpos = false;
    for (Index i = 0; i < m; ++i) {
      stt[size_t(i)] = st.s[size_t(i)] + alpha * dirs.ps[size_t(i)];
      if (stt[size_t(i)] <= 0.0) nonpos = true;
    }
    if (m > 0 && nonpos) continue;
    const double phi = merit(qp, vt, stt, st.mu, rho);
    if (derivative <= 0.0 && phi <= phi0 + opts.armijo_eta * alpha * derivative) {
      *alpha_out = alpha;
      return j;
    }
    if (std::abs(phi - phi0) <= band * (1.0 + std::abs(phi0))) {
      *alpha_out = alpha;
      return j;
    }
  }
  return -1;
}

double update_barrier(const IpmState& st, const Residuals& res, const IpmOptions& opts) {  // :146-151
  if (res.kkt_error <= 10.0 * st.mu) return std::max(opts.tol / 10.0, opts.kappa_mu * st.mu);
  return st.mu;
}

int check_termination(const Residuals& res, const IpmState& st, const IpmOptions& opts) {  // :153-158
  if (res.kkt_error <= opts.tol && st.mu <= opts.tol) return 0;
  if (st.iter >= opts.max_iter) return 1;
  return 2;
}

IpmResult solve(const DenseQp& qp, const IpmOptions& opts) {  // ipm.cpp:160-268
  require(opts.tol > 0.0, "tol must be positive");
  require(opts.kappa_mu > 0.0 && opts.kappa_mu < 1.0, "kappa_mu must lie in (0,1)");
  require(opts.tau > 0.0 && opts.tau < 1.0, "tau must lie in (0,1)");
  require(opts.mu_init > 0.0, "mu_init must be positive");
  require(opts.max_iter >= 1, "max_iter must be at least 1");
  const Index n = qp.H.r, m = qp.J.r;
  require(Index(qp.h.size()) == n, "qp.h length does not match qp.H");
  require(Index(qp.d.size()) == m, "qp.d length does not match qp.J");
  const double start = now_seconds();
  if (opts.backend != "reference" && opts.backend != "eigen")
    throw std::invalid_argument("unknown factorization backend: " + opts.backend);

  IpmState st;
  st.v.assign(size_t(n), 0.0);
  st.s.resize(static_cast<size_t>(m));
  for (Index i = 0; i < m; ++i) st.s[size_t(i)] = std::max(1.0, qp.d[size_t(i)]);
  st.mu = opts.mu_init;
  st.z.resize(static_cast<size_t>(m));
  for (Index i = 0; i < m; ++i) st.z[size_t(i)] = st.mu * (1.0 / st.s[size_t(i)]);
  st.lambda = st.z;
  st.iter = 0;

  IpmResult result;
  ZeroMap zm;
  struct ZGuard {
    ~ZGuard() { g_zmap = nullptr; }
  } zguard;
  if (g_skip_zeros && m > 0) {
    zm = make_zmap(qp.J);
    g_zmap = &zm;
  }
  Residuals res = compute_residuals(qp, st);
  while (true) {
    const int term = check_termination(res, st, opts);
    if (term == 0) {
      result.status = IpmStatus::converged;
      break;
    }
    if (term == 1) {
      result.status = IpmStatus::max_iter;
      break;
    }
    const double mu_next = update_barrier(st, res, opts);
    if (mu_next != st.mu) {
      st.mu = mu_next;
      res = compute_residuals(qp, st);
    }
    const double ls = now_seconds();
    Vec sigma(static_cast<size_t>(m));
    for (Index i = 0; i < m; ++i) sigma[size_t(i)] = st.z[size_t(i)] / st.s[size_t(i)];
    const Mat condensed = assemble_condensed(qp, sigma);
    static constexpr std::array<double, 7> kShifts = {0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1.0, 1e2};
    std::optional<Mat> L;
    double delta_used = 0.0;
    for (double delta : kShifts) {
      try {
        if (delta == 0.0) {
          L.emplace(factorize(opts.backend, condensed));
        } else {
          Mat shifted = condensed;
          for (Index i = 0; i < n; ++i) shifted(i, i) += delta;
          L.emplace(factorize(opts.backend, shifted));
        }
        delta_used = delta;
        break;
      } catch (const NotPositiveDefinite&) {
      }
    }
    result.linalg_seconds += now_seconds() - ls;
    if (!L) {
      result.status = IpmStatus::factorization_failure;
      break;
    }
    const StepDirections dirs = step_directions(qp, st, res, *L);
    if (opts.inspect) opts.inspect(IterationInspection{st, res, dirs, delta_used});
    double alpha_max, alpha_z;
    fraction_to_boundary(st.s, dirs.ps, st.z, dirs.pz, opts.tau, &alpha_max, &alpha_z);
    double alpha = 0.0;
    const int j = line_search(qp, st, dirs, alpha_max, opts, &alpha);
    if (j < 0) {
      result.status = IpmStatus::line_search_failure;
      break;
    }
    const double mu_used = st.mu;
    for (Index i = 0; i < n; ++i) st.v[size_t(i)] += alpha * dirs.pv[size_t(i)];
    for (Index i = 0; i < m; ++i) {
      st.s[size_t(i)] += alpha * dirs.ps[size_t(i)];
      st.lambda[size_t(i)] += alpha * dirs.plambda[size_t(i)];
      st.z[size_t(i)] += alpha_z * dirs.pz[size_t(i)];
    }
    st.iter += 1;
    res = compute_residuals(qp, st);
    if (opts.log) {
      IterationRecord rec;
      rec.iter = st.iter;
      rec.mu = mu_used;
      rec.alpha = alpha;
      rec.alpha_z = alpha_z;
      rec.kkt_error = res.kkt_error;
      rec.objective = dense_objective(qp, st.v);
      rec.delta = delta_used;
      rec.trial = j;
      opts.log(rec);
    }
  }
  result.v = st.v;
  result.s = st.s;
  result.lambda = st.lambda;
  result.z = st.z;
  result.iter = st.iter;
  result.kkt_error = res.kkt_error;
  result.objective = dense_objective(qp, st.v);
  if (qp.has_source && qp.source.A.r > 0 && qp.blocks.bigB.r > 0) {
    result.solution = recover_trajectory(qp, st.v);
  } else {
    result.solution.objective = result.objective;
  }
  result.total_seconds = now_seconds() - start;
  return result;
}

}  // namespace orc
