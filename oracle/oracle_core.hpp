// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference `condmpc` solver (arXiv 2209.13049 re-creation,
// /root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it; the product (the CUDA path
// in paper_2209_13049_b200/) never links or calls it.
//
// Parity status: the reference itself cannot be compiled in this container
// (Eigen3, doctest and CLI11 are absent — SURVEY.md §8(c)), so this restatement
// is pinned against the known-answer values the reference's own tests hold
// (proj/tests/test_ipm.cpp, test_dense_linalg.cpp, test_reduction.cpp,
// test_heat3d.cpp, acceptance.cpp); see tests/test_oracle_kat.py. At the
// BASELINE.json configurations no reference number exists ("parity unpinned"
// there beyond the KATs), so the restatement is the definition of the reference
// CPU path for those sizes.
//
// Column-major dense storage, layout-identical to Eigen::MatrixXd
// (proj/include/condmpc/types.hpp:10-11). Summation orders follow the plain
// loop forms of the Eigen expressions (Eigen's packet order is not observable).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Index = std::int64_t;
constexpr double kInf = std::numeric_limits<double>::infinity();

struct DimensionError : std::runtime_error {
  explicit DimensionError(const std::string& m) : std::runtime_error(m) {}
};
inline void require(bool c, const std::string& m) {
  if (!c) throw DimensionError(m);
}

using Vec = std::vector<double>;

struct Mat {
  Index r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index rows, Index cols, double fill = 0.0) : r(rows), c(cols), a(size_t(rows * cols), fill) {}
  double& operator()(Index i, Index j) { return a[size_t(j * r + i)]; }
  double operator()(Index i, Index j) const { return a[size_t(j * r + i)]; }
  double* col(Index j) { return a.data() + j * r; }
  const double* col(Index j) const { return a.data() + j * r; }
  static Mat identity(Index n) {
    Mat m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

// ---- types.hpp helpers (proj/include/condmpc/types.hpp:21-29)
double inf_norm(const Vec& v);
double max_abs(const Mat& m);

// ---- small BLAS-like helpers with fixed summation order
Vec gemv(const Mat& A, const Vec& x);    // A x, per-row sum in column order
Vec gemv_t(const Mat& A, const Vec& x);  // A' x, per-column dot in row order
double dot(const Vec& a, const Vec& b);
Mat matmul(const Mat& A, const Mat& B);
Mat transpose(const Mat& A);

// ---- dense_linalg (proj/src/dense_linalg.cpp)
struct NotPositiveDefinite : std::runtime_error {
  NotPositiveDefinite(Index p, const std::string& m) : std::runtime_error(m), pivot(p) {}
  Index pivot;
};
// ReferenceBackend::factorize (dense_linalg.cpp:59-77): blocked (64) right-looking
Mat factorize_reference(const Mat& sym);
// EigenLltBackend::factorize (dense_linalg.cpp:86-97): restated as unblocked Cholesky
Mat factorize_llt(const Mat& sym);
Mat factorize(const std::string& backend, const Mat& sym);  // make_backend(name)->factorize
Vec factor_solve(const Mat& L, const Vec& rhs);              // Factor::solve (:102-110)
Mat gram_weighted(const Mat& J, const Vec& sigma);           // (:128-137)

// ---- problem.hpp / problem.cpp
struct LqProblemData {
  Mat A, B, Q, Qf, R, S, E, F;
  Vec gl, gu, xl, xu, ul, uu;
  std::vector<Vec> w;
  Vec x_bar;
  Mat K;
  Index T = 0;
  static LqProblemData basic(Mat A, Mat B, Mat Q, Mat R, Mat Qf, Vec x_bar, Index T);
};
struct Dims {
  Index n_x = 0, n_u = 0, n_c = 0, T = 0;
};
Dims dims(const LqProblemData& d);

// ---- reduction (proj/src/reduction.cpp)
struct BlockMatrices {
  Mat bigA, bigB, bigAtilde, A_K;
};
struct DenseQp {
  Mat H;
  Vec h;
  double h0 = 0.0;
  Mat J;
  Vec d;
  BlockMatrices blocks;
  LqProblemData source;
  bool has_source = false;
};
struct Trajectory {
  std::vector<Vec> x, u, v;
  double objective = 0.0;
};
BlockMatrices build_block_matrices(const LqProblemData& data);
DenseQp build_dense_qp(const LqProblemData& data);
void refresh_initial_state(DenseQp& qp, const Vec& x_bar);
Trajectory recover_trajectory(const DenseQp& qp, const Vec& v);
double dense_objective(const DenseQp& qp, const Vec& v);

// ---- heat3d (proj/src/heat3d.cpp)
struct HeatParams {
  Index N = 4, T = 50;
  double dt = 0.1, dw = 0.02, rho = 8960.0, cp = 386.0, conductivity = 400.0;
  double q_weight = 10.0 * 0.02 * 0.02, r_weight = 0.1 * 0.02 * 0.02;
  double x_min = 200.0, x_max = 550.0, u_min = 300.0, u_max = 500.0, x_init = 300.0,
         setpoint = 350.0;
  double diffusivity() const { return conductivity / (rho * cp); }
  double stability_factor() const { return diffusivity() * dt / (dw * dw); }
};
void laplacian_system(Index N, const HeatParams& p, Mat& A, Mat& B);
LqProblemData build_heat_problem(const HeatParams& p);

// ---- random_problems (proj/src/random_problems.cpp)
struct RandomProblemOptions {
  Index max_n_x = 3, max_n_u = 2, max_n_c = 0, max_T = 4;
  bool cap_rows_for_oracle = true;
  double bound_margin = 0.5;
  double spectral_radius_cap = 1.05;
  // builder extension for BASELINE config 1: fixed dimensions instead of the draw
  bool fixed_dims = false;
  Index n_x = 10, n_u = 2, n_c = 0, T = 10;
};
LqProblemData random_problem(std::mt19937_64& rng, const RandomProblemOptions& o);
std::mt19937_64 instance_rng(std::uint64_t seed, std::uint64_t index);

// ---- enumeration oracle (proj/src/oracle.cpp:34-112)
struct EnumResult {
  int status = 0;  // 0 optimal, 1 infeasible, 2 unbounded_guard
  Vec v;
  double objective = 0.0;
  std::vector<Index> active_set;
  Vec multipliers;
};
EnumResult solve_enumeration(const Mat& H, const Vec& h, double h0, const Mat& J, const Vec& d);

// ---- ipm (proj/src/ipm.cpp)
enum class IpmStatus { converged = 0, max_iter = 1, factorization_failure = 2, line_search_failure = 3 };
struct IpmState {
  Vec v, s, lambda, z;
  double mu = 0.0;
  Index iter = 0;
};
struct Residuals {
  Vec r1, r2, r3;
  double kkt_error = 0.0;
};
struct StepDirections {
  Vec pv, ps, plambda, pz;
};
struct IterationRecord {
  Index iter = 0;
  double mu = 0, alpha = 0, alpha_z = 0, kkt_error = 0, objective = 0;
  double delta = 0;   // extension: shift used
  int trial = 0;      // extension: accepted line-search trial j
};
struct IterationInspection {
  const IpmState& state;
  const Residuals& residuals;
  const StepDirections& dirs;
  double delta;
};
struct IpmOptions {
  double tol = 1e-8, mu_init = 1e-1, kappa_mu = 0.2, tau = 0.995;
  Index max_iter = 200;
  double armijo_eta = 1e-4;
  std::string backend = "reference";
  std::function<void(const IterationRecord&)> log;
  std::function<void(const IterationInspection&)> inspect;
};
struct IpmResult {
  IpmStatus status = IpmStatus::max_iter;
  Trajectory solution;
  Vec v, s, lambda, z;
  Index iter = 0;
  double kkt_error = 0, objective = 0, total_seconds = 0, linalg_seconds = 0;
};

Residuals compute_residuals(const DenseQp& qp, const IpmState& st);
Mat assemble_condensed(const DenseQp& qp, const Vec& sigma);
StepDirections step_directions(const DenseQp& qp, const IpmState& st, const Residuals& res,
                               const Mat& L);
void fraction_to_boundary(const Vec& s, const Vec& ps, const Vec& z, const Vec& pz, double tau,
                          double* alpha, double* alpha_z);
// returns accepted trial j (>=0) and alpha, or -1 when every trial fails
int line_search(const DenseQp& qp, const IpmState& st, const StepDirections& dirs, double alpha_max,
                const IpmOptions& opts, double* alpha);
double merit(const DenseQp& qp, const Vec& v, const Vec& s, double mu, double rho);
double update_barrier(const IpmState& st, const Residuals& res, const IpmOptions& opts);
int check_termination(const Residuals& res, const IpmState& st, const IpmOptions& opts);  // 0 conv, 1 max, 2 go
IpmResult solve(const DenseQp& qp, const IpmOptions& opts);

// number of OpenMP threads the dense kernels use (1 = the reference's single thread)
void set_threads(int n);
// test-speed switch: solve() skips J's all-zero 512-row column chunks in every J product
// (bitwise the same results for finite data; the timed CPU baseline leaves it off)
void set_skip_zeros(bool on);
bool get_skip_zeros();
int get_threads();

}  // namespace orc
