// ORACLE — TEST INFRASTRUCTURE ONLY. Flat C ABI over oracle_core for ctypes
// (oracle/oracle.py). Never linked by the product.
#include <cstring>
#include <string>

#include "oracle_core.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;
template <typename F>
int guard(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
Mat mat_from(const double* p, Index r, Index c) {
  Mat m(r, c);
  if (r * c > 0) std::memcpy(m.a.data(), p, sizeof(double) * size_t(r * c));
  return m;
}
Vec vec_from(const double* p, Index n) { return n > 0 ? Vec(p, p + n) : Vec(); }
void put(double* dst, const Vec& v) {
  if (!v.empty()) std::memcpy(dst, v.data(), sizeof(double) * v.size());
}
void put(double* dst, const Mat& m) {
  if (!m.a.empty()) std::memcpy(dst, m.a.data(), sizeof(double) * m.a.size());
}
IpmState state_from(Index n, Index m, const double* v, const double* s, const double* l,
                    const double* z, double mu) {
  IpmState st;
  st.v = vec_from(v, n);
  st.s = vec_from(s, m);
  st.lambda = vec_from(l, m);
  st.z = vec_from(z, m);
  st.mu = mu;
  return st;
}
}  // namespace

struct orc_rng {
  std::mt19937_64 r;
};
struct orc_problem {
  LqProblemData d;
};
struct orc_qp {
  DenseQp q;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int n) { set_threads(n); }
int orc_get_threads(void) { return get_threads(); }
void orc_set_skip_zeros(int on) { set_skip_zeros(on != 0); }

orc_rng* orc_rng_new(std::uint64_t seed) { return new orc_rng{std::mt19937_64(seed)}; }
orc_rng* orc_rng_instance(std::uint64_t seed, std::uint64_t index) {
  return new orc_rng{instance_rng(seed, index)};
}
void orc_rng_free(orc_rng* r) { delete r; }
double orc_rng_uniform(orc_rng* r, double lo, double hi) {
  std::uniform_real_distribution<double> d(lo, hi);
  return d(r->r);
}
std::int64_t orc_rng_int(orc_rng* r, std::int64_t lo, std::int64_t hi) {
  std::uniform_int_distribution<long> d(lo, hi);
  return d(r->r);
}

// opts_i: max_n_x, max_n_u, max_n_c, max_T, cap_rows, fixed_dims, n_x, n_u, n_c, T
// opts_d: bound_margin, spectral_radius_cap
orc_problem* orc_problem_random(orc_rng* rng, const std::int64_t* oi, const double* od) {
  orc_problem* out = nullptr;
  guard([&] {
    RandomProblemOptions o;
    o.max_n_x = oi[0];
    o.max_n_u = oi[1];
    o.max_n_c = oi[2];
    o.max_T = oi[3];
    o.cap_rows_for_oracle = oi[4] != 0;
    o.fixed_dims = oi[5] != 0;
    o.n_x = oi[6];
    o.n_u = oi[7];
    o.n_c = oi[8];
    o.T = oi[9];
    o.bound_margin = od[0];
    o.spectral_radius_cap = od[1];
    out = new orc_problem{random_problem(rng->r, o)};
    return 0;
  });
  return out;
}

// params: dt, dw, rho, cp, conductivity, q_weight, r_weight, x_min, x_max, u_min, u_max, x_init, setpoint
orc_problem* orc_problem_heat3d(std::int64_t N, std::int64_t T, const double* p) {
  orc_problem* out = nullptr;
  guard([&] {
    HeatParams hp;
    hp.N = N;
    hp.T = T;
    if (p) {
      hp.dt = p[0]; hp.dw = p[1]; hp.rho = p[2]; hp.cp = p[3]; hp.conductivity = p[4];
      hp.q_weight = p[5]; hp.r_weight = p[6]; hp.x_min = p[7]; hp.x_max = p[8];
      hp.u_min = p[9]; hp.u_max = p[10]; hp.x_init = p[11]; hp.setpoint = p[12];
    }
    out = new orc_problem{build_heat_problem(hp)};
    return 0;
  });
  return out;
}

int orc_laplacian_system(std::int64_t N, const double* p, double* A, double* B) {
  return guard([&] {
    HeatParams hp;
    if (p) {
      hp.dt = p[0]; hp.dw = p[1]; hp.rho = p[2]; hp.cp = p[3]; hp.conductivity = p[4];
    }
    Mat a, b;
    laplacian_system(N, hp, a, b);
    put(A, a);
    put(B, b);
    return 0;
  });
}

orc_problem* orc_problem_new(std::int64_t nx, std::int64_t nu, std::int64_t nc, std::int64_t T,
                             const double* A, const double* B, const double* Q, const double* Qf,
                             const double* R, const double* S, const double* E, const double* F,
                             const double* gl, const double* gu, const double* xl, const double* xu,
                             const double* ul, const double* uu, const double* w,
                             const double* x_bar, const double* K) {
  auto* p = new orc_problem;
  LqProblemData& d = p->d;
  d.A = mat_from(A, nx, nx);
  d.B = mat_from(B, nx, nu);
  d.Q = mat_from(Q, nx, nx);
  d.Qf = mat_from(Qf, nx, nx);
  d.R = mat_from(R, nu, nu);
  d.S = mat_from(S, nx, nu);
  d.E = mat_from(E, nc, nx);
  d.F = mat_from(F, nc, nu);
  d.gl = vec_from(gl, nc);
  d.gu = vec_from(gu, nc);
  d.xl = vec_from(xl, nx);
  d.xu = vec_from(xu, nx);
  d.ul = vec_from(ul, nu);
  d.uu = vec_from(uu, nu);
  d.w.clear();
  for (Index t = 0; t < T; ++t) d.w.push_back(vec_from(w + t * nx, nx));
  d.x_bar = vec_from(x_bar, nx);
  d.K = mat_from(K, nu, nx);
  d.T = T;
  return p;
}
void orc_problem_dims(const orc_problem* p, std::int64_t* out) {
  out[0] = p->d.A.r;
  out[1] = p->d.B.c;
  out[2] = p->d.E.r;
  out[3] = p->d.T;
}
int orc_problem_get(const orc_problem* p, const char* f, double* out) {
  const LqProblemData& d = p->d;
  const std::string k(f);
  if (k == "A") put(out, d.A);
  else if (k == "B") put(out, d.B);
  else if (k == "Q") put(out, d.Q);
  else if (k == "Qf") put(out, d.Qf);
  else if (k == "R") put(out, d.R);
  else if (k == "S") put(out, d.S);
  else if (k == "E") put(out, d.E);
  else if (k == "F") put(out, d.F);
  else if (k == "K") put(out, d.K);
  else if (k == "gl") put(out, d.gl);
  else if (k == "gu") put(out, d.gu);
  else if (k == "xl") put(out, d.xl);
  else if (k == "xu") put(out, d.xu);
  else if (k == "ul") put(out, d.ul);
  else if (k == "uu") put(out, d.uu);
  else if (k == "x_bar") put(out, d.x_bar);
  else if (k == "w") {
    for (size_t t = 0; t < d.w.size(); ++t) put(out + t * d.w[t].size(), d.w[t]);
  } else return -1;
  return 0;
}
void orc_problem_free(orc_problem* p) { delete p; }

orc_qp* orc_build_dense_qp(const orc_problem* p) {
  orc_qp* out = nullptr;
  guard([&] {
    out = new orc_qp{build_dense_qp(p->d)};
    return 0;
  });
  return out;
}
orc_qp* orc_qp_new(std::int64_t n, std::int64_t m, const double* H, const double* h, double h0,
                   const double* J, const double* d) {
  auto* q = new orc_qp;
  q->q.H = mat_from(H, n, n);
  q->q.h = vec_from(h, n);
  q->q.h0 = h0;
  q->q.J = mat_from(J, m, n);
  q->q.d = vec_from(d, m);
  q->q.has_source = false;
  return q;
}
void orc_qp_dims(const orc_qp* q, std::int64_t* out) {
  out[0] = q->q.H.r;
  out[1] = q->q.J.r;
}
int orc_qp_get(const orc_qp* q, const char* f, double* out) {
  const std::string k(f);
  if (k == "H") put(out, q->q.H);
  else if (k == "h") put(out, q->q.h);
  else if (k == "h0") out[0] = q->q.h0;
  else if (k == "J") put(out, q->q.J);
  else if (k == "d") put(out, q->q.d);
  else if (k == "bigB") put(out, q->q.blocks.bigB);
  else return -1;
  return 0;
}
int orc_qp_refresh(orc_qp* q, const double* x_bar) {
  return guard([&] {
    refresh_initial_state(q->q, vec_from(x_bar, Index(q->q.source.x_bar.size())));
    return 0;
  });
}
int orc_qp_recover(const orc_qp* q, const double* v, double* xs, double* us, double* obj) {
  return guard([&] {
    const Trajectory tr = recover_trajectory(q->q, vec_from(v, q->q.H.r));
    size_t o = 0;
    for (const auto& x : tr.x) {
      put(xs + o, x);
      o += x.size();
    }
    o = 0;
    for (const auto& u : tr.u) {
      put(us + o, u);
      o += u.size();
    }
    *obj = tr.objective;
    return 0;
  });
}
double orc_dense_objective(const orc_qp* q, const double* v) {
  return dense_objective(q->q, vec_from(v, q->q.H.r));
}
void orc_qp_free(orc_qp* q) { delete q; }

int orc_compute_residuals(const orc_qp* q, const double* v, const double* s, const double* l,
                          const double* z, double mu, double* r1, double* r2, double* r3,
                          double* kkt) {
  return guard([&] {
    const Index n = q->q.H.r, m = q->q.J.r;
    const Residuals r = compute_residuals(q->q, state_from(n, m, v, s, l, z, mu));
    put(r1, r.r1);
    put(r2, r.r2);
    put(r3, r.r3);
    *kkt = r.kkt_error;
    return 0;
  });
}
int orc_assemble_condensed(const orc_qp* q, const double* sigma, double* M) {
  return guard([&] {
    put(M, assemble_condensed(q->q, vec_from(sigma, q->q.J.r)));
    return 0;
  });
}
int orc_gram_weighted(std::int64_t m, std::int64_t n, const double* J, const double* sigma,
                      std::int64_t sigma_len, double* G) {
  return guard([&] {
    put(G, gram_weighted(mat_from(J, m, n), vec_from(sigma, sigma_len)));
    return 0;
  });
}
// 0 ok, 1 not positive definite (pivot), -1 error
int orc_factorize(const char* backend, std::int64_t n, const double* M, double* L,
                  std::int64_t* pivot) {
  try {
    put(L, factorize(backend, mat_from(M, n, n)));
    return 0;
  } catch (const NotPositiveDefinite& e) {
    *pivot = e.pivot;
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
int orc_factor_solve(std::int64_t n, const double* L, const double* b, std::int64_t blen,
                     double* x) {
  return guard([&] {
    put(x, factor_solve(mat_from(L, n, n), vec_from(b, blen)));
    return 0;
  });
}
int orc_step_directions(const orc_qp* q, const double* v, const double* s, const double* l,
                        const double* z, double mu, const double* r1, const double* r2,
                        const double* r3, const double* L, double* pv, double* ps, double* pl,
                        double* pz) {
  return guard([&] {
    const Index n = q->q.H.r, m = q->q.J.r;
    Residuals r;
    r.r1 = vec_from(r1, n);
    r.r2 = vec_from(r2, m);
    r.r3 = vec_from(r3, m);
    const StepDirections d =
        step_directions(q->q, state_from(n, m, v, s, l, z, mu), r, mat_from(L, n, n));
    put(pv, d.pv);
    put(ps, d.ps);
    put(pl, d.plambda);
    put(pz, d.pz);
    return 0;
  });
}
int orc_fraction_to_boundary(std::int64_t m, const double* s, const double* ps, const double* z,
                             const double* pz, double tau, double* out) {
  return guard([&] {
    fraction_to_boundary(vec_from(s, m), vec_from(ps, m), vec_from(z, m), vec_from(pz, m), tau,
                         &out[0], &out[1]);
    return 0;
  });
}
// returns accepted trial (>=0), -2 when every trial fails, -1 on error
int orc_line_search(const orc_qp* q, const double* v, const double* s, const double* l,
                    const double* z, double mu, const double* pv, const double* ps,
                    const double* pl, const double* pz, double alpha_max, double eta,
                    double* alpha) {
  try {
    const Index n = q->q.H.r, m = q->q.J.r;
    StepDirections d;
    d.pv = vec_from(pv, n);
    d.ps = vec_from(ps, m);
    d.plambda = vec_from(pl, m);
    d.pz = vec_from(pz, m);
    IpmOptions o;
    o.armijo_eta = eta;
    const int j = line_search(q->q, state_from(n, m, v, s, l, z, mu), d, alpha_max, o, alpha);
    return j < 0 ? -2 : j;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
double orc_merit(const orc_qp* q, const double* v, const double* s, double mu, double rho) {
  return merit(q->q, vec_from(v, q->q.H.r), vec_from(s, q->q.J.r), mu, rho);
}

typedef void (*orc_log_fn)(void* user, const double* rec);
typedef void (*orc_inspect_fn)(void* user, const double* v, const double* s, const double* l,
                               const double* z, double mu, const double* r1, const double* r2,
                               const double* r3, double kkt, const double* pv, const double* ps,
                               const double* pl, const double* pz, double delta);

// opts_d: tol, mu_init, kappa_mu, tau, armijo_eta. scal_out (8): status, iter, kkt, objective,
// total_seconds, linalg_seconds, solution_objective, has_solution. xs/us optional (trajectory).
int orc_solve(const orc_qp* q, const double* od, std::int64_t max_iter, const char* backend,
              double* v, double* s, double* l, double* z, double* scal, double* xs, double* us,
              orc_log_fn logf, orc_inspect_fn inspf, void* user) {
  return guard([&] {
    IpmOptions o;
    o.tol = od[0];
    o.mu_init = od[1];
    o.kappa_mu = od[2];
    o.tau = od[3];
    o.armijo_eta = od[4];
    o.max_iter = max_iter;
    o.backend = backend;
    if (logf) {
      o.log = [&](const IterationRecord& r) {
        const double rec[8] = {double(r.iter), r.mu, r.alpha, r.alpha_z,
                               r.kkt_error,    r.objective, r.delta, double(r.trial)};
        logf(user, rec);
      };
    }
    if (inspf) {
      o.inspect = [&](const IterationInspection& in) {
        inspf(user, in.state.v.data(), in.state.s.data(), in.state.lambda.data(), in.state.z.data(),
              in.state.mu, in.residuals.r1.data(), in.residuals.r2.data(), in.residuals.r3.data(),
              in.residuals.kkt_error, in.dirs.pv.data(), in.dirs.ps.data(), in.dirs.plambda.data(),
              in.dirs.pz.data(), in.delta);
      };
    }
    const IpmResult r = solve(q->q, o);
    put(v, r.v);
    put(s, r.s);
    put(l, r.lambda);
    put(z, r.z);
    scal[0] = double(int(r.status));
    scal[1] = double(r.iter);
    scal[2] = r.kkt_error;
    scal[3] = r.objective;
    scal[4] = r.total_seconds;
    scal[5] = r.linalg_seconds;
    scal[6] = r.solution.objective;
    scal[7] = r.solution.x.empty() ? 0.0 : 1.0;
    if (!r.solution.x.empty() && xs && us) {
      size_t o2 = 0;
      for (const auto& x : r.solution.x) {
        put(xs + o2, x);
        o2 += x.size();
      }
      o2 = 0;
      for (const auto& u : r.solution.u) {
        put(us + o2, u);
        o2 += u.size();
      }
    }
    return 0;
  });
}

// returns status (0 optimal, 1 infeasible, 2 unbounded_guard) or -1
int orc_solve_enumeration(const orc_qp* q, double* v, double* obj, std::int64_t* active,
                          std::int64_t* nactive, double* mult) {
  return guard([&] {
    const EnumResult r = solve_enumeration(q->q.H, q->q.h, q->q.h0, q->q.J, q->q.d);
    put(v, r.v);
    *obj = r.objective;
    *nactive = Index(r.active_set.size());
    for (size_t i = 0; i < r.active_set.size(); ++i) active[i] = r.active_set[i];
    put(mult, r.multipliers);
    return r.status;
  });
}

}  // extern "C"
