// The IPM outer loop on the host (C++), driving the device kernels through the launchers
// of internal.cuh. Restates condmpc::ipm::solve (proj/src/ipm.cpp:160-268) decision for
// decision: termination (:153-158), monotone barrier (:146-151), the shift ladder
// (:205-221), fraction to boundary (:105-116), backtracking Armijo with the roundoff band
// (:118-144). The device returns small scalar packets; every branch is evaluated here with
// the reference's rule on the same scalars.
//
// Two host syncs per iteration in the common case:
//   A: after the residual pass (kkt -> termination and barrier decisions)
//   B: after condense + Cholesky + solve + recovery + trial 0 (info, alpha_max, merit)
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <stdexcept>
#include <vector>

#include "../../include/condmpc_cuda.h"
#include "internal.cuh"

namespace cmpc {

namespace {
double now_seconds() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void require(bool c, const char* m) {
  if (!c) throw DimError(m);
}
// wait for publish number `seq` (k_publish wrote the packet into mapped host memory first):
// a spin on the mapped word instead of a stream synchronize plus a D2H copy; the stream is
// polled now and then so a device error surfaces instead of hanging
void wait_published(Ctx& c, unsigned long long seq, long long* syncs) {
  for (long spins = 0;; ++spins) {
    if (*c.pub_host >= seq) break;
    // after the first microseconds, give the core back now and then: with as many solving
    // threads as cores (batch mode) a pure spin starves the driver's own threads
    if (spins > 4096) std::this_thread::yield();
    if ((spins & 0xfff) == 0xfff) {
      const cudaError_t e = cudaStreamQuery(c.stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) CMPC_CUDA(e);
      if (e == cudaSuccess && *c.pub_host < seq)
        throw CudaError("packet publish lost (stream idle, sequence not reached)");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  if (syncs) ++*syncs;
}
void sync_packet(Ctx& c, long long* syncs) { wait_published(c, launch_publish(c), syncs); }
}  // namespace

void drop_graphs(Ctx& c) {
  if (c.g_step) cudaGraphExecDestroy(c.g_step);
  if (c.g_next) cudaGraphExecDestroy(c.g_next);
  c.g_step = c.g_next = nullptr;
  c.g_step_nodes = c.g_next_nodes = 0;
}

namespace {

// timing event: a plain record, or an external event-record node while capturing
void rec(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CMPC_CUDA(cudaStreamIsCapturing(s, &st));
  if (st == cudaStreamCaptureStatusActive)
    CMPC_CUDA(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
  else
    CMPC_CUDA(cudaEventRecord(e, s));
}

// segment A: sigma/omega/q, condensation with the right-hand side J'(r2 - sigma r3) fused
// into the SYRK (its diagonal jobs stream every nonzero row of P), Cholesky (delta = 0)
// fused with the solve, recovery + fraction to boundary, trial 0 and the device's verdict on
// it (trial0_decide), published into the second packet slot
void seg_step(Ctx& c, double tau, double eta) {
  NvtxRange nv("cmpc: condense + factor + step + trial 0");
  rec(c.ev0, c.stream);
  launch_prepare_step(c, nullptr);
  // right-hand side P'q fused into the SYRK's diagonal jobs (with the plan's step weights
  // accounting for it: +4% of the SYRK at n = 500, +2% at n = 2000, against 14% and 3% for a
  // separate pass over P; tools/phases.py condense vs condense_rhs vs Jty).
  // option "rhs_pass" = 2 forces the separate pass (tests/test_gpu_jtl_recurrence.py)
  const bool fused = c.ps > 0 && c.npieces > 0 && c.opt_rhs_pass != 2;
  if (!fused) launch_rhs_partial(c);  // J'(r2 - sigma r3) by its own pass over P
  rec(c.ev2, c.stream);
  launch_condense(c, false, fused, c.ev4);
  rec(c.ev3, c.stream);
  if (c.comm) {  // M = H + sum_g J_g' Sigma_g J_g and J' (r2 - sigma r3) over all ranks
    // only the lower triangle is formed (and factored): it travels packed, n (n + 1) / 2
    launch_pack_lower(c, c.M, c.Mpack, true);
    comm_group(c, true);
    comm_allreduce(c, c.Mpack, (size_t)(c.n * (c.n + 1) / 2), CommType::f64, CommOp::sum);
    comm_allreduce(c, c.tq, (size_t)c.n, CommType::f64, CommOp::sum);
    comm_group(c, false);
    launch_pack_lower(c, c.M, c.Mpack, false);
  }
  if (c.comm || !fused) launch_rhs_final(c);  // (unsharded + fused: done by k_syrk_reduce)
  launch_debug_sum(c, c.M, c.n * c.n, 0);
  launch_debug_sum(c, c.rhs, c.n, 1);
  launch_debug_sum(c, c.omega, c.ldp + c.pz, 4);
  launch_cholesky(c, c.M, c.L, 0.0, c.rhs, c.pv);  // factor + both triangular solves
  launch_debug_sum(c, c.pv, c.n, 2);
  launch_debug_sum(c, c.L, c.n * c.n, 5);
  rec(c.ev1, c.stream);
  launch_recover(c, tau);
  launch_debug_sum(c, c.ps_, c.m, 3);
  launch_trial(c, 0.0, true, /*linear=*/true, /*decide=*/true, eta, /*publish into slot B=*/1);
}

// seg_next may run gated on the device's trial-0 verdict: every kernel in it then checks it
bool seg_next_gated(const Ctx& c) { return !c.comm && (c.m == 0 || c.jtl_recur); }

// segment B: the accepted step (alpha, alpha_z on the device) and the residuals after it;
// nothing runs when d_alpha[2] = 0 (a speculative launch whose trial 0 the device refused)
void seg_next(Ctx& c) {
  NvtxRange nv("cmpc: update + residuals");
  launch_update_dev(c);
  launch_residuals(c, /*reuse_trial=*/true, /*gated=*/seg_next_gated(c), /*publish into slot A=*/0);
}

// run a segment eagerly, or capture it once into a CUDA graph and replay it
template <typename F>
void run_segment(Ctx& c, cudaGraphExec_t& exec, long long& nodes, bool allow_capture, F&& seg) {
  if (exec) {
    CMPC_CUDA(cudaGraphLaunch(exec, c.stream));
    g_launches += nodes;
    ++c.pub_expect;  // every segment graph ends with one k_publish
    return;
  }
  // (a loopback communicator synchronizes the ranks' streams with events across contexts,
  // which a per-context capture cannot hold)
  if (!allow_capture || c.comm_loop || !c.opt_graphs) {
    seg();
    return;
  }
  cudaGraph_t graph = nullptr;
  const long long l0 = g_launches;
  // the captured k_publish advances pub_expect although nothing runs until the launch below:
  // a capture that fails puts it back, or every later wait would be for a publish that never comes
  const unsigned long long pub0 = c.pub_expect;
  CMPC_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  try {
    seg();
    CMPC_CUDA(cudaStreamEndCapture(c.stream, &graph));
    nodes = g_launches - l0;
    g_launches = l0;
    CMPC_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  } catch (...) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(c.stream, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
      cudaGraph_t g2 = nullptr;
      cudaStreamEndCapture(c.stream, &g2);
      if (g2) cudaGraphDestroy(g2);
    }
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    c.pub_expect = pub0;
    g_launches = l0;
    throw;
  }
  cudaGraphDestroy(graph);
  CMPC_CUDA(cudaGraphLaunch(exec, c.stream));
  g_launches += nodes;
}

}  // namespace

// merit phi(v, s) = 0.5 v'Hv + h'v - mu sum log s + rho |Jv - d + s|_1 (ipm.cpp:25-32)
double merit_host(const Packet&, double vhv, double hv, double sum_log, double sum_abs, double mu,
                  double rho, bool has_rows) {
  double phi = 0.5 * vhv + hv;
  if (has_rows) {
    phi -= mu * sum_log;
    phi += rho * sum_abs;
  }
  return phi;
}

namespace {

// the accept loop of line_search (ipm.cpp:129-143). `A` holds the residual packet at the
// current state, `dg`/`dps` the derivative pieces; trial 0 may already be evaluated.
int run_line_search(Ctx& c, const Packet& A, double dg, double dps, double alpha_max, double eta,
                    const Packet* trial0, double* alpha_out, int* ntrials, long long* syncs) {
  const bool rows = rows_all(c) > 0;
  const double rho = 10.0 * A.max_lam + 1.0;
  const double phi0 = merit_host(A, A.obj_vHv, A.obj_hv, A.sum_log_s, A.sum_abs_r3, c.mu, rho, rows);
  double derivative = dg;
  if (rows) {
    derivative -= c.mu * dps;
    derivative -= rho * A.sum_abs_r3;
  }
  constexpr double band = 10.0 * std::numeric_limits<double>::epsilon();
  double alpha = alpha_max;
  for (int j = 0; j <= 30; ++j, alpha *= 0.5) {
    Packet T;
    if (j == 0 && trial0) {
      T = *trial0;
    } else {
      launch_trial(c, alpha, false, /*linear=*/true);
      sync_packet(c, syncs);
      T = *c.pk_host;
    }
    ++*ntrials;
    if (rows && T.any_nonpos) continue;
    const double phi = merit_host(T, T.t_vHv, T.t_hv, T.t_sum_log, T.t_sum_abs, c.mu, rho, rows);
    if (derivative <= 0.0 && phi <= phi0 + eta * alpha * derivative) {
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

}  // namespace

int line_search_host(Ctx& c, double alpha_max, double eta, double* alpha, int* ntrials) {
  const Packet A = *c.pk_host;  // residuals + derivative pieces already in the packet
  // the trials use P v (from the residual pass) and P pv: the direction may have been set
  // from the host, so form P pv here
  launch_Jx(c, c.pv, c.y, nullptr);
  return run_line_search(c, A, A.d_gpv, A.d_ps_s, alpha_max, eta, nullptr, alpha, ntrials, nullptr);
}

int solve_loop(Ctx& c, const double* opts, int64_t max_iter, double* v_out, double* s_out,
               double* lam_out, double* z_out, double* out, cmpc_log_fn log,
               cmpc_inspect_fn inspect, void* user) {
  const double tol = opts[0], mu_init = opts[1], kappa_mu = opts[2], tau = opts[3],
               eta = opts[4];
  // check_options (ipm.cpp:17-23)
  require(tol > 0.0, "tol must be positive");
  require(kappa_mu > 0.0 && kappa_mu < 1.0, "kappa_mu must lie in (0,1)");
  require(tau > 0.0 && tau < 1.0, "tau must lie in (0,1)");
  require(mu_init > 0.0, "mu_init must be positive");
  require(max_iter >= 1, "max_iter must be at least 1");

  NvtxRange nv_solve("cmpc_solve");
  // QPs that fit in one CTA's shared memory: the whole loop on the device (small.cu)
  if (!inspect && c.opt_small && c.Jsmall && !c.comm)
    return small_solve(c, opts, max_iter, v_out, s_out, lam_out, z_out, out, log, user);
  const long long launches0 = g_launches;
  long long syncs = 0, trials = 0;
  const int64_t n = c.n, m = c.m;
  const double start = now_seconds();
  double linalg = 0.0, device_s = 0.0, syrk_s = 0.0, chol_s = 0.0, syrk_k = 0.0;
  long long syrk_launches = 0;
  cudaEvent_t e_start, e_end;
  CMPC_CUDA(cudaEventCreate(&e_start));
  CMPC_CUDA(cudaEventCreate(&e_end));
  CMPC_CUDA(cudaEventRecord(e_start, c.stream));
  static const bool tverb = getenv("CMPC_SOLVE_TIMES") != nullptr;
  const double t_es = now_seconds();

  // init (ipm.cpp:170-177)
  set_mu(c, mu_init);
  launch_init_state(c, c.mu);
  if (c.g_tau != tau || c.g_eta != eta) drop_graphs(c);
  c.g_tau = tau;
  c.g_eta = eta;
  // speculation: seg_next is enqueued right behind seg_step and applies the step only if the
  // device accepted trial 0; an inspect hook needs the state before the step, a communicator
  // allreduces the trial's sums after the verdict would be taken
  const bool spec = c.opt_spec && !inspect && seg_next_gated(c);
  // from here every segment ends in k_publish, which also resets the packet's accumulated
  // maxima / minima: the per-phase reset kernels drop out of the iteration graphs
  launch_reset_packet_all(c);
  struct AutoReset {
    Ctx& c;
    explicit AutoReset(Ctx& cc) : c(cc) { c.pk_autoreset = true; }
    ~AutoReset() { c.pk_autoreset = false; }
  } auto_reset(c);
  launch_residuals(c);
  sync_packet(c, &syncs);
  Packet A = *c.pk_host;
  int64_t iter = 0;
  int status = 1;
  static constexpr std::array<double, 7> kShifts = {0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1.0, 1e2};

  std::vector<double> hv, hs, hl, hz, h1, h2, h3, hpv, hps, hpl, hpz;
  if (inspect) {
    hv.resize(size_t(n)); h1.resize(size_t(n)); hpv.resize(size_t(n));
    for (auto* x : {&hs, &hl, &hz, &h2, &h3, &hps, &hpl, &hpz}) x->resize(size_t(m));
  }

  // CMPC_GAP_TRACE: device-timeline gaps between a segment's end and the next enqueue
  const bool gap_trace = getenv("CMPC_GAP_TRACE") != nullptr;
  cudaEvent_t g_end = nullptr, g_beg = nullptr;
  double gap_ms = 0.0;
  long gap_n = 0;
  if (gap_trace) {
    CMPC_CUDA(cudaEventCreate(&g_end));
    CMPC_CUDA(cudaEventCreate(&g_beg));
  }
  auto gap_mark_end = [&] {
    if (gap_trace) CMPC_CUDA(cudaEventRecord(g_end, c.stream));
  };
  auto gap_mark_begin = [&] {
    if (!gap_trace) return;
    CMPC_CUDA(cudaEventRecord(g_beg, c.stream));
    CMPC_CUDA(cudaEventSynchronize(g_beg));
    float ms = 0.f;
    CMPC_CUDA(cudaEventElapsedTime(&ms, g_end, g_beg));
    gap_ms += ms;
    ++gap_n;
  };
  gap_mark_end();
  while (true) {
    NvtxRange nv_iter("cmpc: IPM iteration");
    // check_termination (ipm.cpp:153-158)
    if (A.kkt <= tol && c.mu <= tol) {
      status = 0;
      break;
    }
    if (iter >= max_iter) {
      status = 1;
      break;
    }
    // update_barrier (ipm.cpp:146-151)
    const double mu_next = (A.kkt <= 10.0 * c.mu) ? std::max(tol / 10.0, kappa_mu * c.mu) : c.mu;
    if (mu_next != c.mu) {
      set_mu(c, mu_next);
      launch_residuals_mu(c, A);
    }
    // sigma, condensed matrix, factorization with the shift ladder (ipm.cpp:200-226), then
    // speculatively: directions, recovery, fraction to boundary, line-search trial 0
    size_t shift = 0;
    gap_mark_begin();
    run_segment(c, c.g_step, c.g_step_nodes, iter >= 1, [&] { seg_step(c, tau, eta); });
    if (spec) run_segment(c, c.g_next, c.g_next_nodes, iter >= 1, [&] { seg_next(c); });
    gap_mark_end();
    wait_published(c, c.pub_expect, &syncs);
    float ms = 0.f;
    CMPC_CUDA(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
    linalg += ms * 1e-3;
    CMPC_CUDA(cudaEventElapsedTime(&ms, c.ev2, c.ev3));
    syrk_s += ms * 1e-3;
    CMPC_CUDA(cudaEventElapsedTime(&ms, c.ev2, c.ev4));
    syrk_k += ms * 1e-3;
    ++syrk_launches;
    CMPC_CUDA(cudaEventElapsedTime(&ms, c.ev3, c.ev1));
    chol_s += ms * 1e-3;
    Packet B = *c.pk_host_b;
    if (spec && B.pad[6] != 0.0) {  // the device took trial 0: the step is already applied
      const double alpha_max = std::min(1.0, B.alpha_s_min);
      double alpha = 0.0;
      int nt = 0;
      // the host's own verdict on the same packet (no launch when it agrees)
      const int j = run_line_search(c, A, B.d_gpv, B.d_ps_s, alpha_max, eta, &B, &alpha, &nt, &syncs);
      if (j != 0 || alpha != alpha_max)
        throw CudaError("speculative step: the device accepted line-search trial 0, the host did not");
      trials += nt;
      const double mu_used = c.mu;
      iter += 1;
      A = *c.pk_host;
      if (log) {
        const double rec[8] = {double(iter), mu_used, alpha, std::min(1.0, B.alpha_z_min), A.kkt, A.objective, 0.0, 0.0};
        log(user, rec);
      }
      continue;
    }
    while (B.info != 0) {
      if (++shift == kShifts.size()) break;
      CMPC_CUDA(cudaEventRecord(c.ev0, c.stream));
      launch_cholesky(c, c.M, c.L, kShifts[shift], c.rhs, c.pv);
      CMPC_CUDA(cudaEventRecord(c.ev1, c.stream));
      launch_recover(c, tau);
      launch_trial(c, 0.0, true, /*linear=*/true);
      sync_packet(c, &syncs);
      B = *c.pk_host;
      CMPC_CUDA(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
      linalg += ms * 1e-3;
    }
    static const bool debug_sums = getenv("CMPC_DEBUG_SUMS") != nullptr;
    if (debug_sums) {  // per-iteration checksums of the step's buffers (tools/race_sums.py)
      const unsigned long long* u = reinterpret_cast<const unsigned long long*>(B.pad);
      fprintf(stderr, "[sums] %p %d M %016llx rhs %016llx pv %016llx ps %016llx omega %016llx L %016llx\n", (void*)&c, (int)iter, u[0], u[1], u[2], u[3], u[4], u[5]);
    }
    A.kkt = B.kkt;  // kkt at the (possibly new) barrier value, as the reference's res
    A.max_comp = B.max_comp;
    if (shift == kShifts.size()) {
      status = 2;
      break;
    }
    const double delta = kShifts[shift];

    if (inspect) {
      const std::pair<double*, const double*> cp[] = {
          {hv.data(), c.v}, {h1.data(), c.r1}, {hpv.data(), c.pv}};
      for (auto& pr : cp)
        if (n > 0) CMPC_CUDA(cudaMemcpyAsync(pr.first, pr.second, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
      const std::pair<double*, const double*> cm[] = {{hs.data(), c.s},   {hl.data(), c.lam},
                                                      {hz.data(), c.z},   {h2.data(), c.r2},
                                                      {h3.data(), c.r3},  {hps.data(), c.ps_},
                                                      {hpl.data(), c.pl}, {hpz.data(), c.pzd}};
      for (auto& pr : cm)
        if (m > 0) CMPC_CUDA(cudaMemcpyAsync(pr.first, pr.second, sizeof(double) * m, cudaMemcpyDeviceToHost, c.stream));
      CMPC_CUDA(cudaStreamSynchronize(c.stream));
      ++syncs;
      inspect(user, hv.data(), hs.data(), hl.data(), hz.data(), c.mu, h1.data(), h2.data(),
              h3.data(), B.kkt, hpv.data(), hps.data(), hpl.data(), hpz.data(), delta);
    }

    const double alpha_max = std::min(1.0, B.alpha_s_min);
    const double alpha_z = std::min(1.0, B.alpha_z_min);
    double alpha = 0.0;
    int nt = 0;
    const int j = run_line_search(c, A, B.d_gpv, B.d_ps_s, alpha_max, eta, &B, &alpha, &nt, &syncs);
    trials += nt;
    if (j < 0) {
      status = 3;
      break;
    }
    const double mu_used = c.mu;
    set_alpha(c, alpha, alpha_z);
    iter += 1;
    gap_mark_begin();
    run_segment(c, c.g_next, c.g_next_nodes, iter >= 2, [&] { seg_next(c); });
    gap_mark_end();
    wait_published(c, c.pub_expect, &syncs);
    A = *c.pk_host;
    if (log) {
      const double rec[8] = {double(iter), mu_used, alpha, alpha_z, A.kkt, A.objective, delta, double(j)};
      log(user, rec);
    }
  }

  if (gap_trace) {
    fprintf(stderr, "[cmpc gaps] %ld host turnarounds, %.1f us average\n", gap_n,
            gap_n ? gap_ms * 1e3 / gap_n : 0.0);
    cudaEventDestroy(g_end);
    cudaEventDestroy(g_beg);
  }
  const double t_loop = now_seconds();
  if (v_out && n > 0) CMPC_CUDA(cudaMemcpyAsync(v_out, c.v, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
  if (m > 0) {
    if (s_out) CMPC_CUDA(cudaMemcpyAsync(s_out, c.s, sizeof(double) * m, cudaMemcpyDeviceToHost, c.stream));
    if (lam_out) CMPC_CUDA(cudaMemcpyAsync(lam_out, c.lam, sizeof(double) * m, cudaMemcpyDeviceToHost, c.stream));
    if (z_out) CMPC_CUDA(cudaMemcpyAsync(z_out, c.z, sizeof(double) * m, cudaMemcpyDeviceToHost, c.stream));
  }
  const double t_copy = now_seconds();
  CMPC_CUDA(cudaEventRecord(e_end, c.stream));
  CMPC_CUDA(cudaStreamSynchronize(c.stream));
  if (tverb)
    fprintf(stderr, "[cmpc solve] to e_start %.3f ms, loop %.3f, copies %.3f, sync %.3f\n",
            (t_es - start) * 1e3, (t_loop - t_es) * 1e3, (t_copy - t_loop) * 1e3, (now_seconds() - t_copy) * 1e3);
  float dms = 0.f;
  CMPC_CUDA(cudaEventElapsedTime(&dms, e_start, e_end));
  device_s = dms * 1e-3;
  cudaEventDestroy(e_start);
  cudaEventDestroy(e_end);
  out[0] = status;
  out[1] = double(iter);
  out[2] = A.kkt;
  out[3] = A.objective;
  out[4] = now_seconds() - start;
  out[5] = linalg;
  out[6] = device_s;
  out[7] = double(g_launches - launches0);
  out[8] = double(syncs);
  out[9] = double(trials);
  out[10] = syrk_s;
  out[11] = chol_s;
  out[12] = double(syrk_launches);
  out[13] = syrk_k;
  return CMPC_OK;
}

}  // namespace cmpc
