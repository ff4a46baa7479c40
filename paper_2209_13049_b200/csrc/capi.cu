// C ABI (include/condmpc_cuda.h): context lifecycle, QP upload, per-step entry points and
// the stand-alone linear algebra of the reference's plug point.
#include <atomic>
#include <csignal>
#include <execinfo.h>
#include <unistd.h>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/condmpc_cuda.h"
#include "internal.cuh"

namespace cmpc {
thread_local long long g_launches = 0;

void pool_init(int device) {
  static std::once_flag flags[kMaxDevices];
  once_per_device(flags, device, [&] {
    cudaMemPool_t pool;
    CMPC_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    unsigned long long keep = ~0ull;  // never hand cached pages back to the OS
    CMPC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  });
}
thread_local std::string g_error;

// host loop (ipm_host.cpp)
int solve_loop(Ctx& c, const double* opts, int64_t max_iter, double* v, double* s, double* lam,
               double* z, double* out, cmpc_log_fn log, cmpc_inspect_fn inspect, void* user);
void drop_graphs(Ctx& c);
int line_search_host(Ctx& c, double alpha_max, double eta, double* alpha, int* ntrials);
double merit_host(const Packet& A, double vhv, double hv, double sum_log, double sum_abs,
                  double mu, double rho, bool has_rows);
}  // namespace cmpc

using namespace cmpc;

struct cmpc_ctx {
  Ctx c;
};

namespace {

template <typename F>
int guard(F&& f) {
  try {
    return f();
  } catch (const DimError& e) {
    g_error = e.what();
    return CMPC_ERR_DIM;
  } catch (const CudaError& e) {
    g_error = e.what();
    return CMPC_ERR_CUDA;
  } catch (const std::exception& e) {
    g_error = e.what();
    return CMPC_ERR_ARG;
  }
}

void sync(Ctx& c) { CMPC_CUDA(cudaStreamSynchronize(c.stream)); }

void d2h(Ctx& c, double* dst, const double* src, int64_t count) {
  if (dst && count > 0)
    CMPC_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyDeviceToHost, c.stream));
}
void h2d(Ctx& c, double* dst, const double* src, int64_t count) {
  if (src && count > 0) upload_h2d(dst, src, sizeof(double) * count, c.stream);
}

void read_packet(Ctx& c) {
  CMPC_CUDA(cudaMemcpyAsync(c.pk_host, c.pk, sizeof(Packet), cudaMemcpyDeviceToHost, c.stream));
  sync(c);
}

void release_qp(Ctx& c) {
  drop_graphs(c);
  vec_free(c);
  syrk_free(c);
  free_structure(c);
  markov_free(c);
  for (double* p : {c.H, c.h, c.d, c.Jsmall, c.small_log, c.small_res}) dev_free(p, c.stream);
  if (c.J && c.owns_J) dev_free(c.J, c.stream);
  c.H = c.h = c.J = c.d = c.Jsmall = c.small_log = c.small_res = nullptr;
  c.small_log_cap = 0;
  c.n = c.m = 0;
}

void require_loaded(Ctx& c) {
  if (!c.pk) throw DimError("no QP loaded on this context");
}

}  // namespace

// Diagnostics: CMPC_SEGV_TRACE=1 prints the native stack on SIGSEGV (addr2line-able offsets)
namespace {
void segv_trace(int sig) {
  void* frames[64];
  const int k = backtrace(frames, 64);
  backtrace_symbols_fd(frames, k, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct SegvInstall {
  SegvInstall() {
    if (getenv("CMPC_SEGV_TRACE")) signal(SIGSEGV, segv_trace);
  }
} g_segv_install;
}  // namespace

namespace {
// load a QP into the context; adopt = take ownership of the device buffers H, h, J, d
// (the device builder) instead of copying them
int load_impl(Ctx& c, int64_t n, int64_t m, const double* H, const double* h, double h0,
              const double* J, const double* d, int on_device, bool adopt) {
  return guard([&] {
    if (n < 0 || m < 0) throw DimError("negative dimensions");
    if (m > (int64_t(1) << 29) || n > (int64_t(1) << 24)) throw DimError("QP too large");
    CMPC_CUDA(cudaSetDevice(c.device));
    NvtxRange nv("cmpc_load_qp (upload, structure analysis, SYRK plan)");
    const double t_in = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    release_qp(c);
    if (getenv("CMPC_VERBOSE"))
      fprintf(stderr, "[cmpc load] release    %8.2f ms\n",
              (std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - t_in) * 1e3);
    c.n = n;
    c.m = m;
    c.h0 = h0;
    const auto kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    c.owns_J = true;
    if (adopt) {
      c.H = const_cast<double*>(H);
      c.h = const_cast<double*>(h);
      c.J = const_cast<double*>(J);
      c.d = const_cast<double*>(d);
    } else {
      c.H = dev_alloc<double>((size_t)(n * n), c.stream);
      c.h = dev_alloc<double>((size_t)n, c.stream);
      c.J = dev_alloc<double>((size_t)(m * n), c.stream);
      c.d = dev_alloc<double>((size_t)m, c.stream);
      auto copy = [&](double* dst, const double* src, int64_t count) {
        if (count <= 0) return;
        if (on_device) CMPC_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * count, kind, c.stream));
        else upload_h2d(dst, src, sizeof(double) * count, c.stream);
      };
      copy(c.H, H, n * n);
      copy(c.h, h, n);
      copy(c.J, J, m * n);
      copy(c.d, d, m);
    }
    const bool verbose = getenv("CMPC_VERBOSE") != nullptr;
    double last = t_in;
    auto tick = [&](const char* what) {
      if (!verbose) return;
      sync(c);
      const double now = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
      if (what) fprintf(stderr, "[cmpc load] %-10s %8.2f ms\n", what, (now - last) * 1e3);
      last = now;
    };
    tick("h2d");
    if (!c.J && prob_rows(c)) analyze_structure_built(c, *prob_rows(c));  // built: J never stored
    else analyze_structure(c);
    tick("analyze");
    // the dense J is not read again by the general path (every product goes through P); a
    // QP small enough for the one-CTA solver keeps it (small.cu)
    if (c.J && small_fits(n, m)) {
      if (c.owns_J) {
        c.Jsmall = c.J;
      } else {
        c.Jsmall = dev_alloc<double>((size_t)std::max<int64_t>(1, m * n), c.stream);
        CMPC_CUDA(cudaMemcpyAsync(c.Jsmall, c.J, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, c.stream));
      }
    } else if (c.owns_J) {
      dev_free(c.J, c.stream);
    }
    c.J = nullptr;
    syrk_plan(c);
    tick("plan");
    vec_alloc(c);
    sync(c);
    tick("alloc");
    return CMPC_OK;
  });
}

}  // namespace

extern "C" {

int cmpc_abi_version(void) { return 1; }
const char* cmpc_last_error(void) { return g_error.c_str(); }
long long cmpc_launch_count(void) { return g_launches; }

int cmpc_ctx_create(cmpc_ctx** out, int device) {
  return guard([&] {
    auto* x = new cmpc_ctx;
    x->c.device = device;
    CMPC_CUDA(cudaSetDevice(device));
    pool_init(device);
    CMPC_CUDA(cudaStreamCreateWithFlags(&x->c.stream, cudaStreamNonBlocking));
    CMPC_CUDA(cudaEventCreate(&x->c.ev0));
    CMPC_CUDA(cudaEventCreate(&x->c.ev1));
    CMPC_CUDA(cudaEventCreate(&x->c.ev2));
    CMPC_CUDA(cudaEventCreate(&x->c.ev3));
    CMPC_CUDA(cudaEventCreate(&x->c.ev4));
    CMPC_CUDA(cudaStreamCreateWithFlags(&x->c.stream2, cudaStreamNonBlocking));
    CMPC_CUDA(cudaEventCreateWithFlags(&x->c.fork, cudaEventDisableTiming));
    CMPC_CUDA(cudaEventCreateWithFlags(&x->c.join, cudaEventDisableTiming));
    *out = x;
    return CMPC_OK;
  });
}

void cmpc_ctx_destroy(cmpc_ctx* x) {
  if (!x) return;
  cudaSetDevice(x->c.device);
  cudaStreamSynchronize(x->c.stream);
  drop_graphs(x->c);
  try {
    comm_detach(x->c);
  } catch (...) {
  }
  release_qp(x->c);
  prob_free(x->c);
  cudaStreamSynchronize(x->c.stream);
  cudaEventDestroy(x->c.ev0);
  cudaEventDestroy(x->c.ev1);
  cudaEventDestroy(x->c.ev2);
  cudaEventDestroy(x->c.ev3);
  cudaEventDestroy(x->c.ev4);
  cudaEventDestroy(x->c.fork);
  cudaEventDestroy(x->c.join);
  cudaStreamDestroy(x->c.stream2);
  cudaStreamDestroy(x->c.stream);
  delete x;
}

int cmpc_load_qp(cmpc_ctx* x, int64_t n, int64_t m, const double* H, const double* h, double h0,
                 const double* J, const double* d, int on_device) {
  if (!x) {
    g_error = "null context (closed?)";
    return CMPC_ERR_DIM;
  }
  prob_free(x->c);  // a bare QP: no structured problem behind it
  return load_impl(x->c, n, m, H, h, h0, J, d, on_device, false);
}

int cmpc_build_qp(cmpc_ctx* x, const cmpc_lq_problem* p) {
  if (!x || !p) {
    g_error = "null context or problem";
    return CMPC_ERR_DIM;
  }
  double *H = nullptr, *h = nullptr, *J = nullptr, *d = nullptr;
  double h0 = 0.0;
  int64_t m = 0;
  const int rc = guard([&] {
    CMPC_CUDA(cudaSetDevice(x->c.device));
    prob_build(x->c, *p, &H, &h, &h0, &J, &d, &m);
    return CMPC_OK;
  });
  if (rc) return rc;
  return load_impl(x->c, p->T * p->nu, m, H, h, h0, J, d, 1, true);
}

int cmpc_get_qp(cmpc_ctx* x, double* H, double* h, double* h0, double* d) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    d2h(c, H, c.H, c.n * c.n);
    d2h(c, h, c.h, c.n);
    d2h(c, d, c.d, c.m);
    if (h0) *h0 = c.h0;
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_refresh_initial_state(cmpc_ctx* x, const double* x_bar) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    prob_refresh(c, x_bar);
    launch_hmax(c);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_recover_trajectory(cmpc_ctx* x, const double* v, double* xs, double* us, double* objective) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    const double* vd = c.v;
    double* tmp = nullptr;
    if (v) {
      tmp = dev_alloc<double>(size_t(std::max<int64_t>(c.n, 1)), c.stream);
      if (c.n > 0) CMPC_CUDA(cudaMemcpyAsync(tmp, v, sizeof(double) * c.n, cudaMemcpyHostToDevice, c.stream));
      vd = tmp;
    }
    prob_recover(c, vd, xs, us, objective);
    dev_free(tmp, c.stream);
    return CMPC_OK;
  });
}

int cmpc_ctx_set_option(cmpc_ctx* x, const char* key, int64_t value) {
  return guard([&] {
    if (!x || !key) throw DimError("null argument");
    Ctx& c = x->c;
    CMPC_CUDA(cudaSetDevice(c.device));
    const std::string k(key);
    if (k == "jtl_recurrence") {
      if (value != 0 && value != 1) throw DimError("jtl_recurrence must be 0 or 1");
      c.opt_jtl_recur = value == 1;
      c.jtl_recur = c.m > 0 && c.opt_jtl_recur;
    } else if (k == "rhs_pass") {
      if (value < 0 || value > 2) throw DimError("rhs_pass must be 0, 1 or 2");
      c.opt_rhs_pass = (int)value;
    } else if (k == "graphs") {
      if (value != 0 && value != 1) throw DimError("graphs must be 0 or 1");
      c.opt_graphs = value == 1;
    } else if (k == "small_path") {
      if (value != 0 && value != 1) throw DimError("small_path must be 0 or 1");
      c.opt_small = value == 1;
    } else if (k == "markov") {
      if (value < 0 || value > 2) throw DimError("markov must be 0, 1 or 2");
      c.opt_markov = (int)value;  // (read when a QP is built: cmpc_build_qp)
    } else if (k == "speculate") {
      if (value != 0 && value != 1) throw DimError("speculate must be 0 or 1");
      c.opt_spec = value == 1;
    } else {
      throw DimError("unknown option: " + k);
    }
    drop_graphs(c);  // captured segments hold the previous form
    return CMPC_OK;
  });
}

int cmpc_ctx_clone(cmpc_ctx* src, cmpc_ctx** out) {
  if (!src || !out) {
    g_error = "cmpc_ctx_clone: null context";
    return CMPC_ERR_ARG;
  }
  cmpc_ctx* x = nullptr;
  int rc = cmpc_ctx_create(&x, src->c.device);
  if (rc) return rc;
  rc = guard([&] {
    const Ctx& s = src->c;
    Ctx& c = x->c;
    require_loaded(const_cast<Ctx&>(s));
    CMPC_CUDA(cudaStreamSynchronize(s.stream));
    c.opt_jtl_recur = s.opt_jtl_recur;
    c.opt_rhs_pass = s.opt_rhs_pass;
    c.opt_graphs = s.opt_graphs;
    c.opt_small = s.opt_small;
    c.opt_spec = s.opt_spec;
    c.opt_markov = s.opt_markov;
    c.n = s.n;
    c.m = s.m;
    c.h0 = s.h0;
    c.ps = s.ps;
    c.pz = s.pz;
    c.p = s.p;
    c.ldp = s.ldp;
    c.zero_k = s.zero_k;
    c.h_start_col = s.h_start_col;
    cudaStream_t st = c.stream;
    auto dup = [&](auto* src_ptr, size_t count) {
      using T = std::remove_const_t<std::remove_pointer_t<decltype(src_ptr)>>;
      T* dst = dev_alloc<T>(count, st);
      if (count > 0 && src_ptr)
        CMPC_CUDA(cudaMemcpyAsync(dst, src_ptr, sizeof(T) * count, cudaMemcpyDeviceToDevice, st));
      return dst;
    };
    c.H = dup(s.H, size_t(s.n * s.n));
    c.h = dup(s.h, size_t(s.n));
    c.d = dup(s.d, size_t(s.m));
    c.J = nullptr;
    c.P = s.P ? dup(s.P, size_t(s.ldp * s.n)) : nullptr;
    if (s.Jsmall) c.Jsmall = dup(s.Jsmall, size_t(std::max<int64_t>(1, s.m * s.n)));
    c.hi = dup(s.hi, size_t(s.ps));
    c.start_col = dup(s.start_col, size_t(s.n + 1));
    c.row_map = dup(s.row_map, size_t(s.m));
    c.mem_ptr = dup(s.mem_ptr, size_t(s.p + 1));
    c.mem_rows = dup(s.mem_rows, size_t(s.m));
    c.sing_col = dup(s.sing_col, size_t(s.pz));
    c.sing_val = dup(s.sing_val, size_t(s.pz));
    if (s.markov) {  // the Markov table and its layout (the plan's chunk lists are rebuilt)
      c.markov = true;
      c.ldmk = s.ldmk;
      c.mk_cols = s.mk_cols;
      c.mk_nq = s.mk_nq;
      c.mk_T = s.mk_T;
      c.mk_nu = s.mk_nu;
      c.mk_nchunks = s.mk_nchunks;
      c.mk_ps = s.mk_ps;
      c.h_mk_chunk = s.h_mk_chunk;
      c.h_mk_width = s.h_mk_width;
      c.mk = dup(s.mk, size_t(s.ldmk * s.mk_cols));
      c.mk_base = dup(s.mk_base, size_t(s.mk_T + 2));
      c.mk_cnt = dup(s.mk_cnt, size_t(s.mk_T + 1));
      c.mk_rbend = dup(s.mk_rbend, size_t(s.ldmk / 32));
      c.mk_chunk = dup(s.mk_chunk, size_t(s.mk_nchunks));
    }
    syrk_plan(c);
    vec_alloc(c);
    sync(c);
    return CMPC_OK;
  });
  if (rc) {
    cmpc_ctx_destroy(x);
    return rc;
  }
  *out = x;
  return CMPC_OK;
}

int cmpc_solve_batch(cmpc_ctx** ctxs, int64_t count, const double* opts, int64_t max_iter,
                     double* v_out, double* scal_out, int threads) {
  if (count <= 0) return CMPC_OK;
  if (threads < 1) threads = 1;
  if (threads > count) threads = (int)count;
  std::atomic<int64_t> next{0};
  std::atomic<int> err{0};
  std::string first_error;
  std::atomic<bool> have_error{false};
  auto worker = [&] {
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= count || err.load() != 0) break;
      Ctx& c = ctxs[i]->c;
      const int rc = guard([&] {
        CMPC_CUDA(cudaSetDevice(c.device));
        require_loaded(c);
        return solve_loop(c, opts, max_iter, v_out ? v_out + i * c.n : nullptr, nullptr, nullptr,
                          nullptr, scal_out + i * 14, nullptr, nullptr, nullptr);
      });
      if (rc < 0 && !have_error.exchange(true)) {
        first_error = g_error;
        err.store(rc);
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  if (err.load() != 0) g_error = first_error;
  return err.load();
}

// A batch of `count` instances that share H and J and differ in (h, h0, d) (config 5,
// refresh_initial_state), solved by `nctx` worker contexts cloned from one analysed QP:
// worker w drives ctxs[w] on its own host thread and takes instances from a shared counter;
// per instance it uploads (h, h0, d) into its context (the captured iteration graphs keep
// pointing at the same buffers) and runs the host loop. Memory and setup cost scale with
// the number of workers, not with the batch.
int cmpc_solve_batch_affine(cmpc_ctx** ctxs, int nctx, int64_t count, const double* h_all,
                            const double* h0_all, const double* d_all, const double* opts,
                            int64_t max_iter, double* v_out, double* scal_out) {
  if (count <= 0 || nctx <= 0) return CMPC_OK;
  std::atomic<int64_t> next{0};
  std::atomic<int> err{0};
  std::string first_error;
  std::atomic<bool> have_error{false};
  auto worker = [&](int w) {
    Ctx& c = ctxs[w]->c;
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= count || err.load() != 0) break;
      const int rc = guard([&] {
        CMPC_CUDA(cudaSetDevice(c.device));
        require_loaded(c);
        if (c.n > 0)
          CMPC_CUDA(cudaMemcpyAsync(c.h, h_all + i * c.n, sizeof(double) * c.n, cudaMemcpyHostToDevice, c.stream));
        if (c.m > 0)
          CMPC_CUDA(cudaMemcpyAsync(c.d, d_all + i * c.m, sizeof(double) * c.m, cudaMemcpyHostToDevice, c.stream));
        c.h0 = h0_all[i];
        launch_hmax(c);
        return solve_loop(c, opts, max_iter, v_out ? v_out + i * c.n : nullptr, nullptr, nullptr,
                          nullptr, scal_out + i * 14, nullptr, nullptr, nullptr);
      });
      if (rc < 0 && !have_error.exchange(true)) {
        first_error = g_error;
        err.store(rc);
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nctx; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  if (err.load() != 0) g_error = first_error;
  return err.load();
}

struct cmpc_batch {
  cmpc::BatchCtx* b = nullptr;
  int device = 0;
};

int cmpc_batch_create(cmpc_ctx* base, int64_t count, cmpc_batch** out) {
  return guard([&] {
    if (!base || !out) throw DimError("null argument");
    Ctx& c = base->c;
    require_loaded(c);
    CMPC_CUDA(cudaSetDevice(c.device));
    auto* x = new cmpc_batch;
    x->device = c.device;
    try {
      x->b = batch_create(c, count);
    } catch (...) {
      delete x;
      throw;
    }
    *out = x;
    return CMPC_OK;
  });
}

int cmpc_batch_set_affine(cmpc_batch* b, const double* h_all, const double* h0_all, const double* d_all) {
  return guard([&] {
    if (!b || !b->b) throw DimError("null batch (closed?)");
    CMPC_CUDA(cudaSetDevice(b->device));
    batch_set_affine(*b->b, h_all, h0_all, d_all);
    return CMPC_OK;
  });
}

int cmpc_batch_solve(cmpc_batch* b, const double* opts, int64_t max_iter, double* v_out, double* scal_out,
                     double* stats) {
  return guard([&] {
    if (!b || !b->b) throw DimError("null batch (closed?)");
    CMPC_CUDA(cudaSetDevice(b->device));
    batch_solve(*b->b, opts, max_iter, v_out, scal_out, stats);
    return CMPC_OK;
  });
}

int cmpc_batch_condense(cmpc_batch* b, const double* sigma_all, const double* w_all, double* M_out,
                        double* tq_out) {
  return guard([&] {
    if (!b || !b->b || !sigma_all || !w_all || !M_out || !tq_out) throw DimError("null argument");
    CMPC_CUDA(cudaSetDevice(b->device));
    batch_condense(*b->b, sigma_all, w_all, M_out, tq_out);
    return CMPC_OK;
  });
}

void cmpc_batch_destroy(cmpc_batch* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  try {
    batch_destroy(b->b);
  } catch (...) {
  }
  delete b;
}

// Page-lock a host buffer for the batch uploads (plain DMA instead of staged copies)
int cmpc_host_register(void* p, int64_t bytes) {
  return guard([&] {
    if (p && bytes > 0) CMPC_CUDA(cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault));
    return CMPC_OK;
  });
}
int cmpc_host_unregister(void* p) {
  return guard([&] {
    if (p) CMPC_CUDA(cudaHostUnregister(p));
    return CMPC_OK;
  });
}

int cmpc_qp_info(cmpc_ctx* x, int64_t* out) {
  const Ctx& c = x->c;
  out[0] = c.n;
  out[1] = c.m;
  out[2] = c.p;
  out[3] = c.ps;
  out[4] = c.pz;
  out[5] = c.nunits;
  out[6] = (int64_t)c.syrk_flops;
  out[7] = (int64_t)c.syrk_bytes;
  return CMPC_OK;
}

int cmpc_qp_layout(cmpc_ctx* x, int64_t* out) {
  if (!x || !out) {
    g_error = "null argument";
    return CMPC_ERR_DIM;
  }
  const Ctx& c = x->c;
  out[0] = c.markov ? 1 : 0;
  out[1] = c.markov ? c.mk_nq : 0;
  out[2] = c.markov ? c.mk_cols : 0;
  out[3] = c.markov ? 8 * c.ldmk * c.mk_cols : (c.P ? 8 * c.ldp * c.n : 0);
  return CMPC_OK;
}

int cmpc_comm_unique_id(void* id128) {
  return guard([&] {
    if (!id128) throw DimError("id buffer is NULL");
    comm_unique_id(id128);
    return CMPC_OK;
  });
}

int cmpc_ctx_attach_comm(cmpc_ctx* x, const void* id128, int nranks, int rank, int64_t m_total) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    if (!id128 || nranks < 1 || rank < 0 || rank >= nranks) throw DimError("bad communicator arguments");
    if (m_total < c.m) throw DimError("m_total is smaller than this shard's rows");
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
    drop_graphs(c);
    comm_attach(c, id128, nranks, rank);
    c.m_all = m_total;
    return CMPC_OK;
  });
}

int cmpc_loop_create(int nranks, int device, void** group) {
  return guard([&] {
    if (!group) throw DimError("null argument");
    *group = comm_loop_create(nranks, device);
    return CMPC_OK;
  });
}

void cmpc_loop_destroy(void* group) {
  try {
    comm_loop_destroy(group);
  } catch (...) {
  }
}

int cmpc_ctx_attach_loop(cmpc_ctx* x, void* group, int rank, int64_t m_total) {
  return guard([&] {
    if (!x || !group) throw DimError("null argument");
    Ctx& c = x->c;
    require_loaded(c);
    if (m_total < c.m) throw DimError("m_total is smaller than this shard's rows");
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
    drop_graphs(c);
    comm_loop_attach(c, group, rank);
    c.m_all = m_total;
    return CMPC_OK;
  });
}

int cmpc_ctx_detach_comm(cmpc_ctx* x) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    drop_graphs(c);
    comm_detach(c);
    c.m_all = -1;
    return CMPC_OK;
  });
}

int cmpc_time_phase(cmpc_ctx* x, int what, int reps, double* ms_per_rep) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    if (reps < 1) throw DimError("reps must be positive");
    auto run = [&] {
      switch (what) {
        case 0: launch_prepare_step(c, nullptr); launch_condense(c, false); break;
        case 1: launch_condense(c, false); break;
        case 2: launch_cholesky(c, c.M, c.L, 0.0); break;
        case 3: launch_chol_solve(c, c.L, c.rhs, c.pv); break;
        case 4: launch_residuals(c); break;
        case 5: launch_recover(c, 0.995); break;
        case 6: launch_trial(c, 0.5, false); break;
        case 7: launch_Jx(c, c.v, c.y, nullptr); break;
        case 8: launch_Jtq(c, c.q, c.Jtl); break;
        case 9: launch_prepare_step(c, nullptr); break;
        case 10: launch_cholesky(c, c.M, c.L, 0.0, c.rhs, c.pv); break;
        case 11: launch_condense(c, false, c.ps > 0 && c.npieces > 0); break;  // + fused P'q
        default: throw DimError("unknown phase");
      }
    };
    run();
    CMPC_CUDA(cudaEventRecord(c.ev2, c.stream));
    for (int r = 0; r < reps; ++r) run();
    CMPC_CUDA(cudaEventRecord(c.ev3, c.stream));
    CMPC_CUDA(cudaEventSynchronize(c.ev3));
    float ms = 0.f;
    CMPC_CUDA(cudaEventElapsedTime(&ms, c.ev2, c.ev3));
    *ms_per_rep = ms / reps;
    return CMPC_OK;
  });
}

// Debug: run the condensation once with a per-piece timeline. out: 8 doubles per piece
// {start us, end us (from the first start), smid, segments, k-steps of the full off-diagonal,
// thin off-diagonal, full diagonal and thin diagonal segments}
int cmpc_debug_syrk_timeline(cmpc_ctx* x, double* out, int64_t cap, int64_t* nctas) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    const int nb = c.npieces;
    long long* buf = dev_alloc<long long>(size_t(3 * std::max(nb, 1)), c.stream);
    c.syrk_prof = buf;
    launch_condense(c, false);
    c.syrk_prof = nullptr;
    std::vector<long long> h(size_t(3 * std::max(nb, 1)));
    CMPC_CUDA(cudaMemcpyAsync(h.data(), buf, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, c.stream));
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
    dev_free(buf, c.stream);
    long long t0 = h.empty() ? 0 : h[0];
    for (int b = 0; b < nb; ++b) t0 = std::min(t0, h[size_t(3 * b)]);
    for (int b = 0; b < nb && b < cap; ++b) {
      out[8 * b] = (h[size_t(3 * b)] - t0) * 1e-3;
      out[8 * b + 1] = (h[size_t(3 * b + 1)] - t0) * 1e-3;
      out[8 * b + 2] = double(h[size_t(3 * b + 2)]);
      for (int q = 0; q < 5; ++q) out[8 * b + 3 + q] = c.syrk_cta_cost[size_t(5 * b + q)];
    }
    *nctas = nb;
    return CMPC_OK;
  });
}

int cmpc_update_qp_affine(cmpc_ctx* x, const double* h, double h0, const double* d, int on_device) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    const auto kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (h && c.n > 0) CMPC_CUDA(cudaMemcpyAsync(c.h, h, sizeof(double) * c.n, kind, c.stream));
    if (d && c.m > 0) CMPC_CUDA(cudaMemcpyAsync(c.d, d, sizeof(double) * c.m, kind, c.stream));
    c.h0 = h0;
    launch_hmax(c);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_set_state(cmpc_ctx* x, const double* v, const double* s, const double* lam,
                   const double* z, double mu) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    h2d(c, c.v, v, c.n);
    h2d(c, c.s, s, c.m);
    h2d(c, c.lam, lam, c.m);
    h2d(c, c.z, z, c.m);
    set_mu(c, mu);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_get_state(cmpc_ctx* x, double* v, double* s, double* lam, double* z) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    d2h(c, v, c.v, c.n);
    d2h(c, s, c.s, c.m);
    d2h(c, lam, c.lam, c.m);
    d2h(c, z, c.z, c.m);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_compute_residuals(cmpc_ctx* x, double* r1, double* r2, double* r3, double* kkt) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    launch_residuals(c);
    d2h(c, r1, c.r1, c.n);
    d2h(c, r2, c.r2, c.m);
    d2h(c, r3, c.r3, c.m);
    read_packet(c);
    if (kkt) *kkt = c.pk_host->kkt;
    return CMPC_OK;
  });
}

int cmpc_set_residuals(cmpc_ctx* x, const double* r1, const double* r2, const double* r3) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    h2d(c, c.r1, r1, c.n);
    h2d(c, c.r2, r2, c.m);
    h2d(c, c.r3, r3, c.m);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_assemble_condensed(cmpc_ctx* x, const double* sigma, double* M) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    if (sigma && c.m > 0) h2d(c, c.sigma, sigma, c.m);
    launch_prepare_step(c, sigma ? c.sigma : nullptr);
    launch_condense(c, true);
    comm_allreduce(c, c.M, (size_t)(c.n * c.n), CommType::f64, CommOp::sum);  // sharded
    d2h(c, M, c.M, c.n * c.n);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_factorize_condensed(cmpc_ctx* x, double delta, int64_t* pivot) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    launch_cholesky(c, c.M, c.L, delta);
    read_packet(c);
    if (c.pk_host->info != 0) {
      if (pivot) *pivot = c.pk_host->info - 1;
      g_error = "cholesky failed: matrix not positive definite at pivot " +
                std::to_string(c.pk_host->info - 1);
      return CMPC_NOT_PD;
    }
    return CMPC_OK;
  });
}

int cmpc_get_factor(cmpc_ctx* x, double* L) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    d2h(c, L, c.L, c.n * c.n);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_set_factor(cmpc_ctx* x, const double* L) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    h2d(c, c.L, L, c.n * c.n);
    launch_factor_inverses(c, c.L);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_step_directions(cmpc_ctx* x, double tau, double* pv, double* ps, double* pl, double* pz,
                         double* alpha) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    if (!(tau > 0.0 && tau < 1.0)) throw DimError("tau must lie in (0,1)");
    launch_prepare_step(c, nullptr);
    launch_rhs_partial(c);
    comm_allreduce(c, c.tq, (size_t)c.n, CommType::f64, CommOp::sum);  // sharded
    launch_rhs_final(c);
    launch_chol_solve(c, c.L, c.rhs, c.pv);
    launch_recover(c, tau);
    d2h(c, pv, c.pv, c.n);
    d2h(c, ps, c.ps_, c.m);
    d2h(c, pl, c.pl, c.m);
    d2h(c, pz, c.pzd, c.m);
    read_packet(c);
    if (alpha) {
      alpha[0] = std::min(1.0, c.pk_host->alpha_s_min);
      alpha[1] = std::min(1.0, c.pk_host->alpha_z_min);
    }
    return CMPC_OK;
  });
}

int cmpc_set_directions(cmpc_ctx* x, const double* pv, const double* ps, const double* pl,
                        const double* pz) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    h2d(c, c.pv, pv, c.n);
    h2d(c, c.ps_, ps, c.m);
    h2d(c, c.pl, pl, c.m);
    h2d(c, c.pzd, pz, c.m);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_line_search(cmpc_ctx* x, double alpha_max, double eta, double* alpha, int* trial) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    if (!(alpha_max > 0.0 && alpha_max <= 1.0)) throw DimError("alpha_max must lie in (0,1]");
    launch_residuals(c);
    launch_ls_pieces(c);
    read_packet(c);
    int nt = 0;
    const int j = line_search_host(c, alpha_max, eta, alpha, &nt);
    if (trial) *trial = j;
    return CMPC_OK;
  });
}

int cmpc_merit(cmpc_ctx* x, double alpha, double rho, double* phi) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    launch_trial(c, alpha, false);
    read_packet(c);
    const Packet& T = *c.pk_host;
    *phi = merit_host(T, T.t_vHv, T.t_hv, T.t_sum_log, T.t_sum_abs, c.mu, rho, c.m > 0);
    return CMPC_OK;
  });
}

int cmpc_apply_step(cmpc_ctx* x, double alpha, double alpha_z) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    launch_update(c, alpha, alpha_z);
    sync(c);
    return CMPC_OK;
  });
}

int cmpc_dense_objective(cmpc_ctx* x, double* obj) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    launch_residuals(c);
    read_packet(c);
    *obj = c.pk_host->objective;
    return CMPC_OK;
  });
}

int cmpc_solve(cmpc_ctx* x, const double* opts, int64_t max_iter, double* v, double* s,
               double* lam, double* z, double* out, cmpc_log_fn log, cmpc_inspect_fn inspect,
               void* user) {
  return guard([&] {
    if (!x) throw DimError("null context (closed?)");
    Ctx& c = x->c;
    require_loaded(c);
    CMPC_CUDA(cudaSetDevice(c.device));
    return solve_loop(c, opts, max_iter, v, s, lam, z, out, log, inspect, user);
  });
}

// ---------------------------------------------------------------- stand-alone linalg
int cmpc_gram_weighted(int device, int64_t m, int64_t n, const double* J, const double* sigma,
                       double* G) {
  cmpc_ctx* x = nullptr;
  int rc = cmpc_ctx_create(&x, device);
  if (rc) return rc;
  rc = guard([&] {
    std::vector<double> zeros(size_t(std::max<int64_t>(1, n * n)), 0.0), d(size_t(std::max<int64_t>(1, m)), 0.0);
    int r = cmpc_load_qp(x, n, m, zeros.data(), zeros.data(), 0.0, J, d.data(), 0);
    if (r) return r;
    return cmpc_assemble_condensed(x, sigma, G);
  });
  cmpc_ctx_destroy(x);
  return rc;
}

int cmpc_cholesky(int device, int64_t n, const double* M, double* L, int64_t* pivot) {
  cmpc_ctx* x = nullptr;
  int rc = cmpc_ctx_create(&x, device);
  if (rc) return rc;
  rc = guard([&] {
    std::vector<double> zeros(size_t(std::max<int64_t>(1, n)), 0.0);
    int r = cmpc_load_qp(x, n, 0, M, zeros.data(), 0.0, nullptr, nullptr, 0);
    if (r) return r;
    Ctx& c = x->c;
    CMPC_CUDA(cudaMemcpyAsync(c.M, M, sizeof(double) * n * n, cudaMemcpyHostToDevice, c.stream));
    r = cmpc_factorize_condensed(x, 0.0, pivot);
    if (r == CMPC_OK) r = cmpc_get_factor(x, L);
    return r;
  });
  cmpc_ctx_destroy(x);
  return rc;
}

int cmpc_fraction_to_boundary(int device, int64_t m, const double* s, const double* ps,
                              const double* z, const double* pz, double tau, double* out) {
  return guard([&] {
    if (!(tau > 0.0 && tau < 1.0)) throw DimError("tau must lie in (0,1)");
    CMPC_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    CMPC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const int64_t mm = std::max<int64_t>(m, 1);
    double* buf = dev_alloc<double>((size_t)(4 * mm + 2), st);
    const double* src[4] = {s, ps, z, pz};
    for (int k = 0; k < 4; ++k)
      if (m > 0)
        CMPC_CUDA(cudaMemcpyAsync(buf + k * mm, src[k], sizeof(double) * m, cudaMemcpyHostToDevice, st));
    launch_fraction_to_boundary(st, m, buf, buf + mm, buf + 2 * mm, buf + 3 * mm, tau, buf + 4 * mm);
    double r[2];
    CMPC_CUDA(cudaMemcpyAsync(r, buf + 4 * mm, sizeof(r), cudaMemcpyDeviceToHost, st));
    dev_free(buf, st);
    CMPC_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    out[0] = std::min(1.0, r[0]);
    out[1] = std::min(1.0, r[1]);
    return CMPC_OK;
  });
}

int cmpc_cholesky_solve(int device, int64_t n, const double* L, const double* b, double* xout) {
  cmpc_ctx* x = nullptr;
  int rc = cmpc_ctx_create(&x, device);
  if (rc) return rc;
  rc = guard([&] {
    std::vector<double> zeros(size_t(std::max<int64_t>(1, n * n)), 0.0);
    int r = cmpc_load_qp(x, n, 0, zeros.data(), zeros.data(), 0.0, nullptr, nullptr, 0);
    if (r) return r;
    Ctx& c = x->c;
    h2d(c, c.L, L, n * n);
    h2d(c, c.rhs, b, n);
    launch_factor_inverses(c, c.L);
    launch_chol_solve(c, c.L, c.rhs, c.pv);
    d2h(c, xout, c.pv, n);
    sync(c);
    return CMPC_OK;
  });
  cmpc_ctx_destroy(x);
  return rc;
}

}  // extern "C"
