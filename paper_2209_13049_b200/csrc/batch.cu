// Lockstep batch: B independent instances that share H and J and differ in (h, h0, d) — the
// receding-horizon case of refresh_initial_state (proj/src/reduction.cpp:270-280) and
// BASELINE.json config 5 (1024 instances). The reference solves them one by one
// (proj/src/verify.cpp:104-111 runs its thread pool over instances); here ONE host loop
// drives all of them, every kernel covering every active instance in one launch:
//   * the condensation (bsyrk.cu) runs one CTA per instance holding its whole lower triangle
//     in registers while P (shared, L2-resident at config 5, 14 MB) streams through TMA;
//     H, the singleton terms and the right-hand side J'w are fused in;
//   * the products with P and H are plain DGEMMs over the B right-hand sides (cuBLAS, loaded
//     at run time): P X, P' Lambda, H V;
//   * the Cholesky of each n x n matrix (n <= kBatchMaxN) and both triangular solves run in
//     one CTA per instance with the trailing matrix in registers (k_b_chol);
//   * the row passes (residuals, sigma, recovery, fraction to boundary, trials, update) are
//     the single-instance formulas with blockIdx.y = instance and per-instance block sums
//     reduced in a fixed order.
// The host loop restates condmpc::ipm::solve (proj/src/ipm.cpp:160-268) for each instance —
// termination, barrier update, shift ladder, backtracking line search with the roundoff band
// — on per-instance packets read back at each sync; instances that are done drop out of the
// active mask. Every decision is taken with the reference's rule on that instance's scalars.
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <vector>

#include "../../include/condmpc_cuda.h"
#include "internal.cuh"

namespace cmpc {

double merit_host(const Packet&, double vhv, double hv, double sum_log, double sum_abs, double mu,
                  double rho, bool has_rows);

namespace {

constexpr int kBT = 256;      // threads of the row / final kernels
constexpr int kStageSlots = 8;  // pinned upload ring (Host::upload_*)
constexpr int kBBlk = 32;     // row-kernel blocks per instance
constexpr int kBatchMaxN = 160;  // the per-instance Cholesky keeps M in shared memory
enum BSlot { kBAbs = 0, kBLog, kBLam, kBS, kBZ, kBR3, kBComp, kBPsS, kBAs, kBAz, kBBad, kBSlots };

// ---------------------------------------------------------------- cuBLAS (plain DGEMMs only)
typedef int (*PFN_cublasCreate)(void**);
typedef int (*PFN_cublasDestroy)(void*);
typedef int (*PFN_cublasSetStream)(void*, cudaStream_t);
typedef int (*PFN_cublasDgemm)(void*, int, int, int, int, int, const double*, const double*, int,
                               const double*, int, const double*, double*, int);
struct Cublas {
  PFN_cublasCreate create = nullptr;
  PFN_cublasDestroy destroy = nullptr;
  PFN_cublasSetStream set_stream = nullptr;
  PFN_cublasDgemm dgemm = nullptr;
};
const Cublas& cublas() {
  static Cublas cb = [] {
    Cublas c;
    void* h = nullptr;
    for (const char* name : {"libcublas.so.12", "libcublas.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) throw CudaError(std::string("batch: cannot load cuBLAS: ") + dlerror());
    c.create = reinterpret_cast<PFN_cublasCreate>(dlsym(h, "cublasCreate_v2"));
    c.destroy = reinterpret_cast<PFN_cublasDestroy>(dlsym(h, "cublasDestroy_v2"));
    c.set_stream = reinterpret_cast<PFN_cublasSetStream>(dlsym(h, "cublasSetStream_v2"));
    c.dgemm = reinterpret_cast<PFN_cublasDgemm>(dlsym(h, "cublasDgemm_v2"));
    if (!c.create || !c.destroy || !c.set_stream || !c.dgemm) throw CudaError("batch: cuBLAS symbols missing");
    return c;
  }();
  return cb;
}
// C (m x n, ldc) = op(A) B, column-major
void dgemm(void* h, bool ta, int m, int n, int k, const double* A, int lda, const double* B, int ldb,
           double* C, int ldc) {
  if (m == 0 || n == 0) return;
  const double one = 1.0, zero = 0.0;
  const int rc = cublas().dgemm(h, ta ? 1 : 0, 0, m, n, k, &one, A, lda, B, ldb, &zero, C, ldc);
  if (rc != 0) throw CudaError("batch: cublasDgemm failed (" + std::to_string(rc) + ")");
  g_launches += 1;
}

__device__ __forceinline__ double jrow_b(const double* y, int32_t rm) {
  const double v = y[rm >> 1];
  return (rm & 1) ? -v : v;
}

// per-instance block partials: part[(b * kBBlk + blk) * kBSlots + slot]; the block's sums
// (in the fixed order of block_sums_maxs) and maxima go to the listed slots
template <int NS, int NX>
struct Slots {
  int s[NS > 0 ? NS : 1], x[NX > 0 ? NX : 1];
};
template <int NS, int NX>
__device__ __forceinline__ void block_out(double (&su)[NS], double (&mx)[NX], double* sh, double* part,
                                          const Slots<NS, NX> sl) {
  block_sums_maxs<kBT>(su, mx, sh);
  if (threadIdx.x == 0) {
    double* o = part + ((int64_t)blockIdx.y * kBBlk + blockIdx.x) * kBSlots;
#pragma unroll
    for (int k = 0; k < NS; ++k) o[sl.s[k]] = su[k];
#pragma unroll
    for (int k = 0; k < NX; ++k) o[sl.x[k]] = mx[k];
  }
}

#define B_ROWS_LOOP(m) for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < (m); r += (int64_t)gridDim.x * blockDim.x)

// v = 0, s = max(1, d), z = mu / s, lambda = z (ipm.cpp:170-177)
__global__ void k_b_init(int64_t n, int64_t m, const double* __restrict__ d, const double* __restrict__ mu,
                         double* __restrict__ v, double* __restrict__ s, double* __restrict__ lam,
                         double* __restrict__ z) {
  const int64_t b = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[b * n + i] = 0.0;
  B_ROWS_LOOP(m) {
    const int64_t o = b * m + r;
    const double sr = fmax(1.0, d[o]);
    const double zr = mul(mu[b], dv(1.0, sr));
    s[o] = sr;
    z[o] = zr;
    lam[o] = zr;
  }
}

// singleton prototype values y[ldp + k] = val_k x[col_k] (one block row per instance)
__global__ void k_b_sing(int64_t pz, int64_t n, int64_t py, int64_t ldp, const int32_t* __restrict__ col,
                         const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t b = blockIdx.y;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < pz; k += (int64_t)gridDim.x * blockDim.x)
    y[b * py + ldp + k] = val[k] * x[b * n + col[k]];
}

// max |h_b| (the kkt scaling)
__global__ void k_b_hmax(int64_t n, const double* __restrict__ h, double* __restrict__ hmax) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = fmax(a, fabs(h[blockIdx.x * n + i]));
  a = block_max<kBT>(a, sh);
  if (threadIdx.x == 0) hmax[blockIdx.x] = a;
}

// residual rows: r2 = lambda - mu/s, r3 = Jv - d + s and their sums / maxima. STEP: the
// accepted step of the rows first (s += alpha ps, lambda += alpha pl, z += alpha_z pz, the
// update of ipm.cpp:240-243), so the iterate is read once for both
template <bool STEP>
__global__ void __launch_bounds__(kBT) k_b_res_rows(int64_t m, int64_t py, const int32_t* __restrict__ row_map,
                                                    const double* __restrict__ yv, const double* __restrict__ d,
                                                    double* __restrict__ s, double* __restrict__ lam,
                                                    double* __restrict__ z, const double* __restrict__ mu_p,
                                                    double* __restrict__ r2, double* __restrict__ r3,
                                                    double* __restrict__ part, const int* __restrict__ act,
                                                    const double* __restrict__ alpha,
                                                    const double* __restrict__ alpha_z,
                                                    const double* __restrict__ ps, const double* __restrict__ pl,
                                                    const double* __restrict__ pz, double* __restrict__ sigma) {
  __shared__ double sh[7 * 32];
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  const double mu = mu_p[b];
  const double* y = yv + b * py;
  const double al = STEP ? alpha[b] : 0.0, az = STEP ? alpha_z[b] : 0.0;
  double sabs = 0.0, slog = 0.0, ml = 0.0, mss = 0.0, mz = 0.0, mr3 = 0.0, mc = 0.0;
  B_ROWS_LOOP(m) {
    const int64_t o = b * m + r;
    const double jv = jrow_b(y, row_map[r]);
    double sr = s[o], lr = lam[o], zr = z[o];
    if (STEP) {
      sr = add(sr, mul(al, ps[o]));
      lr = add(lr, mul(al, pl[o]));
      zr = add(zr, mul(az, pz[o]));
      s[o] = sr;
      lam[o] = lr;
      z[o] = zr;
    }
    r2[o] = sub(lr, mul(mu, dv(1.0, sr)));
    const double t3 = add(sub(jv, d[o]), sr);
    r3[o] = t3;
    sigma[o] = dv(zr, sr);  // the next condensation's sigma (s and z stay until then)
    sabs += fabs(t3);
    slog += log(sr);
    ml = fmax(ml, fabs(lr));
    mss = fmax(mss, fabs(sr));
    mz = fmax(mz, fabs(zr));
    mr3 = fmax(mr3, fabs(t3));
    mc = fmax(mc, fabs(sub(mul(sr, zr), mu)));
  }
  double su[2] = {sabs, slog}, mx[5] = {ml, mss, mz, mr3, mc};
  block_out<2, 5>(su, mx, sh, part, Slots<2, 5>{{kBAbs, kBLog}, {kBLam, kBS, kBZ, kBR3, kBComp}});
}

// r1 = H v + h + J'lambda, kkt, objective pieces (ipm.cpp:46-70) -> packet
__global__ void __launch_bounds__(kBT) k_b_res_final(int64_t n, int64_t m, const double* __restrict__ Hv,
                                                     const double* __restrict__ h, const double* __restrict__ Jtl,
                                                     const double* __restrict__ v, double* __restrict__ r1,
                                                     const double* __restrict__ part,
                                                     const double* __restrict__ hmax, const double* __restrict__ h0,
                                                     Packet* pk, const int* __restrict__ act) {
  __shared__ double sh[5 * 32];
  const int64_t b = blockIdx.x;
  if (!act[b]) return;
  double mr1 = 0.0, vhv = 0.0, hv = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t o = b * n + i;
    const double g = add(Hv[o], h[o]);
    const double r = m > 0 ? add(g, Jtl[o]) : g;
    r1[o] = r;
    mr1 = fmax(mr1, fabs(r));
    vhv += v[o] * Hv[o];
    hv += h[o] * v[o];
  }
  double su[2] = {vhv, hv}, mx[1] = {mr1};
  block_sums_maxs<kBT>(su, mx, sh);
  if (threadIdx.x == 0) {
    const double* pp = part + b * kBBlk * kBSlots;
    double sabs = 0.0, slog = 0.0, ml = 0.0, mss = 0.0, mz = 0.0, mr3 = 0.0, mc = 0.0;
    for (int k = 0; k < kBBlk; ++k) {
      const double* q = pp + k * kBSlots;
      sabs += q[kBAbs];
      slog += q[kBLog];
      ml = fmax(ml, q[kBLam]);
      mss = fmax(mss, q[kBS]);
      mz = fmax(mz, q[kBZ]);
      mr3 = fmax(mr3, q[kBR3]);
      mc = fmax(mc, q[kBComp]);
    }
    Packet* p = pk + b;
    p->max_r1 = mx[0];
    p->max_r3 = mr3;
    p->max_comp = mc;
    p->max_lam = ml;
    p->max_s = mss;
    p->max_z = mz;
    p->max_h = hmax[b];
    p->obj_vHv = su[0];
    p->obj_hv = su[1];
    p->sum_abs_r3 = m > 0 ? sabs : 0.0;
    p->sum_log_s = m > 0 ? slog : 0.0;
    p->objective = 0.5 * su[0] + su[1] + h0[b];
    const double ds = fmax(1.0, fmax(hmax[b], ml) / (double)(n + m));
    double kkt = mx[0] / ds;
    if (m > 0) {
      const double cs = fmax(1.0, fmax(mss, mz) / (double)(2 * m));
      kkt = fmax(kkt, mr3);
      kkt = fmax(kkt, mc / cs);
    }
    p->kkt = kkt;
  }
}

// after a barrier change: r2 and the complementarity maximum at the new mu, then kkt
__global__ void __launch_bounds__(kBT) k_b_mu_rows(int64_t m, const double* __restrict__ s,
                                                   const double* __restrict__ lam, const double* __restrict__ z,
                                                   const double* __restrict__ mu_p, double* __restrict__ r2,
                                                   double* __restrict__ part, const int* __restrict__ act) {
  __shared__ double sh[32];
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  const double mu = mu_p[b];
  double mc = 0.0;
  B_ROWS_LOOP(m) {
    const int64_t o = b * m + r;
    const double sr = s[o];
    r2[o] = sub(lam[o], mul(mu, dv(1.0, sr)));
    mc = fmax(mc, fabs(sub(mul(sr, z[o]), mu)));
  }
  mc = block_max<kBT>(mc, sh);
  if (threadIdx.x == 0) part[((int64_t)b * kBBlk + blockIdx.x) * kBSlots + kBComp] = mc;
}
__global__ void k_b_kkt_mu(int64_t B, int64_t n, int64_t m, const double* __restrict__ part, Packet* pk,
                           const int* __restrict__ act) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B || !act[b]) return;
  double mc = 0.0;
  for (int k = 0; k < kBBlk; ++k) mc = fmax(mc, part[(b * kBBlk + k) * kBSlots + kBComp]);
  Packet* p = pk + b;
  p->max_comp = mc;
  const double ds = fmax(1.0, fmax(p->max_h, p->max_lam) / (double)(n + m));
  double kkt = p->max_r1 / ds;
  if (m > 0) {
    const double cs = fmax(1.0, fmax(p->max_s, p->max_z) / (double)(2 * m));
    kkt = fmax(kkt, p->max_r3);
    kkt = fmax(kkt, mc / cs);
  }
  p->kkt = kkt;
}

// per prototype k: out1 = sum over the member rows of x1 (signed when SIGNED1), out2 = signed
// sum of x2 (when x2); members in ascending row order; the all-zero group gives 0
// WR: x2 is not stored but formed per member row as w = r2 - x1 r3 (x1 = sigma; the
// step_directions right-hand side, ipm.cpp:79-103), so no pass over the rows writes it
template <bool SIGNED1, bool WR = false>
__global__ void __launch_bounds__(kBT) k_b_proto(int64_t p, int64_t ps, int64_t ldp, int64_t m, int64_t py,
                                                 int64_t zero_k, const int32_t* __restrict__ mem_ptr,
                                                 const int32_t* __restrict__ mem_rows, const double* __restrict__ x1,
                                                 const double* __restrict__ x2, double* __restrict__ out1,
                                                 double* __restrict__ out2, const int* __restrict__ act,
                                                 const double* __restrict__ r2 = nullptr,
                                                 const double* __restrict__ r3 = nullptr) {
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p; k += (int64_t)gridDim.x * blockDim.x) {
    double s1 = 0.0, s2 = 0.0;
    if (k != zero_k) {
      for (int32_t e = mem_ptr[k]; e < mem_ptr[k + 1]; ++e) {
        const int32_t rm = mem_rows[e];
        const int64_t o = b * m + (rm >> 1);
        const double a = x1[o];
        s1 += (SIGNED1 && (rm & 1)) ? -a : a;
        if (WR) {
          const double c = sub(r2[o], mul(a, r3[o]));
          s2 += (rm & 1) ? -c : c;
        } else if (x2) {
          const double c = x2[o];
          s2 += (rm & 1) ? -c : c;
        }
      }
    }
    const int64_t o = b * py + (k < ps ? k : ldp + (k - ps));
    out1[o] = s1;
    if (WR || x2) out2[o] = s2;
  }
}

// out[j] += sum over the singleton prototypes of column j of val_k q[ldp + k] (P' q finished)
__global__ void k_b_sing_t(int64_t n, int64_t py, int64_t ldp, const int32_t* __restrict__ sing_ptr,
                           const double* __restrict__ val, const double* __restrict__ q, double* __restrict__ out,
                           const int* __restrict__ act) {
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double s = out[b * n + j];
    for (int32_t k = sing_ptr[j]; k < sing_ptr[j + 1]; ++k) s += val[k] * q[b * py + ldp + k];
    out[b * n + j] = s;
  }
}

constexpr int kCholT = 256;   // 8 warps: warp w owns the columns w + 8 c, lane l the rows l + 32 a
constexpr int kCholW = kCholT / 32;
constexpr int kCholA = 5;     // row slots: n <= 160
constexpr int kCholC = 20;    // column slots
// slot (a, c) exists when row block a can reach column w + 8 c (32 a + 31 >= 8 c)
__device__ __forceinline__ constexpr int cslot(int a, int c) { return 2 * a * a + 2 * a + c; }
constexpr int kCholSlots = cslot(kCholA, 0);

__device__ __forceinline__ double b_rsqrt(double x) {  // MUFU seed + two Newton steps
  if (!(x >= 1e-300 && x <= 1e300)) return 1.0 / sqrt(x);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}

// Per-instance Cholesky of M_b + delta_b I and both triangular solves with rhs_b (the
// ReferenceBackend factorize + Factor::solve, proj/src/dense_linalg.cpp:59-77 and :102-110,
// pivot rule "!(d > 0) || !isfinite(d)" with info = first failing pivot + 1), one CTA per
// instance. Right-looking with the trailing matrix in REGISTERS: thread (lane, warp) holds the
// elements (lane + 32 a, warp + 8 c) of its slots (60 doubles). Pivots run in blocks of 8
// columns (one per warp) inside a loop unrolled over the column slot c, so the pivot column's
// slot is a compile-time index. Per pivot j one barrier: the owner warp forms column j (pivot
// by shuffle, l = a * rsqrt(a_jj)), stores it to shared memory and advances the forward solve;
// after the barrier every thread applies it to all its slots — no per-element or per-column
// predicates: entries above the diagonal and of finished columns are updated too and never
// read. L lives in shared memory with an odd leading dimension (n + 1), so the backward solve's
// row reads are conflict-free; it runs right-looking in one warp's registers.
__global__ void __launch_bounds__(kCholT, 1) k_b_chol(int n, const double* __restrict__ M,
                                                   const double* __restrict__ delta, const double* __restrict__ rhs,
                                                   double* __restrict__ x, Packet* pk, const int* __restrict__ act,
                                                   const double* __restrict__ H, const double* __restrict__ tq,
                                                   double* __restrict__ JtPl) {
  extern __shared__ double bsm[];
  const int ld = n + 1;
  double* L = bsm;            // L[i + j * ld], i >= j
  double* y = bsm + n * ld;   // forward-solve vector (rhs, then L^{-1} rhs)
  double* xs = y + n;         // n
  double* rd = xs + n;        // 1 / l_jj
  __shared__ int s_fail;
  const int64_t b = blockIdx.x;
  if (!act[b]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double dl = delta[b];
  const double* Mb = M + b * (int64_t)n * n;
  double r[kCholSlots];
#pragma unroll
  for (int a = 0; a < kCholA; ++a)
#pragma unroll
    for (int c = 0; c <= 4 * a + 3; ++c) {
      const int i = lane + 32 * a, k = warp + kCholW * c;
      double v = 0.0;
      if (i < n && k < n && i >= k) {
        v = Mb[i + (int64_t)k * n];
        if (i == k && dl != 0.0) v = add(v, dl);
      }
      r[cslot(a, c)] = v;
    }
  for (int j = tid; j < n; j += kCholT) y[j] = rhs[b * n + j];
  if (tid == 0) s_fail = -1;
  __syncthreads();

  bool failed = false;
#pragma unroll
  for (int cb = 0; cb < kCholC; ++cb) {
    if (failed || kCholW * cb >= n) break;
    for (int jj = 0; jj < kCholW; ++jj) {
      const int j = kCholW * cb + jj;
      if (j >= n) break;
      if (warp == jj) {  // column j: its slot index cb is a constant here
        const int aj = j >> 5;
        double d = 0.0;
#pragma unroll
        for (int a = 0; a < kCholA; ++a)
          if (cb <= 4 * a + 3 && a == aj) d = r[cslot(a, cb)];
        d = __shfl_sync(0xffffffffu, d, j & 31);
        if (!(d > 0.0) || !isfinite(d)) {
          if (lane == 0) s_fail = j;
        } else {
          const double rl = b_rsqrt(d);
          const double yj = mul(y[j], rl);
          __syncwarp();
#pragma unroll
          for (int a = 0; a < kCholA; ++a) {
            if (cb > 4 * a + 3) continue;
            const int i = lane + 32 * a;
            if (i > j && i < n) {
              const double l = mul(r[cslot(a, cb)], rl);
              L[i + j * ld] = l;
              y[i] = fma(-l, yj, y[i]);
            }
          }
          if (lane == 0) {
            L[j + j * ld] = mul(d, rl);
            rd[j] = rl;
            y[j] = yj;
          }
        }
      }
      __syncthreads();
      if (s_fail >= 0) {
        failed = true;
        break;
      }
      if (j + 1 >= n) break;
      double li[kCholA];
#pragma unroll
      for (int a = 0; a < kCholA; ++a) {
        const int i = lane + 32 * a;
        li[a] = i > j && i < n ? L[i + j * ld] : 0.0;  // finished rows: no update
      }
#pragma unroll
      for (int c = 0; c < kCholC; ++c) {
        const double lk = L[min(warp + kCholW * c, n - 1) + j * ld];
#pragma unroll
        for (int a = 0; a < kCholA; ++a)
          if (c <= 4 * a + 3) r[cslot(a, c)] = fma(-li[a], lk, r[cslot(a, c)]);
      }
    }
  }
  if (s_fail >= 0) {
    if (tid == 0) pk[b].info = s_fail + 1;
    return;
  }
  // backward (one warp, right-looking): x_j = y_j / l_jj, then y_i -= l_ji x_j for i < j; lane
  // l keeps y_i for i = l + 32 a in registers and x_j reaches every lane by one shuffle
  if (warp == 0) {
    double yr[kCholA];
#pragma unroll
    for (int a = 0; a < kCholA; ++a) yr[a] = lane + 32 * a < n ? y[lane + 32 * a] : 0.0;
    for (int j = n - 1; j >= 0; --j) {
      double yj = 0.0;
#pragma unroll
      for (int a = 0; a < kCholA; ++a)
        if (a == (j >> 5)) yj = yr[a];
      yj = __shfl_sync(0xffffffffu, yj, j & 31);
      const double xj = mul(yj, rd[j]);
      if (lane == 0) xs[j] = xj;
#pragma unroll
      for (int a = 0; a < kCholA; ++a) {
        const int i = lane + 32 * a;
        if (i < j) yr[a] = fma(-L[j + i * ld], xj, yr[a]);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += kCholT) x[b * n + i] = xs[i];
  // J' p_lambda = (M - H) pv - tq: step_directions' p_lambda (ipm.cpp:79-103) through the
  // condensed matrix, J'(-r2 + Sigma (r3 + J pv)) = J' Sigma J pv - J'(r2 - Sigma r3), so the step
  // advances J'lambda by alpha J'p_lambda instead of a pass over P (the single-instance path's
  // recurrence, vec.cu k_jtpl_symv); row i of the lower triangle, then column i, ascending j
  for (int i = tid; i < n; i += kCholT) {
    double s = 0.0;
    for (int j = 0; j <= i; ++j) s = add(s, mul(sub(Mb[i + (int64_t)j * n], H[i + (int64_t)j * n]), xs[j]));
    for (int j = i + 1; j < n; ++j) s = add(s, mul(sub(Mb[j + (int64_t)i * n], H[j + (int64_t)i * n]), xs[j]));
    JtPl[b * n + i] = sub(s, tq[b * n + i]);
  }
  if (tid == 0) pk[b].info = 0;
}

// recovery rows: ps = -r3 - Jpv, plambda = -r2 + sigma (r3 + Jpv), pz = mu/s - z - sigma ps (J pv
// itself is not stored: nothing downstream reads it),
// fraction-to-boundary ratios and sum ps/s
__global__ void __launch_bounds__(kBT) k_b_recover_rows(int64_t m, int64_t py, const int32_t* __restrict__ row_map,
                                                        const double* __restrict__ y, const double* __restrict__ s,
                                                        const double* __restrict__ z, const double* __restrict__ sigma,
                                                        const double* __restrict__ r2, const double* __restrict__ r3,
                                                        const double* __restrict__ mu_p, double tau,
                                                        double* __restrict__ ps,
                                                        double* __restrict__ pl, double* __restrict__ pz,
                                                        double* __restrict__ part, const int* __restrict__ act) {
  __shared__ double sh[3 * 32];
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  const double mu = mu_p[b];
  const double* yb = y + b * py;
  double q = 0.0, as = 1e308, az = 1e308;
  B_ROWS_LOOP(m) {
    const int64_t o = b * m + r;
    const double jp = jrow_b(yb, row_map[r]);
    const double sr = s[o], zr = z[o], sg = sigma[o], t3 = r3[o];
    const double p_s = sub(-t3, jp);
    const double p_l = add(-r2[o], mul(sg, add(t3, jp)));
    const double p_z = sub(sub(mul(mu, dv(1.0, sr)), zr), mul(sg, p_s));
    ps[o] = p_s;
    pl[o] = p_l;
    pz[o] = p_z;
    q += dv(p_s, sr);
    if (p_s < 0.0) as = fmin(as, mul(tau, dv(-sr, p_s)));
    if (p_z < 0.0) az = fmin(az, mul(tau, dv(-zr, p_z)));
  }
  double su[1] = {q}, mx[2] = {-as, -az};  // minima as maxima of the negations (exact)
  block_out<1, 2>(su, mx, sh, part, Slots<1, 2>{{kBPsS}, {kBAs, kBAz}});
}

// (Hv + h) . pv, sum ps/s, alpha minima -> packet
__global__ void __launch_bounds__(kBT) k_b_recover_final(int64_t n, const double* __restrict__ Hv,
                                                         const double* __restrict__ h, const double* __restrict__ pv,
                                                         const double* __restrict__ part, Packet* pk,
                                                         const int* __restrict__ act) {
  __shared__ double sh[32];
  const int64_t b = blockIdx.x;
  if (!act[b]) return;
  double g = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) g += add(Hv[b * n + i], h[b * n + i]) * pv[b * n + i];
  g = block_sum<kBT>(g, sh);
  if (threadIdx.x == 0) {
    double q = 0.0, as = -1e308, az = -1e308;
    for (int k = 0; k < kBBlk; ++k) {
      const double* p = part + (b * kBBlk + k) * kBSlots;
      q += p[kBPsS];
      as = fmax(as, p[kBAs]);
      az = fmax(az, p[kBAz]);
    }
    Packet* p = pk + b;
    p->d_gpv = g;
    p->d_ps_s = q;
    p->alpha_s_min = -as < 1e308 ? -as : __longlong_as_double(0x7ff0000000000000ll);
    p->alpha_z_min = -az < 1e308 ? -az : __longlong_as_double(0x7ff0000000000000ll);
  }
}

// trial step lengths: alpha_b = min(1, alpha_s_min) (trial 0) or the host's value
__global__ void k_b_alpha0(int64_t B, const Packet* pk, double* __restrict__ alpha, const int* __restrict__ act) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < B && act[b]) alpha[b] = fmin(1.0, pk[b].alpha_s_min);
}
__global__ void k_b_vt(int64_t n, const double* __restrict__ v, const double* __restrict__ pv,
                       const double* __restrict__ alpha, double* __restrict__ vt, const int* __restrict__ act) {
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    vt[b * n + i] = add(v[b * n + i], mul(alpha[b], pv[b * n + i]));
}
// trial rows: s_t = s + alpha ps, J v_t = J v + alpha J pv (prototype values), merit sums
__global__ void __launch_bounds__(kBT) k_b_trial_rows(int64_t m, int64_t py, const int32_t* __restrict__ row_map,
                                                      const double* __restrict__ yv, const double* __restrict__ y,
                                                      const double* __restrict__ d, const double* __restrict__ s,
                                                      const double* __restrict__ ps, const double* __restrict__ alpha,
                                                      double* __restrict__ part, const int* __restrict__ act) {
  __shared__ double sh[3 * 32];
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  const double al = alpha[b];
  const double* yvb = yv + b * py;
  const double* yb = y + b * py;
  double sabs = 0.0, slog = 0.0, bad = 0.0;
  B_ROWS_LOOP(m) {
    const int64_t o = b * m + r;
    const double st = add(s[o], mul(al, ps[o]));
    if (st <= 0.0) bad = 1.0;
    slog += log(st);
    const int32_t rm = row_map[r];
    const double u = add(yvb[rm >> 1], mul(al, yb[rm >> 1]));
    const double jv = (rm & 1) ? -u : u;
    sabs += fabs(add(sub(jv, d[o]), st));
  }
  double su[2] = {sabs, slog}, mx[1] = {bad};
  block_out<2, 1>(su, mx, sh, part, Slots<2, 1>{{kBAbs, kBLog}, {kBBad}});
}
__global__ void __launch_bounds__(kBT) k_b_trial_final(int64_t n, int64_t m, const double* __restrict__ vt,
                                                       const double* __restrict__ Hvt, const double* __restrict__ h,
                                                       const double* __restrict__ part, Packet* pk,
                                                       const int* __restrict__ act) {
  __shared__ double sh[3 * 32];
  const int64_t b = blockIdx.x;
  if (!act[b]) return;
  double aa = 0.0, bb = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    aa += vt[b * n + i] * Hvt[b * n + i];
    bb += h[b * n + i] * vt[b * n + i];
  }
  double su[2] = {aa, bb}, mx[1] = {0.0};
  block_sums_maxs<kBT>(su, mx, sh);
  if (threadIdx.x == 0) {
    double sabs = 0.0, slog = 0.0, bad = 0.0;
    for (int k = 0; k < kBBlk; ++k) {
      const double* p = part + (b * kBBlk + k) * kBSlots;
      sabs += p[kBAbs];
      slog += p[kBLog];
      bad = fmax(bad, p[kBBad]);
    }
    Packet* p = pk + b;
    p->t_vHv = su[0];
    p->t_hv = su[1];
    p->t_sum_abs = m > 0 ? sabs : 0.0;
    p->t_sum_log = m > 0 ? slog : 0.0;
    p->any_nonpos = bad > 0.0 ? 1 : 0;
  }
}

// the accepted step (ipm.cpp:240-243)
// the accepted step of v (ipm.cpp:240-243) and what the accepted trial already formed at the
// new point: P v + alpha P pv (the trial's J v_t, k_b_trial_rows: the same operations) and
// H v_t (the trial's product; later trial rounds of other instances recompute it from the same
// v_t). The rows' step rides on the residual pass (k_b_res_rows<true>).
__global__ void k_b_step_v(int64_t n, int64_t py, const double* __restrict__ alpha, double* __restrict__ v,
                           const double* __restrict__ pv, double* __restrict__ yv, const double* __restrict__ y,
                           double* __restrict__ Hv, const double* __restrict__ Hvt, double* __restrict__ Jtl,
                           const double* __restrict__ JtPl, const int* __restrict__ act) {
  const int64_t b = blockIdx.y;
  if (!act[b]) return;
  const double al = alpha[b];
  const int64_t k = n > py ? n : py;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      v[b * n + i] = add(v[b * n + i], mul(al, pv[b * n + i]));
      Hv[b * n + i] = Hvt[b * n + i];
      Jtl[b * n + i] = add(Jtl[b * n + i], mul(al, JtPl[b * n + i]));  // J'(lambda + alpha p_lambda)
    }
    if (i < py) yv[b * py + i] = add(yv[b * py + i], mul(al, y[b * py + i]));
  }
}

}  // namespace

struct BatchCtx {
  Ctx* base = nullptr;
  int64_t B = 0, n = 0, m = 0, py = 0;
  cudaStream_t st = nullptr;
  void* blas = nullptr;
  BatchSyrk syrk;
  // per instance
  double *h = nullptr, *h0 = nullptr, *d = nullptr, *hmax = nullptr;
  double *v = nullptr, *s = nullptr, *lam = nullptr, *z = nullptr, *r1 = nullptr, *r2 = nullptr, *r3 = nullptr;
  double *sigma = nullptr, *w = nullptr, *omega = nullptr, *qw = nullptr, *lp = nullptr, *tq = nullptr;
  double *rhs = nullptr, *M = nullptr, *pv = nullptr, *ps = nullptr, *pl = nullptr, *pz = nullptr;
  double *yv = nullptr, *y = nullptr, *Hv = nullptr, *Hvt = nullptr, *vt = nullptr, *Jtl = nullptr;
  double* JtPl = nullptr;  // J' p_lambda of the step (k_b_chol's epilogue)
  double *part = nullptr, *mu = nullptr, *alpha = nullptr, *alpha_z = nullptr, *delta = nullptr;
  int* act = nullptr;
  Packet* pk = nullptr;
  Packet* pk_host = nullptr;
  double* hstage = nullptr;  // pinned staging ring for the per-instance scalars (mu, alpha, delta)
  int* istage = nullptr;     // pinned staging for the masks
  std::vector<double*> owned;
};

namespace {
template <typename T>
T* balloc(BatchCtx& b, size_t count, bool zero = false) {
  T* p = zero ? dev_zeros<T>(count, b.st) : dev_alloc<T>(count, b.st);
  b.owned.push_back(reinterpret_cast<double*>(p));
  return p;
}
unsigned bgrid(int64_t len) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(kBBlk, ceil_div(len, kBT))); }
}  // namespace

BatchCtx* batch_create(Ctx& base, int64_t B) {
  if (base.markov) throw DimError("batch mode reads the materialised prototypes: build the base QP with option markov = 0");
  if (B < 1) throw DimError("batch: count must be positive");
  if (base.n > kBatchMaxN) throw DimError("batch: the lockstep batch supports n <= 160");
  if (base.m == 0 || base.ps == 0) throw DimError("batch: the lockstep batch needs inequality rows");
  if (base.comm) throw DimError("batch: a sharded context cannot batch");
  auto* b = new BatchCtx;
  b->base = &base;
  b->B = B;
  b->n = base.n;
  b->m = base.m;
  b->py = (base.ldp + base.pz + 3) / 4 * 4;  // per-instance prototype vectors 32-byte aligned (bulk copies)
  b->st = base.stream;
  try {
    const int64_t n = b->n, m = b->m, py = b->py;
    b->h = balloc<double>(*b, B * n);
    b->h0 = balloc<double>(*b, B);
    b->d = balloc<double>(*b, B * m);
    b->hmax = balloc<double>(*b, B);
    for (double** p : {&b->v, &b->r1, &b->rhs, &b->pv, &b->Hv, &b->Hvt, &b->vt, &b->Jtl, &b->tq, &b->JtPl})
      *p = balloc<double>(*b, B * n, true);
    for (double** p : {&b->s, &b->lam, &b->z, &b->r2, &b->r3, &b->sigma, &b->w, &b->ps, &b->pl, &b->pz})
      *p = balloc<double>(*b, B * m, true);
    for (double** p : {&b->omega, &b->qw, &b->lp, &b->yv, &b->y}) *p = balloc<double>(*b, B * py, true);
    b->M = balloc<double>(*b, B * n * n, true);
    b->part = balloc<double>(*b, B * kBBlk * kBSlots, true);
    for (double** p : {&b->mu, &b->alpha, &b->alpha_z, &b->delta}) *p = balloc<double>(*b, B, true);
    b->act = balloc<int>(*b, B, true);
    b->pk = balloc<Packet>(*b, B, true);
    CMPC_CUDA(cudaMallocHost(&b->pk_host, sizeof(Packet) * B));
    CMPC_CUDA(cudaMallocHost(&b->hstage, sizeof(double) * kStageSlots * B));
    CMPC_CUDA(cudaMallocHost(&b->istage, sizeof(int) * kStageSlots * B));
    CMPC_CUDA(cudaFuncSetAttribute(k_b_chol, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * (kBatchMaxN * (kBatchMaxN + 1) + 3 * kBatchMaxN))));
    syrk_plan_batch(base, B, b->syrk, b->st);
    if (cublas().create(&b->blas) != 0) throw CudaError("batch: cublasCreate failed");
    cublas().set_stream(b->blas, b->st);
    CMPC_CUDA(cudaStreamSynchronize(b->st));
  } catch (...) {
    batch_destroy(b);
    throw;
  }
  return b;
}

void batch_destroy(BatchCtx* b) {
  if (!b) return;
  if (b->st) cudaStreamSynchronize(b->st);
  if (b->blas) cublas().destroy(b->blas);
  syrk_free_batch(b->syrk, b->st);
  for (double* p : b->owned) dev_free(p, b->st);
  if (b->pk_host) cudaFreeHost(b->pk_host);
  if (b->hstage) cudaFreeHost(b->hstage);
  if (b->istage) cudaFreeHost(b->istage);
  if (b->st) cudaStreamSynchronize(b->st);
  delete b;
}

void batch_set_affine(BatchCtx& b, const double* h, const double* h0, const double* d) {
  upload_h2d(b.h, h, sizeof(double) * b.B * b.n, b.st);
  upload_h2d(b.h0, h0, sizeof(double) * b.B, b.st);
  upload_h2d(b.d, d, sizeof(double) * b.B * b.m, b.st);
  k_b_hmax<<<(unsigned)b.B, kBT, 0, b.st>>>(b.n, b.h, b.hmax);
  CMPC_LAUNCHED();
  CMPC_CUDA(cudaStreamSynchronize(b.st));
}

namespace {

struct Host {
  BatchCtx& b;
  Ctx& c;
  // CMPC_BATCH_TIMES: device time per phase (events around each phase; diagnostics only)
  bool timed = getenv("CMPC_BATCH_TIMES") != nullptr;
  std::vector<std::pair<const char*, double>> acc;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  // device time of the condensation kernel (the bench's roofline), read after each sync
  cudaEvent_t sy0 = nullptr, sy1 = nullptr;
  double syrk_ms = 0.0, syrk_inst = 0.0;
  long long syrk_launches = 0;
  explicit Host(BatchCtx& bb) : b(bb), c(*bb.base) {
    CMPC_CUDA(cudaEventCreate(&sy0));
    CMPC_CUDA(cudaEventCreate(&sy1));
    if (timed) {
      cudaEventCreate(&t0);
      cudaEventCreate(&t1);
    }
  }
  void syrk_account(int64_t active) {  // after a sync: the iteration's condensation has run
    float ms = 0.f;
    CMPC_CUDA(cudaEventElapsedTime(&ms, sy0, sy1));
    syrk_ms += ms;
    syrk_inst += (double)active;
    ++syrk_launches;
  }
  ~Host() {
    cudaEventDestroy(sy0);
    cudaEventDestroy(sy1);
    if (timed) {
      for (auto& a : acc) fprintf(stderr, "[batch phase] %-10s %9.3f ms\n", a.first, a.second);
      cudaEventDestroy(t0);
      cudaEventDestroy(t1);
    }
  }
  template <typename F>
  void phase(const char* name, F&& f) {
    NvtxRange nv(name);
    if (!timed) {
      f();
      return;
    }
    cudaEventRecord(t0, b.st);
    f();
    cudaEventRecord(t1, b.st);
    cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    for (auto& a : acc)
      if (a.first == name) {
        a.second += ms;
        return;
      }
    acc.push_back({name, ms});
  }
  // exactly kBBlk blocks per instance: the final kernels read every block's partials (a block
  // without rows writes the neutral sums and maxima)
  dim3 rows() const { return dim3(kBBlk, (unsigned)b.B); }
  dim3 vecs() const { return dim3(bgrid(b.n), (unsigned)b.B); }
  dim3 protos() const { return dim3(bgrid(c.p), (unsigned)b.B); }
  // uploads go through a ring of kStageSlots pinned slots without a synchronize: at most four
  // uploads happen between two packet reads (which synchronize the stream), so a slot is never
  // rewritten while its copy is pending
  int hslot = 0, islot = 0;
  void upload_scalars(double* dst, const std::vector<double>& x) {
    double* st = b.hstage + (size_t)(hslot++ % kStageSlots) * b.B;
    std::memcpy(st, x.data(), sizeof(double) * b.B);
    CMPC_CUDA(cudaMemcpyAsync(dst, st, sizeof(double) * b.B, cudaMemcpyHostToDevice, b.st));
  }
  void upload_mask(const std::vector<int>& x) {
    int* st = b.istage + (size_t)(islot++ % kStageSlots) * b.B;
    std::memcpy(st, x.data(), sizeof(int) * b.B);
    CMPC_CUDA(cudaMemcpyAsync(b.act, st, sizeof(int) * b.B, cudaMemcpyHostToDevice, b.st));
  }
  void read_packets(long long* syncs) {
    CMPC_CUDA(cudaMemcpyAsync(b.pk_host, b.pk, sizeof(Packet) * b.B, cudaMemcpyDeviceToHost, b.st));
    CMPC_CUDA(cudaStreamSynchronize(b.st));
    ++*syncs;
  }
  // Y = P X (+ the singleton prototypes' values)
  void px(const double* X, double* Y) {
    dgemm(b.blas, false, (int)c.ldp, (int)b.B, (int)b.n, c.P, (int)c.ldp, X, (int)b.n, Y, (int)b.py);
    if (c.pz > 0) {
      k_b_sing<<<dim3(bgrid(c.pz), (unsigned)b.B), kBT, 0, b.st>>>(c.pz, b.n, b.py, c.ldp, c.sing_col, c.sing_val, X, Y);
      CMPC_LAUNCHED();
    }
  }
  // residuals at the current point (ipm.cpp:46-70) -> packets of the active instances
  // step: the accepted step's rows are applied by the residual row pass (v, P v, H v and J'lambda
  // by k_b_step_v before it)
  void residuals(bool step = false) {
    if (!step) {  // (after a step, k_b_step_v carried P v and H v)
      phase("res:Pv", [&] { px(b.v, b.yv); });
      phase("res:Hv", [&] {
        dgemm(b.blas, false, (int)b.n, (int)b.B, (int)b.n, c.H, (int)b.n, b.v, (int)b.n, b.Hv, (int)b.n);
      });
    }
    phase("res:rows", [&] {  // (before lamP: with a step it writes the new lambda)
      if (step)
        k_b_res_rows<true><<<rows(), kBT, 0, b.st>>>(b.m, b.py, c.row_map, b.yv, b.d, b.s, b.lam, b.z, b.mu, b.r2,
                                                     b.r3, b.part, b.act, b.alpha, b.alpha_z, b.ps, b.pl, b.pz,
                                                     b.sigma);
      else
        k_b_res_rows<false><<<rows(), kBT, 0, b.st>>>(b.m, b.py, c.row_map, b.yv, b.d, b.s, b.lam, b.z, b.mu, b.r2,
                                                      b.r3, b.part, b.act, nullptr, nullptr, nullptr, nullptr,
                                                      nullptr, b.sigma);
      CMPC_LAUNCHED();
    });
    if (!step) {  // (after a step, k_b_step_v advanced J'lambda by alpha J'p_lambda)
      phase("res:lamP", [&] {
        k_b_proto<true><<<protos(), kBT, 0, b.st>>>(c.p, c.ps, c.ldp, b.m, b.py, c.zero_k, c.mem_ptr, c.mem_rows,
                                                    b.lam, nullptr, b.lp, nullptr, b.act);
        CMPC_LAUNCHED();
      });
      phase("res:Jtl", [&] {
        dgemm(b.blas, true, (int)b.n, (int)b.B, (int)c.ldp, c.P, (int)c.ldp, b.lp, (int)b.py, b.Jtl, (int)b.n);
        k_b_sing_t<<<vecs(), kBT, 0, b.st>>>(b.n, b.py, c.ldp, c.sing_ptr, c.sing_val, b.lp, b.Jtl, b.act);
        CMPC_LAUNCHED();
      });
    }
    phase("res:final", [&] {
      k_b_res_final<<<(unsigned)b.B, kBT, 0, b.st>>>(b.n, b.m, b.Hv, b.h, b.Jtl, b.v, b.r1, b.part, b.hmax, b.h0,
                                                     b.pk, b.act);
      CMPC_LAUNCHED();
    });
  }
  void residuals_mu() {
    k_b_mu_rows<<<rows(), kBT, 0, b.st>>>(b.m, b.s, b.lam, b.z, b.mu, b.r2, b.part, b.act);
    CMPC_LAUNCHED();
    k_b_kkt_mu<<<(unsigned)ceil_div(b.B, 128), 128, 0, b.st>>>(b.B, b.n, b.m, b.part, b.pk, b.act);
    CMPC_LAUNCHED();
  }
  // sigma, omega, q, condensation with the right-hand side -r1 + J'(r2 - sigma r3)
  void condense() {
    // sigma = z / s came with the last residual pass; w = r2 - sigma r3 is formed inside the
    // prototype sums (r2 is current: a barrier update recomputes it)
    phase("omegaP", [&] {
      k_b_proto<false, true><<<protos(), kBT, 0, b.st>>>(c.p, c.ps, c.ldp, b.m, b.py, c.zero_k, c.mem_ptr,
                                                         c.mem_rows, b.sigma, nullptr, b.omega, b.qw, b.act, b.r2,
                                                         b.r3);
      CMPC_LAUNCHED();
    });
    phase("syrk", [&] {
      CMPC_CUDA(cudaEventRecord(sy0, b.st));
      launch_condense_batch(c, b.syrk, b.st, b.omega, b.qw, b.py, b.M, b.tq, b.rhs, b.r1, b.act);
      CMPC_CUDA(cudaEventRecord(sy1, b.st));
    });
  }
  void cholesky() {
    phase("chol", [&] {
      const size_t sm = sizeof(double) * ((size_t)b.n * (b.n + 1) + 3 * b.n);
      k_b_chol<<<(unsigned)b.B, kCholT, sm, b.st>>>((int)b.n, b.M, b.delta, b.rhs, b.pv, b.pk, b.act, c.H, b.tq,
                                                    b.JtPl);
      CMPC_LAUNCHED();
    });
  }
  // directions, fraction to boundary, line-search derivative pieces
  void recover(double tau) {
    phase("rec:Ppv", [&] { px(b.pv, b.y); });
    phase("rec:rows", [&] { recover_rows(tau); });
  }
  void recover_rows(double tau) {
    k_b_recover_rows<<<rows(), kBT, 0, b.st>>>(b.m, b.py, c.row_map, b.y, b.s, b.z, b.sigma, b.r2, b.r3, b.mu, tau,
                                               b.ps, b.pl, b.pz, b.part, b.act);
    CMPC_LAUNCHED();
    k_b_recover_final<<<(unsigned)b.B, kBT, 0, b.st>>>(b.n, b.Hv, b.h, b.pv, b.part, b.pk, b.act);
    CMPC_LAUNCHED();
  }
  // merit pieces at v + alpha pv, s + alpha ps (alpha from the device array)
  void trial(bool first) {
    phase("trial", [&] { trial_(first); });
  }
  void trial_(bool first) {
    if (first) {
      k_b_alpha0<<<(unsigned)ceil_div(b.B, 128), 128, 0, b.st>>>(b.B, b.pk, b.alpha, b.act);
      CMPC_LAUNCHED();
    }
    k_b_vt<<<vecs(), kBT, 0, b.st>>>(b.n, b.v, b.pv, b.alpha, b.vt, b.act);
    CMPC_LAUNCHED();
    dgemm(b.blas, false, (int)b.n, (int)b.B, (int)b.n, c.H, (int)b.n, b.vt, (int)b.n, b.Hvt, (int)b.n);
    k_b_trial_rows<<<rows(), kBT, 0, b.st>>>(b.m, b.py, c.row_map, b.yv, b.y, b.d, b.s, b.ps, b.alpha, b.part,
                                             b.act);
    CMPC_LAUNCHED();
    k_b_trial_final<<<(unsigned)b.B, kBT, 0, b.st>>>(b.n, b.m, b.vt, b.Hvt, b.h, b.part, b.pk, b.act);
    CMPC_LAUNCHED();
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

void batch_condense(BatchCtx& b, const double* sigma, const double* w, double* M_out, double* tq_out) {
  Ctx& c = *b.base;
  const int64_t B = b.B, n = b.n, m = b.m;
  upload_h2d(b.sigma, sigma, sizeof(double) * B * m, b.st);
  upload_h2d(b.w, w, sizeof(double) * B * m, b.st);
  std::vector<int> all(size_t(B), 1);
  std::memcpy(b.istage, all.data(), sizeof(int) * B);
  CMPC_CUDA(cudaMemcpyAsync(b.act, b.istage, sizeof(int) * B, cudaMemcpyHostToDevice, b.st));
  k_b_proto<false><<<dim3(bgrid(c.p), (unsigned)B), kBT, 0, b.st>>>(c.p, c.ps, c.ldp, m, b.py, c.zero_k, c.mem_ptr,
                                                                    c.mem_rows, b.sigma, b.w, b.omega, b.qw, b.act);
  CMPC_LAUNCHED();
  launch_condense_batch(c, b.syrk, b.st, b.omega, b.qw, b.py, b.M, b.tq, b.rhs, nullptr, b.act);
  CMPC_CUDA(cudaMemcpyAsync(M_out, b.M, sizeof(double) * B * n * n, cudaMemcpyDeviceToHost, b.st));
  CMPC_CUDA(cudaMemcpyAsync(tq_out, b.tq, sizeof(double) * B * n, cudaMemcpyDeviceToHost, b.st));
  CMPC_CUDA(cudaStreamSynchronize(b.st));
}

// the lockstep host loop: ipm::solve (ipm.cpp:160-268) for every instance, decision for decision
void batch_solve(BatchCtx& b, const double* opts, int64_t max_iter, double* v_out, double* scal, double* stats) {
  const double tol = opts[0], mu_init = opts[1], kappa_mu = opts[2], tau = opts[3], eta = opts[4];
  if (!(tol > 0.0)) throw DimError("tol must be positive");
  if (!(kappa_mu > 0.0 && kappa_mu < 1.0)) throw DimError("kappa_mu must lie in (0,1)");
  if (!(tau > 0.0 && tau < 1.0)) throw DimError("tau must lie in (0,1)");
  if (!(mu_init > 0.0)) throw DimError("mu_init must be positive");
  if (max_iter < 1) throw DimError("max_iter must be at least 1");
  NvtxRange nv("cmpc_batch_solve");
  Host H(b);
  const int64_t B = b.B, n = b.n, m = b.m;
  const long long launches0 = g_launches;
  long long syncs = 0, rounds = 0;
  const double t0 = now_s();
  cudaEvent_t e0, e1;
  CMPC_CUDA(cudaEventCreate(&e0));
  CMPC_CUDA(cudaEventCreate(&e1));
  CMPC_CUDA(cudaEventRecord(e0, b.st));

  std::vector<double> mu(B, mu_init), alpha(B, 0.0), alpha_z(B, 0.0), delta(B, 0.0), phi0(B), deriv(B);
  std::vector<int> status(B, -1), iter(B, 0), all(B, 1), shift(B, 0), trial_j(B, 0);
  std::vector<Packet> A(B);
  static constexpr std::array<double, 7> kShifts = {0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1.0, 1e2};
  constexpr double band = 10.0 * std::numeric_limits<double>::epsilon();

  H.upload_scalars(b.mu, mu);
  H.upload_mask(all);
  k_b_init<<<H.rows(), kBT, 0, b.st>>>(n, m, b.d, b.mu, b.v, b.s, b.lam, b.z);
  CMPC_LAUNCHED();
  H.residuals();
  H.read_packets(&syncs);
  for (int64_t i = 0; i < B; ++i) A[i] = b.pk_host[i];

  int64_t batch_iters = 0;
  while (true) {
    // check_termination (ipm.cpp:153-158), update_barrier (:146-151)
    std::vector<int> run(B, 0), chg(B, 0);
    bool any = false, any_chg = false;
    for (int64_t i = 0; i < B; ++i) {
      if (status[i] >= 0) continue;
      if (A[i].kkt <= tol && mu[i] <= tol) {
        status[i] = 0;
        continue;
      }
      if (iter[i] >= max_iter) {
        status[i] = 1;
        continue;
      }
      run[i] = 1;
      any = true;
      const double mn = (A[i].kkt <= 10.0 * mu[i]) ? std::max(tol / 10.0, kappa_mu * mu[i]) : mu[i];
      if (mn != mu[i]) {
        mu[i] = mn;
        chg[i] = 1;
        any_chg = true;
      }
    }
    if (!any) break;
    ++batch_iters;
    H.upload_scalars(b.mu, mu);
    if (any_chg) {
      H.upload_mask(chg);
      H.residuals_mu();
    }
    H.upload_mask(run);
    std::fill(delta.begin(), delta.end(), 0.0);
    H.upload_scalars(b.delta, delta);
    H.condense();
    H.cholesky();
    H.recover(tau);
    H.trial(true);
    H.read_packets(&syncs);
    ++rounds;
    H.syrk_account(std::count(run.begin(), run.end(), 1));
    std::vector<Packet> Bp(b.pk_host, b.pk_host + B);
    // shift ladder (ipm.cpp:205-221): re-factor the failed instances with the next shift
    for (int64_t i = 0; i < B; ++i) shift[i] = 0;
    while (true) {
      std::vector<int> retry(B, 0);
      bool any_r = false;
      for (int64_t i = 0; i < B; ++i)
        if (run[i] && Bp[i].info != 0 && shift[i] + 1 < (int)kShifts.size()) {
          ++shift[i];
          retry[i] = 1;
          any_r = true;
          delta[i] = kShifts[shift[i]];
        } else if (run[i] && Bp[i].info != 0) {
          shift[i] = (int)kShifts.size();  // every shift failed
        }
      if (!any_r) break;
      H.upload_scalars(b.delta, delta);
      H.upload_mask(retry);
      H.cholesky();
      H.recover(tau);
      H.trial(true);
      H.read_packets(&syncs);
      ++rounds;
      for (int64_t i = 0; i < B; ++i)
        if (retry[i]) Bp[i] = b.pk_host[i];
    }
    // line search (ipm.cpp:118-144) per instance: trial 0 evaluated; further trials in rounds
    std::vector<int> searching(B, 0);
    for (int64_t i = 0; i < B; ++i) {
      if (!run[i]) continue;
      A[i].kkt = Bp[i].kkt;  // kkt at the (possibly new) barrier value, as the reference's res
      A[i].max_comp = Bp[i].max_comp;
      if (shift[i] >= (int)kShifts.size() || Bp[i].info != 0) {
        status[i] = 2;  // factorization_failure
        run[i] = 0;
        continue;
      }
      const bool rows = m > 0;
      const double rho = 10.0 * A[i].max_lam + 1.0;
      phi0[i] = merit_host(A[i], A[i].obj_vHv, A[i].obj_hv, A[i].sum_log_s, A[i].sum_abs_r3, mu[i], rho, rows);
      double der = Bp[i].d_gpv;
      if (rows) {
        der -= mu[i] * Bp[i].d_ps_s;
        der -= rho * A[i].sum_abs_r3;
      }
      deriv[i] = der;
      alpha[i] = std::min(1.0, Bp[i].alpha_s_min);
      alpha_z[i] = std::min(1.0, Bp[i].alpha_z_min);
      trial_j[i] = 0;
      searching[i] = 1;
    }
    std::vector<int> accept(B, 0);
    for (int j = 0; j <= 30; ++j) {
      bool more = false;
      std::vector<int> next(B, 0);
      for (int64_t i = 0; i < B; ++i) {
        if (!searching[i]) continue;
        const Packet& T = b.pk_host[i];
        const bool rows = m > 0;
        const double rho = 10.0 * A[i].max_lam + 1.0;
        bool ok = false;
        if (!(rows && T.any_nonpos)) {
          const double phi = merit_host(T, T.t_vHv, T.t_hv, T.t_sum_log, T.t_sum_abs, mu[i], rho, rows);
          if (deriv[i] <= 0.0 && phi <= phi0[i] + eta * alpha[i] * deriv[i]) ok = true;
          else if (std::abs(phi - phi0[i]) <= band * (1.0 + std::abs(phi0[i]))) ok = true;
        }
        if (ok) {
          accept[i] = 1;
          trial_j[i] = j;
          searching[i] = 0;
        } else if (j == 30) {
          status[i] = 3;  // line_search_failure
          searching[i] = 0;
          run[i] = 0;
        } else {
          alpha[i] *= 0.5;
          next[i] = 1;
          more = true;
        }
      }
      if (!more) break;
      H.upload_scalars(b.alpha, alpha);
      H.upload_mask(next);
      H.trial(false);
      H.read_packets(&syncs);
      ++rounds;
    }
    // the accepted steps, then the residuals at the new points
    bool any_acc = false;
    for (int64_t i = 0; i < B; ++i)
      if (accept[i]) {
        any_acc = true;
        iter[i] += 1;
      }
    if (!any_acc) continue;
    H.upload_scalars(b.alpha, alpha);
    H.upload_scalars(b.alpha_z, alpha_z);
    H.upload_mask(accept);
    k_b_step_v<<<dim3(bgrid(std::max(n, b.py)), (unsigned)B), kBT, 0, b.st>>>(n, b.py, b.alpha, b.v, b.pv, b.yv, b.y,
                                                                          b.Hv, b.Hvt, b.Jtl, b.JtPl, b.act);
    CMPC_LAUNCHED();
    H.residuals(/*step=*/true);
    H.read_packets(&syncs);
    for (int64_t i = 0; i < B; ++i)
      if (accept[i]) A[i] = b.pk_host[i];
    static const char* dbg = getenv("CMPC_BATCH_DEBUG");  // instance whose iterations are printed
    if (dbg) {
      const int64_t q = atoll(dbg);
      if (q < B && accept[q])
        fprintf(stderr, "[batch %lld] iter %d mu %.6g alpha %.10g alpha_z %.10g kkt %.10g obj %.12g j %d\n",
                (long long)q, iter[q], mu[q], alpha[q], alpha_z[q], A[q].kkt, A[q].objective, trial_j[q]);
    }
  }
  CMPC_CUDA(cudaEventRecord(e1, b.st));
  if (v_out) CMPC_CUDA(cudaMemcpyAsync(v_out, b.v, sizeof(double) * B * n, cudaMemcpyDeviceToHost, b.st));
  CMPC_CUDA(cudaStreamSynchronize(b.st));
  float dms = 0.f;
  CMPC_CUDA(cudaEventElapsedTime(&dms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (int64_t i = 0; i < B; ++i) {
    double* o = scal + 14 * i;
    std::fill(o, o + 14, 0.0);
    o[0] = status[i] < 0 ? 1 : status[i];
    o[1] = iter[i];
    o[2] = A[i].kkt;
    o[3] = A[i].objective;
  }
  if (stats) {
    stats[0] = (double)batch_iters;
    stats[1] = dms * 1e-3;
    stats[2] = now_s() - t0;
    stats[3] = double(g_launches - launches0);
    stats[4] = double(syncs);
    stats[5] = double(rounds);
    stats[6] = H.syrk_ms * 1e-3;
    stats[7] = double(H.syrk_launches);
    stats[8] = H.syrk_inst;
    stats[9] = b.syrk.flops_per_instance;
  }
}

}  // namespace cmpc
