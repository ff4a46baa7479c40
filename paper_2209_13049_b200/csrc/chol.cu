// K2/K3/K4: Cholesky of the condensed matrix with the reference's failure rule, and
// the two triangular solves.
//
// Reference: ReferenceBackend::factorize (proj/src/dense_linalg.cpp:59-77: potf2 :24-40,
// trsm :43-51, trailing rankUpdate), failure "!(diag > 0) || !isfinite" at the first
// pivot; Factor::solve (:102-110). The shift ladder (proj/src/ipm.cpp:205-221) re-factors
// M + delta I; here M is kept intact and L written separately, so a retry never repeats the
// SYRK. info = failing pivot + 1 (0 = success).
//
// One persistent dataflow kernel (k_chol_df) factors the matrix in 32 x 32 tiles (lower
// tiles only), left-looking, and fuses both triangular solves:
//   diagonal task d   A_{d,d-1} <- M_{d,d-1} - sum_{k<d-1} L_dk L_{d-1,k}^T   (DMMA, registers)
//                     A_dd      <- M_dd + delta I - sum_{k<d-1} L_dk L_dk^T
//                     then, once diagonal d-1 is published: the sub-diagonal panel
//                     L_{d,d-1} = A_{d,d-1} W_{d-1}^T (published at once), A_dd -= L L^T,
//                     and the 32 x 32 factor: warp 0 runs the pivot chain (row i of the
//                     tile in lane i's registers; the next pivot travels by one shuffle,
//                     each finished column through shared memory) while warp 1 forms
//                     W_d = L_dd^{-1} column by column right behind it; forward solve
//                     y_d = W_d (b_d - sum_k L_dk y_k) rides along.
//   panel task (i, j), i >= j + 2:   L_ij = (M_ij - sum_{k<j} L_ik L_jk^T) W_j^T
//   backward task i:  x_i = W_i^T (y_i - sum_{j>i} L_ji^T x_j)
// So each column of the factor costs one inter-CTA hop on the critical path (diagonal d-1
// -> diagonal d), not two: the sub-diagonal panel is formed by the CTA that needs it next.
// Every finished tile publishes a per-tile flag (release/acquire at GPU scope) stamped with
// the launch's generation number, so flags never need resetting. CTAs grab tasks from an
// atomic counter in an order where a task only waits for tasks earlier in that order,
// which were grabbed by CTAs that are already running: the kernel cannot deadlock whatever
// the residency. The last CTA out publishes info and advances the generation. The W blocks
// are kept, so a later stand-alone solve (k_trsv) is block GEMVs.
#include <algorithm>

#include "internal.cuh"
#include "ptx.cuh"

namespace cmpc {

namespace {

#ifdef CMPC_CHOL_TRACE
// tools/exp/chol_trace.cu: per task, clock64 stamps kept in shared memory while the task runs
// (no global traffic inside the timed region) and flushed with a %globaltimer stamp at its end
__device__ unsigned long long g_ctrace[4096 * 10];
__shared__ unsigned long long s_ctrace[8];
__device__ __forceinline__ void ctrace(int slot) {
  if (threadIdx.x == 0) s_ctrace[slot] = clock64();
}
__device__ __forceinline__ void ctrace_flush(int task) {
  if (threadIdx.x == 0 && task < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long c = clock64();
    for (int k = 0; k < 8; ++k) g_ctrace[task * 10 + k] = s_ctrace[k] ? c - s_ctrace[k] : 0ull;
    g_ctrace[task * 10 + 8] = t;
    for (int k = 0; k < 8; ++k) s_ctrace[k] = 0;
  }
}
#define CTRACE(task, slot) ctrace(slot)
#define CTRACE_FLUSH(task) ctrace_flush(task)
#else
#define CTRACE(task, slot) \
  do {                     \
  } while (0)
#define CTRACE_FLUSH(task) \
  do {                     \
  } while (0)
#endif

constexpr int kB = 32;           // tile edge
constexpr int kLD = 36;          // staged-tile leading dimension (conflict-free DMMA fragments)
constexpr int kTS = kB * kLD;    // doubles per staged tile
constexpr int kT = 128;          // threads per CTA (4 warps)
constexpr unsigned kFull = 0xffffffffu;

// shared memory (doubles)
constexpr int kOffStage = 0;              // 2 stages x {X, Y}
constexpr int kOffA = 4 * kTS;            // -acc of a panel / the factor's input and L
constexpr int kOffW = 5 * kTS;            // a staged W / the new W of a diagonal tile
constexpr int kOffP = 6 * kTS;            // the panel product
constexpr int kOffCol = 7 * kTS;          // 32 x 32 finished factor columns (pivot chain)
constexpr int kOffRR = kOffCol + kB * kB; // 1 / l_pp
constexpr int kOffYs = kOffRR + kB;       // 2 staged y_k
constexpr int kOffYp = kOffYs + 2 * kB;   // y_{d-1}
constexpr int kOffTv = kOffYp + kB;       // b_d - sum_k L_dk y_k
constexpr int kOffRed = kOffTv + kB;      // 4 x 32 quarter partial sums
constexpr int kSmemDoubles = kOffRed + 4 * kB;
constexpr int kDfSmem = kSmemDoubles * 8;
static_assert((kOffCol * 8) % 16 == 0, "16-byte aligned factor columns");

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// polling load: relaxed (an acquire load compiles to LDG.STRONG + CCTL.IVALL, and a spinning
// CTA's stream of L1 invalidations slows the shared-memory pipe of its SM neighbour, e.g. a
// diagonal tile's pivot chain); the acquire fence follows once the flag is seen
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// 1/sqrt(x): MUFU.RSQ64H seed + two Newton steps (~1/3 the latency of the exact sequence);
// flushes subnormals, so the caller re-factors exactly when a pivot leaves [1e-300, 1e300]
__device__ __forceinline__ double rsqrt_mufu(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// stage a packed 32 x 32 tile (column-major, 32 contiguous doubles per column) into
// x[k * kLD + i] with 16-byte cp.async (L2 only: tiles written by other CTAs)
__device__ __forceinline__ void stage_tile(double* x, const double* src) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int ch = threadIdx.x + kT * u;
    const int k = ch >> 4, i2 = (ch & 15) * 2;
    cp_async16(x + k * kLD + i2, src + k * kB + i2);
  }
}
__device__ __forceinline__ void stage_vec(double* x, const double* src) {
  if (threadIdx.x < 16) cp_async16(x + 2 * threadIdx.x, src + 2 * threadIdx.x);
}

// Warp w owns the 16 x 16 block (rows 16 (w & 1) + [0,16), columns 16 (w >> 1) + [0,16)) of a
// 32 x 32 tile as two m16n8 fragments: acc[ni][e] is element
// (16 (w & 1) + g + 8 (e >> 1), 16 (w >> 1) + 8 ni + 2 t + (e & 1)).
struct Frag {
  int m0, n0, g, t;
  __device__ Frag() {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    m0 = 16 * (warp & 1);
    n0 = 16 * (warp >> 1);
    g = lane >> 2;
    t = lane & 3;
  }
  __device__ int row(int e) const { return m0 + g + 8 * (e >> 1); }
  __device__ int col(int ni, int e) const { return n0 + 8 * ni + 2 * t + (e & 1); }
};

// acc += X Y^T (k = 0..31) for this warp's block; X, Y staged as x[k * kLD + row]
__device__ __forceinline__ void gemm_xyt(const Frag& f, const double* x, const double* y, double (&acc)[2][4]) {
  const double* xa = x + f.t * kLD + f.m0 + f.g;
  const double* yb = y + f.t * kLD + f.n0 + f.g;
#pragma unroll
  for (int ks = 0; ks < kB; ks += 4) {
    const int o = ks * kLD;
    const double af[2] = {xa[o], xa[o + 8]};
    dmma1684(acc[0], af, yb[o]);
    dmma1684(acc[1], af, yb[o + 8]);
  }
}

__device__ __forceinline__ void frag_store(const Frag& f, double* x, const double (&acc)[2][4], double sign) {
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int e = 0; e < 4; ++e) x[f.col(ni, e) * kLD + f.row(e)] = sign * acc[ni][e];
}

struct DfArgs {
  const double* M;  // n x n, lower part read
  double* L;        // n x n column-major factor (lower tiles and diagonal tiles written)
  double* Lt;       // nt x nt packed 32 x 32 tiles of L (off-diagonal tiles), read by other CTAs
  double* W;        // nt packed 32 x 32 inverses of the diagonal tiles
  int64_t n;
  double delta;
  int nt, ntasks;
  unsigned* flags;  // nt x nt per-tile done flags (== generation when done)
  unsigned* ctl;    // [0] generation, [1] exit count, [2] failure generation, [3] pivot + 1, [4] task counter
  long long* info;
  const double* rhs;  // n (nullptr: factor only)
  double* x;          // n (may alias rhs: rhs is read before any block of x is written)
  double* ybuf;       // nt * 32
  double* xbuf;       // nt * 32
  unsigned* xflags;   // nt
  int nback;          // nt when solving, else 0
};

// thread 0: spin until both flags carry the generation; false on a published failure
__device__ __forceinline__ bool wait_flags(const unsigned* f1, const unsigned* f2, const unsigned* fail,
                                           unsigned target) {
  while (true) {
    if (ld_relaxed(f1) == target && ld_relaxed(f2) == target) {
      fence_acquire();
      return true;
    }
    if (ld_relaxed(fail) == target) {
      fence_acquire();
      return false;
    }
  }
}
__device__ __forceinline__ unsigned* tile_flag(const DfArgs& A, int i, int j) { return A.flags + i * A.nt + j; }
__device__ __forceinline__ const double* tile_src(const DfArgs& A, int i, int j) {
  return A.Lt + ((size_t)i * A.nt + j) * (kB * kB);
}
__device__ __forceinline__ void publish(unsigned* flag, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(flag, target);
  }
}

// acc = -(M block at (r0, c0)) (+ -delta on the diagonal); lower part only when diag
__device__ __forceinline__ void load_neg_m(const Frag& f, const DfArgs& A, int64_t r0, int64_t c0, bool diag,
                                           double (&acc)[2][4]) {
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = f.row(e), c = f.col(ni, e);
      double v = 0.0;
      if (r0 + r < A.n && c0 + c < A.n && (!diag || r >= c)) {
        v = A.M[(r0 + r) + (c0 + c) * A.n];
        if (diag && r == c && A.delta != 0.0) v = add(v, A.delta);
      }
      acc[ni][e] = -v;
    }
}

// left-looking updates acc1 += L_{i,k} L_{j1,k}^T and (two) acc2 += L_{i,k} L_{j2,k}^T for
// k < K, double-buffered (tile k+1 prefetched when already published); with fwd also the
// forward-solve partial sum_k L_{i,k} y_k (thread: row tid & 31, columns of quarter tid >> 5).
// Returns false on a published failure.
template <bool TWO>
__device__ bool left_updates(const DfArgs& A, const Frag& f, int i, int j1, int K, bool skip2, unsigned target,
                             double* sm, volatile unsigned* s_flag, double (&acc1)[2][4], double (&acc2)[2][4],
                             bool fwd, double& fpart) {
  if (K <= 0) return true;
  const int tid = threadIdx.x;
  const unsigned* failw = A.ctl + 2;
  // stage s: X at sm + 2 s kTS (rows i), Y at + kTS (rows j1)
  if (tid == 0) *s_flag = wait_flags(tile_flag(A, i, 0), tile_flag(A, j1, 0), failw, target) ? 1u : 2u;
  __syncthreads();
  if (*s_flag == 2u) return false;
  double* ys = sm + kOffYs;
  stage_tile(sm, tile_src(A, i, 0));
  stage_tile(sm + kTS, tile_src(A, j1, 0));
  if (fwd) stage_vec(ys, A.ybuf);
  cp_commit();
  const int fr = tid & 31, qd = tid >> 5;
  for (int k = 0; k < K; ++k) {
    const int s = k & 1;
    double* xs = sm + 2 * s * kTS;
    double* xo = sm + 2 * (s ^ 1) * kTS;
    const bool more = k + 1 < K;
    if (tid == 0) {
      const bool ready =
          more && ld_relaxed(tile_flag(A, i, k + 1)) == target && ld_relaxed(tile_flag(A, j1, k + 1)) == target;
      if (ready) fence_acquire();
      *s_flag = ready ? 1u : 0u;
    }
    __syncthreads();  // buffer s^1 is free (gemm k-1 done); s_flag visible
    const bool pre = *s_flag == 1u;
    if (pre) {
      stage_tile(xo, tile_src(A, i, k + 1));
      stage_tile(xo + kTS, tile_src(A, j1, k + 1));
      if (fwd) stage_vec(ys + kB * (s ^ 1), A.ybuf + kB * (k + 1));
    }
    cp_commit();
    cp_wait1();
    __syncthreads();  // tile k visible to every warp
    if (TWO) {
      if (!skip2) gemm_xyt(f, xs, xs, acc2);   // the diagonal block's own update
      gemm_xyt(f, xs, xs + kTS, acc1);
    } else {
      gemm_xyt(f, xs, xs + kTS, acc1);
    }
    if (fwd) {
      const double* yk = ys + kB * s;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) fpart = fma(xs[(8 * qd + kk) * kLD + fr], yk[8 * qd + kk], fpart);
    }
    if (more && !pre) {
      if (tid == 0)
        *s_flag = wait_flags(tile_flag(A, i, k + 1), tile_flag(A, j1, k + 1), failw, target) ? 1u : 2u;
      __syncthreads();
      if (*s_flag == 2u) return false;
      stage_tile(xo, tile_src(A, i, k + 1));
      stage_tile(xo + kTS, tile_src(A, j1, k + 1));
      if (fwd) stage_vec(ys + kB * (s ^ 1), A.ybuf + kB * (k + 1));
      cp_commit();
    }
  }
  __syncthreads();  // staging buffers free
  return true;
}

// L_ij = (-acc) W_j^T: waits for diagonal j, stages W_j (and y_j into yprev when fwd), leaves
// the product in the P region and writes it to Lt and L. Returns false on a failure.
__device__ bool panel(const DfArgs& A, const Frag& f, int i, int j, unsigned target, double* sm,
                      volatile unsigned* s_flag, const double (&acc)[2][4], bool fwd) {
  const int tid = threadIdx.x;
  if (tid == 0) *s_flag = wait_flags(tile_flag(A, j, j), tile_flag(A, j, j), A.ctl + 2, target) ? 1u : 2u;
  frag_store(f, sm + kOffA, acc, -1.0);
  __syncthreads();
  CTRACE(0, 7);
  if (*s_flag == 2u) return false;
  stage_tile(sm + kOffW, A.W + (size_t)j * (kB * kB));
  if (fwd) stage_vec(sm + kOffYp, A.ybuf + kB * j);
  cp_commit();
  cp_wait0();
  __syncthreads();
  double out[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  gemm_xyt(f, sm + kOffA, sm + kOffW, out);
  frag_store(f, sm + kOffP, out, 1.0);
  __syncthreads();
  double* Lt = A.Lt + ((size_t)i * A.nt + j) * (kB * kB);
  const int64_t r0 = (int64_t)kB * i, c0 = (int64_t)kB * j;
  for (int e = tid; e < kB * kB; e += kT) {
    const int r = e & 31, c = e >> 5;
    const double v = sm[kOffP + c * kLD + r];
    Lt[e] = v;
    if (r0 + r < A.n) A.L[(r0 + r) + (c0 + c) * A.n] = v;
  }
  return true;
}

// warp 0: the 32 x 32 factor of a (column-major lower input, kLD) in place, row i in lane i's
// registers. Pivot p: l_ip = a_ip / sqrt(a_pp); the next pivot a_{p+1,p+1} - l^2 is formed in
// lane p+1 and shuffled to all lanes (the critical chain); column p goes to shared memory
// (col) for the rank-1 update of every row and for warp 1's inverse. Returns the first
// failing pivot (< b) or -1; *odd when a pivot left the fast rsqrt's range.
#ifdef CMPC_CHOL_NOINLINE
#define CHOL_FACTOR_INLINE __noinline__
#else
#define CHOL_FACTOR_INLINE
#endif
template <bool EXACT>
__device__ CHOL_FACTOR_INLINE int factor_rows(double* a_sm, double* col, double* rr, volatile int* cnt, int b, bool* odd) {
  const int lane = threadIdx.x & 31;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = (c <= lane) ? a_sm[c * kLD + lane] : 0.0;
  double dcur = __shfl_sync(kFull, a[0], 0);
  int fail = -1;
  bool bad = false;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    if (fail < 0 && p < b && (!(dcur > 0.0) || !isfinite(dcur))) fail = p;
    bad |= !(dcur >= 1e-300 && dcur <= 1e300);
    const double r = EXACT ? 1.0 / sqrt(dcur) : rsqrt_mufu(dcur);
    const double l = (lane >= p) ? a[p] * r : 0.0;
    a[p] = l;
    if (p < 31) {
      const double dn = fma(-l, l, a[p + 1]);  // lane p+1: its next pivot
      dcur = __shfl_sync(kFull, dn, p + 1);
    }
    col[p * kB + lane] = l;
    if (lane == 0) rr[p] = r;
    __syncwarp();
    if (lane == 0) {
#ifndef CMPC_CHOL_NOFENCE
      __threadfence_block();
#endif
      *cnt = p + 1;
    }
#pragma unroll
    for (int c = (p + 1) & ~1; c < 32; c += 2) {
      const double2 lc = ld2(col + p * kB + c);
      if (c > p) a[c] = fma(-l, lc.x, a[c]);
      if (c + 1 > p) a[c + 1] = fma(-l, lc.y, a[c + 1]);
    }
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) a_sm[c * kLD + lane] = (c <= lane) ? a[c] : 0.0;
  *odd = bad;
  return fail;
}

// warp 1: W = L^{-1} column by column (lane c = column c), one pivot behind warp 0:
// w_p = s_p / l_pp, s_i -= l_ip w_p (i > p). Column-major into w_sm.
__device__ CHOL_FACTOR_INLINE void inverse_cols(double* w_sm, const double* col, const double* rr, volatile int* cnt) {
  const int lane = threadIdx.x & 31;
  double s[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    while (*cnt <= p) __nanosleep(20);
#ifndef CMPC_CHOL_NOFENCE
    __threadfence_block();
#endif
    const double wp = s[p] * rr[p];
    s[p] = wp;
#pragma unroll
    for (int i = (p + 1) & ~1; i < 32; i += 2) {
      const double2 lc = ld2(col + p * kB + i);
      if (i > p) s[i] = fma(-lc.x, wp, s[i]);
      if (i + 1 > p) s[i + 1] = fma(-lc.y, wp, s[i + 1]);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) w_sm[lane * kLD + i] = (i >= lane) ? s[i] : 0.0;
}

// diagonal task d: the sub-diagonal panel L_{d,d-1} and the diagonal tile (see the header)
__device__ bool df_diag(const DfArgs& A, int d, unsigned target, double* sm, volatile unsigned* s_flag,
                        volatile int* cnt, volatile int* s_res) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Frag f;
  const int64_t r0 = (int64_t)kB * d;
  const bool fwd = A.rhs != nullptr;
  const bool has_p = d >= 1;
  const bool upper = warp == 2;  // rows 0..15 x columns 16..31: strictly upper in a diagonal tile
  double accP[2][4], accD[2][4];
  if (has_p) load_neg_m(f, A, r0, r0 - kB, false, accP);
  load_neg_m(f, A, r0, r0, true, accD);
  double fpart = 0.0;
  CTRACE(d, 0);
  if (!left_updates<true>(A, f, d, d - 1, d - 1, upper, target, sm, s_flag, accP, accD, fwd, fpart)) return false;
  CTRACE(d, 1);
  const int fr = tid & 31, qd = tid >> 5;
  if (has_p) {
    if (!panel(A, f, d, d - 1, target, sm, s_flag, accP, fwd)) return false;
    publish(tile_flag(A, d, d - 1), target);
    CTRACE(d, 2);
    if (!upper) gemm_xyt(f, sm + kOffP, sm + kOffP, accD);
    if (fwd) {
      const double* yp = sm + kOffYp;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) fpart = fma(sm[kOffP + (8 * qd + kk) * kLD + fr], yp[8 * qd + kk], fpart);
    }
  }
  double* red = sm + kOffRed;
  double* tv = sm + kOffTv;
  if (fwd) red[qd * kB + fr] = fpart;
  const int b = (int)(A.n - r0 < kB ? A.n - r0 : kB);
  // factor input: -accD, lower, identity padding beyond b
  double* a_sm = sm + kOffA;
  auto store_input = [&] {
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = f.row(e), c = f.col(ni, e);
        double v;
        if (r >= b || c >= b) v = (r == c) ? 1.0 : 0.0;
        else v = (r >= c) ? -accD[ni][e] : 0.0;
        a_sm[c * kLD + r] = v;
      }
  };
  store_input();
  if (tid == 0) *cnt = 0;
  __syncthreads();
  if (fwd && tid < kB) {
    const double bi = r0 + tid < A.n ? A.rhs[r0 + tid] : 0.0;
    tv[tid] = bi - ((red[tid] + red[kB + tid]) + (red[2 * kB + tid] + red[3 * kB + tid]));
  }
  double* col = sm + kOffCol;
  double* rr = sm + kOffRR;
  bool odd = false;
  CTRACE(d, 3);
  if (warp == 0) {
    const int fl = factor_rows<false>(a_sm, col, rr, cnt, b, &odd);
    if (lane == 0) {
      s_res[0] = fl;
      s_res[1] = odd ? 1 : 0;
    }
  } else if (warp == 1) {
    inverse_cols(sm + kOffW, col, rr, cnt);
  }
  __syncthreads();
  CTRACE(d, 6);
  if (s_res[1]) {  // a pivot outside [1e-300, 1e300]: redo the tile with the exact square root
    store_input();
    if (tid == 0) *cnt = 0;
    __syncthreads();
    if (warp == 0) {
      const int fl = factor_rows<true>(a_sm, col, rr, cnt, b, &odd);
      if (lane == 0) s_res[0] = fl;
    } else if (warp == 1) {
      inverse_cols(sm + kOffW, col, rr, cnt);
    }
    __syncthreads();
  }
  CTRACE(d, 4);
  const int fl = s_res[0];
  if (fl >= 0) {
    if (tid == 0) {
      A.ctl[3] = (unsigned)(r0 + fl + 1);
      __threadfence();
      st_release(A.ctl + 2, target);
    }
    return false;
  }
  const double* w_sm = sm + kOffW;
  if (fwd) {  // y_d = W_d t (W lower): quarter sums in a fixed order
    double s = 0.0;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int c = 8 * qd + cc;
      if (c <= fr) s = fma(w_sm[c * kLD + fr], tv[c], s);
    }
    __syncthreads();  // red reused
    red[qd * kB + fr] = s;
    __syncthreads();
    if (tid < kB) A.ybuf[r0 + tid] = (red[tid] + red[kB + tid]) + (red[2 * kB + tid] + red[3 * kB + tid]);
  }
  double* Wd = A.W + (size_t)d * (kB * kB);
  for (int e = tid; e < kB * kB; e += kT) {
    const int r = e & 31, c = e >> 5;
    if (r < b && c < b) A.L[(r0 + r) + (r0 + c) * A.n] = a_sm[c * kLD + r];
    Wd[e] = w_sm[c * kLD + r];
  }
  publish(tile_flag(A, d, d), target);
  CTRACE(d, 5);
  CTRACE_FLUSH(d);
  return true;
}

// panel task (i, j), i >= j + 2
__device__ bool df_panel(const DfArgs& A, int i, int j, unsigned target, double* sm, volatile unsigned* s_flag) {
  const Frag f;
  double acc[2][4], unused[2][4];
  CTRACE(64 + i * 64 + j, 0);
  load_neg_m(f, A, (int64_t)kB * i, (int64_t)kB * j, false, acc);
  double fpart = 0.0;
  if (!left_updates<false>(A, f, i, j, j, true, target, sm, s_flag, acc, unused, false, fpart)) return false;
  CTRACE(64 + i * 64 + j, 1);
  if (!panel(A, f, i, j, target, sm, s_flag, acc, false)) return false;
  publish(tile_flag(A, i, j), target);
  CTRACE(64 + i * 64 + j, 2);
  CTRACE_FLUSH(64 + i * 64 + j);
  return true;
}

// backward block i: x_i = W_i^T (y_i - sum_{j>i} L_ji^T x_j), j from the last block down (the
// tile L_ji is staged before x_j is awaited). Warp w owns columns 8w..8w+7; lane = row;
// fixed-order warp sums.
__device__ bool df_back(const DfArgs& A, int i, unsigned target, double* sm, volatile unsigned* s_flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = A.nt;
  const unsigned* failw = A.ctl + 2;
  CTRACE(2048 + i, 0);
  if (tid == 0) *s_flag = wait_flags(tile_flag(A, i, i), tile_flag(A, i, i), failw, target) ? 1u : 2u;
  __syncthreads();
  if (*s_flag == 2u) return false;
  const double* Wi = A.W + (size_t)i * (kB * kB);
  double wv[8], part[8];
#pragma unroll
  for (int cl = 0; cl < 8; ++cl) {
    wv[cl] = __ldcg(Wi + (8 * warp + cl) * kB + lane);
    part[cl] = 0.0;
  }
  for (int j = nt - 1; j > i; --j) {
    double* xs = sm + (j & 1) * kTS;
    if (tid == 0) *s_flag = wait_flags(tile_flag(A, j, i), tile_flag(A, j, i), failw, target) ? 1u : 2u;
    __syncthreads();
    if (*s_flag == 2u) return false;
    stage_tile(xs, tile_src(A, j, i));
    cp_commit();
    if (tid == 0) *s_flag = wait_flags(A.xflags + j, A.xflags + j, failw, target) ? 1u : 2u;
    cp_wait0();
    __syncthreads();
    if (*s_flag == 2u) return false;
    const double xj = __ldcg(A.xbuf + kB * j + lane);
#pragma unroll
    for (int cl = 0; cl < 8; ++cl) part[cl] = fma(xs[(8 * warp + cl) * kLD + lane], xj, part[cl]);
  }
  double* accv = sm + kOffTv;
  const double* yi = A.ybuf + kB * i;
#pragma unroll
  for (int cl = 0; cl < 8; ++cl) {
    const double s = warp_sum(part[cl]);
    if (lane == 0) accv[8 * warp + cl] = __ldcg(yi + 8 * warp + cl) - s;
  }
  __syncthreads();
  const double a0 = accv[lane];
  const int64_t r0 = (int64_t)kB * i;
#pragma unroll
  for (int cl = 0; cl < 8; ++cl) {
    const int c = 8 * warp + cl;  // x(c) = sum_{r >= c} W(r, c) acc(r)
    const double s = warp_sum(wv[cl] * a0);
    if (lane == 0) {
      A.xbuf[kB * i + c] = s;
      if (r0 + c < A.n) A.x[r0 + c] = s;
    }
  }
  publish(A.xflags + i, target);
  CTRACE(2048 + i, 1);
  CTRACE_FLUSH(2048 + i);
  return true;
}

__global__ void __launch_bounds__(kT) k_chol_df(const DfArgs A) {
  extern __shared__ __align__(16) double sm_df[];
  __shared__ unsigned s_target, s_q, s_flag;
  __shared__ int s_cnt, s_res[2];
  const int tid = threadIdx.x;
  if (tid == 0) s_target = *reinterpret_cast<volatile unsigned*>(A.ctl) + 1u;
  __syncthreads();
  const unsigned target = s_target;
  CTRACE(4095, 0);
  CTRACE_FLUSH(4095);
  while (true) {
    if (tid == 0) s_q = atomicAdd(A.ctl + 4, 1u);
    __syncthreads();
    const int q = (int)s_q;
    if (q >= A.ntasks + A.nback) break;
    bool ok;
    if (q >= A.ntasks) {  // backward solve tasks, last block first
      ok = df_back(A, A.nt - 1 - (q - A.ntasks), target, sm_df, &s_flag);
    } else {
      // column by column: the diagonal task of column j (it also forms L_{j,j-1}), then the
      // panels (i, j), i >= j + 2
      int j = 0, rem = q;
      while (true) {
        const int cnt = 1 + max(0, A.nt - j - 2);
        if (rem < cnt) break;
        rem -= cnt;
        ++j;
      }
      if (rem == 0) ok = df_diag(A, j, target, sm_df, &s_flag, &s_cnt, s_res);
      else ok = df_panel(A, j + 1 + rem, j, target, sm_df, &s_flag);
    }
    if (!ok) break;
    __syncthreads();
  }
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

// inverse of every 32 x 32 diagonal block of an existing factor (one warp per block)
__global__ void __launch_bounds__(32) k_diag_inv(const double* __restrict__ L, int64_t n,
                                                 double* __restrict__ Winv) {
  __shared__ double a[kB][kB + 1];  // a[c][r] = L(k0 + r, k0 + c)
  const int lane = threadIdx.x;
  const int64_t k0 = (int64_t)blockIdx.x * kB;
  const int b = (int)(n - k0 < kB ? n - k0 : kB);
  for (int e = lane; e < kB * kB; e += 32) {
    const int r = e & 31, c = e >> 5;
    a[c][r] = (r < b && c < b) ? (r >= c ? L[(k0 + r) + (k0 + c) * n] : 0.0) : (r == c ? 1.0 : 0.0);
  }
  __syncwarp();
  double s[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    const double wp = s[p] / a[p][p];
    s[p] = wp;
#pragma unroll
    for (int i = p + 1; i < 32; ++i) s[i] = fma(-a[p][i], wp, s[i]);
  }
  double* W = Winv + (size_t)blockIdx.x * kB * kB + lane * kB;
#pragma unroll
  for (int i = 0; i < 32; ++i) W[i] = (i >= lane) ? s[i] : 0.0;
}

// x = L^{-T} L^{-1} b with the 32 x 32 diagonal-block inverses W; one CTA of 512 threads;
// x may alias b. Forward: y_k = W_k (b_k - sum_{j<k} L_kj y_j); backward:
// x_k = W_k^T (y_k - sum_{i>k} L_ik^T x_i).
__global__ void __launch_bounds__(512) k_trsv(const double* __restrict__ L,
                                              const double* __restrict__ W, const double* b,
                                              double* x, int64_t n) {
  extern __shared__ double xs[];
  double* t = xs + n;  // 32 scratch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int64_t i = tid; i < n; i += blockDim.x) xs[i] = b[i];
  __syncthreads();
  const int64_t nb = (n + kB - 1) / kB;
  const int row = tid >> 4, part = tid & 15;  // 32 rows x 16 parts
  auto sum16 = [](double s) {
    s += __shfl_xor_sync(kFull, s, 1);
    s += __shfl_xor_sync(kFull, s, 2);
    s += __shfl_xor_sync(kFull, s, 4);
    s += __shfl_xor_sync(kFull, s, 8);
    return s;
  };
  for (int64_t kb = 0; kb < nb; ++kb) {
    const int64_t r0 = kb * kB;
    const int bs = (int)(n - r0 < kB ? n - r0 : kB);
    const double* Wk = W + kb * kB * kB;
    // y_k = W_k b'_k (W lower: row i uses columns j <= i)
    double s = 0.0;
    if (row < bs)
      for (int j = part; j <= row; j += 16) s += Wk[row + j * kB] * xs[r0 + j];
    s = sum16(s);
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
    const int64_t r0 = kb * kB;
    const int bs = (int)(n - r0 < kB ? n - r0 : kB);
    const int64_t tail = r0 + bs;
    const double* Wk = W + kb * kB * kB;
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
      for (int j = row + part; j < bs; j += 16) s += Wk[j + row * kB] * t[j];
    s = sum16(s);
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
    CMPC_CUDA(cudaFuncSetAttribute(k_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
}

}  // namespace

void chol_alloc(Ctx& c) {
  const int64_t nb = ceil_div(std::max<int64_t>(c.n, 1), kB);
  c.Winv = dev_zeros<double>((size_t)nb * kB * kB, c.stream);
  c.Lt = dev_zeros<double>((size_t)nb * nb * kB * kB, c.stream);
  c.df_flags = dev_zeros<unsigned>((size_t)nb * nb, c.stream);
  c.df_ctl = dev_zeros<unsigned>(8, c.stream);
  c.df_y = dev_zeros<double>((size_t)nb * kB, c.stream);
  c.df_x = dev_zeros<double>((size_t)nb * kB, c.stream);
  c.df_xflags = dev_zeros<unsigned>((size_t)nb, c.stream);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  c.df_grid = 2 * sms;  // two 74 KB CTAs per SM
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
  const int nt = (int)ceil_div(n, kB);
  DfArgs a;
  a.M = M;
  a.L = L;
  a.Lt = c.Lt;
  a.W = c.Winv;
  a.n = n;
  a.delta = delta;
  a.nt = nt;
  a.ntasks = nt + (nt >= 2 ? (nt - 1) * (nt - 2) / 2 : 0);
  a.flags = c.df_flags;
  a.ctl = c.df_ctl;
  a.info = info;
  a.rhs = rhs;
  a.x = x;
  a.ybuf = c.df_y;
  a.xbuf = c.df_x;
  a.xflags = c.df_xflags;
  a.nback = rhs ? nt : 0;
  const int grid = std::min(a.ntasks + a.nback, c.df_grid);
  k_chol_df<<<grid, kT, kDfSmem, c.stream>>>(a);
  CMPC_LAUNCHED();
}

void launch_factor_inverses(Ctx& c, const double* L) {
  if (c.n == 0) return;
  k_diag_inv<<<(unsigned)ceil_div(c.n, kB), 32, 0, c.stream>>>(L, c.n, c.Winv);
  CMPC_LAUNCHED();
}

void launch_chol_solve(Ctx& c, const double* L, const double* b, double* x) {
  if (c.n == 0) return;
  set_attrs(c.device);
  const size_t sm = sizeof(double) * ((size_t)c.n + kB);
  if (sm > 200 * 1024) throw CudaError("chol_solve: n too large for the single-CTA TRSV");
  k_trsv<<<1, 512, sm, c.stream>>>(L, c.Winv, b, x, c.n);
  CMPC_LAUNCHED();
}

}  // namespace cmpc
