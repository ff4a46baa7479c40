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
// tiles only) and fuses both triangular solves. The column-to-column chain runs inside ONE
// CTA, the spine, so it never waits for another CTA's flag (an inter-CTA hop through L2 costs
// ~1.3 us with its data: tools/exp/hop_bench.cu, as much as a third of a column); the rest of
// the work is spread over the other CTAs and reaches the spine ahead of time:
//   pre-diagonal task d   A_{d,d-1} = M_{d,d-1} - sum_{k<=d-3} L_dk L_{d-1,k}^T,
//                         A_dd = M_dd + delta I - sum_{k<=d-3} L_dk L_dk^T,
//                         t_d = b_d - sum_{k<=d-3} L_dk y_k          (DMMA, published)
//                         (only columns <= d-3: it never waits for the spine's last two steps,
//                         which would put two inter-CTA hops into every other step)
//   panel task (i, j), i >= j + 2:   L_ij = (M_ij - sum_{k<j} L_ik L_jk^T) W_j^T
//   spine step d (compute warps 0-3): the column d-2 terms (L_{d,d-2} from a panel task,
//                         L_{d-1,d-2} kept from step d-1), the sub-diagonal panel L_{d,d-1} =
//                         A_{d,d-1} W_{d-1}^T (W_{d-1} kept from step d-1), A_dd -= L L^T, then
//                         the 32 x 32 factor: warp 0 runs the pivot chain (row i of the tile in
//                         lane i's registers; the next pivot travels by one shuffle, each
//                         finished column through shared memory) while warp 1 forms
//                         W_d = L_dd^{-1} column by column right behind it; y_d = W_d t_d.
//   spine publisher warps 4-5: store + publish each step's panel and diagonal tile;
//   spine prefetcher warps 6-7: stage the next steps' inputs as soon as they are published,
//                         so neither the flag waits nor the global stores sit on the chain.
//   backward solve (spine, after the factor): x_i = W_i^T (y_i - L_{>i,i}^T x_{>i}).
// Every finished tile publishes a per-tile flag (release/acquire at GPU scope) stamped with
// the launch's generation number, so flags never need resetting. CTAs grab tasks from an
// atomic counter in an order where a task only waits for tasks earlier in that order or for
// the spine's earlier steps, and the spine only for tasks that need nothing from its later
// steps: the kernel cannot deadlock whatever the residency. The last CTA out publishes info
// and advances the generation. The W blocks are kept, so a later stand-alone solve
// (k_trsv) is block GEMVs.
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
  if ((threadIdx.x & 127) == 0) s_ctrace[slot] = clock64();
}
__device__ __forceinline__ void ctrace_flush(int task) {
  if ((threadIdx.x & 127) == 0 && task < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long c = clock64();
    for (int k = 0; k < 8; ++k) g_ctrace[task * 10 + k] = s_ctrace[k] ? c - s_ctrace[k] : 0ull;
    g_ctrace[task * 10 + 8] = t;
    for (int k = 0; k < 8; ++k) s_ctrace[k] = 0;
  }
}
#define CTRACE(slot) ctrace(slot)
#define CTRACE_FLUSH(task) ctrace_flush(task)
// spine: clock64 per step k and event e into shared memory, flushed after the factor
__shared__ long long s_sptrace[64][8];
#define STRACE(k, e)                                              \
  do {                                                            \
    if ((threadIdx.x & 127) == 0 && (k) < 64) s_sptrace[(k)][(e)] = clock64(); \
  } while (0)
#define STRACE_FLUSH()                                                           \
  do {                                                                           \
    __syncthreads();                                                             \
    for (int e_ = threadIdx.x; e_ < 64 * 8; e_ += blockDim.x)                    \
      g_ctrace[3000 * 10 + e_] = (unsigned long long)s_sptrace[e_ / 8][e_ % 8];  \
  } while (0)
#else
#define STRACE(k, e) \
  do {               \
  } while (0)
#define STRACE_FLUSH() \
  do {                 \
  } while (0)
#define CTRACE(slot) \
  do {               \
  } while (0)
#define CTRACE_FLUSH(task) \
  do {                     \
  } while (0)
#endif

constexpr int kB = 32;           // tile edge
constexpr int kLD = 36;          // staged-tile leading dimension (conflict-free DMMA fragments)
constexpr int kTS = kB * kLD;    // doubles per staged tile
constexpr int kT = 256;          // threads per CTA: warps 0-3 compute, 4-7 I/O (spine) / staging
constexpr int kCT = 128;         // compute threads
constexpr int kMaxFusedN = 768;  // the spine runs the backward solve up to this n (bundled bulk
                                 // copies: n = 500 156 us vs 170 with per-block tasks; n = 1000
                                 // 330 vs 321: beyond, the per-block tasks win)
constexpr int kPartLen = 2 * 1024 + kB;  // pre-diagonal results: A_{d,d-1}, A_dd (fragment order), t_d
constexpr unsigned kFull = 0xffffffffu;

// named barriers (0 is __syncthreads). Spine warp groups: compute 0-3 (128 threads),
// publishers 4-5 (64), prefetchers 6-7 (64)
constexpr int kBarInput = 1;     // + parity: prefetchers -> compute, step inputs staged
constexpr int kBarPready = 3;    // + parity: compute -> publishers, the sub-diagonal panel is in smem
constexpr int kBarCompute = 5;   // compute warps only
constexpr int kBarPub = 6;       // publisher warps only
constexpr int kBarSdone = 7;     // + parity: compute -> publishers, L_dd, W_d, y_d are in smem
constexpr int kBarConsumed = 9;  // + parity: compute -> prefetchers, an input set may be overwritten
constexpr int kBarPre = 11;      // prefetcher warps only
constexpr int kPairCount = 192;  // compute (128) + one 64-thread I/O group
constexpr int kIOT = 64;         // threads per I/O group

// shared memory (doubles): the spine's layout ...
constexpr int kSXin = 0;                 // -A_{d,d-1} (panel input)
constexpr int kSP = kTS;                 // 2 (parity): L_{d,d-1}
constexpr int kSW = 3 * kTS;             // 2: W_d
constexpr int kSF = 5 * kTS;             // 2: factor input / L_dd
constexpr int kST2 = 7 * kTS;            // 2: prefetched L_{d,d-2}
constexpr int kSPP = 9 * kTS;            // 2 x 1024: prefetched A_{d,d-1} partial (fragment order)
constexpr int kSPD = kSPP + 2048;        // 2 x 1024: prefetched A_dd partial
constexpr int kSTP = kSPD + 2048;        // 2 x 32: prefetched t_d partial
constexpr int kSCol = kSTP + 64;         // 32 x 32 finished factor columns (pivot chain)
constexpr int kSRR = kSCol + kB * kB;    // 1 / l_pp
constexpr int kSYR = kSRR + kB;          // 4 x 32: y ring
constexpr int kSTV = kSYR + 4 * kB;      // t_d
constexpr int kSRed = kSTV + kB;         // 8 x 32 partial sums
constexpr int kSEnd = kSRed + 8 * kB;
// ... and a task's (the same memory)
constexpr int kTStage = 0;               // 2 stages x {X, Y}
constexpr int kTA = 4 * kTS;             // -acc of a panel
constexpr int kTW = 5 * kTS;             // staged W_j
constexpr int kTP = 6 * kTS;             // the panel product
constexpr int kTYs = 7 * kTS;            // 2 staged y_k
constexpr int kTRed = kTYs + 2 * kB;     // 8 x 32 partial sums
constexpr int kTEnd = kTRed + 8 * kB;
constexpr int kDfSmemFactor = (kSEnd > kTEnd ? kSEnd : kTEnd) * 8;
static_assert((kSCol * 8) % 16 == 0 && (kSPP * 8) % 16 == 0 && (kSTP * 8) % 16 == 0, "16-byte alignment");

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// polling load: relaxed (an acquire load compiles to LDG.STRONG + CCTL.IVALL, an L1
// invalidation per poll); the acquire fence follows once the flag is seen
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
#ifdef CMPC_DIAG_NOREL  // diagnostic only (tools/exp): no ordering, to measure the fence's cost
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
// named barriers between warp groups. bar.sync / bar.arrive are .aligned (the whole warp must
// execute them together); a warp can reach one diverged (lane 0 just spun on a flag), so the
// warp reconverges first and the non-aligned forms count threads, not warps
__device__ __forceinline__ void nbar_sync(int id, int n) {
  __syncwarp();
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  __syncwarp();
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

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
// x[k * kLD + i] with 16-byte cp.async (L2 only: tiles written by other CTAs); thread t of nth
__device__ __forceinline__ void stage_tile(double* x, const double* src, int t, int nth) {
  for (int ch = t; ch < 512; ch += nth) {
    const int k = ch >> 4, i2 = (ch & 15) * 2;
    cp_async16(x + k * kLD + i2, src + k * kB + i2);
  }
}
// a contiguous run of `count` doubles (even)
__device__ __forceinline__ void stage_lin(double* x, const double* src, int count, int t, int nth) {
  for (int ch = t; ch < count / 2; ch += nth) cp_async16(x + 2 * ch, src + 2 * ch);
}

// Compute warp w (0..3) owns the 16 x 16 block (rows 16 (w & 1) + [0,16), columns
// 16 (w >> 1) + [0,16)) of a 32 x 32 tile as two m16n8 fragments: acc[ni][e] is element
// (16 (w & 1) + g + 8 (e >> 1), 16 (w >> 1) + 8 ni + 2 t + (e & 1)).
struct Frag {
  int m0, n0, g, t;
  __device__ Frag() : Frag((threadIdx.x >> 5) & 3) {}
  __device__ explicit Frag(int warp) {
    const int lane = threadIdx.x & 31;
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
  unsigned* flags;   // nt x nt per-tile done flags (== generation when done)
  unsigned* ctl;     // [0] generation, [1] exit count, [2] failure generation, [3] pivot + 1, [4] task counter
  long long* info;
  const double* rhs; // n (nullptr: factor only)
  double* x;         // n (may alias rhs: rhs is read before any block of x is written)
  double* ybuf;      // nt * 32
  double* part;      // nt * kPartLen: pre-diagonal results
  unsigned* pflags;  // nt
  bool back;         // the spine also runs the backward solve (rhs and n <= kMaxFusedN)
  int nback;         // else with rhs: nt backward tasks, one per block
  double* xbuf;      // nt * 32 (backward tasks)
  unsigned* xflags;  // nt
};

// one thread: spin until both flags carry the generation; false on a published failure
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
// packed tiles column-major over the tile grid: tile (i, j) at (j nt + i), so the tiles below a
// diagonal block (one block column) are contiguous for the backward solve's bulk copies
__device__ __forceinline__ double* tile_ptr(const DfArgs& A, int i, int j) {
  return A.Lt + ((size_t)j * A.nt + i) * (kB * kB);
}
__device__ __forceinline__ const double* tile_src(const DfArgs& A, int i, int j) { return tile_ptr(A, i, j); }
// all threads of the CTA: the global writes before it become visible with the flag. The
// barrier orders every thread's writes before thread 0's release store, which is cumulative;
// no sequentially-consistent fence (MEMBAR.SC.GPU drains the SM's memory pipe and stalls the
// neighbouring warps' shared-memory work)
__device__ __forceinline__ void publish(unsigned* flag, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(flag, target);
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

// fixed-order sum of the 8 partial rows red[0..7][r]
__device__ __forceinline__ double sum8(const double* red, int r) {
  return ((red[r] + red[kB + r]) + (red[2 * kB + r] + red[3 * kB + r])) +
         ((red[4 * kB + r] + red[5 * kB + r]) + (red[6 * kB + r] + red[7 * kB + r]));
}

// task CTAs (256 threads, the DMMA on warps 0-3): left-looking updates acc1 += L_{i,k}
// L_{j1,k}^T and (TWO) acc2 += L_{i,k} L_{i,k}^T for k < K, double-buffered (tile k+1 prefetched
// when already published); with fwd also the forward partial sum_k L_{i,k} y_k (thread: row
// tid & 31, columns 4 (tid >> 5) + [0, 4)). Returns false on a published failure.
template <bool TWO>
__device__ bool left_updates(const DfArgs& A, const Frag& f, int i, int j1, int K, bool skip2, unsigned target,
                             double* sm, volatile unsigned* s_flag, double (&acc1)[2][4], double (&acc2)[2][4],
                             bool fwd, double& fpart) {
  if (K <= 0) return true;
  const int tid = threadIdx.x;
  const bool mma = tid < kCT;
  const unsigned* failw = A.ctl + 2;
  auto need_j1 = [&](int) { return true; };
  auto flag_j1 = [&](int k) { return tile_flag(A, j1, k); };
  if (tid == 0) *s_flag = wait_flags(tile_flag(A, i, 0), flag_j1(0), failw, target) ? 1u : 2u;
  __syncthreads();
  if (*s_flag == 2u) return false;
  double* ys = sm + kTYs;
  stage_tile(sm + kTStage, tile_src(A, i, 0), tid, kT);
  if (need_j1(0)) stage_tile(sm + kTStage + kTS, tile_src(A, j1, 0), tid, kT);
  if (fwd) stage_lin(ys, A.ybuf, kB, tid, kT);
  cp_commit();
  const int fr = tid & 31, q8 = tid >> 5;
  for (int k = 0; k < K; ++k) {
    const int s = k & 1;
    double* xs = sm + kTStage + 2 * s * kTS;
    double* xo = sm + kTStage + 2 * (s ^ 1) * kTS;
    const bool more = k + 1 < K;
    if (tid == 0) {
      const bool ready =
          more && ld_relaxed(tile_flag(A, i, k + 1)) == target && ld_relaxed(flag_j1(k + 1)) == target;
      if (ready) fence_acquire();
      *s_flag = ready ? 1u : 0u;
    }
    __syncthreads();  // buffer s^1 is free (gemm k-1 done); s_flag visible
    const bool pre = *s_flag == 1u;
    if (pre) {
      stage_tile(xo, tile_src(A, i, k + 1), tid, kT);
      if (need_j1(k + 1)) stage_tile(xo + kTS, tile_src(A, j1, k + 1), tid, kT);
      if (fwd) stage_lin(ys + kB * (s ^ 1), A.ybuf + kB * (k + 1), kB, tid, kT);
    }
    cp_commit();
    cp_wait1();
    __syncthreads();  // tile k visible to every warp
    if (mma) {
      if (TWO && !skip2) gemm_xyt(f, xs, xs, acc2);  // the diagonal block's own update
      if (need_j1(k)) gemm_xyt(f, xs, xs + kTS, acc1);
    }
    if (fwd) {
      const double* yk = ys + kB * s;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) fpart = fma(xs[(4 * q8 + kk) * kLD + fr], yk[4 * q8 + kk], fpart);
    }
    if (more && !pre) {
      if (tid == 0) *s_flag = wait_flags(tile_flag(A, i, k + 1), flag_j1(k + 1), failw, target) ? 1u : 2u;
      __syncthreads();
      if (*s_flag == 2u) return false;
      stage_tile(xo, tile_src(A, i, k + 1), tid, kT);
      if (need_j1(k + 1)) stage_tile(xo + kTS, tile_src(A, j1, k + 1), tid, kT);
      if (fwd) stage_lin(ys + kB * (s ^ 1), A.ybuf + kB * (k + 1), kB, tid, kT);
      cp_commit();
    }
  }
  __syncthreads();  // staging buffers free
  return true;
}

// panel task (i, j), i >= j + 2: L_ij = (M_ij - sum_{k<j} L_ik L_jk^T) W_j^T
__device__ bool df_panel(const DfArgs& A, int i, int j, unsigned target, double* sm, volatile unsigned* s_flag) {
  const int tid = threadIdx.x;
  const bool mma = tid < kCT;
  const Frag f;
  double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}}, unused[2][4];
  CTRACE(0);
  if (mma) load_neg_m(f, A, (int64_t)kB * i, (int64_t)kB * j, false, acc);
  double fpart = 0.0;
  if (!left_updates<false>(A, f, i, j, j, true, target, sm, s_flag, acc, unused, false, fpart)) return false;
  CTRACE(1);
  if (tid == 0) *s_flag = wait_flags(tile_flag(A, j, j), tile_flag(A, j, j), A.ctl + 2, target) ? 1u : 2u;
  if (mma) frag_store(f, sm + kTA, acc, -1.0);
  __syncthreads();
  if (*s_flag == 2u) return false;
  stage_tile(sm + kTW, A.W + (size_t)j * (kB * kB), tid, kT);
  cp_commit();
  cp_wait0();
  __syncthreads();
  if (mma) {
    double out[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    gemm_xyt(f, sm + kTA, sm + kTW, out);
    frag_store(f, sm + kTP, out, 1.0);
  }
  __syncthreads();
  double* Lt = tile_ptr(A, i, j);
  const int64_t r0 = (int64_t)kB * i, c0 = (int64_t)kB * j;
  for (int e = tid; e < kB * kB; e += kT) {
    const int r = e & 31, c = e >> 5;
    const double v = sm[kTP + c * kLD + r];
    Lt[e] = v;
    if (r0 + r < A.n) A.L[(r0 + r) + (c0 + c) * A.n] = v;
  }
  publish(tile_flag(A, i, j), target);
  CTRACE(2);
  CTRACE_FLUSH(64 + i * 64 + j);
  return true;
}

// pre-diagonal task d: everything of diagonal step d that needs only columns k <= d-3 (so it
// never waits for the spine's last two steps): A_{d,d-1}, A_dd and t through k = d-3
__device__ bool df_prediag(const DfArgs& A, int d, unsigned target, double* sm, volatile unsigned* s_flag) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool mma = tid < kCT;
  const Frag f;
  const int64_t r0 = (int64_t)kB * d;
  const bool fwd = A.rhs != nullptr;
  double accP[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  double accD[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  CTRACE(0);
  if (mma) {
    if (d >= 1) load_neg_m(f, A, r0, r0 - kB, false, accP);
    load_neg_m(f, A, r0, r0, true, accD);
  }
  double fpart = 0.0;
  if (!left_updates<true>(A, f, d, d - 1, d - 2, warp == 2, target, sm, s_flag, accP, accD, fwd, fpart))
    return false;
  CTRACE(1);
  double* out = A.part + (size_t)d * kPartLen;
  if (mma) {
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        out[(ni * 4 + e) * kCT + tid] = accP[ni][e];
        out[1024 + (ni * 4 + e) * kCT + tid] = accD[ni][e];
      }
  }
  double* red = sm + kTRed;
  red[(tid >> 5) * kB + (tid & 31)] = fpart;
  __syncthreads();
  if (tid < kB) {
    const double bi = (fwd && r0 + tid < A.n) ? A.rhs[r0 + tid] : 0.0;
    out[2048 + tid] = bi - sum8(red, tid);
  }
  publish(A.pflags + d, target);
  CTRACE(2);
  CTRACE_FLUSH(2048 + d);
  return true;
}

// warp 0: the 32 x 32 factor of in_sm (column-major lower, kLD) into a_sm, row i in lane i's
// registers. Pivot p: l_ip = a_ip / sqrt(a_pp); the next pivot a_{p+1,p+1} - l^2 is formed in
// lane p+1 and shuffled to all lanes (the critical chain); column p goes to shared memory
// (col) for the rank-1 update of every row and for warp 1's inverse, which it signals on the
// mbarrier sig[p] (arrive = release, warp 1's wait = acquire: a __threadfence_block per pivot
// instead costs ~60 cycles of the chain each). Returns the first failing pivot (< b) or -1;
// *odd when a pivot left the fast rsqrt's range.
template <bool EXACT>
__device__ int factor_rows(const double* in_sm, double* a_sm, double* col, double* rr, uint64_t* sig, int b,
                           bool* odd) {
  const int lane = threadIdx.x & 31;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = (c <= lane) ? in_sm[c * kLD + lane] : 0.0;
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
#pragma unroll
    for (int c = (p + 1) & ~1; c < 32; c += 2) {
      const double2 lc = ld2(col + p * kB + c);
      if (c > p) a[c] = fma(-l, lc.x, a[c]);
      if (c + 1 > p) a[c + 1] = fma(-l, lc.y, a[c + 1]);
    }
    // signalled after the update has read the column: the arrive's release fence then finds
    // no shared-memory store in flight and costs the chain almost nothing
    if (lane == 0) mbar_arrive(sig + p);
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) a_sm[c * kLD + lane] = (c <= lane) ? a[c] : 0.0;
  *odd = bad;
  return fail;
}

// warp 1: W = L^{-1} column by column (lane c = column c), one pivot behind warp 0:
// w_p = s_p / l_pp, s_i -= l_ip w_p (i > p). Column-major into w_sm. `parity` is the phase
// of the sig barriers this factor pass completes.
__device__ void inverse_cols(double* w_sm, const double* col, const double* rr, uint64_t* sig, uint32_t parity) {
  const int lane = threadIdx.x & 31;
  double s[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    mbar_wait(sig + p, parity);
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

struct SpineShared {
  int passes, res[2], fail, io_flag;
};

// spine compute warps (0-3): the diagonal steps. Step k takes the pre-diagonal task's
// A_{k,k-1}, A_kk and t (through column k-3), adds the column k-2 terms with the prefetched
// L_{k,k-2} (L_{k-1,k-2} is its own previous panel), forms the sub-diagonal panel, its rank
// update and the factor.
__device__ void spine_compute(const DfArgs& A, double* sm, volatile SpineShared* ss, uint64_t* sig) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Frag f;
  const bool fwd = A.rhs != nullptr;
  const bool upper = warp == 2;  // rows 0..15 x columns 16..31: strictly upper in a diagonal tile
  const int fr = lane, q4 = warp;  // forward partials: row, 8-column quarter
  double* xin = sm + kSXin;
  double* col = sm + kSCol;
  double* rr = sm + kSRR;
  double* red = sm + kSRed;
  double* tv = sm + kSTV;
  for (int k = 0; k < A.nt; ++k) {
    const int p = k & 1;
    STRACE(k, 0);
    nbar_sync(kBarInput + p, kPairCount);  // step k's inputs staged by the prefetcher warps
    STRACE(k, 1);
    double accP[2][4], accD[2][4];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        accP[ni][e] = sm[kSPP + p * 1024 + (ni * 4 + e) * kCT + tid];
        accD[ni][e] = sm[kSPD + p * 1024 + (ni * 4 + e) * kCT + tid];
      }
    double fpart = 0.0;
    double* pk = sm + kSP + p * kTS;
    if (k >= 1) {  // the sub-diagonal panel L_{k,k-1} = A_{k,k-1} W_{k-1}^T
      if (k >= 2) gemm_xyt(f, sm + kST2 + p * kTS, sm + kSP + (p ^ 1) * kTS, accP);
      STRACE(k, 6);
      frag_store(f, xin, accP, -1.0);
      nbar_sync(kBarCompute, kCT);
      double out[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
      gemm_xyt(f, xin, sm + kSW + (p ^ 1) * kTS, out);
      frag_store(f, pk, out, 1.0);
      nbar_sync(kBarCompute, kCT);
      nbar_arrive(kBarPready + p, kPairCount);  // the publisher warps store and publish it
      STRACE(k, 2);
      if (k >= 2) {  // the column k-2 terms of A_kk and t
        const double* t2 = sm + kST2 + p * kTS;
        if (!upper) gemm_xyt(f, t2, t2, accD);
        if (fwd) {
          const double* y = sm + kSYR + ((k - 2) & 3) * kB;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) fpart = fma(t2[(8 * q4 + cc) * kLD + fr], y[8 * q4 + cc], fpart);
        }
      }
      if (!upper) gemm_xyt(f, pk, pk, accD);
      if (fwd) {
        const double* y = sm + kSYR + ((k - 1) & 3) * kB;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) fpart = fma(pk[(8 * q4 + cc) * kLD + fr], y[8 * q4 + cc], fpart);
      }
    }
    // the factor's input (xin, kept for an exact redo): -accD, lower, identity padding beyond b
    const int64_t r0 = (int64_t)kB * k;
    const int b = (int)(A.n - r0 < kB ? A.n - r0 : kB);
    double* fk = sm + kSF + p * kTS;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = f.row(e), c = f.col(ni, e);
        double v;
        if (r >= b || c >= b) v = (r == c) ? 1.0 : 0.0;
        else v = (r >= c) ? -accD[ni][e] : 0.0;
        xin[c * kLD + r] = v;
      }
    red[q4 * kB + fr] = fpart;
    nbar_sync(kBarCompute, kCT);
    if (tid < kB)
      tv[tid] = sm[kSTP + p * kB + tid] - ((red[tid] + red[kB + tid]) + (red[2 * kB + tid] + red[3 * kB + tid]));
    nbar_arrive(kBarConsumed + p, kPairCount);  // input set p is read: the prefetchers may refill it
    double* wk = sm + kSW + p * kTS;
    bool odd = false;
    uint32_t parity = (uint32_t)(ss->passes & 1);
    STRACE(k, 3);
    if (warp == 0) {
      const int fl = factor_rows<false>(xin, fk, col, rr, sig, b, &odd);
      if (lane == 0) {
        ss->res[0] = fl;
        ss->res[1] = odd ? 1 : 0;
      }
    } else if (warp == 1) {
      inverse_cols(wk, col, rr, sig, parity);
    }
    nbar_sync(kBarCompute, kCT);
    if (tid == 0) ss->passes = ss->passes + 1;
    STRACE(k, 4);
    if (ss->res[1]) {  // a pivot outside [1e-300, 1e300]: redo the tile with the exact square root
      parity = (uint32_t)(ss->passes & 1);
      if (warp == 0) {
        const int fl = factor_rows<true>(xin, fk, col, rr, sig, b, &odd);
        if (lane == 0) ss->res[0] = fl;
      } else if (warp == 1) {
        inverse_cols(wk, col, rr, sig, parity);
      }
      nbar_sync(kBarCompute, kCT);
      if (tid == 0) ss->passes = ss->passes + 1;
    }
    const int fl = ss->res[0];
    if (fl >= 0) {
      if (tid == 0) ss->fail = (int)(r0 + fl);
      nbar_sync(kBarCompute, kCT);
      nbar_arrive(kBarSdone + p, kPairCount);
      return;
    }
    if (fwd) {  // y_k = W_k t (W lower): quarter sums in a fixed order
      double s = 0.0;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const int c = 8 * q4 + cc;
        if (c <= fr) s = fma(wk[c * kLD + fr], tv[c], s);
      }
      red[q4 * kB + fr] = s;
      nbar_sync(kBarCompute, kCT);
      if (tid < kB)
        sm[kSYR + (k & 3) * kB + tid] = (red[tid] + red[kB + tid]) + (red[2 * kB + tid] + red[3 * kB + tid]);
      nbar_sync(kBarCompute, kCT);
    }
    STRACE(k, 5);
    nbar_arrive(kBarSdone + p, kPairCount);  // L_kk, W_k, y_k ready for the publisher warps
  }
}

// spine prefetcher warps (6-7): stage each step's inputs (pre-diagonal partials and the panel
// L_{k,k-2}) into the input set of its parity as soon as they are published, two steps ahead
// at most (an input set is refilled only after the compute warps have read it)
__device__ void spine_prefetch(const DfArgs& A, unsigned target, double* sm, volatile SpineShared* ss) {
  const int t = threadIdx.x - (kCT + kIOT);  // 0..63
  const unsigned* failw = A.ctl + 2;
  for (int s = 0; s < A.nt; ++s) {
    const int p = s & 1;
    if (s >= 2) {
      nbar_sync(kBarConsumed + p, kPairCount);  // step s-2 has read input set p
      if (ss->fail >= 0) return;
    }
    if (t == 0)
      ss->io_flag = wait_flags(A.pflags + s, s >= 2 ? tile_flag(A, s, s - 2) : A.pflags + s, failw, target) ? 1 : 2;
    nbar_sync(kBarPre, kIOT);
    if (ss->io_flag == 2) return;  // the factorization failed (published by the publishers)
    const double* src = A.part + (size_t)s * kPartLen;
    stage_lin(sm + kSPP + p * 1024, src, 1024, t, kIOT);
    stage_lin(sm + kSPD + p * 1024, src + 1024, 1024, t, kIOT);
    stage_lin(sm + kSTP + p * kB, src + 2048, kB, t, kIOT);
    if (s >= 2) stage_tile(sm + kST2 + p * kTS, tile_src(A, s, s - 2), t, kIOT);
    cp_commit();
    cp_wait0();
    STRACE(s + 32, 0);
    nbar_arrive(kBarInput + p, kPairCount);
  }
}

// spine publisher warps (4-5): store and publish each step's sub-diagonal panel and diagonal
// tile (L_kk, W_k, y_k) as soon as the compute warps have them, so nothing waits on the
// prefetches
__device__ bool spine_publish(const DfArgs& A, unsigned target, double* sm, volatile SpineShared* ss) {
  const int t = threadIdx.x - kCT;  // 0..63
  auto publish_pub = [&](unsigned* flag) {  // as publish(), over the publisher warps' barrier
    nbar_sync(kBarPub, kIOT);
    if (t == 0) st_release(flag, target);
  };
  for (int k = 0; k < A.nt; ++k) {
    const int p = k & 1;
    const int64_t r0 = (int64_t)kB * k;
    if (k >= 1) {  // L_{k,k-1}
      nbar_sync(kBarPready + p, kPairCount);
      STRACE(k + 32, 1);
      const double* pk = sm + kSP + p * kTS;
      double* Lt = tile_ptr(A, k, k - 1);
      for (int e = t; e < kB * kB; e += kIOT) {
        const int r = e & 31, c = e >> 5;
        const double v = pk[c * kLD + r];
        Lt[e] = v;
        if (r0 + r < A.n) A.L[(r0 + r) + (r0 - kB + c) * A.n] = v;
      }
      publish_pub(tile_flag(A, k, k - 1));
    }
    nbar_sync(kBarSdone + p, kPairCount);
    STRACE(k + 32, 2);
    if (ss->fail >= 0) {
      if (t == 0) {
        A.ctl[3] = (unsigned)(ss->fail + 1);
        st_release(A.ctl + 2, target);
      }
      return false;
    }
    const int b = (int)(A.n - r0 < kB ? A.n - r0 : kB);
    const double* fk = sm + kSF + p * kTS;
    const double* wk = sm + kSW + p * kTS;
    double* Wd = A.W + (size_t)k * (kB * kB);
    for (int e = t; e < kB * kB; e += kIOT) {
      const int r = e & 31, c = e >> 5;
      if (r < b && c < b) A.L[(r0 + r) + (r0 + c) * A.n] = fk[c * kLD + r];
      Wd[e] = wk[c * kLD + r];
    }
    if (A.rhs && t < kB) A.ybuf[r0 + t] = sm[kSYR + (k & 3) * kB + t];
    publish_pub(tile_flag(A, k, k));
    STRACE(k, 7);
  }
  return true;
}

// backward solve on the spine: x_i = W_i^T (y_i - sum_{j>i} L_ji^T x_j), block i from the last
// down, from the packed tiles of L. Per block the stream holds W_i (with y_i) and then the tiles
// (j, i), j = nt-1 .. i+1, in BUNDLES of up to kBG tiles (one block column is contiguous, so a
// bundle is one 1-D bulk copy): the items (independent of x) flow through a ring of kBSlots
// slots (one elected thread, full/empty mbarriers), so neither the L2 latency nor CTA-wide
// barriers are paid per tile, and the per-item cost (~0.2 us: wait, release, refill) is paid
// per bundle (tools/exp/l2_stream.cu: one SM streams 1 MB in 10 us from 16 KB copies, 41 us
// from 4 KB ones). The loop issues no global load of its own: the empty barrier's arrive is a
// release, and its fence would wait for any global load in flight. Per tile, warp w sums
// columns 4w..4w+3 over the 32 rows (lane = row), tiles in decreasing j; per block, fixed-order
// warp sums, then x_i = W_i^T t.
#ifndef CMPC_DIAG_BACK
#define CMPC_DIAG_BACK 0
#endif
constexpr int kBG = 4;        // tiles per bundle (32 KB)
constexpr int kBSlots = 6;
constexpr int kBLag = 2;      // a slot is refilled kBLag items after it was read (no wait)
constexpr int kBSlot = kBG * kB * kB;     // doubles per slot
constexpr int kBYs = kBSlots * kBSlot;    // y_i beside its W item: one 32-vector per slot
constexpr int kBRed = kBYs + kBSlots * kB;
constexpr int kBTv = kBRed + 8 * kB;
constexpr int kBXs = kBTv + kB;
constexpr int kBEnd = kBXs + kMaxFusedN;
constexpr int kDfSmem = kDfSmemFactor > kBEnd * 8 ? kDfSmemFactor : kBEnd * 8;
static_assert(kDfSmem <= 227 * 1024, "shared memory per CTA");
__device__ void spine_back(const DfArgs& A, double* sm, uint64_t* full, uint64_t* empty) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* xs = sm + kBXs;
  double* red = sm + kBRed;
  double* tv = sm + kBTv;
  const int64_t n = A.n;
  const int nt = A.nt;
  int total = 0;  // one W item per block + its bundles
  for (int i = 0; i < nt; ++i) total += 1 + (nt - 1 - i + kBG - 1) / kBG;
  int pi = nt - 1, pj = nt;  // producer cursor: block pi, next tile row pj (pj == nt: the W item)
  auto issue = [&](int sl) {
    if (pj == nt) {
      mbar_expect_tx(full + sl, kB * kB * 8 + kB * 8);
      bulk_load(sm + sl * kBSlot, A.W + (size_t)pi * (kB * kB), kB * kB * 8, full + sl);
      bulk_load(sm + kBYs + sl * kB, A.ybuf + (size_t)kB * pi, kB * 8, full + sl);
      pj = nt - 1;
    } else {  // tiles (lo .. pj, pi): contiguous
      const int lo = max(pi + 1, pj - kBG + 1), cnt = pj - lo + 1;
      mbar_expect_tx(full + sl, (uint32_t)(cnt * kB * kB * 8));
      bulk_load(sm + sl * kBSlot, tile_src(A, lo, pi), (uint32_t)(cnt * kB * kB * 8), full + sl);
      pj = lo - 1;
    }
    if (pj == pi) {  // block pi done: the next block's W item
      --pi;
      pj = nt;
    }
  };
  if (tid == 0) {
    for (int sl = 0; sl < kBSlots; ++sl) {
      mbar_init(full + sl, 1);
      mbar_init(empty + sl, kT / 32);
    }
    fence_barrier_init();
    // the tiles, W and y were written through the generic proxy (other CTAs, the publishers)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int q = 0; q < total && q < kBSlots; ++q) issue(q);
  }
  __syncthreads();
  int q = 0;  // consumer's item sequence number
  auto consumed = [&] {  // this item's slot is read; refill the slot read kBLag items ago
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + q % kBSlots);
    const int qo = q - kBLag;
    if (tid == 0 && qo >= 0 && qo + kBSlots < total) {
      const int so = qo % kBSlots;
      mbar_wait(empty + so, (uint32_t)((qo / kBSlots) & 1));
#if CMPC_DIAG_BACK != 3
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
      issue(so);
    }
    ++q;
  };
  for (int i = nt - 1; i >= 0; --i) {
    const int64_t c0 = (int64_t)kB * i;
    double wv[4], yv;
    {  // the W item: W_i (column-major) and y_i
      const int sl = q % kBSlots;
      mbar_wait(full + sl, (uint32_t)((q / kBSlots) & 1));
      const double* X = sm + sl * kBSlot;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) wv[cc] = X[(4 * warp + cc) * kB + lane];
      yv = sm[kBYs + sl * kB + lane];
      consumed();
    }
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int hi = nt - 1; hi > i; hi -= kBG) {
      const int lo = max(i + 1, hi - kBG + 1);
      const int sl = q % kBSlots;
      mbar_wait(full + sl, (uint32_t)((q / kBSlots) & 1));
      for (int j = hi; j >= lo; --j) {
        const double* X = sm + sl * kBSlot + (j - lo) * (kB * kB);  // column-major 32 x 32
        const double xr = xs[(int64_t)kB * j + lane];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) s4[cc] = fma(X[(4 * warp + cc) * kB + lane], xr, s4[cc]);
      }
      consumed();
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const double t = warp_sum(s4[cc]);
      if (lane == 0) red[4 * warp + cc] = t;
    }
    __syncthreads();
    if (tid < kB) tv[tid] = yv - red[tid];
    __syncthreads();
    const double tl = tv[lane];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int c = 4 * warp + cc;  // x(c) = sum_{r >= c} W(r, c) t(r)
      const double t = warp_sum(wv[cc] * tl);
      if (lane == 0) {
        xs[c0 + c] = t;
        if (c0 + c < n) A.x[c0 + c] = t;
      }
    }
    __syncthreads();
  }
}

// distributed backward task i (n > kMaxFusedN): x_i = W_i^T (y_i - sum_{j>i} L_ji^T x_j), j from
// the last block down as the x_j are published; the tiles are final once the last diagonal
// block is (it needed them all), so they are staged one ahead without waiting. Warp w sums
// columns 4w..4w+3 (lane = row); fixed-order warp sums.
__device__ bool df_back(const DfArgs& A, int i, unsigned target, double* sm, volatile unsigned* s_flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = A.nt;
  const unsigned* failw = A.ctl + 2;
  if (tid == 0) *s_flag = wait_flags(tile_flag(A, nt - 1, nt - 1), tile_flag(A, i, i), failw, target) ? 1u : 2u;
  __syncthreads();
  if (*s_flag == 2u) return false;
  const double* Wi = A.W + (size_t)i * (kB * kB);
  double wv[4], part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) wv[cc] = __ldcg(Wi + (4 * warp + cc) * kB + lane);
  const double yv = tid < kB ? __ldcg(A.ybuf + (int64_t)kB * i + tid) : 0.0;
  double* red = sm + 2 * kB * kB;
  double* tv = red + 8 * kB;
  if (nt - 1 > i) stage_lin(sm, tile_src(A, nt - 1, i), kB * kB, tid, kT);
  cp_commit();
  for (int j = nt - 1; j > i; --j) {
    const int s = (nt - 1 - j) & 1;
    const bool next = j - 1 > i;
    if (next) stage_lin(sm + (s ^ 1) * (kB * kB), tile_src(A, j - 1, i), kB * kB, tid, kT);
    cp_commit();
    if (tid == 0) *s_flag = wait_flags(A.xflags + j, A.xflags + j, failw, target) ? 1u : 2u;
    cp_wait1();
    __syncthreads();
    if (*s_flag == 2u) return false;
    const double xj = __ldcg(A.xbuf + kB * j + lane);
    const double* X = sm + s * (kB * kB);  // packed column-major
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) part[cc] = fma(X[(4 * warp + cc) * kB + lane], xj, part[cc]);
    __syncthreads();  // the buffer is refilled two tiles later
  }
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    const double t = warp_sum(part[cc]);
    if (lane == 0) red[4 * warp + cc] = t;
  }
  __syncthreads();
  if (tid < kB) tv[tid] = yv - red[tid];
  __syncthreads();
  const double tl = tv[lane];
  const int64_t r0 = (int64_t)kB * i;
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    const int c = 4 * warp + cc;  // x(c) = sum_{r >= c} W(r, c) t(r)
    const double t = warp_sum(wv[cc] * tl);
    if (lane == 0) {
      A.xbuf[kB * i + c] = t;
      if (r0 + c < A.n) A.x[r0 + c] = t;
    }
  }
  publish(A.xflags + i, target);
  return true;
}

__device__ bool df_spine(const DfArgs& A, unsigned target, double* sm) {
  __shared__ SpineShared ss_;
  __shared__ __align__(8) uint64_t sig[kB];  // pivot p's column published (factor -> inverse warp)
  __shared__ __align__(8) uint64_t bfull[kBSlots], bempty[kBSlots];  // backward tile ring
  volatile SpineShared* ss = &ss_;
  if (threadIdx.x == 0) {
    ss->fail = -1;
    ss->passes = 0;
    for (int p = 0; p < kB; ++p) mbar_init(sig + p, 1);
    fence_barrier_init();
  }
  __syncthreads();
  bool ok = true;
  if (threadIdx.x < kCT) spine_compute(A, sm, ss, sig);
  else if (threadIdx.x < kCT + kIOT) ok = spine_publish(A, target, sm, ss);
  else spine_prefetch(A, target, sm, ss);
  __syncthreads();
  if (ss->fail >= 0) return false;
  (void)ok;
  STRACE(63, 0);
  if (A.back) spine_back(A, sm, bfull, bempty);
  STRACE(63, 1);
  STRACE_FLUSH();
  return true;
}

__global__ void __launch_bounds__(kT, 1) k_chol_df(const DfArgs A) {
  extern __shared__ __align__(16) double sm_df[];
  __shared__ unsigned s_target, s_q, s_flag;
  const int tid = threadIdx.x;
  if (tid == 0) s_target = *reinterpret_cast<volatile unsigned*>(A.ctl) + 1u;
  __syncthreads();
  const unsigned target = s_target;
  while (true) {
    if (tid == 0) s_q = atomicAdd(A.ctl + 4, 1u);
    __syncthreads();
    const int q = (int)s_q;
    if (q >= A.ntasks + A.nback) break;
    bool ok;
    if (q >= A.ntasks) {  // backward tasks, last block first
      ok = df_back(A, A.nt - 1 - (q - A.ntasks), target, sm_df, &s_flag);
    } else if (q == 0) {
      ok = df_spine(A, target, sm_df);
    } else {
      // the pre-diagonal tasks without dependencies (d < 3), then column by column: the
      // panels (i, j), i >= j + 2, and the pre-diagonal task j + 3 (which needs columns <= j)
      const int n0 = min(A.nt, 3);
      int r = q - 1;
      if (r < n0) {
        ok = df_prediag(A, r, target, sm_df, &s_flag);
      } else {
        r -= n0;
        int j = 0;
        while (true) {
          const int np = max(0, A.nt - j - 2);
          const int cnt = np + (j + 3 < A.nt ? 1 : 0);
          if (r < cnt) break;
          r -= cnt;
          ++j;
        }
        if (r < max(0, A.nt - j - 2)) ok = df_panel(A, j + 2 + r, j, target, sm_df, &s_flag);
        else ok = df_prediag(A, j + 3, target, sm_df, &s_flag);
      }
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
  c.df_part = dev_zeros<double>((size_t)nb * kPartLen, c.stream);
  c.df_pflags = dev_zeros<unsigned>((size_t)nb, c.stream);
  c.df_x = dev_zeros<double>((size_t)nb * kB, c.stream);
  c.df_xflags = dev_zeros<unsigned>((size_t)nb, c.stream);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  c.df_grid = sms;  // one 141 KB CTA of 256 threads per SM
}

void chol_free(Ctx& c) {
  for (void* p : {(void*)c.Winv, (void*)c.Lt, (void*)c.df_flags, (void*)c.df_ctl, (void*)c.df_y,
                  (void*)c.df_part, (void*)c.df_pflags, (void*)c.df_x, (void*)c.df_xflags})
    dev_free(p, c.stream);
  c.Winv = c.Lt = c.df_y = c.df_part = c.df_x = nullptr;
  c.df_flags = c.df_ctl = c.df_pflags = c.df_xflags = nullptr;
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
  a.ntasks = 1 + nt + (nt >= 2 ? (nt - 1) * (nt - 2) / 2 : 0);
  a.flags = c.df_flags;
  a.ctl = c.df_ctl;
  a.info = info;
  a.rhs = rhs;
  a.x = x;
  a.ybuf = c.df_y;
  a.part = c.df_part;
  a.pflags = c.df_pflags;
  a.back = rhs != nullptr && n <= kMaxFusedN;
  a.nback = (rhs != nullptr && !a.back) ? nt : 0;
  a.xbuf = c.df_x;
  a.xflags = c.df_xflags;
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
