// K1: condensed KKT assembly  M = H + J' diag(sigma) J  on FP64 tensor cores.
//
// Reference: gram_weighted (proj/src/dense_linalg.cpp:128-137) forms the scaled copy
// W = diag(sqrt(sigma)) J and a lower rankUpdate over all m rows; assemble_condensed
// (proj/src/ipm.cpp:72-77) adds H. Here the SYRK runs over the distinct prototype rows P
// (structure.cu) with merged weights omega = Pi' sigma:
//     M_lower = H + P' diag(omega) P + diag(singleton terms)
// * operands: 64-column x 32-row K-major tiles of P staged by TMA (128B swizzle) through a
//   3-stage mbarrier pipeline fed by one producer warp; omega rides the same barrier as a
//   1-D bulk copy; the diagonal weight is applied to the B fragment in registers, so a
//   diagonal tile loads its operand once.
// * math: mma.sync m16n8k16 f64 (DMMA.8x8x4), 4 consumer warps per 64x64 tile, each owning
//   an equal share of the tile's useful 16x8 fragments.
// * zero-block skipping: rows are sorted by nonzero prefix width; tile (I,J) (I>=J) only
//   visits the rows whose prefix reaches column 64*I, and the rows whose prefix ends inside
//   block I only compute the output rows they can reach: off-diagonal segments in 8-row
//   steps (rows 0..8q-1, q = 1..8; up to 32 rows only the A operand's first 32 columns are
//   loaded), diagonal ones THIN (rows 0..31) or FULL.
// * scheduling: one persistent CTA pair per SM grabs PIECES from an atomic counter: first one
//   equal-cost body piece each, then tail pieces of decreasing cost so the CTAs finish
//   together; a piece holds one or more SEGMENTS (a k range of one tile).
// * reduction: every segment stores a partial tile; k_syrk_reduce sums a tile's partials in
//   the plan's k order and adds H and the singleton diagonal (M bitwise reproducible).
#include <cuda.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.cuh"
#include "ptx.cuh"

namespace cmpc {

namespace {

constexpr int kStages = 3;
constexpr int kBoxBytes = 16 * 64 * 8;          // {16 k, 64 cols} FP64 box
constexpr int kOpBytes = 2 * kBoxBytes;         // 32 k x 64 cols
constexpr int kStageBytes = 2 * kOpBytes + 1024;  // A, B, omega (256 B, padded to 1 KB)
constexpr int kSyrkSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers, ring*/;
constexpr int kConsumerWarps = 4;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kSyrkThreads = kConsumers + 32;
// relative cost of one k step per segment shape: a diagonal step also forms its rows' share
// of the fused right-hand side P'q (swept with CMPC_SYRK_COST and tools/phases.py: at C3 the
// fused condensation 297 us with these, 315 us with the weights measured without it,
// 1 / 0.6 / 0.85 / 0.35; C4 and C5 improve too)
constexpr double kCostDiag = 1.1, kCostDiagThin = 0.5;
// off-diagonal segments by output rows / 8 (index 1..8): 16 rows 0.4, 32 rows 0.65 (THIN),
// 48 rows 0.85, 64 rows 1.0 (FULL) as measured; the 8-row steps interpolated
constexpr double kCostRows[9] = {0.0, 0.25, 0.4, 0.55, 0.65, 0.75, 0.85, 0.93, 1.0};

struct SyrkArgs {
  const double* omega;
  const int4* segs;          // {ti | tj << 10 | shape << 20, k0, k1, tile index}
  const int32_t* piece_ptr;  // npieces + 1 into segs
  int npieces;
  unsigned* ctl;             // [0] next piece, [1] retired CTAs (both 0 between launches)
  double* partial;           // per segment: 64 x 64 column-major partial tile
  const double* q;           // fused right-hand side: P' q over the diagonal jobs (null: off)
  double* rhs_part;          // per segment: 2 x 64 half-sums of P' q (diagonal segments)
  long long* prof;           // debug: per piece {start ns, end ns, smid}
  int static_sched;          // debug: CTA b takes pieces b, b + grid, ... (no counter)
  // Markov layout (markov.cu): a segment's k range indexes the chunk lists; chunk ch covers
  // prototype rows [32 ch, 32 ch + 32) and reads table rows cinfo.x.. at column shift cinfo.y
  const int4* clist;         // per position {table row, column shift, prototype row}; null:
                             // P materialised, k = prototype row
};

// byte offset of element (col c, k) inside a 32 x 64 operand tile (two swizzled boxes)
__device__ __forceinline__ uint32_t op_off(int c, int k) {
  const int kk = k & 15;
  return (uint32_t)((k >> 4) * kBoxBytes + c * 128 + ((((kk >> 1) ^ (c & 7)) << 4) | ((kk & 1) << 3)));
}

// Segment epilogue: store the accumulators as the segment's partial tile.
template <int NF>
__device__ __forceinline__ void store_partial(const SyrkArgs& a, int sg,
                                              const double (&acc)[NF][2][4], const int* fr,
                                              const int* fn, int lane) {
  double* out = a.partial + (size_t)sg * (kTile * kTile);
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r = 32 * fr[f] + 16 * mi + g;
      const int c = 8 * fn[f] + 2 * t;
      __stcg(out + c * kTile + r, acc[f][mi][0]);
      __stcg(out + (c + 1) * kTile + r, acc[f][mi][1]);
      __stcg(out + c * kTile + r + 8, acc[f][mi][2]);
      __stcg(out + (c + 1) * kTile + r + 8, acc[f][mi][3]);
    }
}

// Consumer work of one segment. Each segment covers a k range of one 64x64 output tile in
// one of four shapes; the 4 consumer warps split the useful 8-column fragments evenly:
//   FULL (off-diagonal): 2 x 8 fragments (row halves r = 0,1) -> 4 per warp
//   THIN (off-diagonal): rows 0..31 only                      -> 2 per warp
//   FULL (diagonal):     the 12 fragments on or below the diagonal 32x32 blocks -> 3 per warp
//   THIN (diagonal):     the lower-left 32x32 block           -> 1 per warp
template <int NF, bool DIAG, bool THIN>
__device__ __forceinline__ void syrk_segment(const SyrkArgs& a, unsigned char* smem, uint64_t* full,
                                             uint64_t* empty, int it0, int sg, const int4 u,
                                             int warp, int lane) {
  const int nsteps = (u.z - u.y) / kBK;
  const int g = lane >> 2, t = lane & 3;
  // fragment i covers output rows 32*r(i).. and columns 8*fn(i)..; MIXED: the one diagonal
  // warp whose fragments straddle both row halves (fragment 0 in half 0, the rest in half 1)
  const bool mixed = DIAG && !THIN && warp == 1;
  int r0, fn0;
  if (DIAG && !THIN) {
    r0 = warp >= 2 ? 1 : 0;
    fn0 = warp == 0 ? 0 : warp == 1 ? 3 : warp == 2 ? 2 : 5;
  } else if (THIN) {
    r0 = 0;
    fn0 = NF * warp;
  } else {
    r0 = warp & 1;
    fn0 = 4 * (warp >> 1);
  }
  int fr[NF], fn[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    fr[i] = mixed ? (i == 0 ? 0 : 1) : r0;
    fn[i] = mixed ? (i == 0 ? 3 : i - 1) : fn0 + i;
  }

  double acc[NF][2][4];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[f][b][c] = 0.0;
  // fused right-hand side: a diagonal job streams every nonzero row of its column block, so
  // thread (kh, cc) also sums P(k, cc) q(k) over its half of each stage's 32 rows: after the
  // stage's MMAs are issued (the FMAs overlap the tensor pipe), 16-byte loads of row pairs into
  // two accumulators (even and odd rows, added at the end)
  double rq[2] = {0.0, 0.0};
  const bool do_rq = DIAG && a.q != nullptr && (!THIN || (threadIdx.x & 63) < 32);

  for (int it = it0; it < it0 + nsteps; ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (it / kStages) & 1);
    // explicit 32-bit shared addresses: the aligned generic pointer would compile to LD
    // (global-load scoreboard latency) instead of LDS
    const uint32_t sA = smem_u32(smem + s * kStageBytes);
    const uint32_t sB = DIAG ? sA : sA + kOpBytes;
    const uint32_t sW = sA + 2 * kOpBytes;
#pragma unroll
    for (int ks = 0; ks < kBK; ks += 16) {
      double af[2][8], ax[2][8];  // A fragments of half r0 (ax: half 0 for the mixed warp)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const int c = 16 * mi + g + 8 * (x & 1);
          const int k = ks + t + 4 * (x >> 1);
          af[mi][x] = lds64(sA + op_off(32 * (mixed ? 1 : r0) + c, k));
          if (DIAG && !THIN) {
            if (mixed) ax[mi][x] = lds64(sA + op_off(c, k));
          }
        }
      double w[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) w[x] = lds64(sW + 8 * (ks + t + 4 * x));
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        double bf[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) bf[x] = w[x] * lds64(sB + op_off(8 * fn[i] + g, ks + t + 4 * x));
        // as four k4 steps with the two row halves interleaved: four independent DMMA chains
        // between dependent steps instead of the two inside one m16n8k16 (same k order)
        if (DIAG && !THIN && i == 0 && mixed) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) dmma1684(acc[i][mi], ax[mi] + 2 * q, bf[q]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) dmma1684(acc[i][mi], af[mi] + 2 * q, bf[q]);
        }
      }
    }
    if (DIAG && do_rq) {
      const int cc = threadIdx.x & 63, k0 = 16 * (threadIdx.x >> 6);
      const uint32_t sQ = sW + 256;
#pragma unroll
      for (int kk = 0; kk < 16; kk += 2) {  // rows k, k+1 of column cc share one 16-byte chunk
        const double2 pa = lds128(sA + op_off(cc, k0 + kk));
        const double2 qq = lds128(sQ + 8 * (k0 + kk));
        rq[0] = fma(pa.x, qq.x, rq[0]);
        rq[1] = fma(pa.y, qq.y, rq[1]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  store_partial<NF>(a, sg, acc, fr, fn, lane);
  if (DIAG && a.q) a.rhs_part[(size_t)sg * 128 + threadIdx.x] = rq[0] + rq[1];
}

// Off-diagonal segments whose rows end inside the tile's block row at a row count that is not
// 32 or 64: 16 R16 (+ 8 with HALF) output rows x 64 columns, warp w owning column groups 2w, 2w + 1
// (so the four warps stay balanced; the 8-row block runs on m8n8k4); the tile's other rows are
// zero for these prototype rows and are neither computed nor stored (k_syrk_reduce skips them)
template <int R16, bool HALF>
__device__ __forceinline__ void syrk_segment_q(const SyrkArgs& a, unsigned char* smem, uint64_t* full,
                                               uint64_t* empty, int it0, int sg, const int4 u, int warp,
                                               int lane) {
  constexpr int RA = R16 > 0 ? R16 : 1;  // (array extent; R16 = 0 uses only the 8-row block)
  const int nsteps = (u.z - u.y) / kBK;
  const int g = lane >> 2, t = lane & 3;
  const int cg0 = 2 * warp;
  double acc[RA][2][4], acc8[2][2];
#pragma unroll
  for (int rb = 0; rb < RA; ++rb)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[rb][b][c] = 0.0;
#pragma unroll
  for (int b = 0; b < 2; ++b) acc8[b][0] = acc8[b][1] = 0.0;
  for (int it = it0; it < it0 + nsteps; ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (it / kStages) & 1);
    const uint32_t sA = smem_u32(smem + s * kStageBytes);
    const uint32_t sB = sA + kOpBytes;
    const uint32_t sW = sA + 2 * kOpBytes;
#pragma unroll
    for (int ks = 0; ks < kBK; ks += 16) {
      double af[RA][8], a8[4];
#pragma unroll
      for (int rb = 0; rb < R16; ++rb)
#pragma unroll
        for (int x = 0; x < 8; ++x)
          af[rb][x] = lds64(sA + op_off(16 * rb + g + 8 * (x & 1), ks + t + 4 * (x >> 1)));
      if (HALF)
#pragma unroll
        for (int q = 0; q < 4; ++q) a8[q] = lds64(sA + op_off(16 * R16 + g, ks + t + 4 * q));
      double w[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) w[x] = lds64(sW + 8 * (ks + t + 4 * x));
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double bf[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) bf[x] = w[x] * lds64(sB + op_off(8 * (cg0 + i) + g, ks + t + 4 * x));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int rb = 0; rb < R16; ++rb) dmma1684(acc[rb][i], af[rb] + 2 * q, bf[q]);
          if (HALF) dmma884(acc8[i], a8[q], bf[q]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  double* out = a.partial + (size_t)sg * (kTile * kTile);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int c = 8 * (cg0 + i) + 2 * t;
#pragma unroll
    for (int rb = 0; rb < R16; ++rb) {
      const int r = 16 * rb + g;
      __stcg(out + c * kTile + r, acc[rb][i][0]);
      __stcg(out + (c + 1) * kTile + r, acc[rb][i][1]);
      __stcg(out + c * kTile + r + 8, acc[rb][i][2]);
      __stcg(out + (c + 1) * kTile + r + 8, acc[rb][i][3]);
    }
    if (HALF) {
      const int r = 16 * R16 + g;
      __stcg(out + c * kTile + r, acc8[i][0]);
      __stcg(out + (c + 1) * kTile + r, acc8[i][1]);
    }
  }
}

// 2 CTAs per SM: 168 registers (each SM sub-partition holds 3 warps of 168 x 32; the few
// spilled values live outside the k loops)
__global__ void __launch_bounds__(kSyrkThreads, 2)
    k_syrk(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmP32,
           const SyrkArgs a) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* pfull = empty + kStages;  // piece ring: producer -> consumers
  uint64_t* pempty = pfull + 2;
  volatile int* ring = reinterpret_cast<volatile int*>(pempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&pfull[s], 1);
      mbar_init(&pempty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer: grab pieces, stream their segments' stages
    if (lane == 0) {
      int it = 0;
      for (int i = 0;; ++i) {
        const int slot = i & 1;
        if (i >= 2) mbar_wait(&pempty[slot], ((i >> 1) & 1) ^ 1);
        int pg = a.static_sched ? (int)(blockIdx.x + (unsigned)i * gridDim.x) : (int)atomicAdd(a.ctl, 1u);
        if (pg >= a.npieces) pg = -1;
        ring[slot] = pg;
        mbar_arrive(&pfull[slot]);
        if (pg < 0) break;
        const int p = pg;
        const double* omega = a.omega;
        const double* qv = a.q;
        for (int sg = a.piece_ptr[p]; sg < a.piece_ptr[p + 1]; ++sg) {
          const int4 u = a.segs[sg];
          const int ti = u.x & 1023, tj = (u.x >> 10) & 1023;
          const int shape = (u.x >> 20) & 15, diag = ti == tj;  // output rows / 8 (1..8)
          const bool thin = shape <= 4;  // the A operand's first 32 columns suffice
          const uint32_t abytes = thin ? kOpBytes / 2 : kOpBytes;
          const bool with_q = diag && a.q != nullptr;
          const uint32_t bytes = abytes + (diag ? 0u : (uint32_t)kOpBytes) + kBK * 8 + (with_q ? kBK * 8 : 0u);
          const void* tmA = thin ? (const void*)&tmP32 : (const void*)&tmP;
          // operand rows / column offset / prototype row of each k step; Markov layout: the
          // position's entry, loaded one step ahead so its latency overlaps the current step
          int4 nx4 = make_int4(u.y, 0, u.y, 0);
          if (a.clist && u.y < u.z) nx4 = __ldg(a.clist + u.y / kBK);
          for (int kk = u.y; kk < u.z; kk += kBK, ++it) {
            const int s = it % kStages;
            const int ra = a.clist ? nx4.x : kk, cs = a.clist ? nx4.y : 0, pr = a.clist ? nx4.z : kk;
            if (a.clist && kk + kBK < u.z) nx4 = __ldg(a.clist + (kk + kBK) / kBK);
            if (it >= kStages) {
              mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
              // the consumers' generic-proxy reads of this stage (ordered before us by the
              // barrier) must also precede our async-proxy (TMA) rewrite of it: without this
              // fence a slow lane could still read the stage as the next tile lands (seen
              // under SM contention, tests/test_gpu_concurrency.py)
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            unsigned char* st = smem + s * kStageBytes;
            mbar_expect_tx(&full[s], bytes);
            // a 32-column box lands exactly where the first 32 columns of a 64-column box would
            tma_load_2d(st, tmA, ra, cs + 64 * ti, &full[s]);
            tma_load_2d(st + kBoxBytes, tmA, ra + 16, cs + 64 * ti, &full[s]);
            if (!diag) {
              tma_load_2d(st + kOpBytes, &tmP, ra, cs + 64 * tj, &full[s]);
              tma_load_2d(st + kOpBytes + kBoxBytes, &tmP, ra + 16, cs + 64 * tj, &full[s]);
            }
            bulk_load(st + 2 * kOpBytes, omega + pr, kBK * 8, &full[s]);
            if (with_q) bulk_load(st + 2 * kOpBytes + 256, qv + pr, kBK * 8, &full[s]);
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers
  int it0 = 0;
  for (int i = 0;; ++i) {
    const int slot = i & 1;
    mbar_wait(&pfull[slot], (i >> 1) & 1);
    const int pg = ring[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&pempty[slot]);
    if (pg < 0) break;
    const int p = pg;
    long long t_start = 0;
    if (a.prof && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    for (int sg = a.piece_ptr[p]; sg < a.piece_ptr[p + 1]; ++sg) {
      const int4 u = a.segs[sg];
      const int shape = (u.x >> 20) & 15;  // output rows / 8
      const bool diag = (u.x & 1023) == ((u.x >> 10) & 1023);
      if (diag) {
        if (shape == 4) syrk_segment<1, true, true>(a, smem, full, empty, it0, sg, u, warp, lane);
        else syrk_segment<3, true, false>(a, smem, full, empty, it0, sg, u, warp, lane);
      } else {
        switch (shape) {
          case 1: syrk_segment_q<0, true>(a, smem, full, empty, it0, sg, u, warp, lane); break;
          case 2: syrk_segment_q<1, false>(a, smem, full, empty, it0, sg, u, warp, lane); break;
          case 3: syrk_segment_q<1, true>(a, smem, full, empty, it0, sg, u, warp, lane); break;
          case 4: syrk_segment<2, false, true>(a, smem, full, empty, it0, sg, u, warp, lane); break;
          case 5: syrk_segment_q<2, true>(a, smem, full, empty, it0, sg, u, warp, lane); break;
          case 6: syrk_segment_q<3, false>(a, smem, full, empty, it0, sg, u, warp, lane); break;
          case 7: syrk_segment_q<3, true>(a, smem, full, empty, it0, sg, u, warp, lane); break;
          default: syrk_segment<4, false, false>(a, smem, full, empty, it0, sg, u, warp, lane); break;
        }
      }
      it0 += (u.z - u.y) / kBK;
    }
    if (a.prof && threadIdx.x == 0) {  // debug timeline (cmpc_debug_syrk_timeline)
      long long t_end;
      unsigned smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.prof[3 * pg] = t_start;
      a.prof[3 * pg + 1] = t_end;
      a.prof[3 * pg + 2] = smid;
    }
  }
  // the last CTA out resets the piece counter for the next launch (every producer has made
  // its final grab before its consumers saw the end marker)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.ctl + 1, 1u) == gridDim.x - 1) {
      a.ctl[0] = 0;
      a.ctl[1] = 0;
      __threadfence();
    }
  }
}

// M(i,j) = H(i,j) + (sum of the tile's partials [+ singleton diagonal]), lower (+ mirrored
// upper); grid (tiles, 64): 64 elements of one tile per block, four threads per element
// ("ways"), way w summing the chunks of eight segments w, w + 4, ... (eight loads in flight)
// and way 0 adding the four in order (deterministic). The first tile column's tiles collect
// partials from nearly every segment; four ways cut that critical chain by four. Thin
// partials hold rows 0..31 only (flag bit 31 of their id); a warp's 32 elements share one
// row half, so the skip is warp-uniform.
constexpr int kRedWays = 4;
__global__ void __launch_bounds__(256)
    k_syrk_reduce(const double* __restrict__ partial, const int2* __restrict__ tiles,
                  const int32_t* __restrict__ tile_ptr, const int32_t* __restrict__ tile_segs,
                  const double* __restrict__ H, const double* __restrict__ omega_s, int64_t n,
                  double* __restrict__ M, int mirror, const double* __restrict__ rp,
                  const double* __restrict__ qs, const int32_t* __restrict__ sing_ptr,
                  const double* __restrict__ sing_val, double* __restrict__ tq,
                  double* __restrict__ rhs, const double* __restrict__ r1) {
  __shared__ double red[kRedWays][64];
  const int2 tl = tiles[blockIdx.x];
  const int u0 = tile_ptr[blockIdx.x], u1 = tile_ptr[blockIdx.x + 1];
  const int t64 = threadIdx.x & 63, way = threadIdx.x >> 6;
  if (rp && tl.x == tl.y && blockIdx.y == 0) {
    // fused right-hand side of the block: P' q from the diagonal segments' half-sums + the
    // singleton rows of its columns
    const int64_t col = (int64_t)kTile * tl.x + t64;
    double s = 0.0;
    if (col < n) {
      for (int q = u0 + 8 * way; q < u1; q += 8 * kRedWays) {
        double x[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          x[b] = 0.0;
          if (q + b < u1) {
            const int32_t id = tile_segs[q + b] & 0x0fffffff;
            x[b] = __ldcg(rp + (size_t)id * 128 + t64) + __ldcg(rp + (size_t)id * 128 + 64 + t64);
          }
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) s += x[b];
      }
    }
    red[way][t64] = s;
    __syncthreads();
    if (way == 0 && col < n) {
      s = ((red[0][t64] + red[1][t64]) + red[2][t64]) + red[3][t64];
      for (int32_t k = sing_ptr[col]; k < sing_ptr[col + 1]; ++k) s += sing_val[k] * qs[k];
      // unsharded: the final -r1 + J'(r2 - sigma r3) here (k_rhs's rounding, no extra launch)
      tq[col] = s;
      if (r1) rhs[col] = __dadd_rn(-r1[col], s);
    }
    __syncthreads();
  }
  const int e = blockIdx.y * 64 + t64;
  const int rl = e & (kTile - 1), cl = e >> 6;
  const int64_t i = (int64_t)kTile * tl.x + rl, j = (int64_t)kTile * tl.y + cl;
  const bool live = i < n && j < n && i >= j;  // (no early exit: every thread reaches the barrier)
  // a partial's valid rows: 8 x code (id bits 28-31)
  double s = 0.0;
  if (live) {
    for (int q = u0 + 8 * way; q < u1; q += 8 * kRedWays) {
      double x[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        x[b] = 0.0;
        if (q + b < u1) {
          const int32_t id = __ldg(tile_segs + q + b);
          const int code = (int)((unsigned)id >> 28);
          if (rl < 8 * code) x[b] = __ldcg(partial + (size_t)(id & 0x0fffffff) * (kTile * kTile) + e);
        }
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) s += x[b];
    }
  }
  red[way][t64] = s;
  __syncthreads();
  if (way != 0 || !live) return;
  s = ((red[0][t64] + red[1][t64]) + red[2][t64]) + red[3][t64];
  if (i == j) {  // + sum over the singleton rows at column i of omega a^2
    double ds = 0.0;
    for (int32_t k = sing_ptr[i]; k < sing_ptr[i + 1]; ++k) ds += omega_s[k] * (sing_val[k] * sing_val[k]);
    s += ds;
  }
  const double v = H ? H[i + j * n] + s : s;  // H on one rank only when sharded
  M[i + j * n] = v;
  if (mirror && i != j) M[j + i * n] = v;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CMPC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

}  // namespace

void syrk_free(Ctx& c) {
  for (void* p : {(void*)c.units, (void*)c.cta_ptr, (void*)c.syrk_ctl, (void*)c.tiles,
                  (void*)c.tile_ptr, (void*)c.tile_units, (void*)c.partial, (void*)c.rhs_part})
    dev_free(p, c.stream);
  c.units = nullptr;
  c.cta_ptr = nullptr;
  c.syrk_ctl = nullptr;
  c.tiles = nullptr;
  c.tile_ptr = c.tile_units = nullptr;
  c.partial = nullptr;
  c.rhs_part = nullptr;
  delete[] reinterpret_cast<unsigned char*>(c.tmap_P);
  delete[] reinterpret_cast<unsigned char*>(c.tmap_P32);
  c.tmap_P = c.tmap_P32 = nullptr;
}

void syrk_plan(Ctx& c) {
  syrk_free(c);
  const int64_t n = c.n;
  const int nt = (int)ceil_div(n, kTile);
  const int k_end = (int)c.ldp;
  // algorithmic work of one condensation: lower triangle of P' diag(omega) P
  {
    std::vector<int32_t> hh(size_t(std::max<int64_t>(c.ps, 1)));
    if (c.ps > 0) {
      CMPC_CUDA(cudaMemcpyAsync(hh.data(), c.hi, sizeof(int32_t) * c.ps, cudaMemcpyDeviceToHost, c.stream));
      CMPC_CUDA(cudaStreamSynchronize(c.stream));
    }
    double f = 0.0, b = 0.0;
    for (int64_t k = 0; k < c.ps; ++k) {
      f += double(hh[size_t(k)]) * double(hh[size_t(k)] + 1);
      b += 8.0 * hh[size_t(k)];
    }
    c.syrk_flops = f;
    c.syrk_bytes = b;
  }
  // first P row (kBK-aligned down) whose prefix reaches column col
  auto kstart = [&](int64_t col) {
    if (c.ps == 0) return k_end;
    return c.h_start_col[size_t(std::min<int64_t>(n, col))] / kBK * kBK;
  };
  // jobs: per lower tile (I,J), the rows whose prefix ends in the first half of column block I
  // (THIN: only output rows 0..31 are nonzero) and the rest (FULL)
  // shape = the output rows a segment computes / 8 (1..8): off-diagonal tiles in 8-row steps,
  // diagonal tiles 4 (rows 0..31) or 8
  struct Job { int tile, ti, tj, shape, kb, ke; double w; int split; };
  // step weights per segment shape (measured with tools/syrk_timeline.py and the bench)
  const double cost_d = kCostDiag, cost_dt = kCostDiagThin;
  std::vector<Job> jobs;
  std::vector<int2> tiles;
  // Markov layout: the k axis of a job is a list of chunks (stage-major prototype rows are
  // not sorted by width). Column block ti's lists, in order: the chunks whose widest row ends
  // in (64 ti + 8 (q - 1), 64 ti + 8 q], q = 1..8 (the last list: everything beyond); a
  // diagonal tile's thin job spans the first four, its full job the rest. kb/ke index clist.
  std::vector<int32_t> clist;
  std::vector<std::array<int, 9>> mk_lists((size_t)nt);  // list boundaries per column block
  if (c.markov) {
    for (int ti = 0; ti < nt; ++ti) {
      const int lo = kTile * ti;
      mk_lists[size_t(ti)][0] = (int)clist.size();
      for (int q = 1; q <= 8; ++q) {
        const int e0 = lo + 8 * (q - 1), e1 = q == 8 ? (1 << 30) : lo + 8 * q;
        for (int ch = 0; ch < c.mk_nchunks; ++ch) {
          const int w = c.h_mk_width[size_t(ch)];
          if (w > e0 && w <= e1) clist.push_back(ch);
        }
        mk_lists[size_t(ti)][size_t(q)] = (int)clist.size();
      }
    }
  }
  for (int tj = 0; tj < nt; ++tj)
    for (int ti = tj; ti < nt; ++ti) {
      const int tile = (int)tiles.size();
      tiles.push_back({ti, tj});
      const bool dg = ti == tj;
      // the job boundaries along k: rows ending in (lo + 8 (q-1), lo + 8 q], q = 1..8
      int b[9];
      if (c.markov) {
        for (int q = 0; q < 9; ++q) b[q] = mk_lists[size_t(ti)][size_t(q)] * kBK;
      } else {
        b[0] = kstart((int64_t)kTile * ti);
        for (int q = 1; q < 8; ++q) b[q] = std::max(b[q - 1], kstart((int64_t)kTile * ti + 8 * q));
        b[8] = std::max(b[7], k_end);
      }
      if (dg) {
        if (b[4] > b[0]) jobs.push_back({tile, ti, tj, 4, b[0], b[4], cost_dt, 0});
        if (b[8] > b[4]) jobs.push_back({tile, ti, tj, 8, b[4], b[8], cost_d, 0});
      } else {
        for (int q = 1; q <= 8; ++q)
          if (b[q] > b[q - 1]) jobs.push_back({tile, ti, tj, q, b[q - 1], b[q], kCostRows[q], 0});
      }
    }
  // k step of a job position: the prototype row step, or (Markov) the chunk id
  auto step_of = [&](int pos) { return c.markov ? clist[size_t(pos)] : pos; };
  // Pieces. The k axis is split where the cumulative weighted work reaches (1 - tail_frac).
  // The body [0, K) is laid out job after job and cut into one equal-cost piece per CTA slot
  // (every CTA starts with one; few segments, so few partial tiles). The tail [K, end) is laid
  // out the same way and cut into pieces of decreasing cost (remaining / slots, at least
  // min_piece steps) that the CTAs grab as they finish: the dynamic tail absorbs the run-time
  // spread of the body pieces so the CTAs finish together.
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const int slots = sms * 2;
  const int nsteps_all = c.markov ? c.mk_nchunks : k_end / kBK;
  std::vector<double> dens(size_t(std::max(nsteps_all, 1)), 0.0);  // weighted cost per k step
  for (const Job& jb : jobs)
    for (int q = jb.kb / kBK; q < jb.ke / kBK; ++q) dens[size_t(step_of(q))] += jb.w;
  double work = 0.0;
  for (double x : dens) work += x;
  // small problems (C2, C5: ~2 steps per slot) run fewer, longer pieces: fewer partial tiles
  // to reduce, and no dynamic tail
  const double tail_frac = work >= 16.0 * slots ? 0.1 : 0.0, min_piece = 3.0, min_body = 8.0;
  int ksplit = nsteps_all;  // body = steps [0, ksplit)
  {
    double acc = 0.0;
    for (int q = 0; q < nsteps_all; ++q) {
      if (acc >= work * (1.0 - tail_frac)) {
        ksplit = q;
        break;
      }
      acc += dens[size_t(q)];
    }
  }
  // a job's positions before / after the split step (its list is in step order)
  for (Job& jb : jobs) {
    int q = jb.kb / kBK;
    while (q < jb.ke / kBK && step_of(q) < ksplit) ++q;
    jb.split = q;
  }
  auto range = [&](const Job& jb, int region, int& a, int& b) {
    a = region == 0 ? jb.kb / kBK : jb.split;
    b = region == 0 ? jb.split : jb.ke / kBK;
  };
  std::vector<int4> segs;
  std::vector<int32_t> pptr{0};
  std::vector<std::vector<int32_t>> per_tile(tiles.size());
  auto emit = [&](const Job& jb, int a, int b) {
    const int id = (int)segs.size();
    // k_syrk_reduce's row code (bits 28-31): valid rows 8 x code
    per_tile[size_t(jb.tile)].push_back((int32_t)((unsigned)id | ((unsigned)jb.shape << 28)));
    segs.push_back({jb.ti | jb.tj << 10 | jb.shape << 20, a * kBK, b * kBK, jb.tile});
  };
  auto close_piece = [&]() {
    if (pptr.back() != (int32_t)segs.size()) pptr.push_back((int32_t)segs.size());
  };
  for (int region = 0; region < 2; ++region) {
    double cw = 0.0;
    int64_t steps = 0;
    for (const Job& jb : jobs) {
      int a, b;
      range(jb, region, a, b);
      if (a < b) {
        cw += (b - a) * jb.w;
        steps += b - a;
      }
    }
    if (steps == 0) continue;
    double remaining = cw, in_piece = 0.0;
    auto target = [&] {
      return region == 0 ? std::max(std::min(min_body, cw), cw / double(std::min<int64_t>(slots, steps)))
                         : std::max(min_piece, remaining / slots);
    };
    double tgt = target();
    for (const Job& jb : jobs) {
      const double w = jb.w;
      int a, b;
      range(jb, region, a, b);
      while (a < b) {
        const int need = std::max(1, (int)std::ceil((tgt - in_piece) / w - 1e-9));
        const int take = std::min(b - a, need);
        emit(jb, a, a + take);
        in_piece += take * w;
        remaining -= take * w;
        a += take;
        if (in_piece >= tgt - 1e-9) {
          close_piece();
          in_piece = 0.0;
          tgt = target();
        }
      }
    }
    close_piece();
  }
  const int npieces = (int)pptr.size() - 1;
  c.syrk_cta_cost.assign(size_t(5 * npieces), 0.0);  // per piece: segments, steps per shape
  for (int p = 0; p < npieces; ++p)
    for (int q = pptr[size_t(p)]; q < pptr[size_t(p) + 1]; ++q) {
      const int4 u = segs[size_t(q)];
      const int thin = ((u.x >> 20) & 15) < 8 ? 1 : 0, dg = (u.x & 1023) == ((u.x >> 10) & 1023);
      c.syrk_cta_cost[size_t(5 * p)] += 1.0;
      c.syrk_cta_cost[size_t(5 * p + 1 + thin + 2 * dg)] += double(u.z - u.y) / kBK;
    }
  if (getenv("CMPC_SYRK_PLAN"))
    fprintf(stderr, "[syrk plan] jobs %zu tail from step %d of %d, pieces %d segments %zu weighted steps %.0f (%.1f per slot)\n",
            jobs.size(), ksplit, nsteps_all, npieces, segs.size(), work, work / slots);
  std::vector<int32_t> tptr(tiles.size() + 1, 0), tsegs;
  for (size_t t = 0; t < tiles.size(); ++t) {
    tptr[t + 1] = tptr[t] + (int32_t)per_tile[t].size();
    for (int32_t u : per_tile[t]) tsegs.push_back(u);
  }
  c.nunits = (int)segs.size();
  c.npieces = npieces;
  c.nctas = std::min(npieces, slots);
  c.ntiles = (int)tiles.size();
  cudaStream_t st = c.stream;
  c.units = dev_alloc<int4>(segs.size(), st);
  c.cta_ptr = dev_alloc<int32_t>(pptr.size(), st);
  c.syrk_ctl = dev_zeros<unsigned>(2, st);
  c.tiles = dev_alloc<int2>(tiles.size(), st);
  c.tile_ptr = dev_alloc<int32_t>(tptr.size(), st);
  c.tile_units = dev_alloc<int32_t>(std::max<size_t>(1, tsegs.size()), st);
  c.partial = dev_alloc<double>((size_t)kTile * kTile * std::max<size_t>(1, segs.size()), st);
  c.rhs_part = dev_zeros<double>((size_t)128 * std::max<size_t>(1, segs.size()), st);
  if (!segs.empty())
    CMPC_CUDA(cudaMemcpyAsync(c.units, segs.data(), sizeof(int4) * segs.size(), cudaMemcpyHostToDevice, st));
  CMPC_CUDA(cudaMemcpyAsync(c.cta_ptr, pptr.data(), sizeof(int32_t) * pptr.size(), cudaMemcpyHostToDevice, st));
  CMPC_CUDA(cudaMemcpyAsync(c.tiles, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice, st));
  CMPC_CUDA(cudaMemcpyAsync(c.tile_ptr, tptr.data(), sizeof(int32_t) * tptr.size(), cudaMemcpyHostToDevice, st));
  if (!tsegs.empty())
    CMPC_CUDA(cudaMemcpyAsync(c.tile_units, tsegs.data(), sizeof(int32_t) * tsegs.size(), cudaMemcpyHostToDevice, st));
  dev_free(c.mk_clist, st);
  c.mk_clist = nullptr;
  std::vector<int4> cl4;
  if (c.markov) {
    cl4.reserve(clist.size());
    for (int32_t ch : clist) {
      const int2 ci = c.h_mk_chunk[size_t(ch)];
      cl4.push_back({ci.x, ci.y, ch * kBK, 0});
    }
    c.mk_clist = dev_alloc<int4>(std::max<size_t>(1, cl4.size()), st);
    if (!cl4.empty())
      CMPC_CUDA(cudaMemcpyAsync(c.mk_clist, cl4.data(), sizeof(int4) * cl4.size(), cudaMemcpyHostToDevice, st));
  }
  CMPC_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope

  // TMA descriptors over P (ldp rows x n cols, column-major) or, Markov layout, over the
  // table (ldmk rows x T nu cols: a window past the last column reads zeros), boxes
  // {16 rows, 64 | 32 cols}
  auto encode = [&](int cols) {
    auto* tm = new unsigned char[sizeof(CUtensorMap)];
    const int64_t rows = c.markov ? c.ldmk : std::max<int64_t>(c.ldp, 1);
    const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)(c.markov ? c.mk_cols : n)};
    const cuuint64_t strides[1] = {(cuuint64_t)rows * sizeof(double)};
    const cuuint32_t box[2] = {16, (cuuint32_t)cols};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(reinterpret_cast<CUtensorMap*>(tm), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                              c.markov ? (void*)c.mk : (void*)c.P, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      delete[] tm;
      throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    }
    return tm;
  };
  c.tmap_P = encode(64);
  c.tmap_P32 = encode(32);
  static std::once_flag flags[kMaxDevices];  // per device: the attributes live in its context
  once_per_device(flags, c.device, [] {
    CMPC_CUDA(cudaFuncSetAttribute(k_syrk, cudaFuncAttributeMaxDynamicSharedMemorySize, kSyrkSmem));
    // two 99 KB CTAs per SM need the largest shared-memory carveout
    CMPC_CUDA(cudaFuncSetAttribute(k_syrk, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  });
}

void launch_condense(Ctx& c, bool mirror, bool with_rhs, cudaEvent_t after_syrk) {
  with_rhs = with_rhs && c.ps > 0 && c.npieces > 0;
  SyrkArgs a;
  a.omega = c.omega;
  a.q = with_rhs ? c.q : nullptr;
  a.rhs_part = c.rhs_part;
  a.segs = c.units;
  a.piece_ptr = c.cta_ptr;
  a.npieces = c.npieces;
  a.ctl = c.syrk_ctl;
  a.partial = c.partial;
  a.prof = c.syrk_prof;
  a.static_sched = 0;
  a.clist = c.markov ? c.mk_clist : nullptr;
  if (c.npieces > 0) {
    const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(c.tmap_P);
    const CUtensorMap* tm32 = reinterpret_cast<const CUtensorMap*>(c.tmap_P32);
    k_syrk<<<c.nctas, kSyrkThreads, kSyrkSmem, c.stream>>>(*tm, *tm32, a);
    CMPC_LAUNCHED();
  }
  if (after_syrk) {  // the SYRK kernel's own time (roofline); an event node when capturing
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CMPC_CUDA(cudaStreamIsCapturing(c.stream, &cs));
    if (cs == cudaStreamCaptureStatusActive) CMPC_CUDA(cudaEventRecordWithFlags(after_syrk, c.stream, cudaEventRecordExternal));
    else CMPC_CUDA(cudaEventRecord(after_syrk, c.stream));
  }
  // sharded: every rank's partial J_g' Sigma_g J_g, H added by rank 0; the caller allreduces
  k_syrk_reduce<<<dim3(c.ntiles, kTile * kTile / 64), 64 * kRedWays, 0, c.stream>>>(
      c.partial, c.tiles, c.tile_ptr, c.tile_units, c.rank == 0 ? c.H : nullptr, c.omega + c.ldp, c.n, c.M,
      mirror ? 1 : 0, with_rhs ? c.rhs_part : nullptr, c.q + c.ldp, c.sing_ptr, c.sing_val, c.tq,
      c.rhs, with_rhs && !c.comm ? c.r1 : nullptr);
  CMPC_LAUNCHED();
}

}  // namespace cmpc
