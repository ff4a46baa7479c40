// K5-K9: the bandwidth-bound passes of one IPM iteration.
//
// Reference (proj/src/ipm.cpp): compute_residuals :46-70, step_directions :79-103,
// fraction_to_boundary :105-116, line_search + merit :118-144 / :25-32, the iterate
// update :240-243. Every J product goes through the prototype matrix P (structure.cu):
//   (J x)_r = sign_r (P x)_{proto(r)}    J' y = P' (Pi' y)
// Elementwise formulas keep the reference's separate multiply/add rounding (no FMA);
// every sum is a fixed-order two-stage reduction, every max/min an order-free atomic,
// so two runs are bitwise identical (proj/tests/test_ipm.cpp:432-457).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace cmpc {

namespace {

constexpr int kRowT = 256;
constexpr int kLaneMembers = 8;  // prototypes with more member rows take the warp path of k_proto_reduce
enum Slot { kSumAbs = 0, kSumLog = 1, kSumPsS = 2, kSlots = 16 };

// packet -> mapped host memory, then the sequence number (system-scope fence between them, so a
// host that sees the new sequence sees the packet); with reset, the accumulated maxima / minima
// start over (host loop). One warp. k_publish alone, or at the end of a segment's last kernel
// (PubArgs.out non-null: one launch less per segment)
struct PubArgs {
  Packet* out;
  unsigned long long* dev_seq;
  unsigned long long* host_seq;
  int reset;
};
__device__ __forceinline__ void publish_warp(Packet* pk, const PubArgs& pa, int lane) {
  constexpr int kWords = sizeof(Packet) / 8;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(pk);
  volatile unsigned long long* dst = reinterpret_cast<volatile unsigned long long*>(pa.out);
  for (int i = lane; i < kWords; i += 32) dst[i] = src[i];
  __threadfence_system();
  __syncwarp();
  if (lane == 0 && pa.reset) {
    pk->max_r1 = pk->max_r3 = pk->max_comp = pk->max_lam = pk->max_s = pk->max_z = 0.0;
    pk->alpha_s_min = pk->alpha_z_min = __longlong_as_double(0x7ff0000000000000ll);
    pk->any_nonpos = 0;
  }
  if (lane == 0) {
    const unsigned long long q = *pa.dev_seq + 1;
    *pa.dev_seq = q;
    *reinterpret_cast<volatile unsigned long long*>(pa.host_seq) = q;
  }
}


inline unsigned part_blocks(int64_t m) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(kPartBlocks, ceil_div(m, kRowT)));
}

// y[k] = sum_{j < hi_k} A[k + j*lda] x[j]; 32 rows x 8 column slices per block
__global__ void __launch_bounds__(256) k_rows_gemv(const double* __restrict__ A, int64_t lda,
                                                   int64_t rows, int64_t ncols,
                                                   const int32_t* __restrict__ hi,
                                                   const double* __restrict__ x, double* __restrict__ y) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = blockIdx.x * 32ll + lane;
  const int width = (r < rows) ? (hi ? hi[r] : (int)ncols) : 0;
  int wmax = width;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  double s0 = 0.0, s1 = 0.0;
  int64_t j = w;
  for (; j + 8 < wmax; j += 16) {
    const double a0 = (j < width) ? A[r + j * lda] : 0.0;
    const double a1 = (j + 8 < width) ? A[r + (j + 8) * lda] : 0.0;
    s0 += a0 * x[j];
    s1 += a1 * x[j + 8];
  }
  if (j < wmax) s0 += ((j < width) ? A[r + j * lda] : 0.0) * x[j];
  red[w][lane] = s0 + s1;
  __syncthreads();
  if (w == 0 && r < rows) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q][lane];
    y[r] = s;
  }
}

// y[k] = sum_{j < hi_k} P[k + j*ldp] x[j] for the SYRK prototypes: 64 rows per block (two
// per lane, 16-byte loads), the eight warps take interleaved column slices with four loads
// in flight each, then a fixed-order reduction of the slices. ldp is even (a multiple of
// kBK), so every row pair is 16-byte aligned. HBM-bound: P is read once.
template <int D>
__global__ void __launch_bounds__(256) k_proto_gemv(const double* __restrict__ P, int64_t ldp, int64_t rows,
                                                    const int32_t* __restrict__ hi,
                                                    const double* __restrict__ x, double* __restrict__ y,
                                                    int gblocks, const int32_t* __restrict__ sing_col,
                                                    const double* __restrict__ sing_val, int64_t pz,
                                                    double* __restrict__ ys) {
  __shared__ double2 red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if ((int)blockIdx.x >= gblocks) {  // the singleton prototypes: y_k = a_k x[col_k]
    const int64_t k = ((int64_t)blockIdx.x - gblocks) * 256 + threadIdx.x;
    if (k < pz) ys[k] = sing_val[k] * x[sing_col[k]];
    return;
  }
  // widest rows first (rows are sorted by width): the heavy blocks start in the first wave
  const int64_t r = (int64_t)(gblocks - 1 - blockIdx.x) * 64 + 2 * lane;
  const int w0 = r < rows ? hi[r] : 0, w1 = r + 1 < rows ? hi[r + 1] : 0;
  int wmax = max(w0, w1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  const double2* col = reinterpret_cast<const double2*>(P + r);
  const int64_t ld2 = ldp / 2;
  int j = w;
  for (; j + 8 * (D - 1) < wmax; j += 8 * D) {
    double2 v[D];
    double xv[D];
#pragma unroll
    for (int u = 0; u < D; ++u) {
      v[u] = r < rows ? __ldcs(col + (j + 8 * u) * ld2) : make_double2(0.0, 0.0);
      xv[u] = x[j + 8 * u];
    }
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int jj = j + 8 * u;
      const double p0 = jj < w0 ? v[u].x : 0.0, p1 = jj < w1 ? v[u].y : 0.0;
      if (u & 1) {
        b0 += p0 * xv[u];
        b1 += p1 * xv[u];
      } else {
        a0 += p0 * xv[u];
        a1 += p1 * xv[u];
      }
    }
  }
  for (; j < wmax; j += 8) {
    const double2 v = r < rows ? __ldcs(col + j * ld2) : make_double2(0.0, 0.0);
    a0 += (j < w0 ? v.x : 0.0) * x[j];
    a1 += (j < w1 ? v.y : 0.0) * x[j];
  }
  red[w][lane] = make_double2(a0 + b0, a1 + b1);
  __syncthreads();
  if (w == 0 && r < rows) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s0 += red[q][lane].x;
      s1 += red[q][lane].y;
    }
    y[r] = s0;
    if (r + 1 < rows) y[r + 1] = s1;
  }
}

// J' p_lambda without a pass over J (J'lambda carried along). With
// p_lambda = -w + sigma o (J pv) (w = r2 - sigma r3),
//     J' p_lambda = (J' Sigma J) pv - J' w = (M - H) pv - tq,
// M the condensed matrix of this step (lower triangle, k_syrk_reduce) and tq = J' w its fused
// right-hand side part. (M - H) pv has the rounding of the direct P'(omega o P pv) in the
// worst case (both are bounded by eps |P|' Omega |P| |pv|). One warp per output i: lanes
// stride j, the lower-triangle element of (i, j) is read from M and H alike.
__device__ __forceinline__ void jtpl_symv_body(int64_t blk, const double* __restrict__ M,
                                               const double* __restrict__ H, int64_t n,
                                               const double* __restrict__ pv, const double* __restrict__ tq,
                                               double* __restrict__ out) {
  // a CTA owns 32 outputs i0 .. i0 + 31. Part A (j <= i: row i of the lower triangle): lane =
  // output, the 32 warps stride j, so each load is 32 consecutive rows of one column. Part B
  // (j > i: column i below the diagonal): warp w takes output i0 + w, lanes stride j along
  // the column. Loads four at a time; the pieces are added in a fixed order.
  __shared__ double ra[32][33], rb[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i0 = blk * 32, ia = i0 + lane, ib = i0 + w;
  double sa = 0.0, sb = 0.0;
  if (ia < n) {
    int64_t j = w;
    for (; j + 96 <= ia; j += 128) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = ia + (j + 32 * u) * n;
        x[u] = sub(M[e], H[e]) * pv[j + 32 * u];
      }
      sa += (x[0] + x[1]) + (x[2] + x[3]);
    }
    for (; j <= ia; j += 32) {
      const int64_t e = ia + j * n;
      sa += sub(M[e], H[e]) * pv[j];
    }
  }
  if (ib < n) {
    int64_t j = ib + 1 + lane;
    for (; j + 96 < n; j += 128) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = j + 32 * u + ib * n;
        x[u] = sub(M[e], H[e]) * pv[j + 32 * u];
      }
      sb += (x[0] + x[1]) + (x[2] + x[3]);
    }
    for (; j < n; j += 32) {
      const int64_t e = j + ib * n;
      sb += sub(M[e], H[e]) * pv[j];
    }
  }
  ra[w][lane] = sa;
  sb = warp_sum(sb);
  if (lane == 0) rb[w] = sb;
  __syncthreads();
  if (w != 0 || ia >= n) return;
  double s = 0.0;
#pragma unroll 8
  for (int q = 0; q < 32; ++q) s += ra[q][lane];
  out[ia] = sub(s + rb[lane], tq[ia]);
}

__global__ void __launch_bounds__(1024) k_jtpl_symv(const double* __restrict__ M, const double* __restrict__ H,
                                                    int64_t n, const double* __restrict__ pv,
                                                    const double* __restrict__ tq, double* __restrict__ out) {
  jtpl_symv_body(blockIdx.x, M, H, n, pv, tq, out);
}

__global__ void k_sing_x(const int32_t* __restrict__ col, const double* __restrict__ val, int64_t pz,
                         const double* __restrict__ x, double* __restrict__ y) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < pz) y[k] = val[k] * x[col[k]];
}

__device__ __forceinline__ double jrow(const double* y, int32_t rm) {
  const double v = y[rm >> 1];
  return (rm & 1) ? -v : v;
}

// out[j] partial over a chunk of rc P rows: colpart[chunk*n + j]; one warp per (chunk,
// column), 16-byte loads (two rows per lane) with four in flight. Column j's nonzeros are
// the rows >= start_col[j]; the pair containing start_col[j] is read whole and masked.
template <int MINB, int D>
__global__ void __launch_bounds__(256, MINB) k_ptq_partial(const double* __restrict__ P, int64_t ldp,
                                                     int64_t ps, int64_t n,
                                                     const int32_t* __restrict__ start_col,
                                                     const double* __restrict__ q, int rc,
                                                     double* __restrict__ colpart) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = blockIdx.y * 8ll + w;
  if (j >= n) return;
  const int64_t k0 = (int64_t)blockIdx.x * rc, k1 = (ps < k0 + rc ? ps : k0 + rc);
  const int64_t kb = (k0 > (int64_t)start_col[j] ? k0 : (int64_t)start_col[j]);
  const int64_t ka = kb & ~int64_t(1);
  const double* col = P + j * ldp;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t k = ka + 2 * lane;
  for (; k + 64 * (D - 1) < k1; k += 64 * D) {
    double2 v[D], qq[D];
#pragma unroll
    for (int u = 0; u < D; ++u) {
      v[u] = __ldcs(reinterpret_cast<const double2*>(col + k + 64 * u));
      qq[u] = *reinterpret_cast<const double2*>(q + k + 64 * u);
    }
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int64_t kk = k + 64 * u;
      const double e0 = kk >= kb ? v[u].x * qq[u].x : 0.0;
      const double e1 = (kk + 1 >= kb && kk + 1 < k1) ? v[u].y * qq[u].y : 0.0;
      if (u & 1) {
        s2 += e0;
        s3 += e1;
      } else {
        s0 += e0;
        s1 += e1;
      }
    }
  }
  for (; k < k1; k += 64) {
    const double2 v = __ldcs(reinterpret_cast<const double2*>(col + k));
    const double2 qq = *reinterpret_cast<const double2*>(q + k);
    if (k >= kb) s0 += v.x * qq.x;
    if (k + 1 >= kb && k + 1 < k1) s1 += v.y * qq.y;
  }
  const double s = warp_sum((s0 + s1) + (s2 + s3));
  if (lane == 0) colpart[blockIdx.x * n + j] = s;
}

// out[j] = sum_chunks colpart + singleton scatter (singletons sorted by column); one warp
// per column, lanes stride the chunks, fixed-order warp sum
__global__ void __launch_bounds__(256) k_ptq_final(const double* __restrict__ colpart, int nchunks, int64_t n,
                                                   const int32_t* __restrict__ sing_ptr,
                                                   const double* __restrict__ sing_val,
                                                   const double* __restrict__ qs, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x * 8ll + (threadIdx.x >> 5);
  if (j >= n) return;
  double s = 0.0;
  for (int c = lane; c < nchunks; c += 32) s += colpart[(int64_t)c * n + j];
  s = warp_sum(s);
  if (lane == 0) {
    for (int32_t k = sing_ptr[j]; k < sing_ptr[j + 1]; ++k) s += sing_val[k] * qs[k];
    out[j] = s;
  }
}

// ---------------------------------------------------------------- residuals
__global__ void __launch_bounds__(kRowT) k_res_rows(int64_t m, const int32_t* __restrict__ row_map,
                                                    const double* __restrict__ y,
                                                    const double* __restrict__ d,
                                                    const double* __restrict__ s,
                                                    const double* __restrict__ lam,
                                                    const double* __restrict__ z,
                                                    const double* __restrict__ mu_p,
                                                    double* __restrict__ r2, double* __restrict__ r3,
                                                    double* __restrict__ part, Packet* pk,
                                                    const double* __restrict__ gate) {
  __shared__ double sh[7 * 32];
  if (gate && gate[2] == 0.0) return;  // (speculative segment whose step was not taken)
  const double mu = *mu_p;
  double sabs = 0.0, slog = 0.0, ml = 0.0, mss = 0.0, mz = 0.0, mr3 = 0.0, mc = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double jv = jrow(y, row_map[r]);
    const double sr = s[r], lr = lam[r], zr = z[r];
    r2[r] = sub(lr, mul(mu, dv(1.0, sr)));
    const double t3 = add(sub(jv, d[r]), sr);
    r3[r] = t3;
    sabs += fabs(t3);
    slog += log(sr);
    ml = fmax(ml, fabs(lr));
    mss = fmax(mss, fabs(sr));
    mz = fmax(mz, fabs(zr));
    mr3 = fmax(mr3, fabs(t3));
    mc = fmax(mc, fabs(sub(mul(sr, zr), mu)));
  }
  double su[2] = {sabs, slog}, mx[5] = {ml, mss, mz, mr3, mc};
  block_sums_maxs<kRowT>(su, mx, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * kSlots + kSumAbs] = su[0];
    part[blockIdx.x * kSlots + kSumLog] = su[1];
    atomic_max_nonneg(&pk->max_lam, mx[0]);
    atomic_max_nonneg(&pk->max_s, mx[1]);
    atomic_max_nonneg(&pk->max_z, mx[2]);
    atomic_max_nonneg(&pk->max_r3, mx[3]);
    atomic_max_nonneg(&pk->max_comp, mx[4]);
  }
}

// r2 and complementarity at a new barrier value (r1, r3 unchanged)
__global__ void __launch_bounds__(kRowT) k_mu_rows(int64_t m, const double* __restrict__ s,
                                                   const double* __restrict__ lam,
                                                   const double* __restrict__ z,
                                                   const double* __restrict__ mu_p,
                                                   double* __restrict__ r2, Packet* pk) {
  const double mu = *mu_p;
  double mc = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double sr = s[r];
    r2[r] = sub(lam[r], mul(mu, dv(1.0, sr)));
    mc = fmax(mc, fabs(sub(mul(sr, z[r]), mu)));
  }
  mc = warp_max(mc);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(&pk->max_comp, mc);
}

// Per prototype k (rows of J that equal +-P_k): out1[k] = sum of x1 over the member rows
// (signed when SIGNED1), out2[k] = signed sum of x2; members in ascending row order.
// One lane per prototype, members in fixed (ascending) order; the all-zero row group
// (if any) contributes nothing and is skipped.
// SIGMA: the member values are formed here from the rows' state (k_sigma_rows folded in):
// x1 = sigma = z / s (also stored per row), x2 = w = r2 - sigma r3; the zero prototype's rows
// get their sigma from the extra CTAs after the warp path (they add nothing to the sums).
struct SigmaRows {
  const double *s, *z, *r2, *r3;
  double* sigma;
  int zero_blocks;
  int big_blocks;
};

template <bool SIGMA>
__device__ __forceinline__ void member_values(const SigmaRows& sr, const double* x1, const double* x2, int32_t r,
                                              double& a, double& b) {
  if (SIGMA) {
    const double sg = dv(sr.z[r], sr.s[r]);
    sr.sigma[r] = sg;
    a = sg;
    b = sub(sr.r2[r], mul(sg, sr.r3[r]));
  } else {
    a = x1[r];
    b = x2 ? x2[r] : 0.0;
  }
}

template <bool SIGNED1, bool HAS2, bool SIGMA = false>
__global__ void __launch_bounds__(256) k_proto_reduce(int64_t p, const int32_t* __restrict__ mem_ptr,
                                                      const int32_t* __restrict__ mem_rows,
                                                      const double* __restrict__ x1,
                                                      const double* __restrict__ x2,
                                                      double* __restrict__ out1,
                                                      double* __restrict__ out2, int64_t ps,
                                                      int64_t ldp, int64_t zero_k,
                                                      const int32_t* __restrict__ big, int nbig,
                                                      int lane_blocks, SigmaRows sr) {
  const int lane = threadIdx.x & 31;
  if (SIGMA && (int)blockIdx.x >= lane_blocks + sr.big_blocks) {  // the zero prototype's rows
    const int64_t e = (int64_t)mem_ptr[zero_k] + ((int64_t)blockIdx.x - lane_blocks - sr.big_blocks) * 256 + threadIdx.x;
    if (e < mem_ptr[zero_k + 1]) {
      const int32_t r = mem_rows[e] >> 1;
      sr.sigma[r] = dv(sr.z[r], sr.s[r]);
    }
    return;
  }
  if ((int)blockIdx.x >= lane_blocks) {
    // a prototype with more than kLaneMembers members: one warp, lanes stride the members
    // (ascending per lane), fixed butterfly sum across the lanes
    const int wi = ((int)blockIdx.x - lane_blocks) * 8 + (threadIdx.x >> 5);
    if (wi >= nbig) return;
    const int64_t k = big[wi];
    const int32_t b0 = mem_ptr[k], b1 = mem_ptr[k + 1];
    double s1 = 0.0, s2 = 0.0;
    for (int32_t e = b0 + lane; e < b1; e += 32) {
      const int32_t rm = mem_rows[e];
      const int32_t r = rm >> 1;
      double a, bb;
      member_values<SIGMA>(sr, x1, HAS2 ? x2 : nullptr, r, a, bb);
      s1 += (SIGNED1 && (rm & 1)) ? -a : a;
      if (HAS2) s2 += (rm & 1) ? -bb : bb;
    }
    s1 = warp_sum(s1);
    if (HAS2) s2 = warp_sum(s2);
    if (lane == 0) {
      const int64_t o = k < ps ? k : ldp + (k - ps);
      out1[o] = s1;
      if (HAS2) out2[o] = s2;
    }
    return;
  }
  const int64_t base = (blockIdx.x * 8ll + (threadIdx.x >> 5)) * 32;
  const int64_t k = base + lane;
  int32_t b0 = 0, b1 = 0;
  if (k < p && k != zero_k) {
    b0 = mem_ptr[k];
    b1 = mem_ptr[k + 1];
  }
  if (b1 - b0 > kLaneMembers) return;  // the warp path above owns it
  // every lane sums its own prototype: member loads are independent, so they are issued
  // together ahead of the (ordered) accumulation
  double s1 = 0.0, s2 = 0.0;
  {
    double v1[kLaneMembers], v2[kLaneMembers];
#pragma unroll
    for (int u = 0; u < kLaneMembers; ++u) {
      v1[u] = 0.0;
      v2[u] = 0.0;
      if (b0 + u < b1) {
        const int32_t rm = mem_rows[b0 + u];
        const int32_t r = rm >> 1;
        double a, bb;
        member_values<SIGMA>(sr, x1, HAS2 ? x2 : nullptr, r, a, bb);
        v1[u] = (SIGNED1 && (rm & 1)) ? -a : a;
        if (HAS2) v2[u] = (rm & 1) ? -bb : bb;
      }
    }
#pragma unroll
    for (int u = 0; u < kLaneMembers; ++u) {
      if (b0 + u < b1) {
        s1 += v1[u];
        if (HAS2) s2 += v2[u];
      }
    }
  }
  if (k < p) {
    const int64_t o = k < ps ? k : ldp + (k - ps);
    out1[o] = s1;
    if (HAS2) out2[o] = s2;
  }
}

constexpr int kFinT = 1024;

// finalize packet A: r1 = (Hv + h) + J'lambda, max|r1|, kkt, dots for objective and merit.
// mode 0: everything; 1: only this context's row sums into the packet (sharded: they are
// allreduced next); 2: everything, with the (allreduced) row sums taken from the packet.
// m_all = rows of the whole QP (the kkt scaling), nparts = 0 when this context has no rows.
__global__ void __launch_bounds__(kFinT) k_res_final(int64_t n, int64_t m_all, int nparts,
                                                     const double* __restrict__ Hv,
                                                     const double* __restrict__ h,
                                                     const double* __restrict__ Jtl,
                                                     const double* __restrict__ v,
                                                     double* __restrict__ r1,
                                                     const double* __restrict__ part,
                                                     const double* __restrict__ hmax, Packet* pk,
                                                     int mode, const double* __restrict__ gate,
                                                     double* __restrict__ snap, PubArgs pub) {
  __shared__ double sh[5 * 32];
  if (gate && gate[2] == 0.0) {  // (a refused speculative step: nothing but the publish)
    if (pub.out && threadIdx.x < 32) publish_warp(pk, pub, threadIdx.x);
    return;
  }
  double sabs = 0.0, slog = 0.0;
  if (mode != 2)
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
      sabs += part[b * kSlots + kSumAbs];
      slog += part[b * kSlots + kSumLog];
    }
  double mr1 = 0.0, vhv = 0.0, hv = 0.0;
  if (mode != 1)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double g = add(Hv[i], h[i]);
      const double r = m_all > 0 ? add(g, Jtl[i]) : g;
      r1[i] = r;
      mr1 = fmax(mr1, fabs(r));
      vhv += v[i] * Hv[i];
      hv += h[i] * v[i];
    }
  double su[4] = {sabs, slog, vhv, hv}, mx[1] = {mr1};
  block_sums_maxs<kFinT>(su, mx, sh);
  sabs = su[0];
  slog = su[1];
  vhv = su[2];
  hv = su[3];
  if (mode == 1) {
    if (threadIdx.x == 0) {
      pk->sum_abs_r3 = sabs;
      pk->sum_log_s = slog;
    }
    return;
  }
  if (threadIdx.x == 0) {
    if (mode == 2) {
      sabs = pk->sum_abs_r3;
      slog = pk->sum_log_s;
    }
    pk->max_r1 = mx[0];
    pk->obj_vHv = vhv;
    pk->obj_hv = hv;
    pk->sum_abs_r3 = m_all > 0 ? sabs : 0.0;
    pk->sum_log_s = m_all > 0 ? slog : 0.0;
    pk->max_h = *hmax;
    pk->objective = 0.5 * vhv + hv + hmax[1];  // h0 on the device: graphs outlive an h0 change
    const double ds = fmax(1.0, fmax(*hmax, pk->max_lam) / (double)(n + m_all));
    double kkt = mx[0] / ds;
    if (m_all > 0) {
      const double cs = fmax(1.0, fmax(pk->max_s, pk->max_z) / (double)(2 * m_all));
      kkt = fmax(kkt, pk->max_r3);
      kkt = fmax(kkt, pk->max_comp / cs);
    }
    pk->kkt = kkt;
    if (snap) {  // the merit pieces of this point for trial0_decide
      snap[0] = pk->max_lam;
      snap[1] = vhv;
      snap[2] = hv;
      snap[3] = pk->sum_log_s;
      snap[4] = pk->sum_abs_r3;
    }
  }
  if (pub.out) {  // the segment's publish
    __syncthreads();
    if (threadIdx.x < 32) publish_warp(pk, pub, threadIdx.x);
  }
}

// kkt after a barrier change: the residual maxima of the current point come in as arguments
// (the host loop's packet A: k_publish has reset the device packet's accumulators since) and
// are written back, so the packet is whole again; only max_comp was recomputed at the new mu
__global__ void k_kkt_only(int64_t n, int64_t m, const double* __restrict__ hmax, Packet* pk,
                           double max_r1, double max_r3, double max_lam, double max_s, double max_z) {
  pk->max_r1 = max_r1;
  pk->max_r3 = max_r3;
  pk->max_lam = max_lam;
  pk->max_s = max_s;
  pk->max_z = max_z;
  const double ds = fmax(1.0, fmax(*hmax, pk->max_lam) / (double)(n + m));
  double kkt = pk->max_r1 / ds;
  if (m > 0) {
    const double cs = fmax(1.0, fmax(pk->max_s, pk->max_z) / (double)(2 * m));
    kkt = fmax(kkt, pk->max_r3);
    kkt = fmax(kkt, pk->max_comp / cs);
  }
  pk->kkt = kkt;
}

__global__ void k_absmax(const double* __restrict__ x, int64_t n, double* out) {
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a = fmax(a, fabs(x[i]));
  a = warp_max(a);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, a);
}

// ---------------------------------------------------------------- step
// sigma = z/s, w = r2 - sigma r3
__global__ void k_sigma_rows(int64_t m, const double* __restrict__ s, const double* __restrict__ z,
                             const double* __restrict__ r2, const double* __restrict__ r3,
                             const double* __restrict__ sig_in, double* __restrict__ sigma,
                             double* __restrict__ w) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const double sg = sig_in ? sig_in[r] : dv(z[r], s[r]);
  sigma[r] = sg;
  if (w) w[r] = sub(r2[r], mul(sg, r3[r]));
}

__global__ void k_rhs(int64_t n, const double* __restrict__ r1, const double* __restrict__ t,
                      int64_t m, double* __restrict__ rhs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  rhs[i] = m > 0 ? add(-r1[i], t[i]) : -r1[i];
}

// ps, plambda, pz, fraction-to-boundary minima, sum ps/s
__global__ void __launch_bounds__(kRowT) k_recover_rows(
    int64_t m, const int32_t* __restrict__ row_map, const double* __restrict__ y,
    const double* __restrict__ s, const double* __restrict__ z, const double* __restrict__ sigma,
    const double* __restrict__ r2, const double* __restrict__ r3, const double* __restrict__ mu_p,
    double tau, double* __restrict__ Jpv, double* __restrict__ ps, double* __restrict__ pl,
    double* __restrict__ pz, double* __restrict__ part, Packet* pk) {
  __shared__ double sh[3 * 32];
  const double mu = *mu_p;
  double q = 0.0, as = 1e308, az = 1e308;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double jp = jrow(y, row_map[r]);
    const double sr = s[r], zr = z[r], sg = sigma[r], t3 = r3[r];
    Jpv[r] = jp;
    const double p_s = sub(-t3, jp);
    const double p_l = add(-r2[r], mul(sg, add(t3, jp)));
    const double p_z = sub(sub(mul(mu, dv(1.0, sr)), zr), mul(sg, p_s));
    ps[r] = p_s;
    pl[r] = p_l;
    pz[r] = p_z;
    q += dv(p_s, sr);
    if (p_s < 0.0) as = fmin(as, mul(tau, dv(-sr, p_s)));
    if (p_z < 0.0) az = fmin(az, mul(tau, dv(-zr, p_z)));
  }
  double su[1] = {q}, mx[2] = {-as, -az};  // minima as maxima of the negations (exact)
  block_sums_maxs<kRowT>(su, mx, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * kSlots + kSumPsS] = su[0];
    as = -mx[0];
    az = -mx[1];
    if (as < 1e308) atomic_min_nonneg(&pk->alpha_s_min, as);
    if (az < 1e308) atomic_min_nonneg(&pk->alpha_z_min, az);
  }
}

__global__ void __launch_bounds__(kFinT) k_recover_final(int64_t n, int nparts,
                                                         const double* __restrict__ Hv,
                                                         const double* __restrict__ h,
                                                         const double* __restrict__ pv,
                                                         const double* __restrict__ part, Packet* pk) {
  __shared__ double sh[32];
  double g = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) g += add(Hv[i], h[i]) * pv[i];
  g = block_sum<kFinT>(g, sh);
  __syncthreads();
  double q = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) q += part[b * kSlots + kSumPsS];
  q = block_sum<kFinT>(q, sh);
  if (threadIdx.x == 0) {
    pk->d_gpv = g;
    pk->d_ps_s = q;
  }
}

__global__ void __launch_bounds__(kRowT) k_pss_rows(int64_t m, const double* __restrict__ s,
                                                    const double* __restrict__ ps,
                                                    double* __restrict__ part) {
  __shared__ double sh[32];
  double q = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x)
    q += dv(ps[r], s[r]);
  const double t = block_sum<kRowT>(q, sh);
  if (threadIdx.x == 0) part[blockIdx.x * kSlots + kSumPsS] = t;
}

__global__ void k_init_state(int64_t m, const double* __restrict__ d, double mu,
                             double* __restrict__ s, double* __restrict__ lam,
                             double* __restrict__ z) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const double sr = fmax(1.0, d[r]);
  const double zr = mul(mu, dv(1.0, sr));
  s[r] = sr;
  z[r] = zr;
  lam[r] = zr;
}

// ---------------------------------------------------------------- line-search trial
// trial step length: host value, or alpha_max = min(1, tau-ratio minimum) from the device
__device__ __forceinline__ double trial_alpha(double a, const Packet* pk) {
  return pk ? fmin(1.0, pk->alpha_s_min) : a;
}

__global__ void k_axpy_n(int64_t n, const double* __restrict__ x, double a, const Packet* apk,
                         const double* __restrict__ p, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double al = trial_alpha(a, apk);
  if (i < n) out[i] = add(x[i], mul(al, p[i]));
}

// J v_t rows: from yt = P v_t (exact pass), or, when yt is null, from the prototype values of
// the current point and the direction, yv + alpha y (J is linear; the accepted trial's
// values are carried into yv by k_update with the same rounding, so no P pass is needed)
__global__ void __launch_bounds__(kRowT) k_trial_rows(int64_t m, const int32_t* __restrict__ row_map,
                                                      const double* __restrict__ yt,
                                                      const double* __restrict__ yv,
                                                      const double* __restrict__ y,
                                                      const double* __restrict__ d,
                                                      const double* __restrict__ s,
                                                      const double* __restrict__ ps, double alpha_h,
                                                      const Packet* apk, double* __restrict__ part,
                                                      Packet* pk) {
  __shared__ double sh[32];
  double sabs = 0.0, slog = 0.0;
  const double alpha = trial_alpha(alpha_h, apk);
  int bad = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double st = add(s[r], mul(alpha, ps[r]));
    if (st <= 0.0) bad = 1;
    slog += log(st);
    const int32_t rm = row_map[r];
    double jv;
    if (yt) {
      jv = jrow(yt, rm);
    } else {
      const double u = add(yv[rm >> 1], mul(alpha, y[rm >> 1]));
      jv = (rm & 1) ? -u : u;
    }
    sabs += fabs(add(sub(jv, d[r]), st));
  }
  double t = block_sum<kRowT>(sabs, sh);
  if (threadIdx.x == 0) part[blockIdx.x * kSlots + kSumAbs] = t;
  t = block_sum<kRowT>(slog, sh);
  if (threadIdx.x == 0) part[blockIdx.x * kSlots + kSumLog] = t;
  if (__syncthreads_or(bad) && threadIdx.x == 0) pk->any_nonpos = 1;
}

// speculative acceptance of trial 0 (host loop, seg_step): the first pass of the reference's
// accept loop (ipm.cpp:129-143) exactly as run_line_search evaluates it on the host, same
// operations in the same order, from the step packet and the residual snapshot dec[3..7]
// that k_res_final left ({max_lam, v'Hv, h'v, sum log s, sum |r3|} of the current point).
// Writes dec = {alpha, alpha_z, go}: with go != 0 the update + residual segment the host
// enqueued behind this one applies the step; with go = 0 it does nothing and the host runs
// the rest of the line search (or the shift ladder) and sets go itself (set_alpha).
__device__ void trial0_decide(Packet* pk, bool rows, double mu, double eta, double* dec) {
  const double alpha = fmin(1.0, pk->alpha_s_min), alpha_z = fmin(1.0, pk->alpha_z_min);
  int go = 0;
  if (pk->info == 0 && !(rows && pk->any_nonpos)) {
    const double rho = add(mul(10.0, dec[3]), 1.0);
    double phi0 = add(mul(0.5, dec[4]), dec[5]);
    double derivative = pk->d_gpv;
    double phi = add(mul(0.5, pk->t_vHv), pk->t_hv);
    if (rows) {
      phi0 = sub(phi0, mul(mu, dec[6]));
      phi0 = add(phi0, mul(rho, dec[7]));
      derivative = sub(derivative, mul(mu, pk->d_ps_s));
      derivative = sub(derivative, mul(rho, dec[7]));
      phi = sub(phi, mul(mu, pk->t_sum_log));
      phi = add(phi, mul(rho, pk->t_sum_abs));
    }
    constexpr double band = 10.0 * 2.220446049250313080847e-16;  // 10 DBL_EPSILON
    if (derivative <= 0.0 && phi <= add(phi0, mul(mul(eta, alpha), derivative)))
      go = 1;
    else if (fabs(sub(phi, phi0)) <= mul(band, add(1.0, fabs(phi0))))
      go = 1;
  }
  dec[0] = alpha;
  dec[1] = alpha_z;
  dec[2] = go ? 1.0 : 0.0;
  pk->pad[6] = go ? 1.0 : 0.0;
}

__global__ void __launch_bounds__(kFinT) k_trial_final(int64_t n, int64_t m, int nparts,
                                                       const double* __restrict__ vt,
                                                       const double* __restrict__ Hvt,
                                                       const double* __restrict__ h,
                                                       const double* __restrict__ part, Packet* pk,
                                                       const double* __restrict__ mu_p,
                                                       double* dec, double eta, PubArgs pub) {
  __shared__ double sh[5 * 32];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    a += vt[i] * Hvt[i];
    b += h[i] * vt[i];
  }
  double sabs = 0.0, slog = 0.0;
  for (int q = threadIdx.x; q < nparts; q += blockDim.x) {
    sabs += part[q * kSlots + kSumAbs];
    slog += part[q * kSlots + kSumLog];
  }
  double su[4] = {a, b, sabs, slog}, dummy[1] = {0.0};
  block_sums_maxs<kFinT>(su, dummy, sh);
  if (threadIdx.x == 0) {
    pk->t_vHv = su[0];
    pk->t_hv = su[1];
    pk->t_sum_abs = m > 0 ? su[2] : 0.0;
    pk->t_sum_log = m > 0 ? su[3] : 0.0;
    if (dec) trial0_decide(pk, m > 0, *mu_p, eta, dec);
  }
  if (pub.out) {  // the segment's publish
    __syncthreads();
    if (threadIdx.x < 32) publish_warp(pk, pub, threadIdx.x);
  }
}

__global__ void k_update(int64_t n, int64_t m, const double* __restrict__ ap, double* __restrict__ v,
                         const double* __restrict__ pv, double* __restrict__ s,
                         const double* __restrict__ ps, double* __restrict__ lam,
                         const double* __restrict__ pl, double* __restrict__ z,
                         const double* __restrict__ pz, int64_t py, double* __restrict__ yv,
                         const double* __restrict__ y, double* __restrict__ Jtl,
                         const double* __restrict__ JtPl, double* __restrict__ Hv,
                         const double* __restrict__ Hvt) {
  if (ap[2] == 0.0) return;  // trial 0 not accepted: the host finishes the line search first
  const double alpha = ap[0], alpha_z = ap[1];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = add(v[i], mul(alpha, pv[i]));
  // H v of the new point: the accepted (= last) trial's H v_t, same kernel and inputs, bit for
  // bit (a residual pass that recomputes H v overwrites it)
  if (i < n) Hv[i] = Hvt[i];
  if (Jtl && i < n) Jtl[i] = add(Jtl[i], mul(alpha, JtPl[i]));  // J'(lambda + alpha p_lambda)
  if (i < py) yv[i] = add(yv[i], mul(alpha, y[i]));  // P v of the new point (see k_trial_rows)
  if (i < m) {
    s[i] = add(s[i], mul(alpha, ps[i]));
    lam[i] = add(lam[i], mul(alpha, pl[i]));
    z[i] = add(z[i], mul(alpha_z, pz[i]));
  }
}

// stand-alone fraction_to_boundary minima (out[0..1] pre-set to +inf)
__global__ void k_ftb(int64_t m, const double* __restrict__ s, const double* __restrict__ ps,
                      const double* __restrict__ z, const double* __restrict__ pz, double tau,
                      double* out) {
  double as = 1e308, az = 1e308;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (ps[r] < 0.0) as = fmin(as, mul(tau, dv(-s[r], ps[r])));
    if (pz[r] < 0.0) az = fmin(az, mul(tau, dv(-z[r], pz[r])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    as = fmin(as, __shfl_xor_sync(0xffffffffu, as, o));
    az = fmin(az, __shfl_xor_sync(0xffffffffu, az, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (as < 1e308) atomic_min_nonneg(&out[0], as);
    if (az < 1e308) atomic_min_nonneg(&out[1], az);
  }
}

__global__ void k_reset_packet(Packet* pk, int which) {
  if (which == 0) {  // residual maxima
    pk->max_r1 = pk->max_r3 = pk->max_comp = pk->max_lam = pk->max_s = pk->max_z = 0.0;
  } else if (which == 1) {  // recovery minima
    pk->alpha_s_min = __longlong_as_double(0x7ff0000000000000ll);
    pk->alpha_z_min = __longlong_as_double(0x7ff0000000000000ll);
  } else if (which == 2) {
    pk->any_nonpos = 0;
  } else if (which == 3) {
    pk->max_comp = 0.0;
  }
}



// sing_ptr[j] = first singleton prototype with column >= j (singletons sorted by column)
__global__ void k_sing_ptr(const int32_t* __restrict__ sing_col, int64_t pz, int64_t n,
                           int32_t* __restrict__ ptr) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j > n) return;
  int64_t lo = 0, hi = pz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (sing_col[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  ptr[j] = (int32_t)lo;
}

// any H(i, j) != H(j, i) -> *bad = 1 (once per load: picks the column-dot form of H x)
__global__ void k_sym_check(const double* __restrict__ H, int64_t n, unsigned* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    if (i > j && H[i + j * n] != H[j + i * n]) atomicOr(bad, 1u);
  }
}

// y = H x for a symmetric H as column dots (H' x): one warp per column, contiguous 16-byte
// loads when n is even, fixed-order warp sum
// x = v + alpha p when v is given (the line-search trial point, k_axpy_n's rounding; warp j
// also stores x_j), else x as passed
__device__ __forceinline__ void hcol_body(int64_t j, const double* __restrict__ H, int64_t n,
                                          const double* __restrict__ x, double* __restrict__ y,
                                          const double* __restrict__ v, const double* __restrict__ p,
                                          double alpha_h, const Packet* apk, double* __restrict__ xt) {
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double al = v ? trial_alpha(alpha_h, apk) : 0.0;
  const double* col = H + j * n;
  double s0 = 0.0, s1 = 0.0;
  if ((n & 1) == 0) {
    const double2* c2 = reinterpret_cast<const double2*>(col);
    const double2* x2 = reinterpret_cast<const double2*>(v ? v : x);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    for (int64_t i = lane; i < n / 2; i += 32) {
      const double2 a = c2[i];
      double2 b = x2[i];
      if (v) {
        const double2 q = p2[i];
        b.x = add(b.x, mul(al, q.x));
        b.y = add(b.y, mul(al, q.y));
      }
      s0 = fma(a.x, b.x, s0);
      s1 = fma(a.y, b.y, s1);
    }
  } else {
    for (int64_t i = lane; i < n; i += 32) {
      const double b = v ? add(v[i], mul(al, p[i])) : x[i];
      s0 = fma(col[i], b, s0);
    }
  }
  const double s = warp_sum(s0 + s1);
  if (lane == 0) {
    y[j] = s;
    if (v) xt[j] = add(v[j], mul(al, p[j]));
  }
}

__global__ void __launch_bounds__(256) k_hcol_gemv(const double* __restrict__ H, int64_t n,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   const double* __restrict__ v, const double* __restrict__ p,
                                                   double alpha_h, const Packet* apk, double* __restrict__ xt) {
  hcol_body(blockIdx.x * 8ll + (threadIdx.x >> 5), H, n, x, y, v, p, alpha_h, apk, xt);
}

// the trial's H v_t (CTAs below hblocks, a warp per column) and, beside it, J' p_lambda
// (k_jtpl_symv's CTAs; JtPl null: none) in one launch
__global__ void __launch_bounds__(1024) k_trial_hv(const double* __restrict__ H, int64_t n,
                                                   double* __restrict__ Hvt, const double* __restrict__ v,
                                                   const double* __restrict__ pv, double alpha_h,
                                                   const Packet* apk, double* __restrict__ vt, int hblocks,
                                                   const double* __restrict__ M, const double* __restrict__ tq,
                                                   double* __restrict__ JtPl) {
  if ((int)blockIdx.x < hblocks) {
    hcol_body(blockIdx.x * 32ll + (threadIdx.x >> 5), H, n, nullptr, Hvt, v, pv, alpha_h, apk, vt);
    return;
  }
  jtpl_symv_body((int64_t)blockIdx.x - hblocks, M, H, n, pv, tq, JtPl);
}

}  // namespace

// Mapped pinned blocks (packet, sequence word, 64-double staging ring) are recycled across
// loads and contexts: cudaHostAlloc costs milliseconds, a load should not.
namespace {
// [packet A][sequence word][packet B (seg_step's publish)][staging ring]
constexpr size_t kPkBOff = (sizeof(Packet) + 64 + 127) / 128 * 128;
constexpr size_t kStageOff = (kPkBOff + sizeof(Packet) + 127) / 128 * 128;
constexpr size_t kPinnedBytes = kStageOff + 128 * sizeof(double);
std::mutex g_pinned_mu;
std::vector<void*> g_pinned_free;

void* pinned_take() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      void* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  CMPC_CUDA(cudaHostAlloc(&p, kPinnedBytes, cudaHostAllocMapped | cudaHostAllocPortable));
  return p;
}

void pinned_give(void* p) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}
}  // namespace

// column j of the lower triangle at packed offset j n - j (j - 1) / 2
__global__ void k_pack_lower(int64_t n, double* __restrict__ M, double* __restrict__ pk, int to_packed) {
  const int64_t j = blockIdx.y;
  const int64_t base = j * n - j * (j - 1) / 2;
  for (int64_t i = j + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (to_packed) pk[base + (i - j)] = M[i + j * n];
    else M[i + j * n] = pk[base + (i - j)];
  }
}

void launch_pack_lower(Ctx& c, double* M, double* packed, bool to_packed) {
  if (c.n == 0) return;
  if (!packed) throw CudaError("pack_lower: no packed buffer (allocated when a communicator attaches)");
  k_pack_lower<<<dim3((unsigned)std::min<int64_t>(8, ceil_div(c.n, 256)), (unsigned)c.n), 256, 0, c.stream>>>(
      c.n, M, packed, to_packed ? 1 : 0);
  CMPC_LAUNCHED();
}

void vec_alloc(Ctx& c) {
  if (c.comm) comm_buffers(c);  // a sharded context reloaded with its communicator attached
  const size_t n = (size_t)c.n, m = (size_t)c.m;
  const size_t py = (size_t)(c.ldp + c.pz);  // prototype-indexed arrays
  const bool verbose = getenv("CMPC_VERBOSE") != nullptr;
  auto wall = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double last = wall();
  auto tick = [&](const char* what) {
    if (!verbose) return;
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
    const double now = wall();
    fprintf(stderr, "[cmpc alloc] %-10s %8.2f ms\n", what, (now - last) * 1e3);
    last = now;
  };
  c.v = dev_zeros<double>(n, c.stream); c.s = dev_zeros<double>(m, c.stream); c.lam = dev_zeros<double>(m, c.stream); c.z = dev_zeros<double>(m, c.stream);
  c.r1 = dev_zeros<double>(n, c.stream); c.r2 = dev_zeros<double>(m, c.stream); c.r3 = dev_zeros<double>(m, c.stream);
  c.Hv = dev_zeros<double>(n, c.stream); c.Jtl = dev_zeros<double>(n, c.stream); c.y = dev_zeros<double>(py, c.stream); c.sigma = dev_zeros<double>(m, c.stream);
  c.omega = dev_zeros<double>(py, c.stream); c.q = dev_zeros<double>(py, c.stream); c.tq = dev_zeros<double>(n, c.stream); c.JtPl = dev_zeros<double>(n, c.stream); c.rhs = dev_zeros<double>(n, c.stream);
  c.M = dev_zeros<double>(n * n, c.stream); c.L = dev_zeros<double>(n * n, c.stream);
  c.pv = dev_zeros<double>(n, c.stream); c.ps_ = dev_zeros<double>(m, c.stream); c.pl = dev_zeros<double>(m, c.stream); c.pzd = dev_zeros<double>(m, c.stream);
  c.Jpv = dev_zeros<double>(m, c.stream); c.vt = dev_zeros<double>(n, c.stream); c.yt = dev_zeros<double>(py, c.stream); c.yv = dev_zeros<double>(py, c.stream); c.Hvt = dev_zeros<double>(n, c.stream);
  c.part = dev_zeros<double>((size_t)kPartBlocks * kSlots, c.stream);
  const int rc = 2048;
  c.colchunks = (int)std::max<int64_t>(1, ceil_div(c.ps, rc));
  c.colpart = dev_zeros<double>((size_t)c.colchunks * n, c.stream);
  // (and no communicator: checked at use); option "jtl_recurrence" = 0: the direct pass
  c.jtl_recur = c.m > 0 && c.opt_jtl_recur;
  c.hmax = dev_zeros<double>(2, c.stream);  // max|h|, h0
  c.d_mu = dev_zeros<double>(1, c.stream);
  c.d_alpha = dev_zeros<double>(8, c.stream);  // alpha, alpha_z, go, residual snapshot[5]
  c.pk = dev_zeros<Packet>(1, c.stream);
  tick("vectors");
  {  // packet + sequence word + staging ring: one mapped pinned block from the process pool
    void* blk = pinned_take();
    c.pk_host = static_cast<Packet*>(blk);
    c.stage = reinterpret_cast<double*>(static_cast<char*>(blk) + kStageOff);
  }
  c.stage_i = 0;
  CMPC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.pk_map), c.pk_host, 0));
  c.pub_host = reinterpret_cast<volatile unsigned long long*>(reinterpret_cast<char*>(c.pk_host) + sizeof(Packet));
  c.pub_map = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(c.pk_map) + sizeof(Packet));
  c.pk_host_b = reinterpret_cast<Packet*>(reinterpret_cast<char*>(c.pk_host) + kPkBOff);
  c.pk_map_b = reinterpret_cast<Packet*>(reinterpret_cast<char*>(c.pk_map) + kPkBOff);
  *c.pub_host = 0;
  c.pub_dev = dev_zeros<unsigned long long>(1, c.stream);
  c.pub_expect = 0;
  tick("pinned");
  chol_alloc(c);
  tick("chol");
  launch_hmax(c);  // max|h| and h0 on the device
  {  // prototypes with many member rows (duplicates of symmetric segments): warp path
    std::vector<int32_t> mp(size_t(c.p + 1), 0), big;
    if (c.p > 0) {
      CMPC_CUDA(cudaMemcpyAsync(mp.data(), c.mem_ptr, sizeof(int32_t) * (c.p + 1), cudaMemcpyDeviceToHost, c.stream));
      CMPC_CUDA(cudaStreamSynchronize(c.stream));
    }
    for (int64_t k = 0; k < c.p; ++k)
      if (k != c.zero_k && mp[size_t(k + 1)] - mp[size_t(k)] > kLaneMembers) big.push_back((int32_t)k);
    c.nbig = (int)big.size();
    c.nzero = c.zero_k >= 0 ? mp[size_t(c.zero_k + 1)] - mp[size_t(c.zero_k)] : 0;
    c.proto_big = dev_alloc<int32_t>(std::max<size_t>(1, big.size()), c.stream);
    if (!big.empty())
      CMPC_CUDA(cudaMemcpyAsync(c.proto_big, big.data(), sizeof(int32_t) * big.size(), cudaMemcpyHostToDevice, c.stream));
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
  }
  tick("big");
  c.sing_ptr = dev_alloc<int32_t>((size_t)n + 1, c.stream);
  k_sing_ptr<<<(unsigned)ceil_div((int64_t)n + 1, 256), 256, 0, c.stream>>>(c.sing_col, c.pz, c.n, c.sing_ptr);
  CMPC_LAUNCHED();
  c.h_symmetric = false;
  if (c.n > 0) {
    unsigned* bad = dev_zeros<unsigned>(1, c.stream);
    k_sym_check<<<(unsigned)std::min<int64_t>(592, ceil_div(c.n * c.n, 256)), 256, 0, c.stream>>>(c.H, c.n, bad);
    CMPC_LAUNCHED();
    unsigned hb = 1;
    CMPC_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, c.stream));
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
    dev_free(bad, c.stream);
    c.h_symmetric = hb == 0;
  }
  tick("sym");
}

void vec_free(Ctx& c) {
  for (void* p : {(void*)c.v, (void*)c.s, (void*)c.lam, (void*)c.z, (void*)c.r1, (void*)c.r2,
                  (void*)c.r3, (void*)c.Hv, (void*)c.Jtl, (void*)c.y, (void*)c.sigma,
                  (void*)c.omega, (void*)c.q, (void*)c.tq, (void*)c.JtPl, (void*)c.rhs, (void*)c.M,
                  (void*)c.L, (void*)c.pv, (void*)c.ps_, (void*)c.pl, (void*)c.pzd, (void*)c.Jpv,
                  (void*)c.vt, (void*)c.yt, (void*)c.yv, (void*)c.Hvt, (void*)c.part, (void*)c.colpart,
                  (void*)c.hmax, (void*)c.pk, (void*)c.d_mu, (void*)c.d_alpha, (void*)c.Mpack})
    dev_free(p, c.stream);
  if (c.pk_host) {
    CMPC_CUDA(cudaStreamSynchronize(c.stream));  // no staged upload still reading the ring
    pinned_give(c.pk_host);
  }
  c.stage = nullptr;
  dev_free(c.sing_ptr, c.stream);
  c.sing_ptr = nullptr;
  dev_free(c.proto_big, c.stream);
  c.proto_big = nullptr;
  c.nbig = 0;
  dev_free(c.pub_dev, c.stream);
  c.pub_dev = nullptr;
  c.pk_map = c.pk_map_b = nullptr;
  c.pub_host = nullptr;
  c.pub_map = nullptr;
  chol_free(c);
  c.v = c.s = c.lam = c.z = c.r1 = c.r2 = c.r3 = c.Hv = c.Jtl = c.y = c.sigma = nullptr;
  c.omega = c.q = c.tq = c.JtPl = c.rhs = c.M = c.L = c.pv = c.ps_ = c.pl = c.pzd = nullptr;
  c.Jpv = c.vt = c.yt = c.yv = c.Hvt = c.part = c.colpart = c.hmax = c.d_mu = c.d_alpha = nullptr;
  c.pk = nullptr;
  c.pk_host = c.pk_host_b = nullptr;
  c.Mpack = nullptr;
}

// one warp: the packet published on its own (publish_warp)
__global__ void k_publish(Packet* pk, PubArgs pa) { publish_warp(pk, pa, threadIdx.x); }

// the publish arguments of slot A (residual packet) or B (seg_step's packet); counts the publish
PubArgs pub_args(Ctx& c, bool slot_b) {
  ++c.pub_expect;
  return PubArgs{slot_b ? c.pk_map_b : c.pk_map, c.pub_dev, c.pub_map, c.pk_autoreset ? 1 : 0};
}

unsigned long long launch_publish(Ctx& c, bool slot_b) {
  k_publish<<<1, 32, 0, c.stream>>>(c.pk, pub_args(c, slot_b));
  CMPC_LAUNCHED();
  return c.pub_expect;
}

template <bool SIGNED1, bool HAS2>
void launch_proto_reduce(Ctx& c, const double* x1, const double* x2, double* out1, double* out2) {
  const int lane_blocks = (int)ceil_div(c.p, 256);
  const int grid = lane_blocks + (int)ceil_div(c.nbig, 8);
  k_proto_reduce<SIGNED1, HAS2><<<(unsigned)grid, 256, 0, c.stream>>>(
      c.p, c.mem_ptr, c.mem_rows, x1, x2, out1, out2, c.ps, c.ldp, c.zero_k, c.proto_big, c.nbig,
      lane_blocks, SigmaRows{});
  CMPC_LAUNCHED();
}

// sigma = z / s per row, then omega (prototype sums of sigma) and q (signed prototype sums of
// r2 - sigma r3) in one launch (k_sigma_rows + k_proto_reduce<false, true>)
void launch_sigma_reduce(Ctx& c) {
  const int lane_blocks = (int)ceil_div(c.p, 256);
  const int big_blocks = (int)ceil_div(c.nbig, 8);
  const int zero_blocks = c.zero_k >= 0 ? (int)ceil_div(c.nzero, 256) : 0;
  const SigmaRows sr{c.s, c.z, c.r2, c.r3, c.sigma, zero_blocks, big_blocks};
  k_proto_reduce<false, true, true><<<(unsigned)(lane_blocks + big_blocks + zero_blocks), 256, 0, c.stream>>>(
      c.p, c.mem_ptr, c.mem_rows, nullptr, nullptr, c.omega, c.q, c.ps, c.ldp, c.zero_k, c.proto_big, c.nbig,
      lane_blocks, sr);
  CMPC_LAUNCHED();
}

// debug (CMPC_DEBUG_SUMS): order-free XOR checksum of a buffer's bit patterns into pk->pad[slot]
__global__ void k_xorsum(const double* __restrict__ x, int64_t n, Packet* pk, int slot) {
  unsigned long long v = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v ^= (unsigned long long)__double_as_longlong(x[i]) * (unsigned long long)(2 * i + 1);
  for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicXor(reinterpret_cast<unsigned long long*>(&pk->pad[slot]), v);
}
void launch_debug_sum(Ctx& c, const double* x, int64_t n, int slot) {
  static const bool on = getenv("CMPC_DEBUG_SUMS") != nullptr;
  if (!on || n <= 0) return;
  CMPC_CUDA(cudaMemsetAsync(&c.pk->pad[slot], 0, sizeof(double), c.stream));
  k_xorsum<<<64, 256, 0, c.stream>>>(x, n, c.pk, slot);
  CMPC_LAUNCHED();
}

void launch_reset_packet_all(Ctx& c) {
  for (int w = 0; w < 3; ++w) {
    k_reset_packet<<<1, 1, 0, c.stream>>>(c.pk, w);
    CMPC_LAUNCHED();
  }
}

void launch_zero_packet(Ctx& c) {
  CMPC_CUDA(cudaMemsetAsync(c.pk, 0, sizeof(Packet), c.stream));
}

void launch_Hx(Ctx& c, const double* x, double* out) {
  if (c.n == 0) return;
  if (c.h_symmetric) {
    k_hcol_gemv<<<(unsigned)ceil_div(c.n, 8), 256, 0, c.stream>>>(c.H, c.n, x, out, nullptr, nullptr,
                                                                     0.0, nullptr, nullptr);
  } else {
    k_rows_gemv<<<(unsigned)ceil_div(c.n, 32), 256, 0, c.stream>>>(c.H, c.n, c.n, c.n, nullptr, x, out);
  }
  CMPC_LAUNCHED();
}

void launch_Jx(Ctx& c, const double* x, double* y, double* Jx) {
  if (c.markov) {  // P x from the Markov table (markov.cu)
    launch_markov_gemv(c, x, y);
    return;
  }
  // eight 16-byte loads in flight per lane (79% of HBM at config 3; four: 67%); the singleton
  // prototypes ride along as extra CTAs
  const int gblocks = (int)ceil_div(c.ps, 64);
  const int sblocks = (int)ceil_div(c.pz, 256);
  if (gblocks + sblocks > 0) {
    k_proto_gemv<8><<<(unsigned)(gblocks + sblocks), 256, 0, c.stream>>>(c.P, c.ldp, c.ps, c.hi, x, y, gblocks,
                                                                        c.sing_col, c.sing_val, c.pz, y + c.ldp);
    CMPC_LAUNCHED();
  }
  (void)Jx;
}

// prototype-indexed y (SYRK part at [0,ldp), singletons at [ldp, ldp+pz)) -> row values:
// the row kernels address y with proto index k < ps directly and singletons at ldp + (k - ps);
// to keep one index space the row_map stores the compact index (see compact_row_map).

void launch_Jtq(Ctx& c, const double* q, double* out) {
  if (c.n == 0) return;
  if (c.markov) {  // P' q from the Markov table into chunk 0 of colpart
    launch_markov_ptq(c, q, c.colpart);
    k_ptq_final<<<(unsigned)ceil_div(c.n, 8), 256, 0, c.stream>>>(c.colpart, 1, c.n, c.sing_ptr, c.sing_val,
                                                                q + c.ldp, out);
    CMPC_LAUNCHED();
    return;
  }
  if (c.ps > 0) {
    const int rc = 2048;
    dim3 g((unsigned)c.colchunks, (unsigned)ceil_div(c.n, 8));
    // <= 64 registers: four CTAs per SM (74% of HBM at config 3; 102 registers: 61%)
    k_ptq_partial<4, 4><<<g, 256, 0, c.stream>>>(c.P, c.ldp, c.ps, c.n, c.start_col, q, rc, c.colpart);
    CMPC_LAUNCHED();
  }
  k_ptq_final<<<(unsigned)ceil_div(c.n, 8), 256, 0, c.stream>>>(
      c.colpart, c.ps > 0 ? c.colchunks : 0, c.n, c.sing_ptr, c.sing_val, q + c.ldp, out);
  CMPC_LAUNCHED();
}

void launch_residuals(Ctx& c, bool reuse_trial, bool gated, int publish) {
  const double* gate = gated ? c.d_alpha : nullptr;
  const unsigned pb = part_blocks(c.m);
  const int64_t m_all = rows_all(c);
  if (!c.pk_autoreset) {  // (in the host loop, k_publish starts every segment clean)
    k_reset_packet<<<1, 1, 0, c.stream>>>(c.pk, 0);
    CMPC_LAUNCHED();
  }
  // reuse_trial: v was just set to the accepted trial point v + alpha pv; k_update copied the
  // trial's H v_t into H v and carried P v along as yv + alpha P pv, the values the trial's
  // merit used
  if (!reuse_trial) launch_Hx(c, c.v, c.Hv);
  if (c.m > 0) {
    if (!reuse_trial) launch_Jx(c, c.v, c.yv, nullptr);
    k_res_rows<<<pb, kRowT, 0, c.stream>>>(c.m, c.row_map, c.yv, c.d, c.s, c.lam, c.z, c.d_mu, c.r2,
                                           c.r3, c.part, c.pk, gate);
    CMPC_LAUNCHED();
    if (!(reuse_trial && c.jtl_recur && !c.comm)) {
      if (gated) throw CudaError("gated residual pass needs the J'lambda recurrence");  // (after a step: Jtl was advanced by k_update)
      launch_proto_reduce<true, false>(c, c.lam, nullptr, c.q, nullptr);
      launch_Jtq(c, c.q, c.Jtl);
    }
  } else if (c.comm && c.n > 0) {
    CMPC_CUDA(cudaMemsetAsync(c.Jtl, 0, sizeof(double) * c.n, c.stream));
  }
  const int np = c.m > 0 ? (int)pb : 0;
  if (c.comm) {
    // this rank's rows: J_g' lambda_g, the row sums and maxima -> allreduce -> finalize
    k_res_final<<<1, kFinT, 0, c.stream>>>(c.n, m_all, np, c.Hv, c.h, c.Jtl, c.v, c.r1, c.part,
                                           c.hmax, c.pk, 1, gate, nullptr, PubArgs{});
    CMPC_LAUNCHED();
    comm_group(c, true);
    comm_allreduce(c, c.Jtl, (size_t)c.n, CommType::f64, CommOp::sum);
    comm_allreduce(c, &c.pk->sum_log_s, 2, CommType::f64, CommOp::sum);  // sum_log_s, sum_abs_r3
    comm_allreduce(c, &c.pk->max_r3, 5, CommType::f64, CommOp::max);     // max_r3 .. max_z
    comm_group(c, false);
  }
  k_res_final<<<1, kFinT, 0, c.stream>>>(c.n, m_all, np, c.Hv, c.h, c.Jtl, c.v, c.r1, c.part,
                                         c.hmax, c.pk, c.comm ? 2 : 0, gate, c.d_alpha + 3,
                                         publish >= 0 ? pub_args(c, publish == 1) : PubArgs{});
  CMPC_LAUNCHED();
}

void launch_residuals_mu(Ctx& c, const Packet& a) {
  if (c.m > 0 || c.comm) {
    k_reset_packet<<<1, 1, 0, c.stream>>>(c.pk, 3);
    CMPC_LAUNCHED();
  }
  if (c.m > 0) {
    k_mu_rows<<<part_blocks(c.m), kRowT, 0, c.stream>>>(c.m, c.s, c.lam, c.z, c.d_mu, c.r2, c.pk);
    CMPC_LAUNCHED();
  }
  comm_allreduce(c, &c.pk->max_comp, 1, CommType::f64, CommOp::max);
  k_kkt_only<<<1, 1, 0, c.stream>>>(c.n, rows_all(c), c.hmax, c.pk, a.max_r1, a.max_r3, a.max_lam,
                                    a.max_s, a.max_z);
  CMPC_LAUNCHED();
}

void launch_prepare_step(Ctx& c, const double* sigma_override) {
  if (c.m == 0) return;
  if (sigma_override) {
    k_sigma_rows<<<(unsigned)ceil_div(c.m, 256), 256, 0, c.stream>>>(c.m, c.s, c.z, c.r2, c.r3, sigma_override,
                                                                    c.sigma, nullptr);
    CMPC_LAUNCHED();
    launch_proto_reduce<false, false>(c, c.sigma, nullptr, c.omega, nullptr);
  } else {
    launch_sigma_reduce(c);
  }
}

void launch_rhs_partial(Ctx& c) {
  if (c.m > 0) launch_Jtq(c, c.q, c.tq);
  else if (c.n > 0) CMPC_CUDA(cudaMemsetAsync(c.tq, 0, sizeof(double) * c.n, c.stream));
}

void launch_rhs_final(Ctx& c) {
  if (c.n == 0) return;
  k_rhs<<<(unsigned)ceil_div(c.n, 256), 256, 0, c.stream>>>(c.n, c.r1, c.tq, rows_all(c), c.rhs);
  CMPC_LAUNCHED();
}

void launch_rhs(Ctx& c) {
  launch_rhs_partial(c);
  launch_rhs_final(c);
}

// a slot of the pinned staging ring (128 doubles, 4 per slot): the host loop synchronises
// with the stream between segments, so a slot is never reused while its copy is pending
double* stage_slot(Ctx& c, int) {
  double* p = c.stage + 4 * (c.stage_i & 31);
  ++c.stage_i;
  return p;
}

void launch_hmax(Ctx& c) {
  CMPC_CUDA(cudaMemsetAsync(c.hmax, 0, sizeof(double), c.stream));
  double* st = stage_slot(c, 1);
  st[0] = c.h0;
  CMPC_CUDA(cudaMemcpyAsync(c.hmax + 1, st, sizeof(double), cudaMemcpyHostToDevice, c.stream));
  if (c.n > 0) {
    k_absmax<<<(unsigned)std::min<int64_t>(64, ceil_div(c.n, 256)), 256, 0, c.stream>>>(c.h, c.n, c.hmax);
    CMPC_LAUNCHED();
  }
}

void set_mu(Ctx& c, double mu) {
  c.mu = mu;
  double* st = stage_slot(c, 1);
  st[0] = mu;
  CMPC_CUDA(cudaMemcpyAsync(c.d_mu, st, sizeof(double), cudaMemcpyHostToDevice, c.stream));
}

void launch_recover(Ctx& c, double tau) {
  if (!c.pk_autoreset) {  // (in the host loop, k_publish starts every segment clean)
    k_reset_packet<<<1, 1, 0, c.stream>>>(c.pk, 1);
    CMPC_LAUNCHED();
  }
  const unsigned pb = part_blocks(c.m);
  if (c.m > 0) launch_Jx(c, c.pv, c.y, nullptr);
  if (c.m > 0) {
    k_recover_rows<<<pb, kRowT, 0, c.stream>>>(c.m, c.row_map, c.y, c.s, c.z, c.sigma, c.r2, c.r3,
                                               c.d_mu, tau, c.Jpv, c.ps_, c.pl, c.pzd, c.part, c.pk);
    CMPC_LAUNCHED();
  }
  k_recover_final<<<1, kFinT, 0, c.stream>>>(c.n, c.m > 0 ? (int)pb : 0, c.Hv, c.h, c.pv, c.part,
                                             c.pk);
  CMPC_LAUNCHED();
  if (c.comm) {  // step-length minima and sum ps/s over every rank's rows
    comm_group(c, true);
    comm_allreduce(c, &c.pk->alpha_s_min, 2, CommType::f64, CommOp::min);
    comm_allreduce(c, &c.pk->d_ps_s, 1, CommType::f64, CommOp::sum);
    comm_group(c, false);
  }
}

void launch_trial(Ctx& c, double alpha, bool alpha_from_device, bool linear, bool decide, double eta,
                  int publish) {
  const Packet* apk = alpha_from_device ? c.pk : nullptr;
  if (!c.pk_autoreset) {  // (in the host loop, k_publish starts every segment clean)
    k_reset_packet<<<1, 1, 0, c.stream>>>(c.pk, 2);
    CMPC_LAUNCHED();
  }
  // J' p_lambda of the direction (for the step's J'lambda, k_update), formed here beside H v_t
  // (a side-stream branch was no faster alone and cost 45% in batch mode)
  const bool jtpl = c.m > 0 && c.jtl_recur && !c.comm && c.n > 0;
  if (c.n > 0 && c.h_symmetric) {  // v_t = v + alpha pv formed inside H v_t's column dots
    const int hblocks = (int)ceil_div(c.n, 32), sblocks = jtpl ? (int)ceil_div(c.n, 32) : 0;
    k_trial_hv<<<(unsigned)(hblocks + sblocks), 1024, 0, c.stream>>>(c.H, c.n, c.Hvt, c.v, c.pv, alpha, apk, c.vt,
                                                                     hblocks, c.M, c.tq, c.JtPl);
    CMPC_LAUNCHED();
  } else if (c.n > 0) {
    k_axpy_n<<<(unsigned)ceil_div(c.n, 256), 256, 0, c.stream>>>(c.n, c.v, alpha, apk, c.pv, c.vt);
    CMPC_LAUNCHED();
    launch_Hx(c, c.vt, c.Hvt);
    if (jtpl) {
      k_jtpl_symv<<<(unsigned)ceil_div(c.n, 32), 1024, 0, c.stream>>>(c.M, c.H, c.n, c.pv, c.tq, c.JtPl);
      CMPC_LAUNCHED();
    }
  }
  const unsigned pb = part_blocks(c.m);
  if (c.m > 0) {
    if (!linear) launch_Jx(c, c.vt, c.yt, nullptr);
    k_trial_rows<<<pb, kRowT, 0, c.stream>>>(c.m, c.row_map, linear ? nullptr : c.yt, c.yv, c.y,
                                             c.d, c.s, c.ps_, alpha, apk, c.part, c.pk);
    CMPC_LAUNCHED();
  }
  k_trial_final<<<1, kFinT, 0, c.stream>>>(c.n, c.m, c.m > 0 ? (int)pb : 0, c.vt, c.Hvt, c.h,
                                           c.part, c.pk, c.d_mu,
                                           decide && !c.comm ? c.d_alpha : nullptr, eta,
                                           publish >= 0 && !c.comm ? pub_args(c, publish == 1) : PubArgs{});
  CMPC_LAUNCHED();
  if (c.comm) {  // merit row sums and the slack-positivity flag over every rank's rows
    comm_group(c, true);
    comm_allreduce(c, &c.pk->t_sum_log, 2, CommType::f64, CommOp::sum);
    comm_allreduce(c, &c.pk->any_nonpos, 1, CommType::i64, CommOp::max);
    comm_group(c, false);
    if (publish >= 0) launch_publish(c, publish == 1);
  }
}

void launch_fraction_to_boundary(cudaStream_t st, int64_t m, const double* s, const double* ps,
                                 const double* z, const double* pz, double tau, double* out) {
  const double inf = __builtin_huge_val();
  const double init[2] = {inf, inf};
  CMPC_CUDA(cudaMemcpyAsync(out, init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (m > 0) {
    k_ftb<<<part_blocks(m), kRowT, 0, st>>>(m, s, ps, z, pz, tau, out);
    CMPC_LAUNCHED();
  }
}

void launch_ls_pieces(Ctx& c) {
  const unsigned pb = part_blocks(c.m);
  if (c.m > 0) {
    k_pss_rows<<<pb, kRowT, 0, c.stream>>>(c.m, c.s, c.ps_, c.part);
    CMPC_LAUNCHED();
  }
  k_recover_final<<<1, kFinT, 0, c.stream>>>(c.n, c.m > 0 ? (int)pb : 0, c.Hv, c.h, c.pv, c.part,
                                             c.pk);
  CMPC_LAUNCHED();
  comm_allreduce(c, &c.pk->d_ps_s, 1, CommType::f64, CommOp::sum);
}

void launch_init_state(Ctx& c, double mu) {
  if (c.n > 0) CMPC_CUDA(cudaMemsetAsync(c.v, 0, sizeof(double) * c.n, c.stream));
  if (c.m > 0) {
    k_init_state<<<(unsigned)ceil_div(c.m, 256), 256, 0, c.stream>>>(c.m, c.d, mu, c.s, c.lam, c.z);
    CMPC_LAUNCHED();
  }
}

void set_alpha(Ctx& c, double alpha, double alpha_z) {
  double* st = stage_slot(c, 2);
  st[0] = alpha;
  st[1] = alpha_z;
  st[2] = 1.0;  // the step is taken (k_update's gate)
  CMPC_CUDA(cudaMemcpyAsync(c.d_alpha, st, 3 * sizeof(double), cudaMemcpyHostToDevice, c.stream));
}

void launch_update_dev(Ctx& c) {
  const int64_t py = c.m > 0 ? c.ldp + c.pz : 0;
  const int64_t k = std::max(std::max(c.n, c.m), py);
  if (k == 0) return;
  k_update<<<(unsigned)ceil_div(k, 256), 256, 0, c.stream>>>(c.n, c.m, c.d_alpha, c.v, c.pv,
                                                             c.s, c.ps_, c.lam, c.pl, c.z, c.pzd,
                                                             py, c.yv, c.y, c.jtl_recur && !c.comm ? c.Jtl : nullptr,
                                                             c.JtPl, c.Hv, c.Hvt);
  CMPC_LAUNCHED();
}

void launch_update(Ctx& c, double alpha, double alpha_z) {
  set_alpha(c, alpha, alpha_z);
  launch_update_dev(c);
}

}  // namespace cmpc
