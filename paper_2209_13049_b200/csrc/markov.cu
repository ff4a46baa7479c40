// Markov-table prototypes: for a QP built on the device from the
// structured problem, the SYRK prototypes are state rows of J, and state row (t, i) is
//   [G_{t-1} .. G_0] row i,   G_k = A_K^k B   (reduction.cpp:43-60 builds these blocks,
//                                              reduction.cpp:205-248 the rows)
// i.e. a window of one row of the Markov table
//   MK[q, s] = G_{T-1-s/nu}[order(q), s % nu]      (q < nq, s < T nu)
// starting at column (T - t) nu: every row of P is a shifted view of the table, whose
// zero tail ends its nonzero prefix. The table is nq x T nu (10 MB at config 3, 16 MB at
// config 4 T = 200) against 180 MB / 1.53 GB for the materialised P, and it stays in L2.
//
// Prototype layout: stage-major 32-row chunks. States are ordered by the first stage their
// B-response is nonzero (tf), so at stage t the nonzero rows are exactly table rows
// [0, cnt_t) with cnt_t = #{tf < t}; the stage's block is padded to a chunk multiple (the
// padding rows are zero in the stage's window). The structure analysis (structure.cu) moves
// each SYRK prototype to its leader's (stage, table row) slot; the other slots are empty
// prototypes (weight 0). Consumers: the SYRK reads its operand boxes straight from the table
// by TMA (syrk.cu, chunk -> {table row, column shift}); P x and P' q below.
#include <algorithm>
#include <mutex>
#include <numeric>
#include <vector>

#include "internal.cuh"
#include "jrows.cuh"

namespace cmpc {

namespace {

constexpr int kMkKT = 16;  // stages per thread in k_mk_gemv

// states that have a state row in J (only those enter the table)
__global__ void k_mk_used(const RowDesc* rows, int64_t m, int32_t* used) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const RowDesc q = rows[r];
  if (q.kind == 1) used[q.i] = 1;
}

// first k with G_k row i nonzero (T: never) and the last nonzero input of that block (the
// row's nonzero prefix at stage t ends at (t - 1 - tf) nu + lc + 1); G = [G_0 .. G_{T-1}]
// column-major, ld nx
__global__ void k_mk_first(const double* G, int64_t nx, int nu, int T, int32_t* tf, int32_t* lc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nx) return;
  int t = 0, last = -1;
  for (; t < T; ++t) {
    for (int cc = 0; cc < nu; ++cc)
      if (G[i + ((int64_t)t * nu + cc) * nx] != 0.0) last = cc;
    if (last >= 0) break;
  }
  tf[i] = t;
  lc[i] = last;
}

// MK[q + s ldmk] = G[order[q] + ((T-1-s/nu) nu + s%nu) nx]; rows >= nq stay zero
__global__ void k_mk_fill(const double* G, int64_t nx, int nu, int T, const int32_t* order,
                          int64_t nq, int64_t ldmk, double* mk) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s = blockIdx.y;
  if (q >= nq) return;
  const int64_t blk = T - 1 - s / nu, cc = s % nu;
  mk[q + s * ldmk] = G[order[q] + (blk * nu + cc) * nx];
}

// y = P x over the layout: thread (row r of a 32-row table block, warp w) walks the table
// columns s = s0 + w, s0 + w + 8, .. of its block and adds MK[q0 + r, s] x[s - (T - t) nu]
// into one accumulator per stage t of the CTA's stage group (t = g, g + groups, ..): each
// table element is loaded once for up to kMkKT stages; four column loads are in flight per
// thread (the table is L2-resident: latency, not bandwidth, is the limit) and x sits in
// shared memory (SX; global otherwise). Warps reduce in a fixed order.
constexpr int kMkU = 4;
constexpr int kMkW = 8;  // warps per CTA
template <bool SX>
__global__ void __launch_bounds__(kMkW * 32) k_mk_gemv(const double* __restrict__ mk, int64_t ldmk, int nu, int T,
                                                 int groups, const int32_t* __restrict__ rb_end,
                                                 const int32_t* __restrict__ base,
                                                 const int32_t* __restrict__ cnt,
                                                 const double* __restrict__ x, int64_t n,
                                                 double* __restrict__ y) {
  extern __shared__ double xs_dyn[];  // [kMkW][kMkKT][33] reduction, then x
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q0 = (int64_t)blockIdx.x * 32;
  const int g = (int)blockIdx.y + 1;  // first stage of the group (stages are 1..T)
  int nk = 0;
  for (int t = g; t <= T && nk < kMkKT; t += groups) ++nk;
  double (*red)[kMkKT][33] = reinterpret_cast<double (*)[kMkKT][33]>(xs_dyn);
  const double* xv = x;
  if (SX) {
    double* xs = xs_dyn + kMkW * kMkKT * 33;
    for (int64_t i = threadIdx.x; i < n; i += kMkW * 32) xs[i] = x[i];
    __syncthreads();
    xv = xs;
  }
  const int s_end = rb_end[blockIdx.x];
  const int t_max = g + groups * (nk - 1);  // smallest window start: the group's last stage
  const int s_beg = (T - t_max) * nu;
  double acc[kMkKT];
#pragma unroll
  for (int k = 0; k < kMkKT; ++k) acc[k] = 0.0;
  const double* col = mk + q0 + lane;
  int s = s_beg + w;
  for (; s + kMkW * (kMkU - 1) < s_end; s += kMkW * kMkU) {
    double a[kMkU];
#pragma unroll
    for (int u = 0; u < kMkU; ++u) a[u] = __ldg(col + (int64_t)(s + kMkW * u) * ldmk);
#pragma unroll
    for (int u = 0; u < kMkU; ++u)
#pragma unroll
      for (int k = 0; k < kMkKT; ++k) {
        const int c = s + kMkW * u - (T - g - groups * k) * nu;  // column of P (warp-uniform)
        if (k < nk && c >= 0) acc[k] += a[u] * xv[c];
      }
  }
  for (; s < s_end; s += kMkW) {
    const double a = __ldg(col + (int64_t)s * ldmk);
#pragma unroll
    for (int k = 0; k < kMkKT; ++k) {
      const int c = s - (T - g - groups * k) * nu;
      if (k < nk && c >= 0) acc[k] += a * xv[c];
    }
  }
#pragma unroll
  for (int k = 0; k < kMkKT; ++k) red[w][k][lane] = acc[k];
  __syncthreads();
  for (int k = w; k < nk; k += kMkW) {
    const int t = g + groups * k;
    if (q0 >= cnt[t]) continue;
    double sum = 0.0;
#pragma unroll
    for (int u = 0; u < kMkW; ++u) sum += red[u][k][lane];
    y[base[t] + q0 + lane] = sum;
  }
}

__global__ void k_mk_singletons(const int32_t* sing_col, const double* sing_val, int64_t pz,
                                const double* x, double* ys) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < pz) ys[k] = sing_val[k] * x[sing_col[k]];
}

// out[j] = sum over the layout rows of P[row, j] q[row] (P' q without singletons): one CTA
// per column, threads stride every stage's rows, fixed-order block reduction
__global__ void __launch_bounds__(256) k_mk_ptq(const double* __restrict__ mk, int64_t ldmk, int nu, int T,
                                                const int32_t* __restrict__ base,
                                                const int32_t* __restrict__ cnt,
                                                const double* __restrict__ q, double* __restrict__ out) {
  __shared__ double sh[8];
  const int j = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double s = 0.0;
  // warp w takes stages t = t0 + w, t0 + w + 8, ..; P[(t, .), j] nonzero only for j < t nu
  for (int t = j / nu + 1 + w; t <= T; t += 8) {
    const double* colp = mk + (int64_t)((T - t) * nu + j) * ldmk;
    const double* qq = q + base[t];
    for (int r = lane; r < cnt[t]; r += 32) s += colp[r] * qq[r];
  }
  s = warp_sum(s);
  if (lane == 0) sh[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int u = 0; u < 8; ++u) a += sh[u];
    out[j] = a;
  }
}

}  // namespace

void markov_free(Ctx& c) {
  for (void* p : {(void*)c.mk, (void*)c.mk_pos, (void*)c.mk_base, (void*)c.mk_cnt, (void*)c.mk_chunk,
                  (void*)c.mk_clist, (void*)c.mk_rbend})
    dev_free(p, c.stream);
  c.mk = nullptr;
  c.mk_pos = c.mk_base = c.mk_cnt = c.mk_rbend = nullptr;
  c.mk_chunk = nullptr;
  c.mk_clist = nullptr;
  c.h_mk_chunk.clear();
  c.h_mk_width.clear();
  c.ldmk = c.mk_cols = c.mk_nq = c.mk_ps = 0;
  c.mk_T = c.mk_nu = c.mk_nchunks = 0;
  c.markov = false;
}

bool markov_prepare(Ctx& c) {
  markov_free(c);
  const BuiltJ* bj = prob_rows(c);
  if (!c.opt_markov || !bj || c.m == 0 || c.n == 0 || bj->nu <= 0) return false;
  const int64_t nx = bj->nx, m = c.m, n = c.n;
  const int nu = bj->nu;
  const int T = (int)(n / nu);
  if ((int64_t)T * nu != n) return false;
  cudaStream_t st = c.stream;
  int32_t* used = dev_zeros<int32_t>(size_t(nx), st);
  int32_t* tf = dev_alloc<int32_t>(size_t(nx), st);
  int32_t* lc = dev_alloc<int32_t>(size_t(nx), st);
  k_mk_used<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(static_cast<const RowDesc*>(bj->rows), m, used);
  CMPC_LAUNCHED();
  k_mk_first<<<(unsigned)ceil_div(nx, 256), 256, 0, st>>>(bj->G, nx, nu, T, tf, lc);
  CMPC_LAUNCHED();
  std::vector<int32_t> hu((size_t)nx), ht((size_t)nx), hl((size_t)nx);
  CMPC_CUDA(cudaMemcpyAsync(hu.data(), used, sizeof(int32_t) * nx, cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaMemcpyAsync(ht.data(), tf, sizeof(int32_t) * nx, cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaMemcpyAsync(hl.data(), lc, sizeof(int32_t) * nx, cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaStreamSynchronize(st));
  dev_free(used, st);
  dev_free(tf, st);
  dev_free(lc, st);
  std::vector<int32_t> order;
  for (int64_t i = 0; i < nx; ++i)
    if (hu[size_t(i)] && ht[size_t(i)] < T) order.push_back((int32_t)i);
  if (order.empty()) return false;
  // by first nonzero stage, then by the end of that block's nonzeros (descending): a chunk's
  // first row then has the chunk's widest prefix at every stage
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    if (ht[size_t(a)] != ht[size_t(b)]) return ht[size_t(a)] < ht[size_t(b)];
    return hl[size_t(a)] > hl[size_t(b)];
  });
  const int64_t nq = (int64_t)order.size();
  std::vector<int32_t> pos((size_t)nx, -1);
  for (int64_t q = 0; q < nq; ++q) pos[size_t(order[size_t(q)])] = (int32_t)q;
  // per stage t = 1..T: nonzero rows cnt_t = #{tf < t} (order is sorted by tf), padded
  std::vector<int32_t> base(size_t(T + 2), 0), cnt(size_t(T + 1), 0);
  c.h_mk_chunk.clear();
  c.h_mk_width.clear();
  int64_t nz = 0;
  for (int t = 1; t <= T; ++t) {
    while (nz < nq && ht[size_t(order[size_t(nz)])] < t) ++nz;
    const int64_t pc = round_up(nz, kBK);
    cnt[size_t(t)] = (int32_t)pc;
    base[size_t(t + 1)] = base[size_t(t)] + (int32_t)pc;
    for (int64_t q0 = 0; q0 < pc; q0 += kBK) {
      c.h_mk_chunk.push_back({(int)q0, (T - t) * nu});
      const int32_t f = order[size_t(q0)];
      c.h_mk_width.push_back((t - 1 - ht[size_t(f)]) * nu + hl[size_t(f)] + 1);
    }
  }
  const int64_t ps = base[size_t(T + 1)];
  if (ps == 0) return false;
  c.ldmk = round_up(nq, 32);
  c.mk_cols = (int64_t)T * nu;
  c.mk_nq = nq;
  c.mk_T = T;
  c.mk_nu = nu;
  c.mk_ps = ps;
  c.mk_nchunks = (int)c.h_mk_chunk.size();
  // per 32-row table block: end of its nonzero columns, (T - tf of its first row) nu
  std::vector<int32_t> rbend((size_t)(c.ldmk / 32));
  for (size_t b = 0; b < rbend.size(); ++b) {
    const int64_t q = (int64_t)b * 32;
    rbend[b] = q < nq ? (T - ht[size_t(order[size_t(q)])]) * nu : 0;
  }
  auto up = [&](const std::vector<int32_t>& v) {
    int32_t* d = dev_alloc<int32_t>(std::max<size_t>(1, v.size()), st);
    CMPC_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice, st));
    return d;
  };
  c.mk_pos = up(pos);
  c.mk_base = up(base);
  c.mk_cnt = up(cnt);
  c.mk_rbend = up(rbend);
  int32_t* dorder = up(order);
  c.mk_chunk = dev_alloc<int2>(c.h_mk_chunk.size(), st);
  CMPC_CUDA(cudaMemcpyAsync(c.mk_chunk, c.h_mk_chunk.data(), sizeof(int2) * c.h_mk_chunk.size(),
                            cudaMemcpyHostToDevice, st));
  c.mk = dev_zeros<double>(size_t(c.ldmk * c.mk_cols), st);
  k_mk_fill<<<dim3((unsigned)ceil_div(nq, 256), (unsigned)c.mk_cols), 256, 0, st>>>(bj->G, nx, nu, T, dorder, nq,
                                                                                  c.ldmk, c.mk);
  CMPC_LAUNCHED();
  CMPC_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
  dev_free(dorder, st);
  return true;
}

void launch_markov_gemv(Ctx& c, const double* x, double* y) {
  if (c.ps > 0) {
    // stage groups: at most kMkKT stages per thread, and two CTAs per SM for small tables
    const int nrb = (int)(c.ldmk / 32);
    const int groups = std::min(c.mk_T, std::max({4, (int)ceil_div(c.mk_T, kMkKT), (int)ceil_div(296, nrb)}));
    const dim3 grid((unsigned)nrb, (unsigned)groups);
    const size_t sred = sizeof(double) * kMkW * kMkKT * 33, sx = sizeof(double) * (size_t)c.n;
    static std::once_flag flags[kMaxDevices];
    once_per_device(flags, c.device, [] {
      CMPC_CUDA(cudaFuncSetAttribute(k_mk_gemv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      CMPC_CUDA(cudaFuncSetAttribute(k_mk_gemv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    if (sred + sx <= 200 * 1024)
      k_mk_gemv<true><<<grid, kMkW * 32, sred + sx, c.stream>>>(c.mk, c.ldmk, c.mk_nu, c.mk_T, groups, c.mk_rbend,
                                                                c.mk_base, c.mk_cnt, x, c.n, y);
    else
      k_mk_gemv<false><<<grid, kMkW * 32, sred, c.stream>>>(c.mk, c.ldmk, c.mk_nu, c.mk_T, groups, c.mk_rbend,
                                                            c.mk_base, c.mk_cnt, x, c.n, y);
    CMPC_LAUNCHED();
  }
  if (c.pz > 0) {
    k_mk_singletons<<<(unsigned)ceil_div(c.pz, 256), 256, 0, c.stream>>>(c.sing_col, c.sing_val, c.pz, x,
                                                                        y + c.ldp);
    CMPC_LAUNCHED();
  }
}

void launch_markov_ptq(Ctx& c, const double* q, double* out) {
  if (c.n == 0) return;
  k_mk_ptq<<<(unsigned)c.n, 256, 0, c.stream>>>(c.mk, c.ldmk, c.mk_nu, c.mk_T, c.mk_base, c.mk_cnt, q, out);
  CMPC_LAUNCHED();
}

}  // namespace cmpc
