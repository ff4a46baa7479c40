// Markov-table prototypes: for a QP built on the device from the
// structured problem, every row of J is a window of one row of a table of B-responses
// (reduction.cpp:43-60 builds the blocks, reduction.cpp:182-251 the rows):
//   state row (t, i):  [G_{t-1} .. G_0] row i                      G_k = A_K^k B
//   input row (t, i):  [(K G)_{t-1} .. (K G)_0, e_i] row i          (feedback K)
//   mixed row (t, i):  [((E + F K) G)_{t-1} .. , F] row i
// With the Markov blocks in reverse order and the "own stage" block D last, source q (a
// state, input or mixed row index) has the table row
//   MK[q, s] = M_{T-1-s/nu}[i, s % nu]  (s < T nu),   D[i, s % nu]  (T nu <= s < (T+1) nu)
// and row (t, i) of J is the window of MK[q] starting at column (T - t) nu. MK is
// nq x (T+1) nu (10 MB at config 3, 16 MB at config 4 T = 200 against 180 MB / 1.53 GB of
// materialised P) and stays in L2. Input rows without feedback are singletons and stay out.
//
// Prototype layout: stage-major 32-row chunks. Sources are ordered by the last nonzero column
// L_q of their table row (descending): at stage t the window of q is nonzero exactly when
// L_q >= (T - t) nu, so the stage's nonzero rows are table rows [0, cnt_t), and a chunk's
// first row has its widest prefix (L_q - (T - t) nu + 1). Each stage's block is padded to a
// chunk multiple (the padding rows are zero in the stage's window). The structure analysis
// (structure.cu) moves each SYRK prototype to its leader's (stage, table row) slot; the other
// slots are empty prototypes (weight 0). Consumers: the SYRK reads its operand boxes straight
// from the table by TMA (syrk.cu, chunk -> {table row, column shift}); P x and P' q below.
#include <algorithm>
#include <mutex>
#include <numeric>
#include <vector>

#include "internal.cuh"
#include "jrows.cuh"

namespace cmpc {

namespace {

constexpr int kMkKT = 16;  // stages per thread in k_mk_gemv

// the table's sources: states [0, nx), inputs [nx, nx + nu) (feedback only), mixed rows
// [nx + nu, nx + nu + nc); a source enters when J has a row of it
__device__ __forceinline__ int mk_src(const RowDesc q, int nx, int nu, bool inputs) {
  if (q.kind == 1) return q.i;
  if (q.kind == 2) return inputs ? nx + q.i : -1;
  return nx + nu + q.i;
}

__global__ void k_mk_used(const RowDesc* rows, int64_t m, int nx, int nu, bool inputs, int32_t* used) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const int q = mk_src(rows[r], nx, nu, inputs);
  if (q >= 0) used[q] = 1;
}

// MK[q, s] of source q (see the header); G = [G_0 .. G_{T-1}] (ld nx), KG (ld nu), EG and F
// (ld nc), all column-major
struct MkSrc {
  const double *G, *KG, *EG, *F;
  int nx, nu, nc, T;
  __device__ __forceinline__ double operator()(int q, int64_t s) const {
    const int64_t b = s / nu, cc = s - b * nu;
    if (q < nx) return b < T ? G[q + ((T - 1 - b) * nu + cc) * nx] : 0.0;
    if (q < nx + nu) {
      const int i = q - nx;
      return b < T ? KG[i + ((T - 1 - b) * nu + cc) * nu] : (cc == i ? 1.0 : 0.0);
    }
    const int i = q - nx - nu;
    return b < T ? EG[i + ((T - 1 - b) * nu + cc) * nc] : F[i + cc * nc];
  }
};

// last nonzero column of each source's table row (-1: none)
__global__ void k_mk_last(MkSrc src, int nsrc, int32_t* last) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsrc) return;
  int64_t s = (int64_t)(src.T + 1) * src.nu - 1;
  for (; s >= 0; --s)
    if (src(q, s) != 0.0) break;
  last[q] = (int32_t)s;
}

// MK[q + s ldmk] = table row of source order[q]; rows >= nq stay zero
__global__ void k_mk_fill(MkSrc src, const int32_t* order, int64_t nq, int64_t ldmk, double* mk) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s = blockIdx.y;
  if (q >= nq) return;
  mk[q + s * ldmk] = src(order[q], s);
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
  const int g = (int)blockIdx.y;  // first stage of the group (stages are 0..T)
  int nk = 0;
  for (int t = g; t <= T && nk < kMkKT; t += groups) ++nk;
  double (*red)[kMkKT][33] = reinterpret_cast<double (*)[kMkKT][33]>(xs_dyn);
  const double* xv = x;
  if (SX) {
    double* xs = xs_dyn + kMkW * kMkKT * 33;
    // x and nu zeros past it: stage T's windows reach one block past x (the own-stage block of
    // input / mixed sources, which have no row at stage T), so no bound check per product
    for (int64_t i = threadIdx.x; i < n + nu; i += kMkW * 32) xs[i] = i < n ? x[i] : 0.0;
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
        if (k < nk && c >= 0 && (SX || c < n)) acc[k] += a[u] * xv[c];
      }
  }
  for (; s < s_end; s += kMkW) {
    const double a = __ldg(col + (int64_t)s * ldmk);
#pragma unroll
    for (int k = 0; k < kMkKT; ++k) {
      const int c = s - (T - g - groups * k) * nu;
      if (k < nk && c >= 0 && (SX || c < n)) acc[k] += a * xv[c];
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
  // warp w takes stages t = t0 + w, t0 + w + 8, ..; P[(t, .), j] nonzero only for j < (t+1) nu
  for (int t = j / nu + w; t <= T; t += 8) {
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
  c.mk_T = c.mk_nu = c.mk_nchunks = c.mk_nx = 0;
  c.mk_inputs = false;
  c.markov = false;
}

bool markov_prepare(Ctx& c) {
  markov_free(c);
  const BuiltJ* bj = prob_rows(c);
  if (!c.opt_markov || !bj || c.m == 0 || c.n == 0 || bj->nu <= 0) return false;
  const int nx = bj->nx, nu = bj->nu, nc = bj->nc;
  const int64_t m = c.m, n = c.n;
  const int T = (int)(n / nu);
  if ((int64_t)T * nu != n) return false;
  const bool inputs = bj->KG != nullptr;  // without feedback the input rows are singletons
  const int nsrc = nx + nu + nc;
  cudaStream_t st = c.stream;
  const MkSrc src{bj->G, bj->KG, bj->EG, bj->F, nx, nu, nc, T};
  int32_t* used = dev_zeros<int32_t>(size_t(nsrc), st);
  int32_t* last = dev_alloc<int32_t>(size_t(nsrc), st);
  k_mk_used<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(static_cast<const RowDesc*>(bj->rows), m, nx, nu, inputs,
                                                      used);
  CMPC_LAUNCHED();
  k_mk_last<<<(unsigned)ceil_div(nsrc, 128), 128, 0, st>>>(src, nsrc, last);
  CMPC_LAUNCHED();
  std::vector<int32_t> hu((size_t)nsrc), hl((size_t)nsrc);
  CMPC_CUDA(cudaMemcpyAsync(hu.data(), used, sizeof(int32_t) * nsrc, cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaMemcpyAsync(hl.data(), last, sizeof(int32_t) * nsrc, cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaStreamSynchronize(st));
  dev_free(used, st);
  dev_free(last, st);
  std::vector<int32_t> order;
  for (int q = 0; q < nsrc; ++q)
    if (hu[size_t(q)] && hl[size_t(q)] >= 0) order.push_back(q);
  if (order.empty()) return false;
  // widest first: the window of q at stage t ends at L_q - (T - t) nu, so one order sorts
  // every stage by width, and a stage's nonzero rows are a prefix of it
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return hl[size_t(a)] > hl[size_t(b)]; });
  const int64_t nq = (int64_t)order.size();
  std::vector<int32_t> pos((size_t)nsrc, -1);
  for (int64_t q = 0; q < nq; ++q) pos[size_t(order[size_t(q)])] = (int32_t)q;
  // per stage t = 0..T: cnt_t = #{L_q >= (T - t) nu}, padded to chunks
  std::vector<int32_t> base(size_t(T + 2), 0), cnt(size_t(T + 1), 0);
  c.h_mk_chunk.clear();
  c.h_mk_width.clear();
  int64_t nz = 0;
  for (int t = 0; t <= T; ++t) {
    const int64_t lo = (int64_t)(T - t) * nu;
    while (nz < nq && hl[size_t(order[size_t(nz)])] >= lo) ++nz;
    const int64_t pc = round_up(nz, kBK);
    cnt[size_t(t)] = (int32_t)pc;
    base[size_t(t + 1)] = base[size_t(t)] + (int32_t)pc;
    for (int64_t q0 = 0; q0 < pc; q0 += kBK) {
      c.h_mk_chunk.push_back({(int)q0, (int)lo});
      c.h_mk_width.push_back((int32_t)(hl[size_t(order[size_t(q0)])] - lo + 1));
    }
  }
  const int64_t ps = base[size_t(T + 1)];
  if (ps == 0) return false;
  c.ldmk = round_up(nq, 32);
  c.mk_cols = (int64_t)(T + 1) * nu;
  c.mk_nq = nq;
  c.mk_T = T;
  c.mk_nu = nu;
  c.mk_ps = ps;
  c.mk_nchunks = (int)c.h_mk_chunk.size();
  c.mk_nx = nx;
  c.mk_inputs = inputs;
  // per 32-row table block: end of its nonzero columns (its first row's)
  std::vector<int32_t> rbend((size_t)(c.ldmk / 32));
  for (size_t b = 0; b < rbend.size(); ++b) {
    const int64_t q = (int64_t)b * 32;
    rbend[b] = q < nq ? hl[size_t(order[size_t(q)])] + 1 : 0;
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
  k_mk_fill<<<dim3((unsigned)ceil_div(nq, 256), (unsigned)c.mk_cols), 256, 0, st>>>(src, dorder, nq, c.ldmk, c.mk);
  CMPC_LAUNCHED();
  CMPC_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
  dev_free(dorder, st);
  return true;
}

void launch_markov_gemv(Ctx& c, const double* x, double* y) {
  if (c.ps > 0) {
    // stage groups: at most kMkKT stages per thread, and two CTAs per SM for small tables
    const int nrb = (int)(c.ldmk / 32);
    const int groups = std::min(c.mk_T + 1, std::max({4, (int)ceil_div(c.mk_T + 1, kMkKT), (int)ceil_div(296, nrb)}));
    const dim3 grid((unsigned)nrb, (unsigned)groups);
    const size_t sred = sizeof(double) * kMkW * kMkKT * 33, sx = sizeof(double) * (size_t)(c.n + c.mk_nu);
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
