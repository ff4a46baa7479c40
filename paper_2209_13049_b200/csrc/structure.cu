// Exact structure analysis of the constraint Jacobian J (once per loaded QP).
//
// The reference multiplies the dense J in every pass (proj/src/ipm.cpp:53-56, :88,
// :93, :126, :129; proj/src/dense_linalg.cpp:133-134). Its rows repeat with a sign
// flip (upper/lower bounds: proj/src/reduction.cpp:205-248) and most of each row is
// a zero suffix (state row at stage t spans t*n_u columns). This pass finds, bit
// exactly, the distinct rows of J up to sign ("prototypes") so that
//   J v      = Pi (P v),        J' y = P' (Pi' y),        J' S J = P' diag(Pi' sigma) P
// with Pi the signed row->prototype selection. Nothing is assumed about the layout:
// rows are hashed after sign normalisation, grouped by a stable radix sort and every
// group member is verified element by element against its leader; a hash run with any
// mismatch falls back to one prototype per row.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "internal.cuh"
#include "jrows.cuh"

namespace cmpc {

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

// per row: first/last nonzero, count, sign of the first nonzero, hash of the
// sign-normalised row
template <class JA>
__global__ void k_row_summary(JA J, int64_t m, int64_t n, unsigned long long* key, int32_t* lo, int32_t* hi,
                              int32_t* nnz, int8_t* sg, int32_t* idx) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const auto row = J.row(r);
  unsigned long long h = 0x84222325cbf29ce4ull;
  int first = -1, last = -1, cnt = 0;
  double sign = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    const double a = row(j);
    if (a != 0.0) {
      if (first < 0) {
        first = (int)j;
        sign = a > 0.0 ? 1.0 : -1.0;
      }
      last = (int)j;
      ++cnt;
      const unsigned long long bits = (unsigned long long)__double_as_longlong(a * sign);
      h = mix64(h ^ (bits + 0x9e3779b97f4a7c15ull * (unsigned long long)(j + 1)));
    }
  }
  key[r] = mix64(h ^ ((unsigned long long)cnt << 32));
  lo[r] = first;
  hi[r] = last + 1;
  nnz[r] = cnt;
  sg[r] = sign < 0.0 ? -1 : 1;
  idx[r] = (int32_t)r;
}

__global__ void k_head0(const unsigned long long* key, int64_t m, int32_t* head_pos) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  head_pos[i] = (i == 0 || key[i] != key[i - 1]) ? (int32_t)i : 0;
}

// leader row of every row (in original row order) for coalesced verification
__global__ void k_leader_of_row(const int32_t* srow, const int32_t* lead_pos, int64_t m,
                                int32_t* leader_row, int32_t* run_of_row) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int32_t r = srow[i];
  leader_row[r] = srow[lead_pos[i]];
  run_of_row[r] = lead_pos[i];
}

template <class JA>
__global__ void k_verify(JA J, int64_t m, int64_t n, const int32_t* leader_row, const int32_t* run_of_row,
                         const int8_t* sg, int32_t* collide) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const int32_t l = leader_row[r];
  if (l == r) return;
  const double s = (sg[r] == sg[l]) ? 1.0 : -1.0;
  bool eq = true;
  const auto rr = J.row(r), rl = J.row(l);
  for (int64_t j = 0; j < n && eq; ++j) eq = (rr(j) == s * rl(j));
  if (!eq) collide[run_of_row[r]] = 1;
}

__global__ void k_heads(const int32_t* lead_pos, const int32_t* collide, int64_t m,
                        int32_t* head) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  head[i] = (lead_pos[i] == i || collide[lead_pos[i]]) ? 1 : 0;
}

// group info at head positions
__global__ void k_group_info(const int32_t* head, const int32_t* gid, const int32_t* srow,
                             const int32_t* hi, const int32_t* nnz, int64_t m,
                             int32_t* first_pos, unsigned long long* key2, int32_t* gidx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m || !head[i]) return;
  const int32_t g = gid[i] - 1;
  const int32_t r = srow[i];
  first_pos[g] = (int32_t)i;
  const unsigned long long single = nnz[r] <= 1 ? 1ull : 0ull;
  // SYRK prototypes by prefix width, singletons by their column; ties by leader row
  const unsigned long long w = single ? (unsigned long long)(hi[r] > 0 ? hi[r] : 0)
                                      : (unsigned long long)hi[r];
  key2[g] = (single << 62) | (w << 32) | (unsigned long long)r;
  gidx[g] = g;
}

__global__ void k_proto_of_group(const int32_t* gorder, int64_t G, int32_t* proto_of_group) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= G) return;
  proto_of_group[gorder[k]] = (int32_t)k;
}

__global__ void k_group_size(const int32_t* first_pos, int64_t G, int64_t m,
                             const int32_t* proto_of_group, int32_t* size_by_proto) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int32_t end = (g + 1 < G) ? first_pos[g + 1] : (int32_t)m;
  size_by_proto[proto_of_group[g]] = end - first_pos[g];
}

// row_map addresses prototype-indexed vectors: SYRK prototypes at [0, ps), singletons
// at [ldp, ldp + pz)
// gflip (Markov layout, else null): the group's table row is the NEGATED leader (a lower-bound
// leader row is -[G_{t-1} .. G_0] row i; the table holds +G)
__global__ void k_row_map(const int32_t* srow, const int32_t* gid, const int32_t* first_pos,
                          const int32_t* proto_of_group, const int32_t* mem_ptr,
                          const int8_t* sg, int64_t m, int64_t ps, int64_t ldp, int32_t* row_map,
                          int32_t* mem_rows, const int32_t* gflip) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int32_t g = gid[i] - 1;
  const int32_t r = srow[i];
  const int32_t lead = srow[first_pos[g]];
  const int32_t pr = proto_of_group[g];
  const int32_t neg = (sg[r] != sg[lead] ? 1 : 0) ^ (gflip ? gflip[g] : 0);
  const int32_t yi = pr < ps ? pr : (int32_t)(ldp + (pr - ps));
  row_map[r] = (yi << 1) | neg;
  mem_rows[mem_ptr[pr] + (int32_t)(i - first_pos[g])] = (r << 1) | neg;
}

__global__ void k_proto_leader(const int32_t* gorder, const int32_t* first_pos,
                               const int32_t* srow, int64_t G, int32_t* proto_leader) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= G) return;
  proto_leader[k] = srow[first_pos[gorder[k]]];
}

// P[k, j] = J[leader_k, j] for j < hi_k (P pre-zeroed); singletons separately
template <class JA>
__global__ void k_gather_P(JA J, const int32_t* leader, const int32_t* hi_row, int64_t ps, int64_t n,
                           int64_t ldp, double* P, int32_t* hi) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= ps) return;
  const int32_t l = leader[k];
  const int32_t w = hi_row[l];
  hi[k] = w;
  const int64_t j0 = blockIdx.y;
  const auto row = J.row(l);
  for (int64_t j = j0; j < w; j += gridDim.y) P[k + j * ldp] = row(j);
}

template <class JA>
__global__ void k_singletons(JA J, const int32_t* leader, const int32_t* lo_row, int64_t ps, int64_t pz,
                             int32_t* sing_col, double* sing_val) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= pz) return;
  const int32_t l = leader[ps + k];
  const int32_t c = lo_row[l];
  sing_col[k] = c < 0 ? 0 : c;
  sing_val[k] = c < 0 ? 0.0 : J.row(l)(c);
}

// Markov layout: prototype k (standard order, k < ps) -> its leader's row of the table at
// its stage; flags a leader outside the table (then P is materialised after all)
__global__ void k_mk_remap(const int32_t* leader, int64_t ps, const RowDesc* rows,
                           const int32_t* pos, const int32_t* base, int nx, int nu, bool inputs,
                           int32_t* remap, int32_t* flip, int32_t* bad) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= ps) return;
  const RowDesc q = rows[leader[k]];
  // the table's source of the row: state, input (feedback only), mixed
  const int src = q.kind == 1 ? q.i : q.kind == 2 ? (inputs ? nx + q.i : -1) : nx + nu + q.i;
  const int32_t p = src >= 0 ? pos[src] : -1;
  if (p < 0) {
    *bad = 1;
    remap[k] = 0;
    flip[k] = 0;
    return;
  }
  remap[k] = base[q.t] + p;
  flip[k] = q.upper ? 0 : 1;  // the table holds the upper-bound orientation (+G)
}

__global__ void k_mk_groups(const int32_t* proto_of_group, int64_t G, int64_t ps, int64_t ps_mk,
                            const int32_t* remap, const int32_t* flip, int32_t* out, int32_t* gflip) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int32_t k = proto_of_group[g];
  out[g] = k < ps ? remap[k] : (int32_t)(ps_mk + (k - ps));
  gflip[g] = k < ps ? flip[k] : 0;
}

__global__ void k_mk_hi(const int32_t* leader, const int32_t* hi_row, int64_t ps,
                        const int32_t* remap, int32_t* hi) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= ps) return;
  hi[remap[k]] = hi_row[leader[k]];
}

__global__ void k_start_col(const int32_t* hi, int64_t ps, int64_t n, int32_t* start_col) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > n) return;
  int64_t lo = 0, up = ps;  // first k with hi[k] > c
  while (lo < up) {
    const int64_t mid = (lo + up) / 2;
    if (hi[mid] > c) up = mid;
    else lo = mid + 1;
  }
  start_col[c] = (int32_t)lo;
}


}  // namespace

void free_structure(Ctx& c) {
  for (void* p : {(void*)c.P, (void*)c.hi, (void*)c.start_col, (void*)c.row_map,
                  (void*)c.mem_ptr, (void*)c.mem_rows, (void*)c.sing_col, (void*)c.sing_val})
    dev_free(p, c.stream);
  c.P = nullptr;
  c.hi = c.start_col = c.row_map = c.mem_ptr = c.mem_rows = c.sing_col = nullptr;
  c.sing_val = nullptr;
}

template <class JA>
void analyze_impl(Ctx& c, const JA& J, const MarkovRemap* mk) {
  free_structure(c);
  const int64_t m = c.m, n = c.n;
  cudaStream_t st = c.stream;
  (void)0;
  c.start_col = dev_alloc<int32_t>(size_t(n + 1), st);
  if (m == 0) {
    c.ps = c.pz = c.p = 0;
    c.ldp = kBK;
    c.P = dev_alloc<double>(size_t(c.ldp * std::max<int64_t>(n, 1)), st);
    CMPC_CUDA(cudaMemsetAsync(c.P, 0, sizeof(double) * c.ldp * std::max<int64_t>(n, 1), st));
    CMPC_CUDA(cudaMemsetAsync(c.start_col, 0, sizeof(int32_t) * (n + 1), st));
    c.h_start_col.assign(size_t(n + 1), 0);
    c.mem_ptr = dev_alloc<int32_t>(1, st);
    CMPC_CUDA(cudaMemsetAsync(c.mem_ptr, 0, sizeof(int32_t), st));
    return;
  }
  const int T = 256;
  const unsigned gm = unsigned((m + T - 1) / T);

  auto* key = dev_alloc<unsigned long long>(m, st);
  auto* key_s = dev_alloc<unsigned long long>(m, st);
  auto* lo = dev_alloc<int32_t>(m, st);
  auto* hi_row = dev_alloc<int32_t>(m, st);
  auto* nnz = dev_alloc<int32_t>(m, st);
  auto* sg = dev_alloc<int8_t>(m, st);
  auto* idx = dev_alloc<int32_t>(m, st);
  auto* srow = dev_alloc<int32_t>(m, st);
  auto* head_pos = dev_alloc<int32_t>(m, st);
  auto* lead_pos = dev_alloc<int32_t>(m, st);
  auto* leader_row = dev_alloc<int32_t>(m, st);
  auto* run_of_row = dev_alloc<int32_t>(m, st);
  auto* collide = dev_alloc<int32_t>(m, st);
  auto* head = dev_alloc<int32_t>(m, st);
  auto* gid = dev_alloc<int32_t>(m, st);

  k_row_summary<<<gm, T, 0, st>>>(J, m, n, key, lo, hi_row, nnz, sg, idx);
  CMPC_LAUNCHED();

  size_t tmp_bytes = 0, need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, key, key_s, idx, srow, (int)m, 0, 64, st);
  tmp_bytes = std::max(tmp_bytes, need);
  cub::DeviceScan::InclusiveScan(nullptr, need, head_pos, lead_pos, cub::Max(), (int)m, st);
  tmp_bytes = std::max(tmp_bytes, need);
  cub::DeviceScan::InclusiveSum(nullptr, need, head, gid, (int)m, st);
  tmp_bytes = std::max(tmp_bytes, need);
  cub::DeviceScan::ExclusiveSum(nullptr, need, head, gid, (int)m + 1, st);
  tmp_bytes = std::max(tmp_bytes, need);
  // group sort and member pointer scan use at most m items as well
  auto* tmp = dev_alloc<unsigned char>(tmp_bytes + 256, st);

  CMPC_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key_s, idx, srow, (int)m, 0, 64, st));
  k_head0<<<gm, T, 0, st>>>(key_s, m, head_pos);
  CMPC_LAUNCHED();
  CMPC_CUDA(cub::DeviceScan::InclusiveScan(tmp, tmp_bytes, head_pos, lead_pos, cub::Max(), (int)m, st));
  k_leader_of_row<<<gm, T, 0, st>>>(srow, lead_pos, m, leader_row, run_of_row);
  CMPC_LAUNCHED();
  CMPC_CUDA(cudaMemsetAsync(collide, 0, sizeof(int32_t) * m, st));
  k_verify<<<gm, T, 0, st>>>(J, m, n, leader_row, run_of_row, sg, collide);
  CMPC_LAUNCHED();
  k_heads<<<gm, T, 0, st>>>(lead_pos, collide, m, head);
  CMPC_LAUNCHED();
  CMPC_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, head, gid, (int)m, st));
  int32_t G = 0;
  CMPC_CUDA(cudaMemcpyAsync(&G, gid + m - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaStreamSynchronize(st));

  auto* first_pos = dev_alloc<int32_t>(G, st);
  auto* key2 = dev_alloc<unsigned long long>(G, st);
  auto* key2_s = dev_alloc<unsigned long long>(G, st);
  auto* gidx = dev_alloc<int32_t>(G, st);
  auto* gorder = dev_alloc<int32_t>(G, st);
  auto* proto_of_group = dev_alloc<int32_t>(G, st);
  auto* size_by_proto = dev_alloc<int32_t>(G + 1, st);
  auto* leader = dev_alloc<int32_t>(G, st);
  const unsigned gg = unsigned((G + T - 1) / T);
  k_group_info<<<gm, T, 0, st>>>(head, gid, srow, hi_row, nnz, m, first_pos, key2, gidx);
  CMPC_LAUNCHED();
  CMPC_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key2, key2_s, gidx, gorder, G, 0, 64, st));
  k_proto_of_group<<<gg, T, 0, st>>>(gorder, G, proto_of_group);
  CMPC_LAUNCHED();
  CMPC_CUDA(cudaMemsetAsync(size_by_proto, 0, sizeof(int32_t) * (G + 1), st));
  k_group_size<<<gg, T, 0, st>>>(first_pos, G, m, proto_of_group, size_by_proto);
  CMPC_LAUNCHED();
  c.mem_ptr = dev_alloc<int32_t>(G + 1, st);
  CMPC_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, size_by_proto, c.mem_ptr, G + 1, st));
  k_proto_leader<<<gg, T, 0, st>>>(gorder, first_pos, srow, G, leader);
  CMPC_LAUNCHED();

  // split point between SYRK prototypes and singletons
  std::vector<unsigned long long> hk(static_cast<size_t>(G));
  CMPC_CUDA(cudaMemcpyAsync(hk.data(), key2_s, sizeof(unsigned long long) * G,
                            cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaStreamSynchronize(st));
  int64_t ps = std::lower_bound(hk.begin(), hk.end(), 1ull << 62) - hk.begin();
  // the Markov layout (markov.cu) replaces the prototype order of the SYRK part: prototype k
  // moves to its leader's table row at its stage, the layout's other rows are empty
  // prototypes (no member rows: weight 0, zero rows of the table)
  int32_t* remap = nullptr;
  int32_t* gflip = nullptr;
  int64_t ps_l = ps;  // prototype rows of the layout
  if (mk) {
    remap = dev_alloc<int32_t>(size_t(std::max<int64_t>(ps, 1)), st);
    int32_t* flip = dev_alloc<int32_t>(size_t(std::max<int64_t>(ps, 1)), st);
    int32_t* bad = dev_zeros<int32_t>(1, st);
    if (ps > 0) {
      k_mk_remap<<<unsigned((ps + T - 1) / T), T, 0, st>>>(leader, ps, static_cast<const RowDesc*>(mk->rows),
                                                          mk->pos, mk->base, mk->nx, mk->nu, mk->inputs,
                                                          remap, flip, bad);
      CMPC_LAUNCHED();
    }
    int32_t hb = 0;
    CMPC_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CMPC_CUDA(cudaStreamSynchronize(st));
    dev_free(bad, st);
    // declined: a prototype that is not a state row, a layout mostly made of empty rows
    // (duplicate-heavy J: the table would multiply rows the analysis merged), or (option 1)
    // a P small enough to stay in L2
    const double p_bytes = 8.0 * (double)round_up(std::max<int64_t>(ps, 1), kBK) * (double)n;
    if (hb || mk->ps > 2 * ps + 4096 || (!mk->force && p_bytes < kMarkovMinBytes)) {
      dev_free(remap, st);
      remap = nullptr;
    } else {
      ps_l = mk->ps;
      const int64_t Gl = ps_l + (G - ps);
      auto* pog = dev_alloc<int32_t>(G, st);
      gflip = dev_alloc<int32_t>(G, st);
      k_mk_groups<<<gg, T, 0, st>>>(proto_of_group, G, ps, ps_l, remap, flip, pog, gflip);
      CMPC_LAUNCHED();
      dev_free(proto_of_group, st);
      proto_of_group = pog;
      dev_free(size_by_proto, st);
      size_by_proto = dev_zeros<int32_t>(size_t(Gl + 1), st);
      k_group_size<<<gg, T, 0, st>>>(first_pos, G, m, proto_of_group, size_by_proto);
      CMPC_LAUNCHED();
      dev_free(c.mem_ptr, st);
      c.mem_ptr = dev_alloc<int32_t>(size_t(Gl + 1), st);
      size_t need2 = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, need2, size_by_proto, c.mem_ptr, (int)(Gl + 1), st);
      if (need2 > tmp_bytes) {
        dev_free(tmp, st);
        tmp_bytes = need2;
        tmp = dev_alloc<unsigned char>(tmp_bytes + 256, st);
      }
      CMPC_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, size_by_proto, c.mem_ptr, (int)(Gl + 1), st));
    }
    dev_free(flip, st);
  }
  c.markov = remap != nullptr;
  c.ps = ps_l;
  c.p = ps_l + (G - ps);
  c.pz = G - ps;
  c.ldp = round_up(std::max<int64_t>(ps_l, 1), kBK);
  c.row_map = dev_alloc<int32_t>(m, st);
  c.mem_rows = dev_alloc<int32_t>(m, st);
  k_row_map<<<gm, T, 0, st>>>(srow, gid, first_pos, proto_of_group, c.mem_ptr, sg, m, ps_l, c.ldp,
                              c.row_map, c.mem_rows, gflip);
  CMPC_LAUNCHED();
  dev_free(gflip, st);

  if (c.markov) {  // P stays implicit; prefix widths for the work count
    c.hi = dev_zeros<int32_t>(size_t(std::max<int64_t>(ps_l, 1)), st);
    if (ps > 0) {
      k_mk_hi<<<unsigned((ps + T - 1) / T), T, 0, st>>>(leader, hi_row, ps, remap, c.hi);
      CMPC_LAUNCHED();
    }
    dev_free(remap, st);
  } else {
    c.P = dev_alloc<double>(size_t(c.ldp * n), st);
    CMPC_CUDA(cudaMemsetAsync(c.P, 0, sizeof(double) * c.ldp * n, st));
    c.hi = dev_alloc<int32_t>(ps, st);
    if (ps > 0) {
      dim3 grid(unsigned((ps + T - 1) / T), unsigned(std::min<int64_t>(n, 64)));
      k_gather_P<<<grid, T, 0, st>>>(J, leader, hi_row, ps, n, c.ldp, c.P, c.hi);
      CMPC_LAUNCHED();
    }
  }
  c.sing_col = dev_alloc<int32_t>(c.pz, st);
  c.sing_val = dev_alloc<double>(c.pz, st);
  if (c.pz > 0) {
    k_singletons<<<unsigned((c.pz + T - 1) / T), T, 0, st>>>(J, leader, lo, ps, c.pz, c.sing_col,
                                                             c.sing_val);
    CMPC_LAUNCHED();
  }
  // all-zero rows sort first among the singletons (prefix width 0, value 0)
  c.zero_k = -1;
  if (c.pz > 0) {
    double v0 = 1.0;
    CMPC_CUDA(cudaMemcpyAsync(&v0, c.sing_val, sizeof(double), cudaMemcpyDeviceToHost, st));
    CMPC_CUDA(cudaStreamSynchronize(st));
    if (v0 == 0.0) c.zero_k = ps_l;
  }
  if (c.markov) {  // (rows are stage-major, not sorted by width: the plan uses chunk lists)
    CMPC_CUDA(cudaMemsetAsync(c.start_col, 0, sizeof(int32_t) * (n + 1), st));
  } else {
    k_start_col<<<unsigned((n + 1 + T - 1) / T), T, 0, st>>>(c.hi, ps, n, c.start_col);
    CMPC_LAUNCHED();
  }
  c.h_start_col.resize(size_t(n + 1));
  CMPC_CUDA(cudaMemcpyAsync(c.h_start_col.data(), c.start_col, sizeof(int32_t) * (n + 1),
                            cudaMemcpyDeviceToHost, st));
  CMPC_CUDA(cudaStreamSynchronize(st));

  for (void* p : {(void*)key, (void*)key_s, (void*)lo, (void*)hi_row, (void*)nnz, (void*)sg,
                  (void*)idx, (void*)srow, (void*)head_pos, (void*)lead_pos, (void*)leader_row,
                  (void*)run_of_row, (void*)collide, (void*)head, (void*)gid, (void*)tmp,
                  (void*)first_pos, (void*)key2, (void*)key2_s, (void*)gidx, (void*)gorder,
                  (void*)proto_of_group, (void*)size_by_proto, (void*)leader})
    dev_free(p, st);
}

void analyze_structure(Ctx& c) {
  markov_free(c);
  analyze_impl(c, DenseJ{c.J, c.m}, nullptr);
}
void analyze_structure_built(Ctx& c, const BuiltJ& J) {
  c.markov = false;
  const bool mk = markov_prepare(c);  // the table + layout (false: not applicable)
  const MarkovRemap mr{J.rows, c.mk_pos, c.mk_base, c.mk_ps, c.opt_markov == 2, c.mk_nx, c.mk_nu, c.mk_inputs};
  analyze_impl(c, J, mk ? &mr : nullptr);
  if (mk && !c.markov) markov_free(c);  // declined by the analysis
}

}  // namespace cmpc
