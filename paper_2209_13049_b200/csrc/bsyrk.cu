// Lockstep-batch condensation (batch.cu, BASELINE config 5): for every active instance b
//     M_b(lower) = H + P' diag(omega_b) P + diag(singleton terms),   tq_b = P' q_b + singletons,
//     rhs_b = -r1_b + tq_b
// (assemble_condensed + gram_weighted, proj/src/ipm.cpp:72-77 and proj/src/dense_linalg.cpp:
// 128-137, and the right-hand side J'(r2 - sigma r3) of step_directions, ipm.cpp:79-103).
//
// All instances share P (the distinct rows of J, 14 MB at config 5: L2-resident) and its
// prefix-width order; n <= 160. ONE CTA per instance holds the instance's whole lower
// triangle in registers and streams P once:
// * output: the lower triangle in 16 x 16 REGIONS (55 at n = 160), dealt to 15 consumer
//   warps (at most 4 each) by a host plan that balances, SM sub-partition by sub-partition,
//   the work of every prefix of the row stream (rows are sorted by prefix width, so region
//   row I only starts once the rows reach column 16 I); diagonal regions skip their upper
//   8 x 8 block (one m16n8k4 + one m8n8k4);
// * operands: 32-row chunks of P staged by TMA (boxes {16 k, 32 cols}, 128B swizzle) through
//   a 4-stage mbarrier pipeline fed by one producer warp, only the column boxes the chunk's
//   prefix widths reach; omega_b and q_b ride the same barrier as 1-D bulk copies;
// * math: mma.sync m16n8k4 / m8n8k4 f64 (DMMA.8x8x4), omega applied to the A fragment in
//   registers, the diagonal regions' warps also form P'q from their B fragments (DFMA);
// * epilogue: H, the singleton diagonal and the singleton right-hand side added in place —
//   no partial tiles, no reduction kernel.
// Executed DMMA work is ~1.16x the algorithmic count at config 5 (the 64 x 64 tile form of
// syrk.cu executed 1.8x on this shape).
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "ptx.cuh"

namespace cmpc {

namespace {

constexpr int kBsWarps = 15;                       // consumer warps (16 with the producer: 128 registers)
constexpr int kBsThreads = (kBsWarps + 1) * 32;    // + one producer warp
constexpr int kBsRegs = 4;                         // regions per warp (max)
constexpr int kBsKC = 32;                          // P rows per chunk (= kBK, divides ldp)
constexpr int kBsColBoxes = 5;                     // 5 x 32 columns = 160 = kBatchMaxN
constexpr int kBsBox = 16 * 32 * 8;                // one {16 k, 32 cols} FP64 box (4 KB)
constexpr int kBsStageP = 2 * kBsColBoxes * kBsBox;  // 32 k x 160 cols
constexpr int kBsStageBytes = kBsStageP + 1024;      // + omega, q (256 B each), 1 KB aligned
constexpr int kBsStages = 5;
constexpr int kBsSmem = kBsStages * kBsStageBytes + 1024 /*align*/ + 2 * 8 * kBsStages /*barriers*/;
static_assert(kBsStageP % 1024 == 0, "128B-swizzled boxes need 1 KB alignment");
static_assert(kBsKC == kBK, "chunks must tile ldp");

struct BsArgs {
  const double* omega;  // per instance at stride py: ldp prototype weights, then singletons
  const double* q;
  int64_t py;
  const int2* chunks;  // per chunk in processing order: {first row, largest prefix width}
  int nchunks;
  int n;
  int64_t ldp;
  const double* H;
  double* M;  // per instance n x n, column-major (lower triangle written)
  const int32_t* sing_ptr;
  const double* sing_val;
  double* tq;
  double* rhs;
  const double* r1;
  const int* act;
  unsigned char reg[kBsWarps][kBsRegs];  // (I << 4) | J of each warp's regions, 0xff = none
};

// byte offset of the 8 columns starting at col (a multiple of 8) inside a stage's k-half
__device__ __forceinline__ int col_off(int col) { return (col >> 5) * kBsBox + (col & 31) * 128; }

// One chunk's MMAs for a warp whose first NA regions are active (regions sorted by row I, so
// the active ones are a prefix). Each region: 16 x 16 of the output as two m16n8k4 per k4
// step from two A fragments (columns 16I..) and two B fragments (columns 16J..) of the
// sqrt(omega)-scaled rows; a diagonal region computes its upper 8 x 8 block too (discarded).
// The warp's diagonal region (slot dslot) also sums P'q from its B fragments.
template <int NA>
__device__ __forceinline__ void bs_chunk(const unsigned char* st, const int (&offA)[kBsRegs],
                                         const int (&offB)[kBsRegs], int dslot, int g, int t,
                                         double (&acc)[kBsRegs][2][4], double (&rq)[2]) {
  const double* sw = reinterpret_cast<const double*>(st + kBsStageP);
  const double* sq = sw + 32;
#pragma unroll
  for (int k4 = 0; k4 < kBsKC / 4; ++k4) {
    // the k rows of this step: 16-byte chunks c and c ^ 4 of the 128-byte row (c = k4 & 3), so
    // that the lanes of each half-warp (g = 0..3 or 4..7, t = 0..3) hit 16 distinct 8-byte bank
    // pairs through the 128B swizzle (chunk ^ g); rows 4 k4 .. 4 k4 + 3 would give chunks
    // {c', c'+1} ^ g, shared by g and g ^ 1: two-way conflicts on every fragment load (ncu: 44%
    // of the shared wavefronts; removing them did not move the kernel's time). Any assignment of
    // the 32 rows to (k4, t) is valid as long as A, B, omega and q share it.
    const int kk = 2 * (k4 & 3) + (t & 1) + 8 * (t >> 1), k = 16 * (k4 >> 2) + kk;
    // this lane's element (col, k) of an 8-column group: the 128B swizzle XORs the 16-byte
    // chunk index with col & 7 = g
    const unsigned char* base = st + (k4 >> 2) * (kBsColBoxes * kBsBox) + g * 128 +
                                ((((kk >> 1) ^ g) << 4) | ((kk & 1) << 3));
    const double w = sw[k];
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int r = 0; r < NA; ++r) {
      const double b0 = *reinterpret_cast<const double*>(base + offB[r]);
      const double b1 = *reinterpret_cast<const double*>(base + offB[r] + 8 * 128);
      const double av[2] = {w * *reinterpret_cast<const double*>(base + offA[r]),
                            w * *reinterpret_cast<const double*>(base + offA[r] + 8 * 128)};
      dmma1684(acc[r][0], av, b0);
      dmma1684(acc[r][1], av, b1);
      if (r == dslot) {
        d0 = b0;
        d1 = b1;
      }
    }
    if (dslot < NA) {
      const double qk = sq[k];
      rq[0] = fma(qk, d0, rq[0]);
      rq[1] = fma(qk, d1, rq[1]);
    }
  }
}

__global__ void __launch_bounds__(kBsThreads, 1)
    k_bsyrk(const __grid_constant__ CUtensorMap tm, const __grid_constant__ BsArgs a) {
  const int b = blockIdx.x;
  if (!a.act[b]) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBsStages * kBsStageBytes);
  uint64_t* empty = full + kBsStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* omega = a.omega + b * a.py;
  const double* qv = a.q + b * a.py;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBsWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kBsWarps) {  // producer
    if (lane == 0) {
      for (int c = 0; c < a.nchunks; ++c) {
        const int s = c % kBsStages;
        if (c >= kBsStages) mbar_wait(&empty[s], ((c / kBsStages) - 1) & 1);
        const int2 ch = a.chunks[c];
        const int nb = (ch.y + 31) >> 5;
        unsigned char* st = smem + s * kBsStageBytes;
        // the consumers' generic-proxy reads of the stage before the TMA refills it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[s], (uint32_t)(2 * nb * kBsBox + 2 * kBsKC * 8));
        for (int kh = 0; kh < 2; ++kh)
          for (int cb = 0; cb < nb; ++cb)
            tma_load_2d(st + (kh * kBsColBoxes + cb) * kBsBox, &tm, ch.x + 16 * kh, 32 * cb, &full[s]);
        bulk_load(st + kBsStageP, omega + ch.x, kBsKC * 8, &full[s]);
        bulk_load(st + kBsStageP + 256, qv + ch.x, kBsKC * 8, &full[s]);
      }
    }
  } else {
    const int g = lane >> 2, t = lane & 3;
    int rI[kBsRegs], rJ[kBsRegs], offA[kBsRegs], offB[kBsRegs];
    int dslot = kBsRegs;
#pragma unroll
    for (int r = 0; r < kBsRegs; ++r) {
      const int e = a.reg[warp][r];
      rI[r] = e == 0xff ? 1 << 20 : e >> 4;  // never active
      rJ[r] = e == 0xff ? 0 : e & 15;
      offA[r] = e == 0xff ? 0 : col_off(16 * rI[r]);
      offB[r] = col_off(16 * rJ[r]);
      if (e != 0xff && rI[r] == rJ[r]) dslot = r;
    }
    double acc[kBsRegs][2][4];
#pragma unroll
    for (int r = 0; r < kBsRegs; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[r][h][x] = 0.0;
    double rq[2] = {0.0, 0.0};

    int h_next = a.nchunks > 0 ? __ldg(&a.chunks[0].y) : 0;  // read one chunk ahead
    for (int c = 0; c < a.nchunks; ++c) {
      const int s = c % kBsStages;
      const int h = h_next;
      if (c + 1 < a.nchunks) h_next = __ldg(&a.chunks[c + 1].y);
      int na = 0;
#pragma unroll
      for (int r = 0; r < kBsRegs; ++r) na += 16 * rI[r] < h;
      mbar_wait(&full[s], (c / kBsStages) & 1);
      const unsigned char* st = smem + s * kBsStageBytes;
      switch (na) {
        case 4: bs_chunk<4>(st, offA, offB, dslot, g, t, acc, rq); break;
        case 3: bs_chunk<3>(st, offA, offB, dslot, g, t, acc, rq); break;
        case 2: bs_chunk<2>(st, offA, offB, dslot, g, t, acc, rq); break;
        case 1: bs_chunk<1>(st, offA, offB, dslot, g, t, acc, rq); break;
        default: break;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---- epilogue
    asm volatile("bar.sync 1, %0;" ::"n"(kBsWarps * 32) : "memory");  // all stages consumed
    double* sdiag = reinterpret_cast<double*>(smem);  // stage 0 is free now
    double* srq = sdiag + 160;
    const int n = a.n;
    for (int i = threadIdx.x; i < n; i += kBsWarps * 32) {
      double ds = 0.0, dq = 0.0;
      for (int32_t k = a.sing_ptr[i]; k < a.sing_ptr[i + 1]; ++k) {
        const double sv = a.sing_val[k];
        ds += omega[a.ldp + k] * (sv * sv);
        dq += sv * qv[a.ldp + k];
      }
      sdiag[i] = ds;
      srq[i] = dq;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kBsWarps * 32) : "memory");
    double* M = a.M + (int64_t)b * n * n;
#pragma unroll
    for (int r = 0; r < kBsRegs; ++r) {
      if (rI[r] >= 16) continue;
      const int i0 = 16 * rI[r], j0 = 16 * rJ[r];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int i = i0 + g + 8 * (x >> 1);
          const int j = j0 + 8 * hh + 2 * t + (x & 1);
          if (i < n && j < n && i >= j) {
            double v = acc[r][hh][x];
            if (i == j) v += sdiag[i];
            M[i + (int64_t)j * n] = a.H[i + (int64_t)j * n] + v;
          }
        }
    }
    if (dslot < kBsRegs) {
      const int j0 = 16 * rJ[dslot];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        double v = rq[hh];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        const int col = j0 + 8 * hh + g;
        if (t == 0 && col < n) {
          const double s = v + srq[col];
          a.tq[(int64_t)b * n + col] = s;
          if (a.r1) a.rhs[(int64_t)b * n + col] = __dadd_rn(-a.r1[(int64_t)b * n + col], s);
        }
      }
    }
  }
}

}  // namespace

void syrk_plan_batch(Ctx& c, int64_t B, BatchSyrk& out, cudaStream_t st) {
  syrk_free_batch(out, st);
  const int n = (int)c.n;
  if (n > kBsColBoxes * 32) throw DimError("batch condensation: n > 160");
  out.B = B;
  // chunks of 32 rows from the first row with a nonzero prefix to the end of the SYRK rows
  const int ps = (int)c.ps;
  const int k_lo = std::min(ps, c.h_start_col[0]) / kBsKC * kBsKC;
  const int nch = ps > k_lo ? (ps - k_lo + kBsKC - 1) / kBsKC : 0;
  std::vector<int32_t> ch(size_t(std::max(nch, 1)), 0);
  for (int q = 0; q < nch; ++q) {
    const int last = std::min(ps - 1, k_lo + (q + 1) * kBsKC - 1);
    int hi = 0;  // prefix width of row `last`: the columns whose first nonzero row is <= last
    while (hi < n && c.h_start_col[size_t(hi)] <= last) ++hi;
    ch[size_t(q)] = hi;
  }
  // processing order: the widest chunk, then the narrowest, the next widest, ... — the work per
  // chunk stays near its mean, so the TMA runs kBsStages - 1 chunks ahead of compute
  // everywhere instead of the narrow head of the row order being latency-bound
  std::vector<int2> order;
  for (int lo = 0, hi = nch - 1; lo <= hi; --hi, ++lo) {
    order.push_back({k_lo + hi * kBsKC, ch[size_t(hi)]});
    if (lo < hi) order.push_back({k_lo + lo * kBsKC, ch[size_t(lo)]});
  }
  out.nchunks = nch;
  // regions in activation order, dealt to the SM sub-partitions (warp % 4) by least load so far
  // (balancing per warp instead — longest-processing-time over the 15 warps, then the warps
  // over the sub-partitions — left the sub-partitions 8% apart and ran 6% slower)
  const int nr = (n + 15) / 16;
  std::vector<std::pair<int, int>> regs;
  for (int I = 0; I < nr; ++I)
    for (int J = 0; J <= I; ++J) regs.push_back({I, J});
  std::memset(out.reg, 0xff, sizeof(out.reg));
  double load[4] = {0, 0, 0, 0};
  int used[kBsWarps] = {0};
  bool has_diag[kBsWarps] = {false};  // one diagonal region per warp (its P'q accumulators)
  auto fits = [&](int w, bool dg) { return used[w] < kBsRegs && !(dg && has_diag[w]); };
  for (auto [I, J] : regs) {
    const bool dg = I == J;
    double wgt = 0.0;
    for (int q = 0; q < nch; ++q)
      if (16 * I < ch[size_t(q)]) wgt += dg ? 3.0 : 4.0;
    int best = -1;
    for (int p = 0; p < 4; ++p) {
      bool free_slot = false;
      for (int w = p; w < kBsWarps; w += 4) free_slot |= fits(w, dg);
      if (free_slot && (best < 0 || load[p] < load[best])) best = p;
    }
    if (best < 0) throw DimError("batch condensation: no warp slot left for a region");
    int ww = -1;
    for (int w = best; w < kBsWarps; w += 4)
      if (fits(w, dg) && (ww < 0 || used[w] < used[ww])) ww = w;
    out.reg[ww][used[ww]++] = (unsigned char)(I << 4 | J);
    has_diag[ww] |= dg;
    load[best] += wgt;
  }
  for (int w = 0; w < kBsWarps; ++w)  // active regions form a prefix: sort by row I
    std::sort(out.reg[w], out.reg[w] + used[w]);
  if (order.empty()) order.push_back({0, 0});
  out.chunks = dev_alloc<int2>(order.size(), st);
  CMPC_CUDA(cudaMemcpyAsync(out.chunks, order.data(), sizeof(int2) * order.size(), cudaMemcpyHostToDevice, st));
  static std::once_flag flags[kMaxDevices];
  once_per_device(flags, c.device, [] {
    CMPC_CUDA(cudaFuncSetAttribute(k_bsyrk, cudaFuncAttributeMaxDynamicSharedMemorySize, kBsSmem));
  });
  // algorithmic work of one instance: sum over the SYRK rows of hi (hi + 1)
  double f = 0.0;
  for (int64_t k = 0; k < ps; ++k) {
    int hi = 0;
    while (hi < n && c.h_start_col[size_t(hi)] <= k) ++hi;
    f += (double)hi * (hi + 1);
  }
  out.flops_per_instance = f;
  CMPC_CUDA(cudaStreamSynchronize(st));
}

void syrk_free_batch(BatchSyrk& b, cudaStream_t st) {
  dev_free(b.chunks, st);
  b = BatchSyrk{};
}

void launch_condense_batch(Ctx& c, BatchSyrk& bs, cudaStream_t st, const double* omega, const double* q,
                           int64_t s_proto, double* M, double* tq, double* rhs, const double* r1,
                           const int* act) {
  BsArgs a;
  a.omega = omega;
  a.q = q;
  a.py = s_proto;
  a.chunks = bs.chunks;
  a.nchunks = bs.nchunks;
  a.n = (int)c.n;
  a.ldp = c.ldp;
  a.H = c.H;
  a.M = M;
  a.sing_ptr = c.sing_ptr;
  a.sing_val = c.sing_val;
  a.tq = tq;
  a.rhs = rhs;
  a.r1 = r1;
  a.act = act;
  std::memcpy(a.reg, bs.reg, sizeof(a.reg));
  if ((reinterpret_cast<uintptr_t>(omega) | reinterpret_cast<uintptr_t>(q) | (uintptr_t)(s_proto * 8)) & 15)
    throw CudaError("batch condensation: omega/q not 16-byte aligned for the bulk copies (" +
                    std::to_string(reinterpret_cast<uintptr_t>(omega) & 255) + ", " +
                    std::to_string(reinterpret_cast<uintptr_t>(q) & 255) + ")");
  const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(c.tmap_P32);
  k_bsyrk<<<(unsigned)bs.B, kBsThreads, kBsSmem, st>>>(*tm, a);
  CMPC_LAUNCHED();
}

}  // namespace cmpc
