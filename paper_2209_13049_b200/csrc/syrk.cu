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
// * math: mma.sync m16n8k16 f64 (DMMA.8x8x4), 4 consumer warps x (32x32) per 64x64 tile.
// * zero-block skipping: rows are sorted by nonzero prefix width; tile (I,J) (I>=J) only
//   visits the rows whose prefix reaches column 64*I.
// * split-K: (tile, k-chunk) work units with globally aligned chunks so concurrently
//   running units share P rows in L2; partial tiles are summed in a fixed order by
//   k_syrk_reduce (bitwise deterministic run to run).
#include <cuda.h>

#include <algorithm>
#include <functional>
#include <queue>
#include <vector>

#include "internal.cuh"
#include "ptx.cuh"

namespace cmpc {

namespace {

constexpr int kStages = 3;
constexpr int kBoxBytes = 16 * 64 * 8;          // {16 k, 64 cols} FP64 box
constexpr int kOpBytes = 2 * kBoxBytes;         // 32 k x 64 cols
constexpr int kStageBytes = 2 * kOpBytes + 1024;  // A, B, omega (256 B, padded to 1 KB)
constexpr int kSyrkSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kConsumerWarps = 4;
constexpr int kSyrkThreads = (kConsumerWarps + 1) * 32;

// byte offset of element (col c, k) inside a 32 x 64 operand tile (two swizzled boxes)
__device__ __forceinline__ uint32_t op_off(int c, int k) {
  const int kk = k & 15;
  return (uint32_t)((k >> 4) * kBoxBytes + c * 128 + ((((kk >> 1) ^ (c & 7)) << 4) | ((kk & 1) << 3)));
}

__global__ void __launch_bounds__(kSyrkThreads, 2)
    k_syrk(const __grid_constant__ CUtensorMap tmP, const double* __restrict__ omega,
           const int4* __restrict__ units, double* __restrict__ partial) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;

  const int4 u = units[blockIdx.x];
  const int ti = u.x, tj = u.y, k0 = u.z, k1 = u.w;
  const bool diag = ti == tj;
  const int nsteps = (k1 - k0) / kBK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(diag ? kOpBytes : 2 * kOpBytes) + kBK * 8;
      for (int it = 0; it < nsteps; ++it) {
        const int s = it % kStages;
        if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        unsigned char* st = smem + s * kStageBytes;
        const int kk = k0 + it * kBK;
        mbar_expect_tx(&full[s], bytes);
        tma_load_2d(st, &tmP, kk, 64 * ti, &full[s]);
        tma_load_2d(st + kBoxBytes, &tmP, kk + 16, 64 * ti, &full[s]);
        if (!diag) {
          tma_load_2d(st + kOpBytes, &tmP, kk, 64 * tj, &full[s]);
          tma_load_2d(st + kOpBytes + kBoxBytes, &tmP, kk + 16, 64 * tj, &full[s]);
        }
        bulk_load(st + 2 * kOpBytes, omega + kk, kBK * 8, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers: warp (wm, wn) owns rows 32*wm.., cols 32*wn.. of the tile
  const int wm = warp & 1, wn = warp >> 1;
  const bool skip = diag && wm == 0 && wn == 1;  // strictly upper block of a diagonal tile
  const int g = lane >> 2, t = lane & 3;
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  for (int it = 0; it < nsteps; ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (it / kStages) & 1);
    if (!skip) {
      // explicit 32-bit shared addresses: the aligned generic pointer would compile to LD
      // (global-load scoreboard latency) instead of LDS
      const uint32_t sA = smem_u32(smem + s * kStageBytes);
      const uint32_t sB = diag ? sA : sA + kOpBytes;
      const uint32_t sW = sA + 2 * kOpBytes;
#pragma unroll
      for (int ks = 0; ks < kBK; ks += 16) {
        double af[2][8], bf[4][4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            const int c = 32 * wm + 16 * mi + g + 8 * (x & 1);
            const int k = ks + t + 4 * (x >> 1);
            af[mi][x] = lds64(sA + op_off(c, k));
          }
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int c = 32 * wn + 8 * ni + g;
            const int k = ks + t + 4 * x;
            bf[ni][x] = lds64(sW + 8 * k) * lds64(sB + op_off(c, k));
          }
        }
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma16816(acc[mi][ni], af[mi], bf[ni]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (skip) return;
  double* out = partial + (size_t)blockIdx.x * (kTile * kTile);
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int r = 32 * wm + 16 * mi + g;
      const int c = 32 * wn + 8 * ni + 2 * t;
      out[c * kTile + r] = acc[mi][ni][0];
      out[(c + 1) * kTile + r] = acc[mi][ni][1];
      out[c * kTile + r + 8] = acc[mi][ni][2];
      out[(c + 1) * kTile + r + 8] = acc[mi][ni][3];
    }
}

// M(i,j) = H(i,j) + (sum over the tile's units in k order [+ singleton diagonal]), lower;
// grid (tiles, 16): 256 elements of one tile per block
__global__ void k_syrk_reduce(const double* __restrict__ partial, const int2* __restrict__ tiles,
                              const int32_t* __restrict__ tile_ptr,
                              const int32_t* __restrict__ tile_units, const double* __restrict__ H,
                              const double* __restrict__ dsing, int64_t n, double* __restrict__ M,
                              int mirror) {
  const int2 tl = tiles[blockIdx.x];
  const int u0 = tile_ptr[blockIdx.x], u1 = tile_ptr[blockIdx.x + 1];
  const int e = blockIdx.y * blockDim.x + threadIdx.x;
  const int rl = e & (kTile - 1), cl = e >> 6;
  const int64_t i = (int64_t)kTile * tl.x + rl, j = (int64_t)kTile * tl.y + cl;
  if (i >= n || j >= n || i < j) return;
  double s0 = 0.0, s1 = 0.0;
  int q = u0;
  for (; q + 1 < u1; q += 2) {
    s0 += partial[(size_t)tile_units[q] * (kTile * kTile) + e];
    s1 += partial[(size_t)tile_units[q + 1] * (kTile * kTile) + e];
  }
  if (q < u1) s0 += partial[(size_t)tile_units[q] * (kTile * kTile) + e];
  double s = s0 + s1;
  if (i == j) s += dsing[i];
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
  for (void* p : {(void*)c.units, (void*)c.tile_ptr, (void*)c.tile_units, (void*)c.tiles,
                  (void*)c.partial})
    dev_free(p, c.stream);
  c.units = nullptr;
  c.tile_ptr = c.tile_units = nullptr;
  c.tiles = nullptr;
  c.partial = nullptr;
  delete[] reinterpret_cast<unsigned char*>(c.tmap_P);
  c.tmap_P = nullptr;
}

void syrk_plan(Ctx& c) {
  syrk_free(c);
  const int64_t n = c.n;
  const int nt = (int)ceil_div(n, kTile);
  std::vector<int2> tiles;
  std::vector<std::pair<int, int>> range;  // per tile [k_begin, k_end)
  const int k_end = (int)c.ldp;
  int64_t total = 0;
  for (int tj = 0; tj < nt; ++tj)
    for (int ti = tj; ti < nt; ++ti) {
      tiles.push_back({ti, tj});
      int kb = c.ps > 0 ? c.h_start_col[size_t(std::min<int64_t>(n, (int64_t)kTile * ti))] : k_end;
      kb = kb / kBK * kBK;
      if (c.ps == 0) kb = k_end;
      range.push_back({kb, k_end});
      total += std::max(0, k_end - kb);
    }
  // split-K chunk: the (tile, chunk) units run in k-major order (concurrent units share P
  // rows in L2) and the hardware dispatches them in order onto 2 CTAs per SM. Pick the chunk
  // by simulating that list schedule (cost = k-steps + a fixed per-unit overhead for the
  // pipeline fill and the partial-tile store) and keeping the shortest makespan: a chunk
  // that leaves a sliver of a last wave idles most of the chip.
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const int slots = sms * 2;
  auto build = [&](int64_t kc, std::vector<int4>* out, std::vector<std::vector<int>>* pt) {
    const int64_t nchunks = ceil_div(k_end, kc);
    for (int64_t q = 0; q < nchunks; ++q) {
      const int64_t c0 = q * kc, c1 = std::min<int64_t>(k_end, c0 + kc);
      for (size_t t = 0; t < tiles.size(); ++t) {
        const int64_t a = std::max<int64_t>(c0, range[t].first), b = std::min<int64_t>(c1, range[t].second);
        if (a >= b) continue;
        if (pt) (*pt)[t].push_back((int)out->size());
        out->push_back({tiles[t].x, tiles[t].y, (int)a, (int)b});
      }
    }
  };
  auto makespan = [&](const std::vector<int4>& us) {
    std::priority_queue<double, std::vector<double>, std::greater<double>> q;
    for (int s = 0; s < slots; ++s) q.push(0.0);
    double end = 0.0;
    for (const int4& u : us) {
      const double t0 = q.top();
      q.pop();
      // a diagonal tile loads one operand instead of two: ~3/4 of the time per step
      const double steps = double(u.w - u.z) / kBK * (u.x == u.y ? 0.75 : 1.0);
      const double t1 = t0 + steps + 1.5;
      end = std::max(end, t1);
      q.push(t1);
    }
    return end;
  };
  int64_t kc = round_up(std::max<int64_t>(1, total / (int64_t(slots) * 4)), kBK);
  kc = std::max<int64_t>(kc, 8 * kBK);
  {
    double best = 1e300;
    const int64_t hi_kc = std::max<int64_t>(8 * kBK, round_up(std::max<int64_t>(1, total / slots), kBK));
    const int64_t step = std::max<int64_t>(kBK, round_up((hi_kc - 8 * kBK) / 40, kBK));
    for (int64_t cand = 8 * kBK; cand <= hi_kc; cand += step) {
      std::vector<int4> us;
      build(cand, &us, nullptr);
      const double ms = makespan(us);
      if (ms < best * 0.999) {
        best = ms;
        kc = cand;
      }
    }
  }
  std::vector<int4> units;
  std::vector<std::vector<int>> per_tile(tiles.size());
  build(kc, &units, &per_tile);
  std::vector<int32_t> tptr(tiles.size() + 1, 0), tunits;
  for (size_t t = 0; t < tiles.size(); ++t) {
    tptr[t + 1] = tptr[t] + (int32_t)per_tile[t].size();
    for (int u : per_tile[t]) tunits.push_back(u);
  }
  c.nunits = (int)units.size();
  c.ntiles = (int)tiles.size();
  cudaStream_t st = c.stream;
  c.units = dev_alloc<int4>(units.size(), st);
  c.tiles = dev_alloc<int2>(tiles.size(), st);
  c.tile_ptr = dev_alloc<int32_t>(tptr.size(), st);
  c.tile_units = dev_alloc<int32_t>(tunits.size(), st);
  c.partial = dev_alloc<double>((size_t)kTile * kTile * std::max(1, c.nunits), st);
  if (!units.empty())
    CMPC_CUDA(cudaMemcpyAsync(c.units, units.data(), sizeof(int4) * units.size(), cudaMemcpyHostToDevice, st));
  CMPC_CUDA(cudaMemcpyAsync(c.tiles, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice, st));
  CMPC_CUDA(cudaMemcpyAsync(c.tile_ptr, tptr.data(), sizeof(int32_t) * tptr.size(), cudaMemcpyHostToDevice, st));
  if (!tunits.empty())
    CMPC_CUDA(cudaMemcpyAsync(c.tile_units, tunits.data(), sizeof(int32_t) * tunits.size(),
                              cudaMemcpyHostToDevice, st));
  CMPC_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope

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
  // TMA descriptor over P (ldp rows x n cols, column-major), box {16 rows, 64 cols}
  auto* tm = new unsigned char[sizeof(CUtensorMap)];
  c.tmap_P = tm;
  const cuuint64_t dims[2] = {(cuuint64_t)c.ldp, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)c.ldp * sizeof(double)};
  const cuuint32_t box[2] = {16, 64};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(reinterpret_cast<CUtensorMap*>(tm), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                            c.P, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  static bool attr = false;
  if (!attr) {
    CMPC_CUDA(cudaFuncSetAttribute(k_syrk, cudaFuncAttributeMaxDynamicSharedMemorySize, kSyrkSmem));
    // two 99 KB CTAs per SM need the largest shared-memory carveout
    CMPC_CUDA(cudaFuncSetAttribute(k_syrk, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr = true;
  }
}

void launch_condense(Ctx& c, bool mirror) {
  if (c.nunits > 0) {
    const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(c.tmap_P);
    k_syrk<<<c.nunits, kSyrkThreads, kSyrkSmem, c.stream>>>(*tm, c.omega, c.units, c.partial);
    CMPC_LAUNCHED();
  }
  k_syrk_reduce<<<dim3(c.ntiles, kTile * kTile / 256), 256, 0, c.stream>>>(c.partial, c.tiles, c.tile_ptr, c.tile_units, c.rank == 0 ? c.H : nullptr,
                                                 c.dsing, c.n, c.M, mirror ? 1 : 0);
  // (sharded: every rank's partial J_g' Sigma_g J_g, H added by rank 0; the caller allreduces)
  CMPC_LAUNCHED();
}

}  // namespace cmpc
