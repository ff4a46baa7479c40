// %globaltimer timeline of the dataflow Cholesky on one n x n SPD matrix (tools only):
//   nvcc -DCMPC_CHOL_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 chol_trace.cu -o chol_trace
// prints per diagonal task d: start, updates done, sub-diagonal panel published, factor
// start, factor done, published (us from the kernel start); backward tasks start/end.
#include "../../paper_2209_13049_b200/csrc/chol.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cmpc {
thread_local long long g_launches = 0;
namespace {
// spine_back alone, one CTA, on the factor a previous launch left in Lt / W / ybuf
__global__ void __launch_bounds__(256, 1) k_back_only(const DfArgs A, long long* cyc) {
  extern __shared__ __align__(16) double sm_bo[];
  __shared__ __align__(8) uint64_t full[kBSlots], empty[kBSlots];
  __syncthreads();
  const long long t0 = clock64();
  spine_back(A, sm_bo, full, empty);
  __syncthreads();
  if (threadIdx.x == 0) *cyc = clock64() - t0;
}
}  // namespace
}

int main(int argc, char** argv) {
  using namespace cmpc;
  const int64_t n = argc > 1 ? atol(argv[1]) : 500;
  std::vector<double> G(n * n), M(n * n, 0.0);
  srand(1);
  for (auto& g : G) g = rand() / double(RAND_MAX) - 0.5;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      double s = (i == j) ? double(n) : 0.0;
      for (int64_t k = 0; k < n; ++k) s += G[i * n + k] * G[j * n + k];
      M[i + j * n] = M[j + i * n] = s;
    }
  Ctx c;
  c.n = n;
  CMPC_CUDA(cudaStreamCreate(&c.stream));
  double* dM = dev_alloc<double>(n * n, c.stream);
  double* dL = dev_zeros<double>(n * n, c.stream);
  double* db = dev_zeros<double>(n, c.stream);
  double* dx = dev_zeros<double>(n, c.stream);
  c.pk = dev_zeros<Packet>(1, c.stream);
  CMPC_CUDA(cudaMemcpyAsync(dM, M.data(), 8 * n * n, cudaMemcpyHostToDevice, c.stream));
  chol_alloc(c);
  if (argc > 2) c.df_grid = atoi(argv[2]);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) launch_cholesky(c, dM, dL, 0.0, db, dx);
  cudaEventRecord(e0, c.stream);
  const int reps = 20;
  for (int it = 0; it < reps; ++it) launch_cholesky(c, dM, dL, 0.0, db, dx);
  cudaEventRecord(e1, c.stream);
  CMPC_CUDA(cudaStreamSynchronize(c.stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("n=%lld fused factor+solve: %.1f us per launch\n", (long long)n, ms * 1e3 / reps);
  {
    const int nt = (int)((n + 31) / 32);
    DfArgs a{};
    a.M = dM; a.L = dL; a.Lt = c.Lt; a.W = c.Winv; a.n = n; a.nt = nt; a.ybuf = c.df_y; a.x = dx; a.rhs = db;
    long long* dcyc = dev_zeros<long long>(1, c.stream);
    CMPC_CUDA(cudaFuncSetAttribute(k_back_only, cudaFuncAttributeMaxDynamicSharedMemorySize, kDfSmem));
    for (int r = 0; r < (n <= kMaxFusedN ? 3 : 0); ++r) {
      k_back_only<<<1, 256, kDfSmem, c.stream>>>(a, dcyc);
      long long cyc = 0;
      CMPC_CUDA(cudaMemcpyAsync(&cyc, dcyc, 8, cudaMemcpyDeviceToHost, c.stream));
      CMPC_CUDA(cudaStreamSynchronize(c.stream));
      printf("spine_back alone: %.2f us\n", cyc / 1965.0);
    }
  }
  std::vector<unsigned long long> tr(4096 * 10);
#ifdef CMPC_CHOL_TRACE
  CMPC_CUDA(cudaMemcpyFromSymbol(tr.data(), g_ctrace, sizeof(unsigned long long) * tr.size()));
#else
  return 0;
#endif
  // spine: clock64 per step (compute stamps 0-5 on SMSP of warp 0; I/O stamps 6, 7 on warp 4)
  const int nt = (int)((n + 31) / 32);
  const unsigned long long* sp = &tr[3000 * 10];
  auto cy = [&](int k, int e) { return (double)((long long)sp[k * 8 + e] - (long long)sp[0]) / 1965.0; };
  printf("spine (us from step 0 start): wait-in  in-ready  panel-done  factor-start  factor-done  step-done | io: k-2 gemm done | diag-published\n");
  for (int k = 0; k < nt && k < 63; ++k)
    printf("%2d %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f | %7.2f %7.2f\n", k, cy(k, 0), cy(k, 1), cy(k, 2), cy(k, 3), cy(k, 4),
           cy(k, 5), cy(k, 6), cy(k, 7));
  printf("backward: %.2f -> %.2f us\n", cy(63, 0), cy(63, 1));
  printf("io: k  inputs-staged  pready-passed  sdone-passed\n");
  for (int k = 0; k < nt && k < 31; ++k) printf("%2d %7.2f %7.2f %7.2f\n", k, cy(k + 32, 0), cy(k + 32, 1), cy(k + 32, 2));
  return 0;
}
