// clock64 trace of the dataflow Cholesky on one n x n SPD matrix (tools only):
//   nvcc -DCMPC_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include chol_trace.cu -o chol_trace
#include "../../paper_2209_13049_b200/csrc/chol.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cmpc {
thread_local long long g_launches = 0;
namespace {
// the diagonal factor alone (one CTA, the first 64 x 64 block of M)
__global__ void __launch_bounds__(kDfThreads, 1) k_diag_only(const double* M, int64_t n, double* out) {
  extern __shared__ __align__(16) double sm_do[];
  double* a = sm_do;
  double* w = sm_do + kNB * kLD;
  for (int e = threadIdx.x; e < kNB * kNB; e += kDfThreads) {
    const int r = e & 63, c = e >> 6;
    a[r + c * kLD] = (r >= c && r < n && c < n) ? M[r + c * n] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  TRACE(0);
  const int f = diag_factor(a, w, w + kNB * kLD, (int)(n < 64 ? n : 64));
  TRACE(3);
  for (int e = threadIdx.x; e < kNB * kNB; e += kDfThreads) out[e] = a[(e & 63) + (e >> 6) * kLD] + f;
}
}  // namespace
}

int main(int argc, char** argv) {
  using namespace cmpc;
  const int64_t n = argc > 1 ? atol(argv[1]) : 64;
  std::vector<double> G(n * n), M(n * n, 0.0);
  srand(1);
  for (auto& g : G) g = rand() / double(RAND_MAX) - 0.5;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = (i == j) ? double(n) : 0.0;
      for (int64_t k = 0; k < n; ++k) s += G[i * n + k] * G[j * n + k];
      M[i + j * n] = s;
    }
  Ctx c;
  c.n = n;
  CMPC_CUDA(cudaStreamCreate(&c.stream));
  double* dM = dev_alloc<double>(n * n, c.stream);
  double* dL = dev_zeros<double>(n * n, c.stream);
  c.pk = dev_zeros<Packet>(1, c.stream);
  CMPC_CUDA(cudaMemcpyAsync(dM, M.data(), 8 * n * n, cudaMemcpyHostToDevice, c.stream));
  chol_alloc(c);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) launch_cholesky(c, dM, dL, 0.0);
  cudaEventRecord(e0, c.stream);
  const int reps = 20;
  for (int it = 0; it < reps; ++it) launch_cholesky(c, dM, dL, 0.0);
  cudaEventRecord(e1, c.stream);
  CMPC_CUDA(cudaStreamSynchronize(c.stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long tr[256];
  CMPC_CUDA(cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr)));
  long long info = 0;
  CMPC_CUDA(cudaMemcpy(&info, &c.pk->info, 8, cudaMemcpyDeviceToHost));
  std::vector<double> L(n * n);
  CMPC_CUDA(cudaMemcpy(L.data(), dL, 8 * n * n, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      double s = 0;
      for (int64_t k = 0; k <= j; ++k) s += L[i + k * n] * L[j + k * n];
      err = std::max(err, std::abs(s - M[i + j * n]) / M[i + i * n]);
    }
  printf("n=%ld avg %.2f us  info=%lld  max rel err %.2e\n", (long)n, 1e3 * ms / reps, info, err);
  const unsigned long long t0 = tr[0];
  printf("start->diag %llu  diag->end %llu (cycles, CTA 0 of the last launch)\n", tr[2] - t0, tr[3] - tr[2]);
  for (int kb = 0; kb < 8; ++kb)
    printf("kb %d: P1 %6llu  wait-B3 %6llu  P3+P4 %6llu  ->next %6llu\n", kb, tr[11 + 4 * kb] - tr[10 + 4 * kb],
           tr[12 + 4 * kb] - tr[11 + 4 * kb], tr[13 + 4 * kb] - tr[12 + 4 * kb],
           (kb < 7 ? tr[14 + 4 * kb] : tr[3]) - tr[13 + 4 * kb]);
  {
    CMPC_CUDA(cudaFuncSetAttribute(k_diag_only, cudaFuncAttributeMaxDynamicSharedMemorySize, kDfSmem));
    double* dout = dev_alloc<double>(4096, c.stream);
    for (int it = 0; it < 5; ++it) k_diag_only<<<1, kDfThreads, kDfSmem, c.stream>>>(dM, n, dout);
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
    unsigned long long t2[256];
    CMPC_CUDA(cudaMemcpyFromSymbol(t2, g_trace, sizeof(t2)));
    printf("k_diag_only: %llu cycles; per step:\n", t2[3] - t2[0]);
    for (int kb = 0; kb < 7; ++kb)
      printf("  kb %d: P1 %6llu  B3-wait %6llu  P3 %6llu  P4 %6llu\n", kb, t2[11 + 4 * kb] - t2[10 + 4 * kb],
             t2[12 + 4 * kb] - t2[11 + 4 * kb], t2[60 + kb] - t2[12 + 4 * kb], t2[13 + 4 * kb] - t2[60 + kb]);
  }
  printf("worker lane (tid 32), relative to warp-0 P1 start of the same step:\n");
  for (int kb = 0; kb < 8; ++kb)
    printf("kb %d: S3a %5lld S3b %5lld copies %5lld | B1 passed %6lld  W2+X done %6lld  B4 passed %6lld  S3 done %6lld\n", kb,
           (long long)(tr[140 + 2 * kb] - tr[102 + 4 * kb]), (long long)(tr[141 + 2 * kb] - tr[140 + 2 * kb]),
           (long long)(tr[103 + 4 * kb] - tr[141 + 2 * kb]),
           (long long)(tr[100 + 4 * kb] - tr[10 + 4 * kb]), (long long)(tr[101 + 4 * kb] - tr[10 + 4 * kb]),
           (long long)(tr[102 + 4 * kb] - tr[10 + 4 * kb]), (long long)(tr[103 + 4 * kb] - tr[10 + 4 * kb]));
  return 0;
}
