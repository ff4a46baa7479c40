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
// the diagonal factor + inverse alone (one CTA), clock64 around it
__global__ void __launch_bounds__(kT) k_factor_only(const double* M, int64_t n, double* out, long long* cyc) {
  extern __shared__ __align__(16) double sm_fo[];
  __shared__ int s_cnt;
  double* a_sm = sm_fo + kOffA;
  for (int rep = 0; rep < 3; ++rep) {
    for (int e = threadIdx.x; e < kB * kB; e += kT) {
      const int r = e & 31, c = e >> 5;
      a_sm[c * kLD + r] = (r >= c) ? M[r + c * n] : 0.0;
    }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const long long t0 = clock64();
    bool odd = false;
    int f = 0;
    if (threadIdx.x < 32) f = factor_rows<false>(a_sm, sm_fo + kOffCol, sm_fo + kOffRR, &s_cnt, 32, &odd);
    else if (threadIdx.x < 64) inverse_cols(sm_fo + kOffW, sm_fo + kOffCol, sm_fo + kOffRR, &s_cnt);
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[rep] = t1 - t0 + 0 * f;
  }
  for (int e = threadIdx.x; e < kB * kB; e += kT) out[e] = a_sm[(e >> 5) * kLD + (e & 31)] + sm_fo[kOffW + e];
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
    long long* dcyc = dev_zeros<long long>(4, c.stream);
    double* dout = dev_zeros<double>(1024, c.stream);
    CMPC_CUDA(cudaFuncSetAttribute(k_factor_only, cudaFuncAttributeMaxDynamicSharedMemorySize, kDfSmem));
    k_factor_only<<<1, kT, kDfSmem, c.stream>>>(dM, n, dout, dcyc);
    CMPC_CUDA(cudaStreamSynchronize(c.stream));
    long long cyc[3];
    CMPC_CUDA(cudaMemcpy(cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost));
    printf("factor_rows + inverse_cols alone: %lld %lld %lld cycles\n", cyc[0], cyc[1], cyc[2]);
  }
  std::vector<unsigned long long> tr(4096 * 10);
#ifdef CMPC_CHOL_TRACE
  CMPC_CUDA(cudaMemcpyFromSymbol(tr.data(), g_ctrace, sizeof(unsigned long long) * tr.size()));
#else
  return 0;
#endif
  // slots: cycles from the stamp to the task's end; [8] = globaltimer at the end
  const unsigned long long t0 = tr[4095 * 10 + 8];
  const int nt = (int)((n + 31) / 32);
  auto cyc_us = [](unsigned long long c) { return c / 1965.0; };
  printf("diag d: end(us)  [us before the end:] start  updates-done  flag(d-1)-seen  panel-published  factor-start  factor-done(pass 1)  published\n");
  for (int d = 0; d < nt; ++d) {
    const unsigned long long* r = &tr[d * 10];
    printf("%2d end %7.2f | start %6.2f upd %6.2f flag %6.2f panel %6.2f fstart %6.2f fdone %6.2f pub %6.2f\n", d,
           (double)(r[8] - t0) * 1e-3, cyc_us(r[0]), cyc_us(r[1]), cyc_us(r[7]), cyc_us(r[2]), cyc_us(r[3]), cyc_us(r[6]), cyc_us(r[5]));
  }
  printf("backward i: end(us) duration\n");
  for (int i = nt - 1; i >= 0; --i) {
    const unsigned long long* r = &tr[(2048 + i) * 10];
    printf("%2d %7.2f %6.2f\n", i, (double)(r[8] - t0) * 1e-3, cyc_us(r[0]));
  }
  return 0;
}
