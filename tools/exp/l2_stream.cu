// One CTA streaming an L2-resident buffer into shared memory with cp.async.bulk (tools only):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 l2_stream.cu -o l2_stream
// A ring of R slots of S bytes, one mbarrier per slot, a single issuing thread; the consumer
// warps only wait for each slot and release it (no compute): the per-SM bulk-copy bandwidth
// from L2 that a one-CTA backward solve could reach.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra.uni D_%=;\nbra.uni W_%=;\nD_%=:\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void k_stream(const char* src, size_t bytes, int S, int R, long long* out, double* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[32];
  __shared__ int s_done[32];
  if (threadIdx.x == 0) {
    for (int r = 0; r < R; ++r) mbar_init(&full[r], 1), s_done[r] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nch = (int)(bytes / S);
  const long long t0 = clock64();
  double acc = 0.0;
  if (threadIdx.x == 0) {
    for (int c = 0; c < R && c < nch; ++c) {
      mbar_expect_tx(&full[c], S);
      bulk_load(sm + (size_t)c * S, src + (size_t)c * S, S, &full[c]);
    }
  }
  for (int c = 0; c < nch; ++c) {
    const int s = c % R;
    mbar_wait(&full[s], (c / R) & 1);
    acc += *reinterpret_cast<const double*>(sm + (size_t)s * S + 8 * (threadIdx.x & 15));
    __syncthreads();  // everyone has read the slot
    if (threadIdx.x == 0 && c + R < nch) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full[s], S);
      bulk_load(sm + (size_t)s * S, src + (size_t)(c + R) * S, S, &full[s]);
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  if (acc == 1234.5) *sink = acc;
}

int main() {
  const size_t bytes = 1u << 20;  // 1 MB: L of n = 500 is 1 MB
  char* buf;
  long long* out;
  double* sink;
  cudaMalloc(&buf, bytes * 4);
  cudaMalloc(&out, 8);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, bytes * 4);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int S : {2048, 4096, 8192, 16384}) {
    for (int R : {4, 8, 12, 24}) {
      if ((size_t)S * R > 200 * 1024) continue;
      for (int rep = 0; rep < 3; ++rep) k_stream<<<1, 128, S * R>>>(buf, bytes, S, R, out, sink);
      cudaDeviceSynchronize();
      long long cyc = 0;
      cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
      const double us = cyc / 1965.0;
      printf("S %6d R %2d: 1 MB in %7.2f us = %6.1f GB/s %s\n", S, R, us, bytes / us / 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
