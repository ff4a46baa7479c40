// Shared device/host helpers for the B200 condensed-space IPM path.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

namespace cmpc {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
// shape/option precondition failures (the reference's DimensionError, types.hpp:17-19)
struct DimError : std::runtime_error {
  explicit DimError(const std::string& m) : std::runtime_error(m) {}
};

#define CMPC_CUDA(x)                                                                        \
  do {                                                                                      \
    cudaError_t e__ = (x);                                                                  \
    if (e__ != cudaSuccess)                                                                 \
      throw ::cmpc::CudaError(std::string("CUDA error ") + cudaGetErrorString(e__) + " at " + \
                              __FILE__ + ":" + std::to_string(__LINE__));                    \
  } while (0)

// every kernel launch goes through this so the launch count is observable
extern thread_local long long g_launches;
#define CMPC_LAUNCHED()                 \
  do {                                  \
    ++::cmpc::g_launches;               \
    CMPC_CUDA(cudaPeekAtLastError());   \
  } while (0)

// Run f once per device: kernel attributes (large dynamic shared memory opt-in, carveout) and
// memory-pool settings belong to a device's context, not to the process.
constexpr int kMaxDevices = 64;
template <typename F>
void once_per_device(std::once_flag (&flags)[kMaxDevices], int device, F&& f) {
  if (device < 0 || device >= kMaxDevices) throw CudaError("device ordinal out of range");
  std::call_once(flags[device], [&] {
    int cur = 0;
    CMPC_CUDA(cudaGetDevice(&cur));
    if (cur != device) CMPC_CUDA(cudaSetDevice(device));
    f();
    if (cur != device) CMPC_CUDA(cudaSetDevice(cur));
  });
}

// Stream-ordered device allocations from the device's memory pool (kept cached: a
// reloaded QP of similar size reuses the pages instead of re-mapping gigabytes).
void pool_init(int device);
// host -> device copy; large pageable sources are staged through pinned slots by a few host
// threads (upload.cpp). Returns once enqueued on st; the source may then be reused.
void upload_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);
template <typename T>
inline T* dev_alloc(size_t count, cudaStream_t st) {
  void* p = nullptr;
  const size_t bytes = (count == 0 ? 1 : count) * sizeof(T);
  cudaError_t e = cudaMallocAsync(&p, bytes, st);
  if (e != cudaSuccess)
    throw CudaError(std::string("cudaMallocAsync(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  return static_cast<T*>(p);
}
template <typename T>
inline T* dev_zeros(size_t count, cudaStream_t st) {
  T* p = dev_alloc<T>(count, st);
  CMPC_CUDA(cudaMemsetAsync(p, 0, (count == 0 ? 1 : count) * sizeof(T), st));
  return p;
}
inline void dev_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

#ifdef __CUDACC__
// IEEE operations without FMA contraction: elementwise updates follow the
// reference's separate multiply/add rounding (Eigen, SSE2, no -march).
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }

// max/min of non-negative doubles through their ordered bit patterns
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// fixed-order block sum (result valid in thread 0); blockDim.x multiple of 32, <= 1024
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (l < NT / 32) ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// block max / min (result valid in thread 0): one atomic per block instead of one per warp
template <int NT>
__device__ __forceinline__ double block_max(double v, double* sh) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = v;
  if (threadIdx.x < 32) r = warp_max((l < NT / 32) ? sh[l] : v);
  return r;
}
// NS block sums and NX block maxima with one barrier pair (results valid in warp 0); the same
// operations in the same order as NS block_sum and NX block_max calls, so bitwise equal.
// sh: (NS + NX) * 32 doubles.
template <int NT, int NS, int NX>
__device__ __forceinline__ void block_sums_maxs(double (&s)[NS], double (&x)[NX], double* sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NS; ++k) s[k] = warp_sum(s[k]);
#pragma unroll
  for (int k = 0; k < NX; ++k) x[k] = warp_max(x[k]);
  __syncthreads();
  if (l == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) sh[k * 32 + w] = s[k];
#pragma unroll
    for (int k = 0; k < NX; ++k) sh[(NS + k) * 32 + w] = x[k];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = warp_sum((l < NT / 32) ? sh[k * 32 + l] : 0.0);
#pragma unroll
    for (int k = 0; k < NX; ++k) x[k] = warp_max((l < NT / 32) ? sh[(NS + k) * 32 + l] : x[k]);
  }
}
template <int NT>
__device__ __forceinline__ double block_min(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = v;
  if (threadIdx.x < 32) {
    r = (l < NT / 32) ? sh[l] : v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r = fmin(r, __shfl_xor_sync(0xffffffffu, r, o));
  }
  return r;
}

#endif  // __CUDACC__

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline int64_t ceil_div(int64_t x, int64_t a) { return (x + a - 1) / a; }

}  // namespace cmpc
