// Host -> device upload of large pageable buffers (the DenseQp's J and H on cmpc_load_qp, the
// structured problem's A, Q, Qf on cmpc_build_qp).
//
// A plain cudaMemcpyAsync from pageable memory is staged by the driver through one bounce buffer
// on one thread (~11 GB/s on the B200 boxes). Here a pool of host threads copies each chunk into
// one of three pinned slots while the DMA engine drains the previous slot, so the CPU copy and
// the PCIe transfer overlap and the CPU copy itself runs on several cores. Pinned (registered)
// sources and small buffers go straight to cudaMemcpyAsync. The call returns once the last chunk
// is enqueued: the source may be reused immediately (every byte is in a slot or on the device),
// and a slot is only overwritten after its previous DMA's event has completed.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace cmpc {

namespace {

constexpr size_t kSlotBytes = size_t(8) << 20;
constexpr int kSlots = 3;
constexpr size_t kStageMin = size_t(4) << 20;  // smaller uploads: plain cudaMemcpyAsync

struct Stager {
  std::mutex mu;  // one staged upload at a time per process
  char* slot[kSlots] = {};
  cudaEvent_t done[kSlots] = {};
  bool ready = false;
  int device = -1;  // the events belong to this device (recreated when the caller's differs)
};

Stager& stager() {
  static Stager s;
  return s;
}

bool pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

}  // namespace

void upload_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < kStageMin || !pageable(src)) {
    CMPC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  Stager& S = stager();
  std::lock_guard<std::mutex> lk(S.mu);
  if (!S.ready) {
    for (int k = 0; k < kSlots; ++k)
      CMPC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&S.slot[k]), kSlotBytes, cudaHostAllocPortable));
    S.ready = true;
  }
  int dev = 0;
  CMPC_CUDA(cudaGetDevice(&dev));
  if (dev != S.device) {
    for (int k = 0; k < kSlots; ++k)
      if (S.done[k]) {
        CMPC_CUDA(cudaEventSynchronize(S.done[k]));
        cudaEventDestroy(S.done[k]);
      }
    for (int k = 0; k < kSlots; ++k) CMPC_CUDA(cudaEventCreateWithFlags(&S.done[k], cudaEventDisableTiming));
    S.device = dev;
  }
  const size_t nchunks = (bytes + kSlotBytes - 1) / kSlotBytes;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nthr = (int)std::min<unsigned>(8, std::max(1u, hw / 2));
  // chunk c is copied by all threads (stripe t of nthr); go = next chunk released to the workers,
  // copied[c % kSlots] counts finished stripes
  std::atomic<long> go{-1};
  std::atomic<int> copied[kSlots];
  for (auto& a : copied) a.store(0);
  auto stripe = [&](int t, size_t c) {
    const size_t off = c * kSlotBytes, len = std::min(kSlotBytes, bytes - off);
    const size_t per = (len / nthr + 63) / 64 * 64;
    const size_t b = std::min(len, per * t), e = std::min(len, b + per);
    if (e > b) std::memcpy(S.slot[c % kSlots] + b, static_cast<const char*>(src) + off + b, e - b);
  };
  std::atomic<bool> abort{false};
  std::vector<std::thread> pool;
  for (int t = 1; t < nthr; ++t)
    pool.emplace_back([&, t] {
      for (size_t c = 0; c < nchunks; ++c) {
        while (go.load(std::memory_order_acquire) < (long)c) std::this_thread::yield();
        if (abort.load(std::memory_order_acquire)) return;
        stripe(t, c);
        copied[c % kSlots].fetch_add(1, std::memory_order_acq_rel);
      }
    });
  try {
  for (size_t c = 0; c < nchunks; ++c) {
    const int k = (int)(c % kSlots);
    CMPC_CUDA(cudaEventSynchronize(S.done[k]));  // the slot's previous DMA has drained
    copied[k].store(0, std::memory_order_relaxed);
    go.store((long)c, std::memory_order_release);
    stripe(0, c);
    copied[k].fetch_add(1, std::memory_order_acq_rel);
    while (copied[k].load(std::memory_order_acquire) < nthr) std::this_thread::yield();
    const size_t off = c * kSlotBytes, len = std::min(kSlotBytes, bytes - off);
    CMPC_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, S.slot[k], len, cudaMemcpyHostToDevice, st));
    CMPC_CUDA(cudaEventRecord(S.done[k], st));
  }
  } catch (...) {
    abort.store(true, std::memory_order_release);
    go.store(long(nchunks), std::memory_order_release);
    for (auto& th : pool) th.join();
    throw;
  }
  for (auto& th : pool) th.join();
}

}  // namespace cmpc
