// In-process loopback communicator for the row-sharded solve (tests: N ranks on one GPU, one
// host thread each). See comm.cpp for NCCL, which every multi-GPU run uses.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace cmpc {

// ---------------------------------------------------------------- loopback
// An in-process communicator over N contexts on one device, one host thread per rank (the
// shape of one process per GPU): every rank issues the same sequence of allreduces, as with
// NCCL. Per call: each rank records its buffer's ready event and registers (host barrier);
// rank 0's stream waits for every rank's event and reduces all ranks' buffers in rank order
// into the group's result buffer; after a second barrier every rank's stream waits for that
// reduction and copies the result back. Same numbers on every rank, fixed order.
struct LoopGroup {
  int nranks = 0, device = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
  std::vector<void*> bufs;
  std::vector<cudaEvent_t> ready;
  cudaEvent_t done = nullptr;
  double* result = nullptr;  // double-buffered by call parity
  size_t cap = 0;
  unsigned long long calls = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g; });
    }
  }
};

namespace {
template <typename T, int OP>
__global__ void k_loop_reduce(void* const* bufs, int nranks, size_t count, T* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T v = static_cast<const T*>(bufs[0])[i];
    for (int r = 1; r < nranks; ++r) {
      const T x = static_cast<const T*>(bufs[r])[i];
      v = OP == 0 ? v + x : (OP == 1 ? (x > v ? x : v) : (x < v ? x : v));
    }
    out[i] = v;
  }
}
}  // namespace

void* comm_loop_create(int nranks, int device) {
  if (nranks < 1) throw DimError("loopback: nranks must be positive");
  auto* g = new LoopGroup;
  g->nranks = nranks;
  g->device = device;
  g->bufs.assign(size_t(nranks), nullptr);
  g->ready.assign(size_t(nranks), nullptr);
  CMPC_CUDA(cudaSetDevice(device));
  for (auto& e : g->ready) CMPC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CMPC_CUDA(cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming));
  return g;
}

void comm_loop_destroy(void* h) {
  auto* g = static_cast<LoopGroup*>(h);
  if (!g) return;
  cudaDeviceSynchronize();
  for (auto& e : g->ready) cudaEventDestroy(e);
  cudaEventDestroy(g->done);
  if (g->result) cudaFree(g->result);
  delete g;
}

void comm_loop_attach(Ctx& c, void* h, int rank) {
  auto* g = static_cast<LoopGroup*>(h);
  if (!g || rank < 0 || rank >= g->nranks) throw DimError("loopback: bad rank");
  if (c.device != g->device) throw DimError("loopback: every rank must be on the group's device");
  comm_detach(c);
  c.comm = g;
  c.comm_loop = true;
  c.nranks = g->nranks;
  c.rank = rank;
  comm_buffers(c);
}

void comm_loop_allreduce(Ctx& c, void* buf, size_t count, CommType type, CommOp op) {
  auto* g = static_cast<LoopGroup*>(c.comm);
  const size_t es = type == CommType::f64 ? sizeof(double) : sizeof(long long);
  // 1: this rank's contribution is ready on its stream (the call number is read before the
  // first barrier: rank 0 advances it after that barrier)
  const unsigned long long call = g->calls;
  static const bool trace = getenv("CMPC_LOOP_TRACE") != nullptr;
  if (trace) fprintf(stderr, "[loop] rank %d call %llu count %zu op %d\n", c.rank, call, count, (int)op);
  CMPC_CUDA(cudaEventRecord(g->ready[size_t(c.rank)], c.stream));
  g->bufs[size_t(c.rank)] = buf;
  g->barrier();
  // 2: rank 0 reduces (its stream waits for every rank's contribution)
  double* out = nullptr;
  if (c.rank == 0) {
    if (g->cap < 2 * count * es) {
      CMPC_CUDA(cudaStreamSynchronize(c.stream));
      if (g->result) CMPC_CUDA(cudaFree(g->result));
      g->cap = 2 * count * es + 4096;
      CMPC_CUDA(cudaMalloc(&g->result, g->cap));
    }
    for (int r = 0; r < g->nranks; ++r) CMPC_CUDA(cudaStreamWaitEvent(c.stream, g->ready[size_t(r)], 0));
    void** dbufs = nullptr;
    // the buffer pointers travel as kernel data: a small device array per call
    dbufs = dev_alloc<void*>(size_t(g->nranks), c.stream);
    CMPC_CUDA(cudaMemcpyAsync(dbufs, g->bufs.data(), sizeof(void*) * g->nranks, cudaMemcpyHostToDevice, c.stream));
    out = reinterpret_cast<double*>(reinterpret_cast<char*>(g->result) + (call & 1) * (g->cap / 2 / 256 * 256));
    const unsigned grid = (unsigned)std::min<size_t>(1024, (count + 255) / 256 + 1);
    if (type == CommType::f64) {
      if (op == CommOp::sum) k_loop_reduce<double, 0><<<grid, 256, 0, c.stream>>>(dbufs, g->nranks, count, out);
      else if (op == CommOp::max) k_loop_reduce<double, 1><<<grid, 256, 0, c.stream>>>(dbufs, g->nranks, count, out);
      else k_loop_reduce<double, 2><<<grid, 256, 0, c.stream>>>(dbufs, g->nranks, count, out);
    } else {
      long long* o = reinterpret_cast<long long*>(out);
      if (op == CommOp::sum) k_loop_reduce<long long, 0><<<grid, 256, 0, c.stream>>>(dbufs, g->nranks, count, o);
      else if (op == CommOp::max) k_loop_reduce<long long, 1><<<grid, 256, 0, c.stream>>>(dbufs, g->nranks, count, o);
      else k_loop_reduce<long long, 2><<<grid, 256, 0, c.stream>>>(dbufs, g->nranks, count, o);
    }
    CMPC_LAUNCHED();
    dev_free(dbufs, c.stream);
    CMPC_CUDA(cudaEventRecord(g->done, c.stream));
    g->calls = call + 1;
  }
  g->barrier();
  // 3: every rank takes the result (rank 0's event of this call is recorded by now)
  out = reinterpret_cast<double*>(reinterpret_cast<char*>(g->result) + (call & 1) * (g->cap / 2 / 256 * 256));
  if (c.rank != 0) CMPC_CUDA(cudaStreamWaitEvent(c.stream, g->done, 0));
  CMPC_CUDA(cudaMemcpyAsync(buf, out, count * es, cudaMemcpyDeviceToDevice, c.stream));
  // the done event is re-recorded by the next call only after every rank has queued its wait
  g->barrier();
}

}  // namespace cmpc
