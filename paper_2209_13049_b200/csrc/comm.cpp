// NCCL for the row-sharded solve (one process per GPU): the partial sums of the iteration
// (J_g' Sigma_g J_g, J_g' y_g, the per-row maxima / minima / sums of the residual, recovery
// and line-search packets) are combined with allreduces on the solve's stream, so they are
// captured into the iteration's CUDA graphs like every kernel.
//
// libnccl is opened at run time (dlopen "libnccl.so.2": inside a PyTorch process this is the
// copy torch already loaded), so the library loads and runs single-GPU without NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "internal.cuh"

namespace cmpc {



namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (!a.handle) return;
    auto sym = [&](const char* s) { return dlsym(a.handle, s); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!a.handle || !a.AllReduce || !a.CommInitRank || !a.GetUniqueId)
    throw CudaError("NCCL unavailable: dlopen(libnccl.so.2) failed");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    throw CudaError(std::string("NCCL ") + what + ": " + s);
  }
}

}  // namespace

void comm_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  check(api().GetUniqueId(reinterpret_cast<ncclUniqueId*>(out128)), "GetUniqueId");
}

void comm_attach(Ctx& c, const void* id128, int nranks, int rank) {
  comm_detach(c);
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  CMPC_CUDA(cudaSetDevice(c.device));
  ncclComm_t comm = nullptr;
  check(api().CommInitRank(&comm, nranks, id, rank), "CommInitRank");
  c.comm = comm;
  c.nranks = nranks;
  c.rank = rank;
  comm_buffers(c);
}

void comm_buffers(Ctx& c) {
  if (c.n > 0 && !c.Mpack) c.Mpack = dev_alloc<double>((size_t)(c.n * (c.n + 1) / 2), c.stream);
}

void comm_detach(Ctx& c) {
  if (c.comm && !c.comm_loop) {
    cudaStreamSynchronize(c.stream);
    api().CommDestroy(static_cast<ncclComm_t>(c.comm));
  }
  if (c.comm_loop) cudaStreamSynchronize(c.stream);  // the group outlives its ranks
  c.comm = nullptr;
  c.comm_loop = false;
  c.nranks = 1;
  c.rank = 0;
}

void comm_allreduce(Ctx& c, void* buf, size_t count, CommType type, CommOp op) {
  if (!c.comm || count == 0) return;
  if (c.comm_loop) {
    comm_loop_allreduce(c, buf, count, type, op);
    return;
  }
  const ncclDataType_t dt = type == CommType::f64 ? ncclFloat64 : ncclInt64;
  const ncclRedOp_t ro = op == CommOp::sum ? ncclSum : (op == CommOp::max ? ncclMax : ncclMin);
  check(api().AllReduce(buf, buf, count, dt, ro, static_cast<ncclComm_t>(c.comm), c.stream), "AllReduce");
}

void comm_group(Ctx& c, bool start) {
  if (!c.comm || c.comm_loop) return;
  check(start ? api().GroupStart() : api().GroupEnd(), start ? "GroupStart" : "GroupEnd");
}

}  // namespace cmpc
