// Collectives of the buffer manager over NCCL (NVLink 5 / NVSwitch): the
// "gathers or allgathers results and replicated state" step of the north star
// (PageRank rank vector allgather, k-means centroid-sum allreduce, GEMM B
// broadcast) when the partitioned NDRange spans processes (one per GPU).
// The reference has no data collectives (a sequential TCP
// broadcast of DeviceIdRequest only), so these are new.
//
// NCCL is loaded lazily with dlopen("libnccl.so.2"): single-GPU use never
// touches it, and inside a PyTorch process the already-loaded libnccl.so.2 is
// reused (same soname), so both stacks share one NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "haocl/runtime.hpp"
#include "hcl_cabi.h"
#include "hcl_host.h"

namespace hcl {
void set_last_error(const std::string& m);
}

namespace {

struct Nccl {
  void* handle = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

std::mutex g_mu;
Nccl g_nccl;
std::map<int, ncclComm_t> g_comms;  // device index -> communicator
std::map<int, std::pair<int, int>> g_rank;  // device index -> (rank, nranks)

[[noreturn]] void fail(haocl::ErrorCode c, const std::string& m) { throw haocl::Error(c, m); }

Nccl& nccl() {
  if (g_nccl.handle) return g_nccl;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(haocl::ErrorCode::precondition, std::string("libnccl.so.2 not loadable: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) fail(haocl::ErrorCode::precondition, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  g_nccl.getUniqueId = reinterpret_cast<decltype(g_nccl.getUniqueId)>(sym("ncclGetUniqueId"));
  g_nccl.commInitRank = reinterpret_cast<decltype(g_nccl.commInitRank)>(sym("ncclCommInitRank"));
  g_nccl.commDestroy = reinterpret_cast<decltype(g_nccl.commDestroy)>(sym("ncclCommDestroy"));
  g_nccl.broadcast = reinterpret_cast<decltype(g_nccl.broadcast)>(sym("ncclBroadcast"));
  g_nccl.allReduce = reinterpret_cast<decltype(g_nccl.allReduce)>(sym("ncclAllReduce"));
  g_nccl.groupStart = reinterpret_cast<decltype(g_nccl.groupStart)>(sym("ncclGroupStart"));
  g_nccl.groupEnd = reinterpret_cast<decltype(g_nccl.groupEnd)>(sym("ncclGroupEnd"));
  g_nccl.getErrorString = reinterpret_cast<decltype(g_nccl.getErrorString)>(sym("ncclGetErrorString"));
  g_nccl.handle = h;
  return g_nccl;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(haocl::ErrorCode::transport, std::string(what) + ": " + nccl().getErrorString(r));
}

void hcl_check(int rc) {
  if (rc != HCL_OK) {
    int code = rc - HCL_ERR_BASE;
    if (code < 0 || code > 23) code = 0;
    throw haocl::Error(static_cast<haocl::ErrorCode>(code), hcl_last_error());
  }
}

ncclComm_t comm_of(int dev) {
  auto it = g_comms.find(dev);
  if (it == g_comms.end())
    fail(haocl::ErrorCode::precondition, "device " + std::to_string(dev) + " has no NCCL communicator (hcl_nccl_init)");
  return it->second;
}

template <typename F>
int guarded(F&& f) {
  try {
    std::lock_guard<std::mutex> lock(g_mu);
    f();
    return HCL_OK;
  } catch (const haocl::Error& e) {
    hcl::set_last_error(e.what());
    return HCL_ERR_BASE + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    hcl::set_last_error(std::string("internal: ") + e.what());
    return HCL_ERR_BASE;
  }
}

uint8_t* buffer_base(int dev, uint64_t id, uint64_t need_first, uint64_t need_len) {
  void* p = nullptr;
  uint64_t first = 0, bytes = 0;
  hcl_check(hcl_buffer_device_ptr(dev, id, &p, &first, &bytes));
  if (need_first < first || need_first + need_len > first + bytes)
    fail(haocl::ErrorCode::size, "collective range outside the buffer's resident slice");
  return static_cast<uint8_t*>(p) - first;  // logical byte 0
}

cudaStream_t stream_of(int dev) {  // the device's collective stream
  void* s = nullptr;
  hcl_check(hcl_comm_stream(dev, &s));
  return static_cast<cudaStream_t>(s);
}

}  // namespace

extern "C" {

int hcl_nccl_unique_id(uint8_t* out, int cap) {
  return guarded([&] {
    if (cap < static_cast<int>(sizeof(ncclUniqueId))) fail(haocl::ErrorCode::size, "unique id needs 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
  });
}

int hcl_nccl_init(int dev, int nranks, int rank, const uint8_t* id_bytes) {
  return guarded([&] {
    if (g_comms.count(dev)) return;
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    void* s = nullptr;
    hcl_check(hcl_device_stream(dev, &s));  // validates dev
    int ord = 0;  // ncclCommInitRank binds the current device
    if (cudaStreamGetDevice(static_cast<cudaStream_t>(s), &ord) == cudaSuccess) cudaSetDevice(ord);
    ncclComm_t comm;
    nccl_check(nccl().commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    g_comms[dev] = comm;
    g_rank[dev] = {rank, nranks};
  });
}

int hcl_nccl_destroy(int dev) {
  return guarded([&] {
    auto it = g_comms.find(dev);
    if (it == g_comms.end()) return;
    nccl().commDestroy(it->second);
    g_comms.erase(it);
    g_rank.erase(dev);
  });
}

// In-place allgather of uneven byte ranges: rank r owns [bounds[r], bounds[r+1])
// of the buffer; afterwards every rank holds [bounds[0], bounds[nranks]).
int hcl_allgatherv(int dev, uint64_t buffer_id, const uint64_t* bounds) {
  return guarded([&] {
    ncclComm_t comm = comm_of(dev);
    auto [rank, nranks] = g_rank[dev];
    uint8_t* base = buffer_base(dev, buffer_id, bounds[0], bounds[nranks] - bounds[0]);
    cudaStream_t st = stream_of(dev);
    hcl_check(hcl_comm_acquire(dev, buffer_id, 1));
    nccl_check(nccl().groupStart(), "ncclGroupStart");
    for (int r = 0; r < nranks; ++r) {
      size_t n = bounds[r + 1] - bounds[r];
      if (!n) continue;
      nccl_check(nccl().broadcast(base + bounds[r], base + bounds[r], n, ncclUint8, r, comm, st), "ncclBroadcast");
    }
    nccl_check(nccl().groupEnd(), "ncclGroupEnd");
    hcl_check(hcl_comm_release(dev, buffer_id, 1));
  });
}

// In-place sum of `count` int64 at logical byte `offset`.
int hcl_allreduce_sum_i64(int dev, uint64_t buffer_id, uint64_t offset, uint64_t count) {
  return guarded([&] {
    ncclComm_t comm = comm_of(dev);
    uint8_t* base = buffer_base(dev, buffer_id, offset, count * 8);
    hcl_check(hcl_comm_acquire(dev, buffer_id, 1));
    nccl_check(nccl().allReduce(base + offset, base + offset, count, ncclInt64, ncclSum, comm, stream_of(dev)),
               "ncclAllReduce");
    hcl_check(hcl_comm_release(dev, buffer_id, 1));
  });
}

// Stream-ordered barrier across the communicator's ranks on the device's
// kernel stream: a one-element allreduce. Kernels enqueued after it start only
// once every rank's kernels before it have finished -- the ordering a fused
// exchange kernel needs (its NVLink stores into peer buffers must land before
// any rank reads them in the next step).
int hcl_nccl_barrier(int dev) {
  return guarded([&] {
    ncclComm_t comm = comm_of(dev);
    void* s = nullptr;
    hcl_check(hcl_device_stream(dev, &s));
    static std::map<int, void*> scratch;
    void*& p = scratch[dev];
    if (!p) {
      int ord = 0;
      if (cudaStreamGetDevice(static_cast<cudaStream_t>(s), &ord) == cudaSuccess) cudaSetDevice(ord);
      if (cudaMalloc(&p, 8) != cudaSuccess) fail(haocl::ErrorCode::internal, "hcl_nccl_barrier: cudaMalloc");
    }
    nccl_check(nccl().allReduce(p, p, 1, ncclInt64, ncclSum, comm, static_cast<cudaStream_t>(s)), "ncclAllReduce");
  });
}

int hcl_broadcast(int dev, uint64_t buffer_id, uint64_t offset, uint64_t bytes, int root) {
  return guarded([&] {
    ncclComm_t comm = comm_of(dev);
    uint8_t* base = buffer_base(dev, buffer_id, offset, bytes);
    hcl_check(hcl_comm_acquire(dev, buffer_id, 1));
    nccl_check(nccl().broadcast(base + offset, base + offset, bytes, ncclUint8, root, comm, stream_of(dev)),
               "ncclBroadcast");
    hcl_check(hcl_comm_release(dev, buffer_id, 1));
  });
}

}  // extern "C"
