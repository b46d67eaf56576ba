// Device layer of the C-ABI (include/hcl_cabi.h): CUDA device enumeration,
// one stream per device, the per-device buffer store and the launch path.
//
// Replaces the node daemon's BufferStore and do_launch
// (proj/src/daemon.cpp:21-114, 278-352): buffers live in HBM instead of byte
// vectors, DataTransfer chunks become cudaMemcpyAsync, and launch_kernel
// becomes an asynchronous kernel launch bracketed by CUDA events.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <memory>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "../../include/hcl_cabi.h"

namespace hcl {

std::atomic<uint64_t> g_kernel_launches{0};
thread_local uint64_t t_kernel_launches = 0;
thread_local bool t_launch_untimed = false;

const char* error_code_name(ErrorCode code) {
  switch (code) {
    case ErrorCode::internal: return "internal";
    case ErrorCode::protocol: return "protocol";
    case ErrorCode::version: return "version";
    case ErrorCode::malformed: return "malformed";
    case ErrorCode::encoding: return "encoding";
    case ErrorCode::unknown_call: return "unknown_call";
    case ErrorCode::busy: return "busy";
    case ErrorCode::precondition: return "precondition";
    case ErrorCode::reassembly_conflict: return "reassembly_conflict";
    case ErrorCode::argument: return "argument";
    case ErrorCode::name: return "name";
    case ErrorCode::config: return "config";
    case ErrorCode::connect: return "connect";
    case ErrorCode::timeout: return "timeout";
    case ErrorCode::transport: return "transport";
    case ErrorCode::remote: return "remote";
    case ErrorCode::handle: return "handle";
    case ErrorCode::policy: return "policy";
    case ErrorCode::size: return "size";
    case ErrorCode::mapping: return "mapping";
    case ErrorCode::unknown_device: return "unknown_device";
    case ErrorCode::registration: return "registration";
    case ErrorCode::contract: return "contract";
    case ErrorCode::parse: return "parse";
  }
  return "unknown";
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  fail(ErrorCode::internal, std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                                cudaGetErrorString(e) + ") at " + file + ":" +
                                std::to_string(line) + ": " + what);
}

namespace {

// Stream-ordered dependency tracking: every allocation remembers the event of
// its last writer and of its readers per stream, so copies on the H2D / D2H
// streams overlap kernels on the compute stream while RAW and WAR order holds.
struct Dep {
  cudaEvent_t ev = nullptr;
  cudaStream_t st = nullptr;
  cudaStream_t waited = nullptr;  // a stream already ordered after ev (its wait need not repeat)
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  uint64_t work = 0;
  uint64_t kernels = 0;  // kernel launches captured (counted again at every replay)
  bool seen = false;
};

struct DevAlloc {
  uint8_t* ptr = nullptr;
  uint64_t first_byte = 0;
  uint64_t bytes = 0;
  bool external = false;
  uint8_t mem = 0;       // 0 stream-ordered pool, 1 cudaMalloc (IPC-exportable), 2 IPC-mapped peer memory
  uint64_t version = 0;  // bumped on every tracked write (BufView::version)
  Dep last_write;
  std::vector<Dep> reads;  // at most one per stream
};

std::atomic<uint64_t> g_write_version{0};

struct Device {
  int ordinal = 0;
  cudaStream_t stream = nullptr;  // kernels, allocation, peer copies
  cudaStream_t h2d = nullptr;     // host -> device copies
  cudaStream_t d2h = nullptr;     // device -> host copies
  // second copy streams: a large copy is split in two halves on (h2d, h2d2) / (d2h, d2h2)
  // -- one stream's copy does not saturate the PCIe link (measured 47 GB/s H2D with one
  // stream, 55 GB/s with two)
  cudaStream_t h2d2 = nullptr, d2h2 = nullptr;
  cudaStream_t comm = nullptr;    // NCCL collectives (overlap the compute stream)
  int sm_count = 0;      // SM budget the kernels size their grids to
  int sm_physical = 0;   // the GPU's SM count
  uint64_t hbm_bytes = 0;
  std::string name;
  std::mutex mu;
  std::unordered_map<uint64_t, DevAlloc> bufs;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;  // since last finish
  std::vector<cudaEvent_t> spare_events;
  std::vector<cudaEvent_t> spare_sync;  // timing-disabled events for dependencies
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  std::unordered_map<std::string, GraphEntry> graphs;  // captured launches (KernelDef::graphable)

  cudaEvent_t event() {
    if (!spare_events.empty()) {
      cudaEvent_t e = spare_events.back();
      spare_events.pop_back();
      return e;
    }
    cudaEvent_t e;
    HCL_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t sync_event() {
    if (!spare_sync.empty()) {
      cudaEvent_t e = spare_sync.back();
      spare_sync.pop_back();
      return e;
    }
    cudaEvent_t e;
    HCL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
  }
  void drop(Dep& d) {
    if (d.ev) spare_sync.push_back(d.ev);  // waits already enqueued keep their snapshot
    d = Dep{};
  }
  // make `s` wait for the writer (and, for a write, the readers) of `a`
  void wait_for(DevAlloc& a, cudaStream_t s, bool write) {
    auto wait = [&](Dep& d) {
      if (!d.ev || d.st == s || d.waited == s) return;
      HCL_CUDA(cudaStreamWaitEvent(s, d.ev, 0));
      d.waited = s;  // later work on s is stream-ordered after this wait
    };
    wait(a.last_write);
    if (write)
      for (Dep& r : a.reads) wait(r);
  }
  // record that an operation on `s` just read / wrote `a`
  cudaEvent_t note(DevAlloc& a, cudaStream_t s, bool write) {
    cudaEvent_t e = sync_event();
    HCL_CUDA(cudaEventRecord(e, s));
    if (write) {
      if (!a.external) a.version = g_write_version.fetch_add(1) + 1;
      drop(a.last_write);
      for (Dep& r : a.reads) drop(r);
      a.reads.clear();
      a.last_write = Dep{e, s};
    } else {
      for (Dep& r : a.reads)
        if (r.st == s) {  // stream order subsumes the older read
          drop(r);
          r = Dep{e, s};
          return e;
        }
      a.reads.push_back(Dep{e, s});
    }
    return e;
  }
  // before freeing: the compute stream (which frees) waits for every user
  void retire(DevAlloc& a) {
    wait_for(a, stream, true);
    drop(a.last_write);
    for (Dep& r : a.reads) drop(r);
    a.reads.clear();
  }
};

// free an allocation after d.retire(a) (the device stream then follows every use)
void free_alloc(Device& d, DevAlloc& a) {
  if (!a.ptr) return;
  if (a.mem == 1 || a.mem == 2) {  // not stream-ordered: wait for the uses first
    HCL_CUDA(cudaStreamSynchronize(d.stream));
    if (a.mem == 1)
      HCL_CUDA(cudaFree(a.ptr));
    else
      HCL_CUDA(cudaIpcCloseMemHandle(a.ptr));
  } else if (!a.external) {
    HCL_CUDA(cudaFreeAsync(a.ptr, d.stream));
  }
}

std::mutex g_devices_mu;
std::vector<std::unique_ptr<Device>> g_devices;
thread_local std::string g_last_error;

Device& device(int dev) {
  std::lock_guard<std::mutex> lock(g_devices_mu);
  if (dev < 0 || dev >= static_cast<int>(g_devices.size()))
    fail(ErrorCode::unknown_device, "device " + std::to_string(dev) + " (have " +
                                        std::to_string(g_devices.size()) + "; call hcl_init)");
  return *g_devices[dev];
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HCL_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return HCL_ERR_BASE + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_last_error = std::string("internal: ") + e.what();
    return HCL_ERR_BASE + static_cast<int>(ErrorCode::internal);
  }
}

DevAlloc& alloc_of(Device& d, uint64_t id, const char* what) {
  auto it = d.bufs.find(id);
  if (it == d.bufs.end())
    fail(ErrorCode::precondition, std::string(what) + ": buffer " + std::to_string(id) +
                                      " is not allocated on device " + std::to_string(d.ordinal));
  return it->second;
}

uint8_t* range_ptr(DevAlloc& a, uint64_t offset, uint64_t len, uint64_t id, const char* what) {
  if (offset < a.first_byte || offset + len > a.first_byte + a.bytes)
    fail(ErrorCode::size, std::string(what) + ": range [" + std::to_string(offset) + ", " +
                              std::to_string(offset + len) + ") outside the resident slice [" +
                              std::to_string(a.first_byte) + ", " +
                              std::to_string(a.first_byte + a.bytes) + ") of buffer " +
                              std::to_string(id));
  return a.ptr + (offset - a.first_byte);
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HCL_GRAPH");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Everything a graphable launch function's enqueued work depends on: the kernel,
// arguments (device addresses and extents, scalars), the range, the device's SM
// budget and scratch, and the launch-shaping environment knobs.
std::string graph_key(const KernelDef* k, const std::vector<LaunchArg>& la, const LaunchCtx& c, const Device& d) {
  std::string key;
  auto put = [&key](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
  put(&k, sizeof(k));
  for (const LaunchArg& a : la) {
    put(&a.kind, sizeof(a.kind));
    put(&a.scalar, sizeof(a.scalar));
    put(&a.buf.ptr, sizeof(a.buf.ptr));
    put(&a.buf.first_byte, sizeof(a.buf.first_byte));
    put(&a.buf.bytes, sizeof(a.buf.bytes));
  }
  put(c.goff, sizeof(c.goff));
  put(c.gsize, sizeof(c.gsize));
  put(&c.dims, sizeof(c.dims));
  put(&c.whole, sizeof(c.whole));
  put(&d.sm_count, sizeof(d.sm_count));
  put(&d.scratch, sizeof(d.scratch));
  put(&d.scratch_bytes, sizeof(d.scratch_bytes));
  for (const char* v : {"HCL_GEMM_SHAPE", "HCL_GEMM_CG", "HCL_GEMM_B_KMAJOR", "HCL_GEMM_GROUP", "HCL_GEMM_PROMO",
                        "HCL_GEMM_TMAC", "HCL_GEMM_ONE", "HCL_GEMM_PERSIST", "HCL_GEMM_KSPLIT", "HCL_GEMM_PDL", "HCL_GEMM_SEG", "HCL_SIMT_MS", "HCL_SIMT_KSPLIT",
                        "HCL_SIMT_TILE"}) {
    const char* e = std::getenv(v);
    key += '|';
    if (e) key += e;
  }
  return key;
}

void* scratch_for(int dev, size_t bytes) {
  Device& d = device(dev);
  if (d.scratch_bytes < bytes) {
    if (d.scratch) HCL_CUDA(cudaFreeAsync(d.scratch, d.stream));
    HCL_CUDA(cudaMallocAsync(&d.scratch, bytes, d.stream));
    d.scratch_bytes = bytes;
  }
  return d.scratch;
}

template <typename T>
__global__ void local_add_kernel(T* __restrict__ dst, const T* __restrict__ src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = dst[i] + src[i];
}

std::atomic<uint64_t> g_coll_tmp{0};
uint64_t coll_tmp_id() { return 0xC011'0000'0000'0000ULL | g_coll_tmp.fetch_add(1); }

// a nested C-ABI call's failure back into an exception (its message is in g_last_error)
void check_rc(int rc) {
  if (rc != HCL_OK) fail(static_cast<ErrorCode>(rc - HCL_ERR_BASE), g_last_error);
}

}  // namespace

// Shared by the host runtime's C entry points (one last-error channel).
void set_last_error(const std::string& m) { g_last_error = m; }

}  // namespace hcl

using namespace hcl;

extern "C" {

const char* hcl_last_error(void) { return g_last_error.c_str(); }

uint64_t hcl_kernel_launch_count(void) { return g_kernel_launches.load(); }

int hcl_init(const int* cuda_ordinals, int n, int* num_devices) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(g_devices_mu);
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      fail(ErrorCode::precondition, std::string("no CUDA device available (") +
                                        cudaGetErrorString(e) + "); the B200 path has no CPU fallback");
    std::vector<int> want;
    if (cuda_ordinals && n > 0)
      want.assign(cuda_ordinals, cuda_ordinals + n);
    else
      for (int i = 0; i < count; ++i) want.push_back(i);
    if (!g_devices.empty()) {
      bool same = g_devices.size() == want.size();
      for (size_t i = 0; same && i < want.size(); ++i) same = g_devices[i]->ordinal == want[i];
      if (!same) fail(ErrorCode::config, "hcl_init called again with a different device list");
      if (num_devices) *num_devices = static_cast<int>(g_devices.size());
      return;
    }
    for (int ord : want) {
      if (ord < 0 || ord >= count) fail(ErrorCode::unknown_device, "CUDA ordinal " + std::to_string(ord));
      auto d = std::make_unique<Device>();
      d->ordinal = ord;
      HCL_CUDA(cudaSetDevice(ord));
      cudaDeviceProp prop{};
      HCL_CUDA(cudaGetDeviceProperties(&prop, ord));
      if (prop.major != 10)
        fail(ErrorCode::precondition, std::string("device ") + prop.name +
                                          " is not sm_100 (Blackwell B200); this library is built for sm_100a only");
      d->sm_count = d->sm_physical = prop.multiProcessorCount;
      d->hbm_bytes = prop.totalGlobalMem;
      d->name = prop.name;
      HCL_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
      HCL_CUDA(cudaStreamCreateWithFlags(&d->h2d, cudaStreamNonBlocking));
      HCL_CUDA(cudaStreamCreateWithFlags(&d->d2h, cudaStreamNonBlocking));
      HCL_CUDA(cudaStreamCreateWithFlags(&d->h2d2, cudaStreamNonBlocking));
      HCL_CUDA(cudaStreamCreateWithFlags(&d->d2h2, cudaStreamNonBlocking));
      HCL_CUDA(cudaStreamCreateWithFlags(&d->comm, cudaStreamNonBlocking));
      g_devices.push_back(std::move(d));
    }
    // NVLink P2P between every pair (NVSwitch: all-to-all).
    for (size_t i = 0; i < g_devices.size(); ++i)
      for (size_t j = 0; j < g_devices.size(); ++j) {
        if (i == j) continue;
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, g_devices[i]->ordinal, g_devices[j]->ordinal);
        if (ok) {
          cudaSetDevice(g_devices[i]->ordinal);
          cudaError_t pe = cudaDeviceEnablePeerAccess(g_devices[j]->ordinal, 0);
          if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
      }
    if (num_devices) *num_devices = static_cast<int>(g_devices.size());
  });
}

int hcl_device_set_sm_budget(int dev, int sms) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    if (sms <= 0) {  // reset to the whole GPU
      d.sm_count = d.sm_physical;
      return;
    }
    if (sms < 2 || sms > d.sm_physical)
      fail(ErrorCode::argument, "SM budget must be in [2, " + std::to_string(d.sm_physical) + "]");
    d.sm_count = sms & ~1;  // CTA pairs
  });
}

int hcl_device_count(int* n) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(g_devices_mu);
    *n = static_cast<int>(g_devices.size());
  });
}

int hcl_device_info(int dev, int* type, double* relative_throughput, int* sm_count,
                    uint64_t* hbm_bytes, char* name, int name_cap) {
  return guarded([&] {
    Device& d = device(dev);
    if (type) *type = 1;  // wire::DeviceType::gpu
    if (relative_throughput) *relative_throughput = static_cast<double>(d.sm_count) / d.sm_physical;
    if (sm_count) *sm_count = d.sm_count;
    if (hbm_bytes) *hbm_bytes = d.hbm_bytes;
    if (name && name_cap > 0) {
      std::strncpy(name, d.name.c_str(), static_cast<size_t>(name_cap) - 1);
      name[name_cap - 1] = 0;
    }
  });
}

int hcl_device_stream(int dev, void** stream) {
  return guarded([&] { *stream = device(dev).stream; });
}

int hcl_query_registry(const char* bundle, char* names_csv, int names_cap, uint32_t* arities,
                       int arity_cap, int* n) {
  return guarded([&] {
    if (!bundle_exists(bundle)) fail(ErrorCode::name, std::string("unknown bundle '") + bundle + "'");
    std::string csv;
    int count = 0;
    for (const auto& k : registry()) {
      if (std::strcmp(k.bundle, bundle) != 0) continue;
      if (!csv.empty()) csv += ",";
      csv += k.name;
      if (arities && count < arity_cap) arities[count] = static_cast<uint32_t>(k.kinds.size());
      ++count;
    }
    if (names_csv) {
      if (static_cast<int>(csv.size()) + 1 > names_cap) fail(ErrorCode::size, "names buffer too small");
      std::memcpy(names_csv, csv.c_str(), csv.size() + 1);
    }
    *n = count;
  });
}

int hcl_kernel_signature(const char* bundle, const char* kernel, uint8_t* kinds,
                         uint8_t* part_classes, int cap, int* arity) {
  return guarded([&] {
    const KernelDef* k = find_kernel(bundle, kernel);
    if (!k) fail(ErrorCode::name, std::string("unknown kernel '") + kernel + "'");
    *arity = static_cast<int>(k->kinds.size());
    for (int i = 0; i < *arity && i < cap; ++i) {
      if (kinds) kinds[i] = k->kinds[i];
      if (part_classes) part_classes[i] = k->part_classes[i];
    }
  });
}

int hcl_buffer_alloc(int dev, uint64_t id, uint64_t first_byte, uint64_t bytes) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    auto it = d.bufs.find(id);
    if (it != d.bufs.end()) {
      if (it->second.first_byte == first_byte && it->second.bytes == bytes) return;
      d.retire(it->second);
      free_alloc(d, it->second);
      d.bufs.erase(it);
    }
    DevAlloc a;
    a.first_byte = first_byte;
    a.bytes = bytes;
    if (bytes) {
      HCL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.ptr), bytes, d.stream));
      HCL_CUDA(cudaMemsetAsync(a.ptr, 0, bytes, d.stream));  // alloc zero-fills (daemon.cpp:21-69)
    }
    auto [pos, ok] = d.bufs.emplace(id, a);
    if (bytes) d.note(pos->second, d.stream, true);
  });
}

int hcl_buffer_bind_external(int dev, uint64_t id, void* ptr, uint64_t first_byte, uint64_t bytes) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    auto it = d.bufs.find(id);
    if (it != d.bufs.end()) {
      d.retire(it->second);
      free_alloc(d, it->second);
      d.bufs.erase(it);
    }
    DevAlloc a;
    a.ptr = static_cast<uint8_t*>(ptr);
    a.first_byte = first_byte;
    a.bytes = bytes;
    a.external = true;
    d.bufs.emplace(id, a);
  });
}

// Cross-process buffers (fused exchange kernels over NVLink):
// a cudaMalloc allocation whose IPC handle other processes map as peer memory.
int hcl_buffer_alloc_shared(int dev, uint64_t id, uint64_t bytes, uint8_t* ipc_handle) {
  return guarded([&] {
    if (!ipc_handle || !bytes) fail(ErrorCode::argument, "hcl_buffer_alloc_shared: need a handle slot and bytes > 0");
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    auto it = d.bufs.find(id);
    if (it != d.bufs.end()) {
      d.retire(it->second);
      free_alloc(d, it->second);
      d.bufs.erase(it);
    }
    DevAlloc a;
    a.bytes = bytes;
    a.mem = 1;
    HCL_CUDA(cudaMalloc(reinterpret_cast<void**>(&a.ptr), bytes));
    HCL_CUDA(cudaMemsetAsync(a.ptr, 0, bytes, d.stream));
    HCL_CUDA(cudaStreamSynchronize(d.stream));  // zeroed before any peer can store into it
    cudaIpcMemHandle_t h;
    HCL_CUDA(cudaIpcGetMemHandle(&h, a.ptr));
    std::memcpy(ipc_handle, &h, sizeof(h));
    auto [pos, ok] = d.bufs.emplace(id, a);
    d.note(pos->second, d.stream, true);
  });
}

int hcl_buffer_open_shared(int dev, uint64_t id, const uint8_t* ipc_handle, uint64_t bytes) {
  return guarded([&] {
    if (!ipc_handle) fail(ErrorCode::argument, "hcl_buffer_open_shared: handle is NULL");
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    auto it = d.bufs.find(id);
    if (it != d.bufs.end()) {
      d.retire(it->second);
      free_alloc(d, it->second);
      d.bufs.erase(it);
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof(h));
    DevAlloc a;
    a.bytes = bytes;
    a.mem = 2;
    a.external = true;  // another process's memory: writes to it are not versioned here
    HCL_CUDA(cudaIpcOpenMemHandle(reinterpret_cast<void**>(&a.ptr), h, cudaIpcMemLazyEnablePeerAccess));
    d.bufs.emplace(id, a);
  });
}

constexpr uint64_t kSplitCopyBytes = 32ull << 20;

// Host <-> device copies run on the device's H2D / D2H streams, ordered after
// the buffer's last writer (and, for a write, its readers); a blocking call
// waits for its own copy only.
static int buffer_copy(int dev, uint64_t id, uint64_t offset, void* host, uint64_t len, bool write,
                       bool async) {
  return guarded([&] {
    Device& d = device(dev);
    // held through a blocking wait: the event must not be recycled meanwhile
    std::lock_guard<std::mutex> lock(d.mu);
    DevAlloc& a = alloc_of(d, id, write ? "write_buffer" : "read_buffer");
    uint8_t* p = range_ptr(a, offset, len, id, write ? "write_buffer" : "read_buffer");
    if (!len) return;
    HCL_CUDA(cudaSetDevice(d.ordinal));
    cudaStream_t s = write ? d.h2d : d.d2h;
    const cudaMemcpyKind kind = write ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    d.wait_for(a, s, write);
    if (len >= kSplitCopyBytes) {  // two halves on two copy streams, joined on s
      cudaStream_t s2 = write ? d.h2d2 : d.d2h2;
      d.wait_for(a, s2, write);
      const uint64_t h = (len / 2) & ~uint64_t(4095);
      uint8_t* hp = static_cast<uint8_t*>(host);
      HCL_CUDA(cudaMemcpyAsync(write ? p : hp, write ? static_cast<const void*>(hp) : p, h, kind, s));
      HCL_CUDA(cudaMemcpyAsync(write ? p + h : hp + h, write ? static_cast<const void*>(hp + h) : p + h, len - h,
                               kind, s2));
      cudaEvent_t j = d.sync_event();
      HCL_CUDA(cudaEventRecord(j, s2));
      HCL_CUDA(cudaStreamWaitEvent(s, j, 0));
      d.spare_sync.push_back(j);  // the enqueued wait keeps its snapshot
    } else {
      HCL_CUDA(cudaMemcpyAsync(write ? p : host, write ? static_cast<const void*>(host) : p, len, kind, s));
    }
    cudaEvent_t done = d.note(a, s, write);
    if (!async) HCL_CUDA(cudaEventSynchronize(done));
  });
}

int hcl_buffer_write(int dev, uint64_t id, uint64_t offset, const void* src, uint64_t len) {
  return buffer_copy(dev, id, offset, const_cast<void*>(src), len, true, false);
}
int hcl_buffer_read(int dev, uint64_t id, uint64_t offset, void* dst, uint64_t len) {
  return buffer_copy(dev, id, offset, dst, len, false, false);
}
int hcl_buffer_write_async(int dev, uint64_t id, uint64_t offset, const void* src, uint64_t len) {
  return buffer_copy(dev, id, offset, const_cast<void*>(src), len, true, true);
}
int hcl_buffer_read_async(int dev, uint64_t id, uint64_t offset, void* dst, uint64_t len) {
  return buffer_copy(dev, id, offset, dst, len, false, true);
}

int hcl_buffer_copy_peer(int dst_dev, uint64_t dst_id, uint64_t dst_offset, int src_dev,
                         uint64_t src_id, uint64_t src_offset, uint64_t len) {
  return guarded([&] {
    Device& dd = device(dst_dev);
    Device& sd = device(src_dev);
    std::unique_lock<std::mutex> l1(dd.mu, std::defer_lock), l2(sd.mu, std::defer_lock);
    if (&dd == &sd)
      l1.lock();
    else
      std::lock(l1, l2);
    DevAlloc& da = alloc_of(dd, dst_id, "copy_peer dst");
    DevAlloc& sa = alloc_of(sd, src_id, "copy_peer src");
    uint8_t* dp = range_ptr(da, dst_offset, len, dst_id, "copy_peer dst");
    uint8_t* sp = range_ptr(sa, src_offset, len, src_id, "copy_peer src");
    if (!len) return;
    if (&dd == &sd) {
      HCL_CUDA(cudaSetDevice(dd.ordinal));
      dd.wait_for(sa, dd.stream, false);
      dd.wait_for(da, dd.stream, true);
      HCL_CUDA(cudaMemcpyAsync(dp, sp, len, cudaMemcpyDeviceToDevice, dd.stream));
      dd.note(sa, dd.stream, false);
      dd.note(da, dd.stream, true);
      return;
    }
    // the source's compute stream first waits for the source's writer; the copy
    // runs on the destination's compute stream (NVLink P2P through NVSwitch)
    HCL_CUDA(cudaSetDevice(sd.ordinal));
    sd.wait_for(sa, sd.stream, false);
    cudaEvent_t ready = sd.sync_event();
    HCL_CUDA(cudaEventRecord(ready, sd.stream));
    HCL_CUDA(cudaSetDevice(dd.ordinal));
    HCL_CUDA(cudaStreamWaitEvent(dd.stream, ready, 0));
    dd.wait_for(da, dd.stream, true);
    HCL_CUDA(cudaMemcpyPeerAsync(dp, dd.ordinal, sp, sd.ordinal, len, dd.stream));
    dd.note(da, dd.stream, true);
    // the source must not be overwritten before the copy lands
    cudaEvent_t done = dd.sync_event();
    HCL_CUDA(cudaEventRecord(done, dd.stream));
    HCL_CUDA(cudaSetDevice(sd.ordinal));
    HCL_CUDA(cudaStreamWaitEvent(sd.stream, done, 0));
    sd.note(sa, sd.stream, false);
    sd.spare_sync.push_back(ready);
    dd.spare_sync.push_back(done);
  });
}

int hcl_buffer_swap(int dev, uint64_t id_a, uint64_t id_b) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    auto a = d.bufs.find(id_a);
    auto b = d.bufs.find(id_b);
    if (b == d.bufs.end()) fail(ErrorCode::handle, "buffer_swap: buffer " + std::to_string(id_b) + " not on device");
    if (a == d.bufs.end()) {  // id_a had no allocation here: it takes id_b's
      d.bufs.emplace(id_a, b->second);
      d.bufs.erase(b);
      return;
    }
    std::swap(a->second, b->second);
  });
}

int hcl_buffer_release(int dev, uint64_t id) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    auto it = d.bufs.find(id);
    if (it == d.bufs.end()) return;  // idempotent
    HCL_CUDA(cudaSetDevice(d.ordinal));
    d.retire(it->second);
    free_alloc(d, it->second);
    d.bufs.erase(it);
  });
}

int hcl_buffer_device_ptr(int dev, uint64_t id, void** ptr, uint64_t* first_byte, uint64_t* bytes) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    DevAlloc& a = alloc_of(d, id, "device_ptr");
    if (ptr) *ptr = a.ptr;
    if (first_byte) *first_byte = a.first_byte;
    if (bytes) *bytes = a.bytes;
  });
}

int hcl_stream_acquire(int dev, uint64_t id, int write) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    d.wait_for(alloc_of(d, id, "stream_acquire"), d.stream, write != 0);
  });
}

int hcl_comm_stream(int dev, void** stream) {
  return guarded([&] { *stream = device(dev).comm; });
}

int hcl_comm_acquire(int dev, uint64_t id, int write) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    d.wait_for(alloc_of(d, id, "comm_acquire"), d.comm, write != 0);
  });
}

int hcl_comm_release(int dev, uint64_t id, int write) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    d.note(alloc_of(d, id, "comm_release"), d.comm, write != 0);
  });
}

int hcl_stream_release(int dev, uint64_t id, int write) {
  return guarded([&] {
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    d.note(alloc_of(d, id, "stream_release"), d.stream, write != 0);
  });
}

int hcl_launch(int dev, const char* kernel, const hcl_arg* args, uint32_t nargs,
               const uint64_t goff[3], const uint64_t gsize[3], uint32_t dims,
               uint64_t* work_units) {
  return guarded([&] {
    const KernelDef* k = find_kernel_any(kernel ? kernel : "");
    if (!k) fail(ErrorCode::name, std::string("unknown kernel '") + (kernel ? kernel : "") + "'");
    if (nargs != k->kinds.size())
      fail(ErrorCode::argument, std::string(kernel) + ": expected " + std::to_string(k->kinds.size()) +
                                    " arguments, got " + std::to_string(nargs));
    Device& d = device(dev);
    std::lock_guard<std::mutex> lock(d.mu);
    HCL_CUDA(cudaSetDevice(d.ordinal));
    std::vector<LaunchArg> la(nargs);
    for (uint32_t i = 0; i < nargs; ++i) {
      bool want_scalar = k->kinds[i] == HCL_ARG_SCALAR;
      bool is_scalar = args[i].kind == HCL_ARG_SCALAR;
      if (want_scalar != is_scalar)
        fail(ErrorCode::argument, std::string(kernel) + " argument " + std::to_string(i) +
                                      (want_scalar ? ": expected a scalar" : ": expected a buffer"));
      la[i].kind = args[i].kind;
      la[i].scalar = args[i].scalar;
      la[i].id = args[i].buffer_id;
      if (!is_scalar) {
        DevAlloc& a = alloc_of(d, args[i].buffer_id, kernel);
        la[i].buf = BufView{a.ptr, a.first_byte, a.bytes, a.version};
      }
    }
    LaunchCtx c;
    c.dev = dev;
    c.stream = d.stream;
    c.sm_count = d.sm_count;
    c.sm_budgeted = d.sm_count < d.sm_physical;
    c.args = la.data();
    c.nargs = nargs;
    c.dims = dims ? dims : 1;
    c.whole = gsize == nullptr;  // NULL gsize: the kernel's whole range
    for (int i = 0; i < 3; ++i) {
      c.goff[i] = goff ? goff[i] : 0;
      c.gsize[i] = gsize ? gsize[i] : 1;
    }
    c.scratch = scratch_for;
    // order after pending copies of the arguments (RAW; WAR for outputs)
    for (uint32_t i = 0; i < nargs; ++i)
      if (args[i].kind != HCL_ARG_SCALAR)
        d.wait_for(alloc_of(d, args[i].buffer_id, kernel), d.stream, args[i].kind != HCL_ARG_IN);
    const bool timed = !t_launch_untimed;  // hcl_finish's device_ms counts the timed launches
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
      e0 = d.event();
      e1 = d.event();
      HCL_CUDA(cudaEventRecord(e0, d.stream));
    }
    uint64_t w = 0;
    if (k->graphable && graphs_enabled()) {
      // the second identical launch is captured into a CUDA graph, later ones replay it
      // (same kernels, same work -- only the per-kernel launch gaps go)
      GraphEntry& ge = d.graphs[graph_key(k, la, c, d)];
      if (ge.exec) {
        HCL_CUDA(cudaGraphLaunch(ge.exec, d.stream));
        g_kernel_launches += ge.kernels;  // the replay launches the captured kernels again
        w = ge.work;
      } else if (ge.seen) {
        HCL_CUDA(cudaStreamBeginCapture(d.stream, cudaStreamCaptureModeThreadLocal));
        cudaGraph_t g = nullptr;
        const uint64_t k0 = t_kernel_launches;
        try {
          w = k->launch(c);
        } catch (...) {
          cudaStreamEndCapture(d.stream, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        HCL_CUDA(cudaStreamEndCapture(d.stream, &g));
        const cudaError_t ie = cudaGraphInstantiate(&ge.exec, g, 0);
        cudaGraphDestroy(g);
        HCL_CUDA(ie);
        HCL_CUDA(cudaGraphLaunch(ge.exec, d.stream));
        ge.work = w;
        ge.kernels = t_kernel_launches - k0;  // counted once at capture = this launch
      } else {
        w = k->launch(c);
        ge.seen = true;
      }
    } else {
      w = k->launch(c);
    }
    if (timed) {
      HCL_CUDA(cudaEventRecord(e1, d.stream));
      d.timed.emplace_back(e0, e1);
    }
    for (uint32_t i = 0; i < nargs; ++i)
      if (args[i].kind == HCL_ARG_IN) d.note(alloc_of(d, args[i].buffer_id, kernel), d.stream, false);
    for (uint32_t i = 0; i < nargs; ++i)
      if (args[i].kind == HCL_ARG_OUT || args[i].kind == HCL_ARG_INOUT)
        d.note(alloc_of(d, args[i].buffer_id, kernel), d.stream, true);
    if (work_units) *work_units = w;
  });
}

// In-process collective over NVLink peer copies (SURVEY.md §8(b)'s proposed
// hcl_collective): devs[i] holds buffer buf_ids[i].
//   op 0 broadcast:  bytes [0, count*es) of devs[root] to every device
//   op 1 allgather:  device i contributes elements [i*count, (i+1)*count)
//   op 2 allreduce:  element-wise sum in device order (0, 1, ..., ndev-1) on the
//                    root, then broadcast -- deterministic and bit-identical on
//                    every device; dtype 0 int64, 1 fp64, 2 fp32
int hcl_collective(int op, const int* devs, int ndev, const uint64_t* buf_ids, uint64_t count, int dtype, int root) {
  return guarded([&] {
    if (ndev < 1 || !devs || !buf_ids) fail(ErrorCode::argument, "collective: need at least one device");
    if (dtype < 0 || dtype > 2) fail(ErrorCode::argument, "collective: dtype must be 0 (i64), 1 (f64) or 2 (f32)");
    if (root < 0 || root >= ndev) fail(ErrorCode::argument, "collective: root out of range");
    const uint64_t es = dtype == 2 ? 4 : 8, bytes = count * es;
    if (op == 0) {
      for (int i = 0; i < ndev; ++i)
        if (i != root) check_rc(hcl_buffer_copy_peer(devs[i], buf_ids[i], 0, devs[root], buf_ids[root], 0, bytes));
    } else if (op == 1) {
      for (int j = 0; j < ndev; ++j)
        for (int i = 0; i < ndev; ++i)
          if (i != j)
            check_rc(hcl_buffer_copy_peer(devs[i], buf_ids[i], j * bytes, devs[j], buf_ids[j], j * bytes, bytes));
    } else if (op == 2) {
      const int rd = devs[root];
      const uint64_t acc = coll_tmp_id(), tmp = coll_tmp_id();
      check_rc(hcl_buffer_alloc(rd, acc, 0, bytes));
      check_rc(hcl_buffer_alloc(rd, tmp, 0, bytes));
      check_rc(hcl_buffer_copy_peer(rd, acc, 0, devs[0], buf_ids[0], 0, bytes));
      for (int i = 1; i < ndev; ++i) {
        check_rc(hcl_buffer_copy_peer(rd, tmp, 0, devs[i], buf_ids[i], 0, bytes));
        Device& d = device(rd);
        std::lock_guard<std::mutex> lock(d.mu);
        HCL_CUDA(cudaSetDevice(d.ordinal));
        DevAlloc& aa = alloc_of(d, acc, "collective");
        DevAlloc& ta = alloc_of(d, tmp, "collective");
        d.wait_for(aa, d.stream, true);
        d.wait_for(ta, d.stream, false);
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ceil_div(count, 256), 8ull * d.sm_count));
        if (count) {
          if (dtype == 0)
            local_add_kernel<long long><<<grid, 256, 0, d.stream>>>(reinterpret_cast<long long*>(aa.ptr),
                                                                    reinterpret_cast<const long long*>(ta.ptr), count);
          else if (dtype == 1)
            local_add_kernel<double><<<grid, 256, 0, d.stream>>>(reinterpret_cast<double*>(aa.ptr),
                                                                 reinterpret_cast<const double*>(ta.ptr), count);
          else
            local_add_kernel<float><<<grid, 256, 0, d.stream>>>(reinterpret_cast<float*>(aa.ptr),
                                                                reinterpret_cast<const float*>(ta.ptr), count);
          HCL_LAUNCHED();
        }
        d.note(aa, d.stream, true);
        d.note(ta, d.stream, false);
      }
      for (int i = 0; i < ndev; ++i) check_rc(hcl_buffer_copy_peer(devs[i], buf_ids[i], 0, rd, acc, 0, bytes));
      check_rc(hcl_buffer_release(rd, acc));
      check_rc(hcl_buffer_release(rd, tmp));
    } else {
      fail(ErrorCode::argument, "collective: op must be 0 (broadcast), 1 (allgather) or 2 (allreduce)");
    }
  });
}

int hcl_finish(int dev, double* device_ms) {
  return guarded([&] {
    Device& d = device(dev);
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
    {
      std::lock_guard<std::mutex> lock(d.mu);
      timed.swap(d.timed);
    }
    // the streams are fixed for the device's lifetime: synchronize them without
    // the device lock so other threads keep issuing work meanwhile
    HCL_CUDA(cudaSetDevice(d.ordinal));
    HCL_CUDA(cudaStreamSynchronize(d.h2d));
    HCL_CUDA(cudaStreamSynchronize(d.h2d2));
    HCL_CUDA(cudaStreamSynchronize(d.stream));
    HCL_CUDA(cudaStreamSynchronize(d.comm));
    HCL_CUDA(cudaStreamSynchronize(d.d2h));
    HCL_CUDA(cudaStreamSynchronize(d.d2h2));
    double total = 0.0;
    for (auto& [a, b] : timed) {
      float ms = 0.f;
      HCL_CUDA(cudaEventSynchronize(b));
      HCL_CUDA(cudaEventElapsedTime(&ms, a, b));
      total += ms;
    }
    std::lock_guard<std::mutex> lock(d.mu);
    for (auto& [a, b] : timed) {
      d.spare_events.push_back(a);
      d.spare_events.push_back(b);
    }
    if (device_ms) *device_ms = total;
  });
}

}  // extern "C"
