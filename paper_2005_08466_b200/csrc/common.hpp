// Shared internals of libhaocl_b200: error model, launch descriptors and the
// kernel registry types. Nothing here crosses the C-ABI (include/hcl_cabi.h).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace hcl {

// Numeric values mirror haocl::ErrorCode (proj/include/haocl/error.hpp:11-36).
enum class ErrorCode : uint16_t {
  internal = 0,
  protocol = 1,
  version = 2,
  malformed = 3,
  encoding = 4,
  unknown_call = 5,
  busy = 6,
  precondition = 7,
  reassembly_conflict = 8,
  argument = 9,
  name = 10,
  config = 11,
  connect = 12,
  timeout = 13,
  transport = 14,
  remote = 15,
  handle = 16,
  policy = 17,
  size = 18,
  mapping = 19,
  unknown_device = 20,
  registration = 21,
  contract = 22,
  parse = 23,
};

const char* error_code_name(ErrorCode code);

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message)
      : std::runtime_error(std::string(error_code_name(code)) + ": " + message), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] inline void fail(ErrorCode code, const std::string& message) {
  throw Error(code, message);
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define HCL_CUDA(x) ::hcl::cuda_check((x), #x, __FILE__, __LINE__)

// Counts every CUDA kernel this library launches (the bench reports it as
// gpu_launches). Kernel launch sites use HCL_LAUNCHED() right after <<<>>>.
extern std::atomic<uint64_t> g_kernel_launches;
extern thread_local uint64_t t_kernel_launches;  // this thread's share (graph capture counts)
// Set by a caller that times its launches itself (the HostContext runtime records one
// CUDA-event pair per part for the scheduler's rates): hcl_launch then skips its own
// pair (each timing event record serializes the stream's front end, ~2.5 us a record).
extern thread_local bool t_launch_untimed;
#define HCL_LAUNCHED()                                            \
  do {                                                            \
    ::hcl::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
    ++::hcl::t_kernel_launches;                                   \
    HCL_CUDA(cudaGetLastError());                                 \
  } while (0)

// The resident slice of one buffer on one device: `ptr` addresses logical
// byte `first_byte` of the buffer; `bytes` are resident. `logical_size` is
// the size the host created the buffer with.
struct BufView {
  uint8_t* ptr = nullptr;
  uint64_t first_byte = 0;
  uint64_t bytes = 0;
  // changes with every write through this library (copies, peer copies, kernel
  // outputs); 0 for externally bound memory (never assumed unchanged)
  uint64_t version = 0;
};

struct LaunchArg {
  uint32_t kind = 0;  // hcl_arg_kind
  int64_t scalar = 0;
  uint64_t id = 0;
  BufView buf;
};

struct LaunchCtx {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  bool sm_budgeted = false;  // sm_count is a budget below the GPU's SM count (hcl_device_set_sm_budget)
  const LaunchArg* args = nullptr;
  uint32_t nargs = 0;
  uint64_t goff[3] = {0, 0, 0};
  uint64_t gsize[3] = {1, 1, 1};
  uint32_t dims = 1;
  // true when the launch covers the kernel's whole range (the reference's
  // enqueue_ndrange_kernel carries global_size but never splits it,
  // proj/src/daemon.cpp:334); false for one sub-range of a partitioned launch
  bool whole = true;
  // scratch: device memory owned by the device record, grown on demand
  void* (*scratch)(int dev, size_t bytes) = nullptr;
};

// The dim-0 rows [lo, lo+cnt) this launch computes out of `total`.
inline void sub_range(const LaunchCtx& c, uint64_t total, uint64_t& lo, uint64_t& cnt,
                      const char* what) {
  if (c.whole) {
    lo = 0;
    cnt = total;
    return;
  }
  lo = c.goff[0];
  cnt = c.gsize[0];
  if (lo + cnt > total)
    fail(ErrorCode::argument, std::string(what) + ": NDRange sub-range exceeds the global range");
}

using LaunchFn = uint64_t (*)(LaunchCtx&);
// Bytes per dim-0 row of a SPLIT_ROWS argument, from the launch's scalars.
using RowBytesFn = uint64_t (*)(const int64_t* scalars, uint32_t nargs, uint32_t arg_index);
// Global range (dim 0) of the kernel when launched whole.
using RowsFn = uint64_t (*)(const int64_t* scalars, uint32_t nargs);

struct KernelDef {
  const char* bundle;
  const char* name;
  std::vector<uint8_t> kinds;        // hcl_arg_kind per argument
  std::vector<uint8_t> part_classes; // hcl_part_class per argument
  LaunchFn launch;
  RowBytesFn row_bytes;  // may be null when no SPLIT_ROWS argument
  RowsFn rows;           // may be null (then dim 0 must be given)
  // the launch function only enqueues stream work (no host syncs): repeated
  // identical launches are captured once into a CUDA graph and replayed
  bool graphable = false;
};

const std::vector<KernelDef>& registry();
const KernelDef* find_kernel(const std::string& bundle, const std::string& name);
const KernelDef* find_kernel_any(const std::string& name);
bool bundle_exists(const std::string& bundle);

// ---- helpers for launchers --------------------------------------------

inline int64_t scalar_arg(const LaunchCtx& c, uint32_t i, const char* what) {
  if (c.args[i].kind != 0) fail(ErrorCode::argument, std::string(what) + ": expected a scalar argument");
  return c.args[i].scalar;
}

inline const BufView& buffer_arg(const LaunchCtx& c, uint32_t i, const char* what) {
  if (c.args[i].kind == 0) fail(ErrorCode::argument, std::string(what) + ": expected a buffer argument");
  return c.args[i].buf;
}

// Pointer to logical byte `byte` of a buffer, checking that [byte, byte+len)
// is resident on this device.
template <typename T>
T* at_byte(const BufView& b, uint64_t byte, uint64_t len, const char* what) {
  if (byte < b.first_byte || byte + len > b.first_byte + b.bytes)
    fail(ErrorCode::argument, std::string(what) + ": byte range [" + std::to_string(byte) + ", " +
                                  std::to_string(byte + len) + ") not resident on the device (slice [" +
                                  std::to_string(b.first_byte) + ", " +
                                  std::to_string(b.first_byte + b.bytes) + "))");
  return reinterpret_cast<T*>(b.ptr + (byte - b.first_byte));
}

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

}  // namespace hcl
