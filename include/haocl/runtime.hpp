#pragma once

// haocl::HostContext on B200 — the reference's OpenCL-like host API
// (proj/include/haocl/runtime.hpp:97-153) re-targeted from TCP node daemons to
// the in-process CUDA C-ABI (include/hcl_cabi.h).
//
// Kept verbatim in shape: get_device_ids, create_queue, create_buffer,
// create_program, create_kernel, set_kernel_arg, enqueue_write_buffer,
// enqueue_read_buffer, enqueue_ndrange_kernel, submit_task, launch_task,
// finish, release, breakdown, trace, scheduler. Buffers are placed lazily on
// the first queue that touches them and migrate device-to-device over NVLink
// (the reference migrates host-mediated, proj/src/runtime.cpp:220-249).
//
// New: the PARTITIONED NDRange launch. enqueue_ndrange_kernel(kernel, global,
// dims, queues, weights) splits dim 0 of the global range into one sub-range
// per queue (cumulative-floor split by integer weights; equal weights give the
// reference's block_range, proj/src/bench.cpp:31-33), scatters SPLIT_ROWS
// inputs, replicates REPLICATE inputs, launches every part concurrently, and
// leaves SPLIT_ROWS outputs sharded until read (gathered) or used elsewhere.

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <set>
#include <span>
#include <string>
#include <vector>

namespace haocl {

// ---- errors (proj/include/haocl/error.hpp) --------------------------------
enum class ErrorCode : uint16_t {
  internal = 0, protocol = 1, version = 2, malformed = 3, encoding = 4, unknown_call = 5, busy = 6,
  precondition = 7, reassembly_conflict = 8, argument = 9, name = 10, config = 11, connect = 12,
  timeout = 13, transport = 14, remote = 15, handle = 16, policy = 17, size = 18, mapping = 19,
  unknown_device = 20, registration = 21, contract = 22, parse = 23,
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

// ---- handles, timing, trace (proj/include/haocl/runtime.hpp:29-90) -------
enum class HandleKind : uint8_t { context, queue, buffer, program, kernel, event };

struct Handle {
  HandleKind kind = HandleKind::event;
  uint64_t id = 0;
  bool operator==(const Handle&) const = default;
};

enum class DeviceType : uint8_t { cpu = 0, gpu = 1, fpga = 2 };

struct DeviceModel {
  DeviceType type = DeviceType::gpu;
  double relative_throughput = 1.0;
};

struct DeviceEntry {
  int global_id = 0;
  int cuda_ordinal = 0;
  uint32_t local_index = 0;
  std::string name;
  DeviceModel model;
};

struct GlobalDeviceMap {
  std::vector<DeviceEntry> entries;
  const DeviceEntry* find(int global_id) const {
    for (const auto& e : entries)
      if (e.global_id == global_id) return &e;
    return nullptr;
  }
};

struct TimingBreakdown {
  double init_ms = 0.0;
  double data_creation_ms = 0.0;
  double transfer_ms = 0.0;
  double compute_ms = 0.0;
  double modeled_compute_ms = 0.0;
  double total() const { return init_ms + data_creation_ms + transfer_ms + compute_ms; }
};

struct TimingFragment {
  double transfer_ms = 0.0;
  double compute_ms = 0.0;  // CUDA-event kernel time on the device
  double modeled_ms = 0.0;  // work_units / (relative_throughput * baseline rate)
};

// One forwarded operation (the reference records one per ApiCallRequest /
// DataTransfer, proj/src/runtime.cpp:198-503).
struct TraceEvent {
  int device = -1;
  std::string function;  // alloc_buffer | write_buffer | read_buffer | launch_kernel | release_object | query_registry | copy_peer
  uint64_t buffer_id = 0;
};

class MessageTrace {
 public:
  void record(TraceEvent event);
  std::vector<TraceEvent> events() const;
  size_t count_calls(const std::string& function, int device = -1) const;
  void clear();

 private:
  mutable std::mutex mutex_;
  std::vector<TraceEvent> events_;
};

// ---- tasks and the scheduler (proj/include/haocl/api.hpp, scheduler.hpp) ---
inline constexpr double kBaselineWorkRate = 1e9;

struct Placement {
  enum class Mode { explicit_device, auto_policy };
  Mode mode = Mode::explicit_device;
  int device_id = 0;
  std::string policy;
  static Placement explicit_on(int gid) { return Placement{Mode::explicit_device, gid, {}}; }
  static Placement auto_with(std::string policy) { return Placement{Mode::auto_policy, -1, std::move(policy)}; }
};

// A bound argument: scalar_i64 or a buffer handle id (wire::TypedValue's i64 /
// handle cases, the only ones the kernel engine consumes).
struct Arg {
  bool is_buffer = false;
  int64_t scalar = 0;
  uint64_t buffer = 0;
  static Arg of_i64(int64_t v) { return Arg{false, v, 0}; }
  static Arg of_handle(uint64_t id) { return Arg{true, 0, id}; }
};

struct KernelTask {
  std::string kernel_name;
  std::vector<Arg> args;
  std::array<uint64_t, 3> global_size = {1, 1, 1};
  uint32_t dims = 1;
  std::string user_id = "default";
  bool shared_flag = true;
  Placement placement;
};

struct TaskEstimate {
  double work_units = 1.0;
  uint64_t in_bytes = 0;
  uint64_t out_bytes = 0;
};

struct DeviceState {
  int global_id = 0;
  DeviceModel model;
  int outstanding_tasks = 0;
  std::map<std::string, double> profiled_rate;  // kernel -> EMA work-units/s
  std::set<uint64_t> resident_buffers;
};

struct ClusterState {
  std::vector<DeviceState> devices;
  DeviceState* find(int global_id);
  const DeviceState* find(int global_id) const;
};

struct SchedulerOptions {
  double baseline_rate = kBaselineWorkRate;
  double net_bandwidth = 1e8;  // bytes/s charged for non-resident data
  double ema_alpha = 0.3;
};

class Scheduler {
 public:
  using PolicyFn = std::function<int(const KernelTask&, const ClusterState&, const TaskEstimate&)>;

  explicit Scheduler(SchedulerOptions options = {}, std::map<std::string, int> kernel_map = {});
  ~Scheduler();
  void configure(SchedulerOptions options, std::map<std::string, int> kernel_map);
  void register_policy(const std::string& name, PolicyFn policy);
  bool has_policy(const std::string& name) const;
  int schedule(const KernelTask& task, const TaskEstimate& estimate);
  void record_profile(int global_id, const std::string& kernel_name, double work_units, double observed_seconds);
  void sync_devices(const std::vector<std::pair<int, DeviceModel>>& devices);
  void note_dispatch(int global_id);
  void note_complete(int global_id);
  void note_resident(uint64_t buffer_id, const std::vector<int>& device_ids);
  void drop_resident(uint64_t buffer_id);
  ClusterState snapshot() const;
  const SchedulerOptions& options() const;
  static double modeled_cost(const DeviceState& device, const std::string& kernel_name,
                             const TaskEstimate& estimate, const SchedulerOptions& options, bool inputs_resident);

  // New: integer split weights for a partitioned launch over `gids`, proportional
  // to each device's measured (EMA) rate for the kernel, else its modeled rate.
  // Equal rates give equal weights (and so the reference's block_range split).
  std::vector<uint64_t> partition_weights(const std::string& kernel_name, const std::vector<int>& gids) const;
  // Persisted EMA profiles: "gid<TAB>kernel<TAB>rate" lines (exact round trip).
  // import replaces the rates of the listed devices it knows; returns how many.
  std::string export_profiles() const;
  size_t import_profiles(const std::string& text);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// Cumulative-floor split: boundary_i = floor(total * W_{<i} / W) (128-bit).
std::vector<uint64_t> split_ranges(uint64_t total, const std::vector<uint64_t>& weights);
// nnz-balanced split (spmv_partition_ranges, proj/src/kernels.cpp:300-321),
// generalised to weights: part p targets ceil(nnz * w_p / W).
std::vector<int64_t> spmv_partition_ranges(int64_t rows, const int64_t* row_ptr, int64_t parts,
                                           const std::vector<uint64_t>& weights = {});

struct HostOptions {
  SchedulerOptions scheduler;
  std::map<std::string, int> kernel_map;  // static_map table
  std::vector<int> cuda_ordinals;         // empty: every visible GPU
};

class HostContext {
 public:
  // Enumerates CUDA devices through hcl_init (one stream per GPU) and builds the
  // global device map (ascending CUDA ordinal). Replaces connect + DeviceIdRequest.
  static HostContext init(const HostOptions& options = {});

  HostContext(HostContext&&) noexcept;
  HostContext& operator=(HostContext&&) noexcept;
  ~HostContext();

  const GlobalDeviceMap& device_map() const;
  std::vector<int> get_device_ids(std::optional<DeviceType> filter = {}) const;

  Handle create_queue(int global_device_id, std::string user_id = "default", bool shared = true);
  Handle create_buffer(uint64_t size);
  Handle create_program(const std::string& bundle);
  Handle create_kernel(Handle program, const std::string& kernel_name);
  void set_kernel_arg(Handle kernel, uint32_t index, int64_t scalar);
  void set_kernel_arg(Handle kernel, uint32_t index, Handle buffer);

  // blocking = false (OpenCL's blocking_write = CL_FALSE): the copy is queued on
  // the device's H2D stream, ordered against kernels that use the buffer; the
  // host memory must stay valid (and should be pinned) until finish(queue).
  Handle enqueue_write_buffer(Handle queue, Handle buffer, std::span<const uint8_t> data, uint64_t offset = 0,
                              bool blocking = true);
  std::vector<uint8_t> enqueue_read_buffer(Handle queue, Handle buffer);
  // Read into caller memory (pinned memory gives full PCIe/C2C bandwidth).
  // blocking = false: queued on the D2H stream; dst is valid after finish(queue).
  void enqueue_read_buffer_into(Handle queue, Handle buffer, void* dst, uint64_t offset, uint64_t len,
                                bool blocking = true);
  Handle enqueue_ndrange_kernel(Handle queue, Handle kernel, std::array<uint64_t, 3> global_size = {1, 1, 1},
                                uint32_t dims = 1);
  // Partitioned NDRange over several queues (one device each). No weights and
  // no bounds: the split follows the scheduler's EMA-profiled rates per
  // (device, kernel), with 2% hysteresis so profiling noise does not move
  // shards between devices on every launch.
  Handle enqueue_ndrange_kernel(Handle kernel, std::array<uint64_t, 3> global_size, uint32_t dims,
                                const std::vector<Handle>& queues, std::vector<uint64_t> weights = {},
                                std::vector<uint64_t> bounds = {});  // explicit row boundaries (parts+1), e.g. nnz-balanced
  // One sub-range [row_offset, row_offset+rows) of dim 0 of the global range on
  // one queue (clEnqueueNDRangeKernel's global_work_offset): the unit a rank
  // runs when the partitioned NDRange spans processes (one process per GPU).
  // SPLIT_ROWS buffers need only that slice resident on the queue's device.
  Handle enqueue_ndrange_range(Handle queue, Handle kernel, std::array<uint64_t, 3> global_size, uint32_t dims,
                               uint64_t row_offset, uint64_t rows);
  // The split a partitioned launch of `kernel` would use (parts+1 row boundaries).
  std::vector<uint64_t> partition_plan(Handle kernel, std::array<uint64_t, 3> global_size,
                                       const std::vector<Handle>& queues, std::vector<uint64_t> weights = {});

  // ---- collectives across processes (one GPU per rank, NCCL over NVLink) ----
  // Join the communicator for the queue's device (unique id from rank 0).
  void init_collectives(Handle queue, int rank, int nranks, const std::vector<uint8_t>& nccl_unique_id);
  // Rank r holds bytes [bounds[r], bounds[r+1]) of `buffer` on the queue's
  // device; afterwards every rank holds [bounds[0], bounds[nranks]) (uneven
  // allgather: PageRank's rank vector).
  void enqueue_allgather(Handle queue, Handle buffer, const std::vector<uint64_t>& byte_bounds);
  // Element-wise int64 sum of every rank's copy (k-means centroid sums).
  void enqueue_allreduce_sum_i64(Handle queue, Handle buffer);
  // Root's bytes to every rank (GEMM B).
  void enqueue_broadcast(Handle queue, Handle buffer, int root);
  // Fused-exchange plumbing (one process per GPU): back
  // `buffer` on the queue's device with IPC-exportable memory and return its
  // 64-byte handle; map a peer rank's handle on the queue's device and return
  // the mapped device address (kernels such as pagerank_step_exchange store
  // into it over NVLink); a stream-ordered barrier across the communicator,
  // after which `completed` buffers are whole on the queue's device (the
  // peers' stores filled the rows this rank did not write).
  std::vector<uint8_t> share_buffer(Handle queue, Handle buffer);
  // Back `buffer` on the queue's device with caller-owned device memory of at
  // least its size (no copy; the caller keeps ownership and must keep it alive
  // until the buffer is released). Bound as the buffer's whole allocation with
  // nothing valid yet -- e.g. a symmetric-memory tensor whose NVSwitch
  // multicast address a kernel stores through (pagerank_step_binned).
  void bind_external(Handle queue, Handle buffer, uint64_t device_ptr);
  uint64_t open_shared_buffer(Handle queue, const std::vector<uint8_t>& ipc_handle, uint64_t bytes);
  void enqueue_barrier(Handle queue, const std::vector<Handle>& completed = {});

  std::pair<int, Handle> submit_task(const KernelTask& task);
  Handle launch_task(Handle queue, const KernelTask& task);

  // Waits for the queue's device stream and drains its transfer/compute fragment.
  TimingFragment finish(Handle queue);
  void release(Handle handle);

  TimingBreakdown breakdown() const;
  void add_data_creation_ms(double ms);
  MessageTrace& trace();
  Scheduler& scheduler();
  // SM budget of a (logical) device: its kernels size their grids to `sms`
  // SMs, and the scheduler's model relative_throughput becomes sms/SM count
  // (emulated heterogeneous devices on one GPU; hcl_device_set_sm_budget)
  void set_device_sm_budget(int global_device_id, int sms);
  uint64_t buffer_size(Handle buffer) const;
  int queue_device(Handle queue) const;
  // Device pointer of a buffer's resident slice on a device (for zero-copy interop).
  void* buffer_device_ptr(Handle buffer, int global_device_id, uint64_t* first_byte = nullptr,
                          uint64_t* bytes = nullptr) const;

 private:
  HostContext();
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace haocl
