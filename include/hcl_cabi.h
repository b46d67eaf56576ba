/*
 * hcl_cabi.h — device-level C-ABI of the B200 partitioned-NDRange runtime.
 *
 * This is the boundary that replaces the reference's node-side "ICD" layer:
 * the 5-op forwarded-call table served by NodeDaemon
 * (proj/include/haocl/api.hpp:19-21, proj/src/daemon.cpp:159-170) and the
 * kernel engine it dispatches to, haocl::kernels::execute
 * (proj/include/haocl/kernels.hpp:52-55, proj/src/kernels.cpp:268-283).
 * Instead of TCP frames to a daemon, the host runtime calls these functions
 * in-process; each device is one CUDA GPU with one stream.
 *
 * Conventions
 *   - Plain C types only; no torch or C++ types cross this boundary.
 *   - Return 0 on success, otherwise HCL_ERR_BASE + haocl::ErrorCode
 *     (proj/include/haocl/error.hpp:11-36). The offset exists because
 *     ErrorCode::internal == 0. The message of the most
 *     recent failure on the calling thread is hcl_last_error().
 *   - Thread safe across devices; calls for one device are serialized on that
 *     device's stream (the reference serializes per device with a mutex,
 *     proj/src/daemon.cpp:328-332).
 *   - Buffers are identified by (device, 64-bit id). A device may hold the
 *     whole buffer or one byte slice of it (a partition); offsets are always
 *     LOGICAL byte offsets into the whole buffer.
 */
#ifndef HCL_CABI_H
#define HCL_CABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCL_OK 0
#define HCL_ERR_BASE 1000

/* haocl::ErrorCode values (proj/include/haocl/error.hpp:11-36) */
enum hcl_error_code {
  HCL_E_INTERNAL = 0,
  HCL_E_PRECONDITION = 7,
  HCL_E_ARGUMENT = 9,
  HCL_E_NAME = 10,
  HCL_E_HANDLE = 16,
  HCL_E_POLICY = 17,
  HCL_E_SIZE = 18,
  HCL_E_MAPPING = 19,
  HCL_E_UNKNOWN_DEVICE = 20,
  HCL_E_REGISTRATION = 21,
  HCL_E_CONTRACT = 22
};

/* Argument kinds: ArgKind {scalar_i64, buffer_in, buffer_out}
 * (proj/include/haocl/kernels.hpp:24) plus inout. */
enum hcl_arg_kind { HCL_ARG_SCALAR = 0, HCL_ARG_IN = 1, HCL_ARG_OUT = 2, HCL_ARG_INOUT = 3 };

/* Partition class of an argument for a partitioned NDRange launch
 * (generalises ArgKind). */
enum hcl_part_class {
  HCL_PART_NONE = 0,      /* scalar */
  HCL_PART_REPLICATE = 1, /* whole buffer on every device (GEMM B, PageRank x) */
  HCL_PART_SPLIT_ROWS = 2, /* row slice [lo,hi) of dim 0 on each device (GEMM A, C) */
  HCL_PART_REDUCE_SUM = 3, /* each part produces a full-size int64 partial; the
                              runtime sums them (k-means centroid sums) */
  HCL_PART_EXCHANGE = 5,  /* full-size output on every part's device: each part's
                              kernel writes its rows into ALL copies through the
                              PEERS list (pagerank_step_exchange); afterwards the
                              buffer is whole on every participating device */
  HCL_PART_PEERS = 6,     /* input the runtime fills per part (multi-part launches):
                              uint64 device addresses of the EXCHANGE output's copies
                              on the other parts' devices; the next argument is
                              their count (parts - 1) */
  HCL_PART_LOCAL = 7,     /* per-device workspace (inout): allocated whole and
                              zero-filled on every part's device, never copied
                              between devices; its contents are private to the
                              device (pagerank_step_binned's bin values) */
  HCL_PART_MERGE_TOPK = 4  /* each part produces full-size per-query sorted
                              top-k lists (an index and a distance output); the
                              runtime folds them pairwise with the kernel's
                              companion "<name>_merge" (knn reference-set split,
                              proj/src/bench.cpp:367-447 + kernels.cpp:323-361) */
};

/* One bound kernel argument, BoundArg (proj/include/haocl/kernels.hpp:44-50). */
typedef struct hcl_arg {
  uint32_t kind;      /* enum hcl_arg_kind */
  uint32_t reserved;
  int64_t scalar;     /* HCL_ARG_SCALAR */
  uint64_t buffer_id; /* buffer kinds */
} hcl_arg;

/* ---- devices ---------------------------------------------------------- */
/* Enumerate CUDA devices (all visible, or the listed ordinals) and create one
 * stream per device. Idempotent for the same list. Replaces the
 * DeviceIdRequest broadcast (proj/src/runtime.cpp:338-345). */
int hcl_init(const int* cuda_ordinals, int n, int* num_devices);
int hcl_device_count(int* n);
/* type: 1 = gpu (wire::DeviceType, proj/include/haocl/wire.hpp:44) */
int hcl_device_info(int dev, int* type, double* relative_throughput, int* sm_count,
                    uint64_t* hbm_bytes, char* name, int name_cap);
/* SM budget of a logical device: the persistent kernels size their grids to
 * `sms` (even, 2..the GPU's SM count) instead of the whole GPU, so several
 * logical devices on one GPU run concurrently at different rates -- an
 * emulated heterogeneous node set for the rate-proportional split (the
 * reference's DeviceProfile.relative_throughput, proj/src/scheduler.cpp:38-48).
 * relative_throughput becomes sms / SM count; sms <= 0 restores the whole GPU. */
int hcl_device_set_sm_budget(int dev, int sms);

/* ---- registry (query_registry; proj/src/api.cpp:93-117) ---------------- */
/* Kernel names of a bundle as a comma-separated list; arities per kernel. */
int hcl_query_registry(const char* bundle, char* names_csv, int names_cap, uint32_t* arities,
                       int arity_cap, int* n);
/* Per-argument kind (enum hcl_arg_kind) and partition class. */
int hcl_kernel_signature(const char* bundle, const char* kernel, uint8_t* kinds,
                         uint8_t* part_classes, int cap, int* arity);

/* ---- buffers (alloc_buffer / read_buffer / release_object, DataTransfer) */
/* Allocate the logical byte range [first_byte, first_byte+bytes) of buffer `id`
 * on `dev`, zero-filled (proj/src/daemon.cpp:21-69). Idempotent when the same
 * range is already resident; a different range reallocates. */
int hcl_buffer_alloc(int dev, uint64_t id, uint64_t first_byte, uint64_t bytes);
int hcl_buffer_write(int dev, uint64_t id, uint64_t offset, const void* src, uint64_t len);
int hcl_buffer_read(int dev, uint64_t id, uint64_t offset, void* dst, uint64_t len);
/* Asynchronous variants on the device stream (src/dst must be pinned for overlap). */
int hcl_buffer_write_async(int dev, uint64_t id, uint64_t offset, const void* src, uint64_t len);
int hcl_buffer_read_async(int dev, uint64_t id, uint64_t offset, void* dst, uint64_t len);
/* Device-to-device copy over NVLink P2P (replaces host-mediated migration,
 * proj/src/runtime.cpp:237-248). Offsets are logical. */
int hcl_buffer_copy_peer(int dst_dev, uint64_t dst_id, uint64_t dst_offset, int src_dev,
                         uint64_t src_id, uint64_t src_offset, uint64_t len);
int hcl_buffer_release(int dev, uint64_t id); /* idempotent */
/* Exchange the device allocations of two buffer ids (bookkeeping only; their
 * pending-work dependencies travel with the memory). Commits a staged output. */
int hcl_buffer_swap(int dev, uint64_t id_a, uint64_t id_b);
/* Device pointer of the resident slice (ptr addresses logical byte first_byte). */
int hcl_buffer_device_ptr(int dev, uint64_t id, void** ptr, uint64_t* first_byte,
                          uint64_t* bytes);
/* Bind caller-owned device memory as buffer `id` (no copy; caller keeps ownership). */
int hcl_buffer_bind_external(int dev, uint64_t id, void* ptr, uint64_t first_byte,
                             uint64_t bytes);

/* ---- launch (launch_kernel -> kernels::execute) ------------------------ */
/* Launch `kernel` of the built-in bundles on `dev`, asynchronously on the
 * device stream. goff/gsize give the NDRange sub-range (dim 0 = rows) this
 * device computes; gsize == NULL runs the kernel's whole range (what the
 * reference's un-split enqueue_ndrange_kernel does). work_units is the
 * reference's work count for this sub-range (proj/src/kernels.cpp:285-298).
 * Errors: HCL_E_NAME for an unknown kernel, HCL_E_ARGUMENT for arity, size or
 * range violations (as kernels::execute). */
int hcl_launch(int dev, const char* kernel, const hcl_arg* args, uint32_t nargs,
               const uint64_t goff[3], const uint64_t gsize[3], uint32_t dims,
               uint64_t* work_units);

/* ---- completion and timing -------------------------------------------- */
/* Wait for the device stream; device_ms = summed CUDA-event time of kernels
 * launched since the previous finish (may be NULL). */
int hcl_finish(int dev, double* device_ms);
/* Number of CUDA kernels this library has launched (all devices). */
uint64_t hcl_kernel_launch_count(void);
/* Raw CUDA stream of a device (cudaStream_t as void*), for event timing. */
int hcl_device_stream(int dev, void** stream);
/* Interop with work issued directly on the device's compute stream (e.g. an
 * external collective): acquire orders the stream after the buffer's pending
 * copies (write != 0: also after its readers); release records the access so
 * later copies order after it. Copies run on per-device H2D / D2H streams. */
int hcl_stream_acquire(int dev, uint64_t id, int write);
int hcl_stream_release(int dev, uint64_t id, int write);
/* The same for the device's collective stream: NCCL work issued there
 * overlaps kernels on the compute stream, ordered per buffer. */
int hcl_comm_stream(int dev, void** stream);
int hcl_comm_acquire(int dev, uint64_t id, int write);
int hcl_comm_release(int dev, uint64_t id, int write);

/* ---- collectives (NCCL over NVLink 5 / NVSwitch, loaded lazily) ---------- */
int hcl_nccl_unique_id(uint8_t* out, int cap); /* cap >= 128 */
int hcl_nccl_init(int dev, int nranks, int rank, const uint8_t* id);
int hcl_nccl_destroy(int dev);
/* in place: rank r contributes bytes [bounds[r], bounds[r+1]) of the buffer */
int hcl_allgatherv(int dev, uint64_t buffer_id, const uint64_t* bounds);
int hcl_allreduce_sum_i64(int dev, uint64_t buffer_id, uint64_t offset, uint64_t count);
int hcl_broadcast(int dev, uint64_t buffer_id, uint64_t offset, uint64_t bytes, int root);
/* Stream-ordered barrier on the device's kernel stream (a one-element NCCL
 * allreduce): later kernels start after every rank's earlier kernels finished. */
int hcl_nccl_barrier(int dev);

/* In-process collective across this process's devices over NVLink peer
 * copies: devs[i] holds buffer buf_ids[i]. op 0 broadcast
 * count elements from devs[root]; op 1 allgather (device i contributes
 * elements [i*count, (i+1)*count)); op 2 allreduce sum in device order (bit-
 * identical on every device). dtype 0 int64, 1 fp64, 2 fp32. */
int hcl_collective(int op, const int* devs, int ndev, const uint64_t* buf_ids, uint64_t count, int dtype,
                   int root);

/* ---- cross-process peer buffers (fused exchange kernels) -------------- */
/* Allocate buffer `id` on `dev` IPC-exportable (cudaMalloc, zero-filled) and
 * return its 64-byte CUDA IPC handle; another process maps it with
 * hcl_buffer_open_shared as a buffer of its own device, and kernels there
 * store into it over NVLink (pagerank_step_exchange). */
int hcl_buffer_alloc_shared(int dev, uint64_t id, uint64_t bytes, uint8_t* ipc_handle);
int hcl_buffer_open_shared(int dev, uint64_t id, const uint8_t* ipc_handle, uint64_t bytes);

/* ---- remote-node path ------------------------------ */
/* Serve this process's logical devices (hcl_init) to remote hosts over the
 * HaoCL wire protocol: HCL1 frames on TCP `message_port` and message_port+1
 * (data), the daemon side of proj/src/daemon.cpp + net.cpp (Ping/Pong,
 * DeviceIdRequest, DataTransfer/DataAck, the five forwarded ApiCalls,
 * Shutdown). Buffers stay resident in HBM between calls. hcl_node_start
 * returns once both ports listen; hcl_node_wait blocks until a Shutdown
 * message (or hcl_node_stop from another thread); hcl_node_stop drains the
 * connections and frees the daemon. */
int hcl_node_start(const char* host, int message_port, void** node);
int hcl_node_wait(void* node);
int hcl_node_stop(void* node);

const char* hcl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HCL_CABI_H */
