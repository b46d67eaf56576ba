/*
 * hcl_host.h — C-ABI of the host runtime (haocl::HostContext on B200,
 * include/haocl/runtime.hpp). One C entry point per reference HostContext
 * method (proj/include/haocl/runtime.hpp:97-153) plus the partitioned NDRange
 * launch; used by non-C++ callers (the Python package, bench.py) and shown in
 * INTEGRATION.md as the binding a maintainer would add.
 *
 * Return codes follow include/hcl_cabi.h: 0 = OK, else HCL_ERR_BASE +
 * haocl::ErrorCode; message via hcl_last_error(). Handles are session-unique
 * 64-bit ids (the reference's Handle::id, SPEC design decision).
 */
#ifndef HCL_HOST_H
#define HCL_HOST_H

#include <stdint.h>

#include "hcl_cabi.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hcl_context hcl_context;

typedef struct hcl_scheduler_options {
  double baseline_rate; /* work-units/s at relative_throughput 1.0 (1e9) */
  double net_bandwidth; /* bytes/s for non-resident data (1e8) */
  double ema_alpha;     /* 0.3 */
} hcl_scheduler_options;

/* HostContext::init. ordinals: CUDA devices to use (NULL = all). opts may be NULL. */
int hcl_ctx_init(const int* cuda_ordinals, int n, const hcl_scheduler_options* opts, hcl_context** out);
int hcl_ctx_destroy(hcl_context* ctx);

int hcl_ctx_get_device_ids(hcl_context* ctx, int* ids, int cap, int* n);
int hcl_ctx_create_queue(hcl_context* ctx, int global_device_id, const char* user_id, int shared,
                         uint64_t* queue);
int hcl_ctx_create_buffer(hcl_context* ctx, uint64_t size, uint64_t* buffer);
int hcl_ctx_create_program(hcl_context* ctx, const char* bundle, uint64_t* program);
int hcl_ctx_create_kernel(hcl_context* ctx, uint64_t program, const char* name, uint64_t* kernel);
int hcl_ctx_set_kernel_arg_i64(hcl_context* ctx, uint64_t kernel, uint32_t index, int64_t value);
int hcl_ctx_set_kernel_arg_buffer(hcl_context* ctx, uint64_t kernel, uint32_t index, uint64_t buffer);

/* enqueue_write_buffer (proj/src/runtime.cpp:448-483); offset > 0 writes a sub-range. */
int hcl_ctx_enqueue_write_buffer(hcl_context* ctx, uint64_t queue, uint64_t buffer, const void* data,
                                 uint64_t len, uint64_t offset, uint64_t* event);
/* enqueue_read_buffer (proj/src/runtime.cpp:485-514) of [offset, offset+len). */
int hcl_ctx_enqueue_read_buffer(hcl_context* ctx, uint64_t queue, uint64_t buffer, void* dst, uint64_t offset,
                                uint64_t len);
/* Non-blocking variants (OpenCL blocking_write/read = CL_FALSE): queued on the
 * device's copy streams and ordered against kernels using the buffer; host
 * memory (pinned for overlap) must stay valid until hcl_ctx_finish. */
int hcl_ctx_enqueue_write_buffer_async(hcl_context* ctx, uint64_t queue, uint64_t buffer, const void* data,
                                       uint64_t len, uint64_t offset, uint64_t* event);
int hcl_ctx_enqueue_read_buffer_async(hcl_context* ctx, uint64_t queue, uint64_t buffer, void* dst, uint64_t offset,
                                      uint64_t len);
/* enqueue_ndrange_kernel (proj/src/runtime.cpp:516-540). */
int hcl_ctx_enqueue_ndrange_kernel(hcl_context* ctx, uint64_t queue, uint64_t kernel, const uint64_t global[3],
                                   uint32_t dims, uint64_t* event);
/* Partitioned NDRange over nqueues queues; weights NULL = scheduler weights;
 * bounds (nqueues+1 row boundaries, e.g. nnz-balanced) NULL = computed split. */
int hcl_ctx_enqueue_ndrange_partitioned(hcl_context* ctx, uint64_t kernel, const uint64_t global[3], uint32_t dims,
                                        const uint64_t* queues, int nqueues, const uint64_t* weights,
                                        const uint64_t* bounds, uint64_t* event);
/* One sub-range [row_offset, row_offset+rows) of dim 0 on one queue (the part a
 * rank runs when the partitioned NDRange spans processes; OpenCL's global_work_offset). */
int hcl_ctx_enqueue_ndrange_range(hcl_context* ctx, uint64_t queue, uint64_t kernel, const uint64_t global[3],
                                  uint32_t dims, uint64_t row_offset, uint64_t rows, uint64_t* event);
/* Collectives when the partitioned NDRange spans processes (one GPU per rank,
 * NCCL over NVLink; the id comes from hcl_nccl_unique_id on rank 0). */
int hcl_ctx_init_collectives(hcl_context* ctx, uint64_t queue, int rank, int nranks, const uint8_t* nccl_id);
/* rank r owns bytes [bounds[r], bounds[r+1]); afterwards all ranks hold the union */
int hcl_ctx_enqueue_allgather(hcl_context* ctx, uint64_t queue, uint64_t buffer, const uint64_t* bounds, int nranks);
int hcl_ctx_enqueue_allreduce_sum_i64(hcl_context* ctx, uint64_t queue, uint64_t buffer);
int hcl_ctx_enqueue_broadcast(hcl_context* ctx, uint64_t queue, uint64_t buffer, int root);
/* Fused-exchange plumbing (HostContext::share_buffer / open_shared_buffer /
 * enqueue_barrier): 64-byte CUDA IPC handle of a buffer backed on the queue's
 * device; a peer's handle mapped on the queue's device (its device address);
 * a stream-ordered barrier across the NCCL communicator after which the
 * `completed` buffers count as whole on the queue's device. */
int hcl_ctx_share_buffer(hcl_context* ctx, uint64_t queue, uint64_t buffer, uint8_t* ipc_handle);
int hcl_ctx_open_shared_buffer(hcl_context* ctx, uint64_t queue, const uint8_t* ipc_handle, uint64_t bytes,
                               uint64_t* device_address);
int hcl_ctx_enqueue_barrier(hcl_context* ctx, uint64_t queue, const uint64_t* completed, int n);
/* Back a buffer on the queue's device with caller-owned device memory (>= its
 * size; e.g. a symmetric-memory allocation with an NVSwitch multicast mapping). */
int hcl_ctx_bind_external(hcl_context* ctx, uint64_t queue, uint64_t buffer, uint64_t device_ptr);
/* The row boundaries (nqueues+1) the partitioned launch would use. */
int hcl_ctx_partition_plan(hcl_context* ctx, uint64_t kernel, const uint64_t global[3], const uint64_t* queues,
                           int nqueues, const uint64_t* weights, uint64_t* bounds);

/* submit_task with auto placement (proj/src/runtime.cpp:542-594). kind[i]: 0 scalar, 1 buffer. */
int hcl_ctx_submit_task(hcl_context* ctx, const char* kernel, const uint8_t* is_buffer, const int64_t* values,
                        int nargs, const char* policy, int explicit_device, int* chosen, uint64_t* event);

int hcl_ctx_finish(hcl_context* ctx, uint64_t queue, double* transfer_ms, double* compute_ms, double* modeled_ms);
/* release(handle): kind = haocl::HandleKind (1 queue, 2 buffer, 3 program, 4 kernel, 5 event). */
int hcl_ctx_release(hcl_context* ctx, uint8_t kind, uint64_t id);
/* [init, data_creation, transfer, compute, modeled_compute] ms */
int hcl_ctx_breakdown(hcl_context* ctx, double out[5]);
int hcl_ctx_add_data_creation_ms(hcl_context* ctx, double ms);
int hcl_ctx_buffer_size(hcl_context* ctx, uint64_t buffer, uint64_t* size);
int hcl_ctx_buffer_device_ptr(hcl_context* ctx, uint64_t buffer, int global_device_id, void** ptr,
                              uint64_t* first_byte, uint64_t* bytes);
/* Message trace (forwarding fidelity): number of recorded calls named `function` (device -1 = any). */
int hcl_ctx_trace_count(hcl_context* ctx, const char* function, int device, uint64_t* count);
int hcl_ctx_trace_clear(hcl_context* ctx);

/* Scheduler (proj/include/haocl/scheduler.hpp:52-98). */
int hcl_ctx_sched_record_profile(hcl_context* ctx, int global_id, const char* kernel, double work_units,
                                 double seconds);
int hcl_ctx_sched_rate(hcl_context* ctx, int global_id, const char* kernel, double* rate);
int hcl_ctx_sched_schedule(hcl_context* ctx, const char* kernel, const char* policy, int explicit_device,
                           double work_units, uint64_t in_bytes, uint64_t out_bytes, int* chosen);
int hcl_ctx_sched_set_model(hcl_context* ctx, int global_id, double relative_throughput);
int hcl_ctx_sched_save_profiles(hcl_context* ctx, const char* path);
int hcl_ctx_sched_load_profiles(hcl_context* ctx, const char* path, int* loaded);
/* SM budget of a logical device (hcl_device_set_sm_budget) + scheduler model update. */
int hcl_ctx_set_sm_budget(hcl_context* ctx, int global_id, int sms);
int hcl_ctx_sched_partition_weights(hcl_context* ctx, const char* kernel, const int* gids, int n,
                                    uint64_t* weights);

/* Device-free host logic (usable without a GPU). */
int hcl_split_ranges(uint64_t total, const uint64_t* weights, int parts, uint64_t* bounds);
int hcl_spmv_partition_ranges(int64_t rows, const int64_t* row_ptr, int64_t parts, const uint64_t* weights,
                              int64_t* out);
/* A standalone scheduler (no devices needed) for host-logic tests: devices are
 * (gid, relative_throughput) pairs. */
typedef struct hcl_scheduler hcl_scheduler;
int hcl_sched_create(const hcl_scheduler_options* opts, const int* gids, const double* rel_tp, int n,
                     const char* const* map_kernels, const int* map_gids, int nmap, hcl_scheduler** out);
int hcl_sched_destroy(hcl_scheduler* s);
int hcl_sched_schedule(hcl_scheduler* s, const char* kernel, const char* policy, int explicit_device,
                       double work_units, uint64_t in_bytes, uint64_t out_bytes, const uint64_t* buffers,
                       int nbuffers, int* chosen);
int hcl_sched_record_profile(hcl_scheduler* s, int global_id, const char* kernel, double work_units,
                             double seconds);
int hcl_sched_rate(hcl_scheduler* s, int global_id, const char* kernel, double* rate);
int hcl_sched_note_resident(hcl_scheduler* s, uint64_t buffer, const int* gids, int n);
int hcl_sched_register_fixed_policy(hcl_scheduler* s, const char* name, int gid);
int hcl_sched_modeled_cost(hcl_scheduler* s, int global_id, const char* kernel, double work_units,
                           uint64_t in_bytes, uint64_t out_bytes, int resident, double* cost);
int hcl_sched_partition_weights(hcl_scheduler* s, const char* kernel, const int* gids, int n, uint64_t* weights);
/* Persist / restore the EMA profiles (text, one "gid<TAB>kernel<TAB>rate" per line). */
int hcl_sched_save_profiles(hcl_scheduler* s, const char* path);
int hcl_sched_load_profiles(hcl_scheduler* s, const char* path, int* loaded);

#ifdef __cplusplus
}
#endif
#endif /* HCL_HOST_H */
