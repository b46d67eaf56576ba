"""ctypes binding of libhaocl_b200.so (include/hcl_cabi.h, include/hcl_host.h).

The library is built in-tree (``paper_2005_08466_b200/build.py``). There is no
fallback: if it is missing, importing the runtime raises. GPU entry points
fail with ``precondition`` when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libhaocl_b200.so")

HCL_ERR_BASE = 1000

ERROR_NAMES = ["internal", "protocol", "version", "malformed", "encoding", "unknown_call", "busy",
               "precondition", "reassembly_conflict", "argument", "name", "config", "connect", "timeout",
               "transport", "remote", "handle", "policy", "size", "mapping", "unknown_device",
               "registration", "contract", "parse"]

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int)
f64p = C.POINTER(C.c_double)


class HclArg(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("reserved", C.c_uint32), ("scalar", C.c_int64),
                ("buffer_id", C.c_uint64)]


class SchedOptions(C.Structure):
    _fields_ = [("baseline_rate", C.c_double), ("net_bandwidth", C.c_double), ("ema_alpha", C.c_double)]


# (name, restype, argtypes) for every exported symbol the headers declare
CABI = [
    ("hcl_init", C.c_int, [i32p, C.c_int, i32p]),
    ("hcl_device_count", C.c_int, [i32p]),
    ("hcl_device_info", C.c_int, [C.c_int, i32p, f64p, i32p, u64p, C.c_char_p, C.c_int]),
    ("hcl_comm_stream", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("hcl_comm_acquire", C.c_int, [C.c_int, C.c_uint64, C.c_int]),
    ("hcl_comm_release", C.c_int, [C.c_int, C.c_uint64, C.c_int]),
    ("hcl_collective", C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_int]),
    ("hcl_node_start", C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("hcl_node_wait", C.c_int, [C.c_void_p]),
    ("hcl_node_stop", C.c_int, [C.c_void_p]),
    ("hcl_device_set_sm_budget", C.c_int, [C.c_int, C.c_int]),
    ("hcl_query_registry", C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_uint32), C.c_int, i32p]),
    ("hcl_kernel_signature", C.c_int, [C.c_char_p, C.c_char_p, u8p, u8p, C.c_int, i32p]),
    ("hcl_buffer_alloc", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]),
    ("hcl_buffer_write", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64]),
    ("hcl_buffer_read", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64]),
    ("hcl_buffer_write_async", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64]),
    ("hcl_buffer_read_async", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64]),
    ("hcl_buffer_copy_peer", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                       C.c_uint64]),
    ("hcl_buffer_release", C.c_int, [C.c_int, C.c_uint64]),
    ("hcl_buffer_swap", C.c_int, [C.c_int, C.c_uint64, C.c_uint64]),
    ("hcl_buffer_device_ptr", C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_void_p), u64p, u64p]),
    ("hcl_buffer_bind_external", C.c_int, [C.c_int, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64]),
    ("hcl_launch", C.c_int, [C.c_int, C.c_char_p, C.POINTER(HclArg), C.c_uint32, u64p, u64p, C.c_uint32, u64p]),
    ("hcl_finish", C.c_int, [C.c_int, f64p]),
    ("hcl_kernel_launch_count", C.c_uint64, []),
    ("hcl_device_stream", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("hcl_stream_acquire", C.c_int, [C.c_int, C.c_uint64, C.c_int]),
    ("hcl_stream_release", C.c_int, [C.c_int, C.c_uint64, C.c_int]),
    ("hcl_nccl_unique_id", C.c_int, [u8p, C.c_int]),
    ("hcl_nccl_init", C.c_int, [C.c_int, C.c_int, C.c_int, u8p]),
    ("hcl_nccl_destroy", C.c_int, [C.c_int]),
    ("hcl_allgatherv", C.c_int, [C.c_int, C.c_uint64, u64p]),
    ("hcl_allreduce_sum_i64", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]),
    ("hcl_broadcast", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]),
    ("hcl_nccl_barrier", C.c_int, [C.c_int]),
    ("hcl_buffer_alloc_shared", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("hcl_buffer_open_shared", C.c_int, [C.c_int, C.c_uint64, C.c_void_p, C.c_uint64]),
    ("hcl_last_error", C.c_char_p, []),
]

HOST = [
    ("hcl_ctx_init", C.c_int, [i32p, C.c_int, C.POINTER(SchedOptions), C.POINTER(C.c_void_p)]),
    ("hcl_ctx_destroy", C.c_int, [C.c_void_p]),
    ("hcl_ctx_get_device_ids", C.c_int, [C.c_void_p, i32p, C.c_int, i32p]),
    ("hcl_ctx_create_queue", C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_int, u64p]),
    ("hcl_ctx_create_buffer", C.c_int, [C.c_void_p, C.c_uint64, u64p]),
    ("hcl_ctx_create_program", C.c_int, [C.c_void_p, C.c_char_p, u64p]),
    ("hcl_ctx_create_kernel", C.c_int, [C.c_void_p, C.c_uint64, C.c_char_p, u64p]),
    ("hcl_ctx_set_kernel_arg_i64", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int64]),
    ("hcl_ctx_set_kernel_arg_buffer", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64]),
    ("hcl_ctx_enqueue_write_buffer", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64,
                                               C.c_uint64, u64p]),
    ("hcl_ctx_enqueue_read_buffer", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64,
                                              C.c_uint64]),
    ("hcl_ctx_enqueue_write_buffer_async", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64,
                                                     C.c_uint64, u64p]),
    ("hcl_ctx_enqueue_read_buffer_async", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64,
                                                    C.c_uint64]),
    ("hcl_ctx_enqueue_ndrange_kernel", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, u64p, C.c_uint32, u64p]),
    ("hcl_ctx_enqueue_ndrange_partitioned", C.c_int, [C.c_void_p, C.c_uint64, u64p, C.c_uint32, u64p, C.c_int,
                                                      u64p, u64p, u64p]),
    ("hcl_ctx_enqueue_ndrange_range", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, u64p, C.c_uint32,
                                                C.c_uint64, C.c_uint64, u64p]),
    ("hcl_ctx_init_collectives", C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.c_int, u8p]),
    ("hcl_ctx_enqueue_allgather", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, u64p, C.c_int]),
    ("hcl_ctx_enqueue_allreduce_sum_i64", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64]),
    ("hcl_ctx_enqueue_broadcast", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int]),
    ("hcl_ctx_share_buffer", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("hcl_ctx_bind_external", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64]),
    ("hcl_ctx_open_shared_buffer", C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, u64p]),
    ("hcl_ctx_enqueue_barrier", C.c_int, [C.c_void_p, C.c_uint64, u64p, C.c_int]),
    ("hcl_ctx_partition_plan", C.c_int, [C.c_void_p, C.c_uint64, u64p, u64p, C.c_int, u64p, u64p]),
    ("hcl_ctx_submit_task", C.c_int, [C.c_void_p, C.c_char_p, u8p, i64p, C.c_int, C.c_char_p, C.c_int, i32p,
                                      u64p]),
    ("hcl_ctx_finish", C.c_int, [C.c_void_p, C.c_uint64, f64p, f64p, f64p]),
    ("hcl_ctx_release", C.c_int, [C.c_void_p, C.c_uint8, C.c_uint64]),
    ("hcl_ctx_breakdown", C.c_int, [C.c_void_p, f64p]),
    ("hcl_ctx_add_data_creation_ms", C.c_int, [C.c_void_p, C.c_double]),
    ("hcl_ctx_buffer_size", C.c_int, [C.c_void_p, C.c_uint64, u64p]),
    ("hcl_ctx_buffer_device_ptr", C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p), u64p, u64p]),
    ("hcl_ctx_trace_count", C.c_int, [C.c_void_p, C.c_char_p, C.c_int, u64p]),
    ("hcl_ctx_trace_clear", C.c_int, [C.c_void_p]),
    ("hcl_ctx_sched_record_profile", C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_double, C.c_double]),
    ("hcl_ctx_sched_rate", C.c_int, [C.c_void_p, C.c_int, C.c_char_p, f64p]),
    ("hcl_ctx_sched_schedule", C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_uint64,
                                         C.c_uint64, i32p]),
    ("hcl_ctx_sched_set_model", C.c_int, [C.c_void_p, C.c_int, C.c_double]),
    ("hcl_ctx_sched_save_profiles", C.c_int, [C.c_void_p, C.c_char_p]),
    ("hcl_ctx_sched_load_profiles", C.c_int, [C.c_void_p, C.c_char_p, i32p]),
    ("hcl_ctx_set_sm_budget", C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    ("hcl_ctx_sched_partition_weights", C.c_int, [C.c_void_p, C.c_char_p, i32p, C.c_int, u64p]),
    ("hcl_split_ranges", C.c_int, [C.c_uint64, u64p, C.c_int, u64p]),
    ("hcl_spmv_partition_ranges", C.c_int, [C.c_int64, i64p, C.c_int64, u64p, i64p]),
    ("hcl_sched_create", C.c_int, [C.POINTER(SchedOptions), i32p, f64p, C.c_int, C.POINTER(C.c_char_p), i32p,
                                   C.c_int, C.POINTER(C.c_void_p)]),
    ("hcl_sched_destroy", C.c_int, [C.c_void_p]),
    ("hcl_sched_schedule", C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_uint64,
                                     C.c_uint64, u64p, C.c_int, i32p]),
    ("hcl_sched_record_profile", C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_double, C.c_double]),
    ("hcl_sched_rate", C.c_int, [C.c_void_p, C.c_int, C.c_char_p, f64p]),
    ("hcl_sched_note_resident", C.c_int, [C.c_void_p, C.c_uint64, i32p, C.c_int]),
    ("hcl_sched_register_fixed_policy", C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    ("hcl_sched_modeled_cost", C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_double, C.c_uint64, C.c_uint64,
                                         C.c_int, f64p]),
    ("hcl_sched_partition_weights", C.c_int, [C.c_void_p, C.c_char_p, i32p, C.c_int, u64p]),
    ("hcl_sched_save_profiles", C.c_int, [C.c_void_p, C.c_char_p]),
    ("hcl_sched_load_profiles", C.c_int, [C.c_void_p, C.c_char_p, i32p]),
]

DATAGEN = [
    ("hcl_gen_splitmix_at", C.c_uint64, [C.c_uint64, C.c_uint64]),
    ("hcl_gen_doubles", None, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]),
    ("hcl_gen_f32", None, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]),
    ("hcl_gen_bf16", None, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]),
    ("hcl_gen_rmat_edges", None, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int]),
    ("hcl_gen_kmeans_points", None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_void_p,
                                     C.c_int]),
    ("hcl_pagerank_csr", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int]),
    ("hcl_csr_row_blocks", C.c_int64, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]),
    ("hcl_pagerank_units", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, i64p, i64p]),
    ("hcl_pagerank_relabel", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    ("hcl_pagerank_bins_build", C.c_void_p, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                             C.c_int64, C.c_int64, C.c_int64, C.c_void_p]),
    ("hcl_pagerank_bins_export", C.c_int, [C.c_void_p] + [C.c_void_p] * 7),
    ("hcl_pagerank_bins_free", None, [C.c_void_p]),
    ("hcl_counting_order", C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
]


class PrBinsInfo(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("lo", "hi", "bin_rows", "chunk_edges", "span_max", "unit_edges", "n_edges",
                                          "n_chunks", "n_bins", "gstride", "n_entries", "n_src", "n_units",
                                          "n_slots", "n_desc")]

EXTRA = []  # appended by workload modules

_lib = None


class HaoclError(Exception):
    """haocl::Error across the C-ABI: .code is the reference's ErrorCode value."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.name = ERROR_NAMES[code] if 0 <= code < len(ERROR_NAMES) else "unknown"
        super().__init__(message)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in CABI + HOST + DATAGEN + EXTRA:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        code = rc - HCL_ERR_BASE
        msg = lib().hcl_last_error()
        raise HaoclError(code, msg.decode() if msg else f"error {rc}")


def declared_symbols():
    return [n for n, _, _ in CABI + HOST + DATAGEN]
