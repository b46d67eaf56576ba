"""Python front end of haocl::HostContext on B200 (over include/hcl_host.h).

Method names, argument meaning and error behaviour mirror the reference's
C++ HostContext (proj/include/haocl/runtime.hpp:97-153): errors raise
``HaoclError`` carrying the reference's ``ErrorCode`` (e.g. ``name`` 10 for
an unknown kernel, ``argument`` 9 for arity/size violations, ``handle`` 16
for released handles), so parity tests read like the reference's own.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import HaoclError, check


class HandleKind(IntEnum):  # proj/include/haocl/runtime.hpp:29
    context = 0
    queue = 1
    buffer = 2
    program = 3
    kernel = 4
    event = 5


@dataclass(frozen=True)
class Handle:
    kind: HandleKind
    id: int


@dataclass
class TimingFragment:  # runtime.hpp:66-70
    transfer_ms: float = 0.0
    compute_ms: float = 0.0
    modeled_ms: float = 0.0


@dataclass
class TimingBreakdown:  # runtime.hpp:55-64
    init_ms: float = 0.0
    data_creation_ms: float = 0.0
    transfer_ms: float = 0.0
    compute_ms: float = 0.0
    modeled_compute_ms: float = 0.0

    def total(self) -> float:
        return self.init_ms + self.data_creation_ms + self.transfer_ms + self.compute_ms


@dataclass
class SchedulerOptions:  # scheduler.hpp:46-50
    baseline_rate: float = 1e9
    net_bandwidth: float = 1e8
    ema_alpha: float = 0.3

    def c(self) -> N.SchedOptions:
        return N.SchedOptions(self.baseline_rate, self.net_bandwidth, self.ema_alpha)


@dataclass
class KernelTask:  # api.hpp:43-51 (args: int scalars or buffer Handles)
    kernel_name: str
    args: list = field(default_factory=list)
    global_size: tuple = (1, 1, 1)
    dims: int = 1
    policy: Optional[str] = None  # None = explicit placement on `device`
    device: int = 0


def _bytes_view(data) -> tuple[int, int, object]:
    """(address, length, keepalive) of a host buffer without copying."""
    if isinstance(data, np.ndarray):
        a = np.ascontiguousarray(data)
        return a.ctypes.data, a.nbytes, a
    if isinstance(data, (bytes, bytearray, memoryview)):
        a = np.frombuffer(data, np.uint8)
        return a.ctypes.data, a.nbytes, a
    if hasattr(data, "data_ptr") and hasattr(data, "nbytes"):  # torch CPU tensor (pinned or not)
        return int(data.data_ptr()), int(data.nbytes), data
    raise TypeError(f"unsupported host buffer type {type(data)}")


class HostContext:
    """haocl::HostContext::init over the CUDA devices of this process."""

    def __init__(self, cuda_ordinals: Optional[Sequence[int]] = None,
                 scheduler: Optional[SchedulerOptions] = None):
        """HostContext::init (proj/src/runtime.cpp:317-374): CUDA devices instead of a cluster file."""
        L = N.lib()
        self._L = L
        ords = list(cuda_ordinals or [])
        arr = (C.c_int * max(1, len(ords)))(*ords) if ords else None
        opts = (scheduler or SchedulerOptions()).c()
        p = C.c_void_p()
        check(L.hcl_ctx_init(arr, len(ords), C.byref(opts), C.byref(p)))
        self._ctx = p

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._L.hcl_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- devices ---------------------------------------------------------
    def get_device_ids(self) -> list[int]:
        """proj/src/runtime.cpp:378-383."""
        ids = (C.c_int * 64)()
        n = C.c_int()
        check(self._L.hcl_ctx_get_device_ids(self._ctx, ids, 64, C.byref(n)))
        return list(ids[: n.value])

    # -- objects ---------------------------------------------------------
    def create_queue(self, global_device_id: int, user_id: str = "default", shared: bool = True) -> Handle:
        """proj/src/runtime.cpp:385-399."""
        q = C.c_uint64()
        check(self._L.hcl_ctx_create_queue(self._ctx, global_device_id, user_id.encode(), int(shared), C.byref(q)))
        return Handle(HandleKind.queue, q.value)

    def create_buffer(self, size: int) -> Handle:
        """proj/src/runtime.cpp:401-406 (lazy: placed on first use)."""
        b = C.c_uint64()
        check(self._L.hcl_ctx_create_buffer(self._ctx, size, C.byref(b)))
        return Handle(HandleKind.buffer, b.value)

    def create_program(self, bundle: str) -> Handle:
        """proj/src/runtime.cpp:408-417 (query_registry of a bundle)."""
        p = C.c_uint64()
        check(self._L.hcl_ctx_create_program(self._ctx, bundle.encode(), C.byref(p)))
        return Handle(HandleKind.program, p.value)

    def create_kernel(self, program: Handle, kernel_name: str) -> Handle:
        """proj/src/runtime.cpp:419-435 (name error 10 for unknown kernels)."""
        k = C.c_uint64()
        check(self._L.hcl_ctx_create_kernel(self._ctx, program.id, kernel_name.encode(), C.byref(k)))
        return Handle(HandleKind.kernel, k.value)

    def set_kernel_arg(self, kernel: Handle, index: int, value) -> None:
        """proj/src/runtime.cpp:437-446 (int -> i64 scalar, Handle -> buffer)."""
        if isinstance(value, Handle):
            if value.kind != HandleKind.buffer:
                raise HaoclError(16, "handle: argument is not a buffer handle")
            check(self._L.hcl_ctx_set_kernel_arg_buffer(self._ctx, kernel.id, index, value.id))
        else:
            check(self._L.hcl_ctx_set_kernel_arg_i64(self._ctx, kernel.id, index, int(value)))

    # -- transfers -------------------------------------------------------
    def enqueue_write_buffer(self, queue: Handle, buffer: Handle, data, offset: int = 0,
                             blocking: bool = True) -> Handle:
        """proj/src/runtime.cpp:448-483 (size error 18 past the end). blocking=False
        queues the copy on the device's H2D stream (keep `data` alive, ideally
        pinned, until finish(queue))."""
        ptr, n, keep = _bytes_view(data)
        ev = C.c_uint64()
        fn = self._L.hcl_ctx_enqueue_write_buffer if blocking else self._L.hcl_ctx_enqueue_write_buffer_async
        check(fn(self._ctx, queue.id, buffer.id, C.c_void_p(ptr), n, offset, C.byref(ev)))
        del keep
        return Handle(HandleKind.event, ev.value)

    def enqueue_read_buffer(self, queue: Handle, buffer: Handle, offset: int = 0, length: Optional[int] = None,
                            out=None, blocking: bool = True) -> np.ndarray:
        """proj/src/runtime.cpp:485-514 (gathers the buffer's shards). blocking=False queues the copy on the D2H stream; `out` is valid after finish(queue)."""
        if length is None:
            length = self.buffer_size(buffer) - offset
        if out is None:
            out = np.empty(length, np.uint8)
        ptr, n, keep = _bytes_view(out)
        if n < length:
            raise HaoclError(18, "size: output buffer too small")
        fn = self._L.hcl_ctx_enqueue_read_buffer if blocking else self._L.hcl_ctx_enqueue_read_buffer_async
        check(fn(self._ctx, queue.id, buffer.id, C.c_void_p(ptr), offset, length))
        return out

    # -- launches --------------------------------------------------------
    def enqueue_ndrange_kernel(self, queue: Handle, kernel: Handle, global_size=(1, 1, 1), dims: int = 1) -> Handle:
        """proj/src/runtime.cpp:516-540: the whole range on one queue."""
        g = (C.c_uint64 * 3)(*global_size)
        ev = C.c_uint64()
        check(self._L.hcl_ctx_enqueue_ndrange_kernel(self._ctx, queue.id, kernel.id, g, dims, C.byref(ev)))
        return Handle(HandleKind.event, ev.value)

    def enqueue_ndrange_partitioned(self, kernel: Handle, global_size, dims: int, queues: Sequence[Handle],
                                    weights: Optional[Sequence[int]] = None,
                                    bounds: Optional[Sequence[int]] = None) -> Handle:
        """The bench layer's partitioning moved into the runtime (run_matmul /
        run_spmv / run_knn, proj/src/bench.cpp:147-447; block_range 31-33).
        Partitioned NDRange: split dim 0 of global_size over `queues` (by
        `weights`, or at explicit row `bounds`, e.g. nnz-balanced ranges)."""
        g = (C.c_uint64 * 3)(*global_size)
        qs = (C.c_uint64 * len(queues))(*[q.id for q in queues])
        w = (C.c_uint64 * len(queues))(*weights) if weights is not None else None
        b = (C.c_uint64 * (len(queues) + 1))(*[int(x) for x in bounds]) if bounds is not None else None
        ev = C.c_uint64()
        check(self._L.hcl_ctx_enqueue_ndrange_partitioned(self._ctx, kernel.id, g, dims, qs, len(queues), w, b,
                                                          C.byref(ev)))
        return Handle(HandleKind.event, ev.value)

    def enqueue_ndrange_range(self, queue: Handle, kernel: Handle, global_size, dims: int, row_offset: int,
                              rows: int) -> Handle:
        """Rows [row_offset, row_offset+rows) of dim 0 on one queue (a rank's part)."""
        g = (C.c_uint64 * 3)(*global_size)
        ev = C.c_uint64()
        check(self._L.hcl_ctx_enqueue_ndrange_range(self._ctx, queue.id, kernel.id, g, dims, row_offset, rows,
                                                    C.byref(ev)))
        return Handle(HandleKind.event, ev.value)

    # -- collectives across processes (one GPU per rank) --------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(N.lib().hcl_nccl_unique_id(buf, 128))
        return bytes(buf)

    def init_collectives(self, queue: Handle, rank: int, nranks: int, unique_id: bytes) -> None:
        ident = (C.c_uint8 * 128)(*unique_id[:128])
        check(self._L.hcl_ctx_init_collectives(self._ctx, queue.id, rank, nranks, ident))

    def enqueue_allgather(self, queue: Handle, buffer: Handle, byte_bounds: Sequence[int]) -> None:
        b = (C.c_uint64 * len(byte_bounds))(*[int(x) for x in byte_bounds])
        check(self._L.hcl_ctx_enqueue_allgather(self._ctx, queue.id, buffer.id, b, len(byte_bounds) - 1))

    def enqueue_allreduce_sum_i64(self, queue: Handle, buffer: Handle) -> None:
        check(self._L.hcl_ctx_enqueue_allreduce_sum_i64(self._ctx, queue.id, buffer.id))

    def share_buffer(self, queue: Handle, buffer: Handle) -> bytes:
        """Back `buffer` on the queue's device with IPC-exportable memory (zero-filled);
        returns its 64-byte CUDA IPC handle for the other ranks (fused exchange kernels)."""
        h = (C.c_uint8 * 64)()
        check(self._L.hcl_ctx_share_buffer(self._ctx, queue.id, buffer.id, h))
        return bytes(h)

    def bind_external(self, queue: Handle, buffer: Handle, device_ptr: int) -> None:
        """Back `buffer` on the queue's device with caller-owned device memory
        (>= the buffer's size, kept alive by the caller until release), e.g. a
        torch symmetric-memory tensor whose multicast address a kernel stores to."""
        check(self._L.hcl_ctx_bind_external(self._ctx, queue.id, buffer.id, device_ptr))

    def open_shared_buffer(self, queue: Handle, ipc_handle: bytes, nbytes: int) -> int:
        """Map a peer rank's shared buffer on the queue's device; returns its device
        address (what pagerank_step_exchange's peers list holds)."""
        h = (C.c_uint8 * 64)(*ipc_handle[:64])
        addr = C.c_uint64()
        check(self._L.hcl_ctx_open_shared_buffer(self._ctx, queue.id, h, nbytes, C.byref(addr)))
        return addr.value

    def enqueue_barrier(self, queue: Handle, completed: Sequence[Handle] = ()) -> None:
        """Stream-ordered barrier across the NCCL communicator (init_collectives);
        afterwards the `completed` buffers count as whole on the queue's device
        (peer ranks stored the rows this rank did not write)."""
        ids = (C.c_uint64 * max(1, len(completed)))(*[b.id for b in completed])
        check(self._L.hcl_ctx_enqueue_barrier(self._ctx, queue.id, ids, len(completed)))

    def enqueue_broadcast(self, queue: Handle, buffer: Handle, root: int) -> None:
        check(self._L.hcl_ctx_enqueue_broadcast(self._ctx, queue.id, buffer.id, root))

    def partition_plan(self, kernel: Handle, global_size, queues: Sequence[Handle],
                       weights: Optional[Sequence[int]] = None) -> list[int]:
        """Row boundaries a partitioned launch would use: split_ranges of the
        weights (block_range for equal ones, proj/src/bench.cpp:31-33) or of the
        scheduler's EMA rates (proj/src/scheduler.cpp:136-149)."""
        g = (C.c_uint64 * 3)(*global_size)
        qs = (C.c_uint64 * len(queues))(*[q.id for q in queues])
        w = (C.c_uint64 * len(queues))(*weights) if weights is not None else None
        out = (C.c_uint64 * (len(queues) + 1))()
        check(self._L.hcl_ctx_partition_plan(self._ctx, kernel.id, g, qs, len(queues), w, out))
        return list(out)

    def submit_task(self, task: KernelTask) -> tuple[int, Handle]:
        """proj/src/runtime.cpp:542-594 (scheduler placement)."""
        n = len(task.args)
        isb = (C.c_uint8 * max(1, n))()
        vals = (C.c_int64 * max(1, n))()
        for i, a in enumerate(task.args):
            if isinstance(a, Handle):
                isb[i], vals[i] = 1, a.id
            else:
                isb[i], vals[i] = 0, int(a)
        chosen = C.c_int()
        ev = C.c_uint64()
        pol = task.policy.encode() if task.policy else None
        check(self._L.hcl_ctx_submit_task(self._ctx, task.kernel_name.encode(), isb, vals, n, pol, task.device,
                                          C.byref(chosen), C.byref(ev)))
        return chosen.value, Handle(HandleKind.event, ev.value)

    def finish(self, queue: Handle) -> TimingFragment:
        """proj/src/runtime.cpp:606-616 (CUDA-event compute time, EMA profiles)."""
        t, c, m = C.c_double(), C.c_double(), C.c_double()
        check(self._L.hcl_ctx_finish(self._ctx, queue.id, C.byref(t), C.byref(c), C.byref(m)))
        return TimingFragment(t.value, c.value, m.value)

    def release(self, handle: Handle) -> None:
        """proj/src/runtime.cpp:618-666."""
        check(self._L.hcl_ctx_release(self._ctx, int(handle.kind), handle.id))

    # -- observability ---------------------------------------------------
    def breakdown(self) -> TimingBreakdown:
        """proj/src/runtime.cpp:668-671."""
        out = (C.c_double * 5)()
        check(self._L.hcl_ctx_breakdown(self._ctx, out))
        return TimingBreakdown(*list(out))

    def add_data_creation_ms(self, ms: float) -> None:
        check(self._L.hcl_ctx_add_data_creation_ms(self._ctx, ms))

    def buffer_size(self, buffer: Handle) -> int:
        s = C.c_uint64()
        check(self._L.hcl_ctx_buffer_size(self._ctx, buffer.id, C.byref(s)))
        return s.value

    def buffer_device_ptr(self, buffer: Handle, global_device_id: int) -> tuple[int, int, int]:
        p, f, b = C.c_void_p(), C.c_uint64(), C.c_uint64()
        check(self._L.hcl_ctx_buffer_device_ptr(self._ctx, buffer.id, global_device_id, C.byref(p), C.byref(f),
                                                C.byref(b)))
        return p.value or 0, f.value, b.value

    def trace_count(self, function: str, device: int = -1) -> int:
        c = C.c_uint64()
        check(self._L.hcl_ctx_trace_count(self._ctx, function.encode(), device, C.byref(c)))
        return c.value

    def trace_clear(self) -> None:
        check(self._L.hcl_ctx_trace_clear(self._ctx))

    # -- scheduler -------------------------------------------------------
    def record_profile(self, gid: int, kernel: str, work_units: float, seconds: float) -> None:
        check(self._L.hcl_ctx_sched_record_profile(self._ctx, gid, kernel.encode(), work_units, seconds))

    def profiled_rate(self, gid: int, kernel: str) -> float:
        r = C.c_double()
        check(self._L.hcl_ctx_sched_rate(self._ctx, gid, kernel.encode(), C.byref(r)))
        return r.value

    def set_relative_throughput(self, gid: int, rel: float) -> None:
        check(self._L.hcl_ctx_sched_set_model(self._ctx, gid, rel))

    def save_profiles(self, path: str) -> None:
        """Persist the scheduler's EMA rates per (device, kernel) (§8(f) 2)."""
        check(self._L.hcl_ctx_sched_save_profiles(self._ctx, os.fsencode(path)))

    def load_profiles(self, path: str) -> int:
        n = C.c_int()
        check(self._L.hcl_ctx_sched_load_profiles(self._ctx, os.fsencode(path), C.byref(n)))
        return n.value

    def set_sm_budget(self, gid: int, sms: int) -> None:
        """Give logical device `gid` a budget of `sms` SMs (its kernels size their
        grids to it; the scheduler model becomes sms / SM count)."""
        check(self._L.hcl_ctx_set_sm_budget(self._ctx, gid, sms))

    def partition_weights(self, kernel: str, gids: Sequence[int]) -> list[int]:
        g = (C.c_int * len(gids))(*gids)
        w = (C.c_uint64 * len(gids))()
        check(self._L.hcl_ctx_sched_partition_weights(self._ctx, kernel.encode(), g, len(gids), w))
        return list(w)


# ---------------------------------------------------------------------------
# device-free host logic


def split_ranges(total: int, weights: Sequence[int]) -> list[int]:
    w = (C.c_uint64 * len(weights))(*weights)
    out = (C.c_uint64 * (len(weights) + 1))()
    check(N.lib().hcl_split_ranges(total, w, len(weights), out))
    return list(out)


def spmv_partition_ranges(row_ptr: np.ndarray, parts: int, weights: Optional[Sequence[int]] = None) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, np.int64)
    out = np.empty(parts + 1, np.int64)
    w = (C.c_uint64 * parts)(*weights) if weights is not None else None
    check(N.lib().hcl_spmv_partition_ranges(len(rp) - 1, rp.ctypes.data_as(N.i64p), parts, w,
                                            out.ctypes.data_as(N.i64p)))
    return out


class Scheduler:
    """Standalone haocl::Scheduler (no devices needed): devices are
    (global_id, relative_throughput) pairs; `kernel_map` is the static_map table."""

    def __init__(self, devices: Iterable[tuple[int, float]], options: Optional[SchedulerOptions] = None,
                 kernel_map: Optional[dict] = None):
        devs = list(devices)
        gids = (C.c_int * max(1, len(devs)))(*[d[0] for d in devs])
        rel = (C.c_double * max(1, len(devs)))(*[d[1] for d in devs])
        km = kernel_map or {}
        mk = (C.c_char_p * max(1, len(km)))(*[k.encode() for k in km])
        mg = (C.c_int * max(1, len(km)))(*list(km.values()))
        opts = (options or SchedulerOptions()).c()
        p = C.c_void_p()
        check(N.lib().hcl_sched_create(C.byref(opts), gids, rel, len(devs), mk, mg, len(km), C.byref(p)))
        self._s = p

    def __del__(self):
        try:
            N.lib().hcl_sched_destroy(self._s)
        except Exception:
            pass

    def schedule(self, kernel: str, policy: Optional[str] = None, device: int = 0, work_units: float = 1.0,
                 in_bytes: int = 0, out_bytes: int = 0, buffers: Sequence[int] = ()) -> int:
        b = (C.c_uint64 * max(1, len(buffers)))(*buffers)
        c = C.c_int()
        check(N.lib().hcl_sched_schedule(self._s, kernel.encode(), policy.encode() if policy else None, device,
                                         work_units, in_bytes, out_bytes, b, len(buffers), C.byref(c)))
        return c.value

    def record_profile(self, gid: int, kernel: str, work_units: float, seconds: float) -> None:
        check(N.lib().hcl_sched_record_profile(self._s, gid, kernel.encode(), work_units, seconds))

    def rate(self, gid: int, kernel: str) -> float:
        r = C.c_double()
        check(N.lib().hcl_sched_rate(self._s, gid, kernel.encode(), C.byref(r)))
        return r.value

    def note_resident(self, buffer: int, gids: Sequence[int]) -> None:
        g = (C.c_int * max(1, len(gids)))(*gids)
        check(N.lib().hcl_sched_note_resident(self._s, buffer, g, len(gids)))

    def register_fixed_policy(self, name: str, gid: int) -> None:
        check(N.lib().hcl_sched_register_fixed_policy(self._s, name.encode(), gid))

    def modeled_cost(self, gid: int, kernel: str, work_units: float, in_bytes: int = 0, out_bytes: int = 0,
                     resident: bool = True) -> float:
        c = C.c_double()
        check(N.lib().hcl_sched_modeled_cost(self._s, gid, kernel.encode(), work_units, in_bytes, out_bytes,
                                             int(resident), C.byref(c)))
        return c.value

    def partition_weights(self, kernel: str, gids: Sequence[int]) -> list[int]:
        g = (C.c_int * len(gids))(*gids)
        w = (C.c_uint64 * len(gids))()
        check(N.lib().hcl_sched_partition_weights(self._s, kernel.encode(), g, len(gids), w))
        return list(w)

    def save_profiles(self, path: str) -> None:
        check(N.lib().hcl_sched_save_profiles(self._s, os.fsencode(path)))

    def load_profiles(self, path: str) -> int:
        n = C.c_int()
        check(N.lib().hcl_sched_load_profiles(self._s, os.fsencode(path), C.byref(n)))
        return n.value
