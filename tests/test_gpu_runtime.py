"""Host runtime contracts on the GPU: sharded residency (several valid
intervals per device), the data-movement contract of the partition classes
checked through the MessageTrace (each forwarded call is one traced message,
proj/include/haocl/runtime.hpp:80-90), and the locking
discipline (a finish() on one queue does not block the other queues, the
reference's thread-per-part host pattern, proj/src/bench.cpp:107-133)."""
import threading
import time

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


def kernel(ctx, bundle, name, args):
    k = ctx.create_kernel(ctx.create_program(bundle), name)
    for i, a in enumerate(args):
        ctx.set_kernel_arg(k, i, a)
    return k


# ---- residency: disjoint valid intervals -------------------

def test_disjoint_partial_writes_keep_every_byte(ctx, queues):
    """Whole on device 0, then two disjoint partial writes from device 1: the
    bytes between them stay valid on device 0 only, and a read through device
    2 gathers all three pieces."""
    data = np.arange(100, dtype=np.float64)
    b = ctx.create_buffer(data.nbytes)
    ctx.enqueue_write_buffer(queues[0], b, data)
    ctx.enqueue_write_buffer(queues[1], b, np.full(10, -1.0), offset=0)
    ctx.enqueue_write_buffer(queues[1], b, np.full(10, -2.0), offset=90 * 8)
    want = data.copy()
    want[:10] = -1.0
    want[90:] = -2.0
    for q in (queues[2], queues[1], queues[0]):
        assert (ctx.enqueue_read_buffer(q, b).view(np.float64) == want).all()
    # device 1 then needs the middle: it must come from device 0, not stale HBM
    ctx.enqueue_write_buffer(queues[0], b, np.full(5, 7.0), offset=50 * 8)
    want[50:55] = 7.0
    vk = kernel(ctx, "core", "vecadd", [b, b, ctx.create_buffer(data.nbytes), 100])
    out = ctx.create_buffer(data.nbytes)
    ctx.set_kernel_arg(vk, 2, out)
    ctx.enqueue_ndrange_kernel(queues[1], vk, (100, 1, 1), 1)
    ctx.finish(queues[1])
    assert (ctx.enqueue_read_buffer(queues[3], out).view(np.float64) == 2 * want).all()
    ctx.release(b)
    ctx.release(out)


def test_partitioned_then_subrange_launch(ctx, queues):
    """A partitioned launch leaves the output sharded over four devices; a
    sub-range launch on one device then rewrites rows in the middle of another
    device's shard. Every row must read back from its latest writer."""
    n = 4000
    x = O.gen_doubles(n, 5)
    y = O.gen_doubles(n, 6)
    bx, by, bo = ctx.create_buffer(n * 8), ctx.create_buffer(n * 8), ctx.create_buffer(n * 8)
    ctx.enqueue_write_buffer(queues[0], bx, x)
    ctx.enqueue_write_buffer(queues[0], by, y)
    vk = kernel(ctx, "core", "vecadd", [bx, by, bo, n])
    ctx.enqueue_ndrange_partitioned(vk, (n, 1, 1), 1, queues, [1, 1, 1, 1])
    ctx.enqueue_write_buffer(queues[3], bx, np.zeros(n))  # x := 0 (whole, device 3)
    ctx.enqueue_ndrange_range(queues[3], vk, (n, 1, 1), 1, 1500, 200)  # rows of device 1's shard
    for q in queues:
        ctx.finish(q)
    want = x + y
    want[1500:1700] = y[1500:1700]
    for q in queues:
        got = ctx.enqueue_read_buffer(q, bo).view(np.float64)
        assert got.tobytes() == want.tobytes()
    for b in (bx, by, bo):
        ctx.release(b)


# ---- MessageTrace: the partition classes' data movement ------------------------

def test_trace_split_rows_and_replicate(ctx, queues):
    """matmul(A, B, C): A and C are SPLIT_ROWS, B is REPLICATE. Over P devices:
    exactly P launch_kernel messages; each non-owner device pulls only its A
    slice (one copy_peer, allocation = its rows) and B once; a second launch
    moves nothing."""
    n, P = 256, 4
    a = O.gen_doubles(n * n, 42)
    b = O.gen_doubles(n * n, 43)
    ba, bb, bc = ctx.create_buffer(a.nbytes), ctx.create_buffer(b.nbytes), ctx.create_buffer(a.nbytes)
    ctx.enqueue_write_buffer(queues[0], ba, a)
    ctx.enqueue_write_buffer(queues[0], bb, b)
    mk = kernel(ctx, "core", "matmul", [ba, bb, bc, n, n, n])
    ctx.trace_clear()
    ctx.enqueue_ndrange_partitioned(mk, (n, n, 1), 2, queues[:P], [1] * P)
    gids = [ctx.get_device_ids()[i] for i in range(P)]
    assert ctx.trace_count("launch_kernel") == P
    for i, g in enumerate(gids):
        assert ctx.trace_count("launch_kernel", g) == 1
        # device 0 holds A and B already; the others copy their A rows and all of B
        assert ctx.trace_count("copy_peer", g) == (0 if i == 0 else 2)
        if i:
            _, first, nbytes = ctx.buffer_device_ptr(ba, g)
            assert (first, nbytes) == (i * n // P * n * 8, n // P * n * 8)  # only its slice
            _, first, nbytes = ctx.buffer_device_ptr(bb, g)
            assert (first, nbytes) == (0, n * n * 8)  # replicated whole
        _, first, nbytes = ctx.buffer_device_ptr(bc, g)
        assert (first, nbytes) == (i * n // P * n * 8, n // P * n * 8)
    ctx.trace_clear()
    ctx.enqueue_ndrange_partitioned(mk, (n, n, 1), 2, queues[:P], [1] * P)
    assert ctx.trace_count("copy_peer") == 0 and ctx.trace_count("alloc_buffer") == 0
    assert ctx.trace_count("launch_kernel") == P
    # the gather of C reads each shard from its owner: one read per device
    for q in queues[:P]:
        ctx.finish(q)
    ctx.trace_clear()
    c = ctx.enqueue_read_buffer(queues[0], bc).view(np.float64)
    assert ctx.trace_count("read_buffer") == P
    for g in gids:
        assert ctx.trace_count("read_buffer", g) == 1
    assert c.tobytes() == O.matmul_f64(a, b, n, n, n).tobytes()
    for x in (ba, bb, bc):
        ctx.release(x)


def test_trace_reduce_sum_tree(ctx, queues):
    """REDUCE_SUM over 4 parts folds as a binary tree: 3 copy_peer messages
    (device 0 <- 1, 2 <- 3, then 0 <- 2), results equal to the whole launch."""
    from paper_2005_08466_b200 import datagen as G

    n, d, k = 9000, 32, 16
    pts = G.gen_kmeans_points(n, d, k, 42)
    cent = pts[: k * d].copy()
    a = O.kmeans_assign(pts, n, d, cent, k)
    s_want, c_want = O.kmeans_accumulate(pts, n, d, a, k)
    bp, ba, bs, bcn = (ctx.create_buffer(x) for x in (pts.nbytes, n * 4, k * d * 8, k * 8))
    ctx.enqueue_write_buffer(queues[0], bp, pts)
    ctx.enqueue_write_buffer(queues[0], ba, a.astype(np.int32))
    acc = kernel(ctx, "b200", "kmeans_accumulate", [bp, ba, bs, bcn, n, d, k])
    ctx.enqueue_ndrange_partitioned(acc, (n, 1, 1), 1, queues, [1, 1, 1, 1])  # stage inputs first
    ctx.trace_clear()
    ctx.enqueue_ndrange_partitioned(acc, (n, 1, 1), 1, queues, [1, 1, 1, 1])
    g = ctx.get_device_ids()
    assert ctx.trace_count("copy_peer") == 2 * 3  # sums + counts, three folds each
    assert ctx.trace_count("copy_peer", g[0]) == 4 and ctx.trace_count("copy_peer", g[2]) == 2
    for q in queues:
        ctx.finish(q)
    s = ctx.enqueue_read_buffer(queues[1], bs).view(np.int64)
    c = ctx.enqueue_read_buffer(queues[1], bcn).view(np.int64)
    assert (s == s_want).all() and (c == c_want).all()
    for x in (bp, ba, bs, bcn):
        ctx.release(x)


# ---- locking: finish() on one queue does not stall the others -------------------

def test_finish_does_not_block_other_queues(ctx, queues):
    """Thread A waits in finish() on a long fp64 matmul; meanwhile the main
    thread creates, writes and reads back a buffer on another queue. Those
    calls need only copy engines, so they must complete while A still waits
    (with one table lock held across the device sync they would queue behind it)."""
    n = 8192  # zero-filled inputs (never written): no host data needed
    ba, bb, bc = (ctx.create_buffer(n * n * 8) for _ in range(3))
    mk = kernel(ctx, "core", "matmul", [ba, bb, bc, n, n, n])
    ctx.enqueue_ndrange_kernel(queues[0], mk, (n, n, 1), 2)
    ctx.finish(queues[0])  # warm-up: allocation, first launch
    reps = 4
    t_kernel = time.perf_counter()
    for _ in range(reps):
        ctx.enqueue_ndrange_kernel(queues[0], mk, (n, n, 1), 2)
    ctx.finish(queues[0])
    t_kernel = time.perf_counter() - t_kernel
    assert t_kernel > 0.1, f"the blocking kernels are too short to test overlap ({t_kernel:.3f} s)"

    done = {}

    def waiter():
        for _ in range(reps):
            ctx.enqueue_ndrange_kernel(queues[0], mk, (n, n, 1), 2)
        done["enqueued"] = time.perf_counter()
        ctx.finish(queues[0])
        done["finished"] = time.perf_counter()

    th = threading.Thread(target=waiter)
    th.start()
    while "enqueued" not in done:
        time.sleep(0.001)
    time.sleep(0.005)
    t0 = time.perf_counter()
    x = np.arange(1 << 17, dtype=np.float64)
    b = ctx.create_buffer(x.nbytes)
    ctx.enqueue_write_buffer(queues[2], b, x)
    got = ctx.enqueue_read_buffer(queues[2], b).view(np.float64)
    ctx.finish(queues[2])
    t1 = time.perf_counter()
    th.join()
    assert (got == x).all()
    assert t1 < done["finished"], "queue 2's calls waited for queue 0's finish()"
    assert t1 - t0 < 0.5 * t_kernel
    for h in (ba, bb, bc, b):
        ctx.release(h)


def test_bind_external_memory(ctx, queues):
    """bind_external (hcl_ctx_bind_external): a buffer backed by caller-owned
    device memory (here a torch tensor, as bench.py binds symmetric-memory xs'
    buffers) -- a kernel's output lands in that memory, reads go through the
    runtime, the memory is not freed by release, and a second device gets a
    copy through the usual residency rules."""
    import torch

    n = 1000
    dev = ctx.get_device_ids()[0]
    t = torch.full((n,), -1.0, dtype=torch.float64, device="cuda:0")
    torch.cuda.synchronize()
    out = ctx.create_buffer(n * 8)
    ctx.bind_external(queues[0], out, t.data_ptr())
    a = np.arange(n, dtype=np.float64)
    b_a = ctx.create_buffer(n * 8)
    ctx.enqueue_write_buffer(queues[0], b_a, a)
    vk = kernel(ctx, "core", "vecadd", [b_a, b_a, out, n])
    ctx.enqueue_ndrange_kernel(queues[0], vk, (n, 1, 1), 1)
    ctx.finish(queues[0])
    assert (t.cpu().numpy() == 2 * a).all()  # the kernel wrote the caller's memory
    for q in queues:
        assert (ctx.enqueue_read_buffer(q, out).view(np.float64) == 2 * a).all()
    ctx.release(out)
    ctx.release(b_a)
    ctx.release(vk)
    assert (t.cpu().numpy() == 2 * a).all()  # still the caller's (not freed)
    with pytest.raises(Exception):
        ctx.bind_external(queues[0], ctx.create_buffer(8), 0)  # null pointer: argument error
    assert dev == ctx.get_device_ids()[0]


def test_zero_row_parts(ctx, queues):
    """Empty parts: a partitioned launch whose weights give one queue no rows, and
    a rank-style sub-range launch of zero rows, leave the result exactly as the
    whole launch computes it (the empty part launches nothing and moves nothing)."""
    if len(queues) < 2:
        pytest.skip("needs two logical devices")
    m, n, k = 300, 256, 128
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    outs = []
    for mode in ("whole", "zero-weight", "zero-range"):
        kh = kernel(ctx, "b200", "gemm_bf16", [])
        ba, bb, bc = ctx.create_buffer(a.nbytes), ctx.create_buffer(b.nbytes), ctx.create_buffer(m * n * 4)
        ctx.enqueue_write_buffer(queues[0], ba, a)
        ctx.enqueue_write_buffer(queues[0], bb, b)
        for i, v in enumerate([ba, bb, bc, m, k, n, 1]):
            ctx.set_kernel_arg(kh, i, v)
        if mode == "whole":
            ctx.enqueue_ndrange_kernel(queues[0], kh, (m, n, 1), 2)
        elif mode == "zero-weight":
            ctx.enqueue_ndrange_partitioned(kh, (m, n, 1), 2, queues[:2], [0, 1])
        else:
            ctx.enqueue_ndrange_range(queues[1], kh, (m, n, 1), 2, 0, 0)  # nothing
            ctx.enqueue_ndrange_range(queues[0], kh, (m, n, 1), 2, 0, m)
        for q in queues[:2]:
            ctx.finish(q)
        outs.append(ctx.enqueue_read_buffer(queues[0], bc).tobytes())
        for x in (ba, bb, bc, kh):
            ctx.release(x)
    assert outs[1] == outs[0] and outs[2] == outs[0]
