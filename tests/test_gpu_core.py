"""GPU parity of the reference's "core" bundle through the host API and the
C-ABI: outputs must be BIT-IDENTICAL to the reference (FNV-1a digests of
tests/golden/reference_golden.json, measured by running the reference), for
every partition P in {1, 2, 4} of the NDRange."""
import numpy as np
import pytest

import oracle as O
from paper_2005_08466_b200 import HaoclError
from paper_2005_08466_b200 import _native as N

pytestmark = pytest.mark.gpu


def h(x):
    return "%016x" % x


def run(ctx, kernel, args, outs, queues, global_rows=None, partitioned=False, weights=None, bundle="core"):
    """Bind args (ints or np arrays for inputs; ('out', nbytes) for outputs), launch
    whole on queues[0] or partitioned over queues, and return output arrays (uint8)."""
    prog = ctx.create_program(bundle)
    k = ctx.create_kernel(prog, kernel)
    bufs = {}
    for i, a in enumerate(args):
        if isinstance(a, tuple) and a[0] == "out":
            b = ctx.create_buffer(a[1])
            bufs[i] = b
            ctx.set_kernel_arg(k, i, b)
        elif isinstance(a, np.ndarray):
            b = ctx.create_buffer(a.nbytes)
            ctx.enqueue_write_buffer(queues[0], b, a)
            bufs[i] = b
            ctx.set_kernel_arg(k, i, b)
        else:
            ctx.set_kernel_arg(k, i, int(a))
    if partitioned:
        ctx.enqueue_ndrange_partitioned(k, (global_rows, 1, 1), 1, queues, weights)
    else:
        ctx.enqueue_ndrange_kernel(queues[0], k, (global_rows or 1, 1, 1), 1)
    for q in queues:
        ctx.finish(q)
    res = {i: ctx.enqueue_read_buffer(queues[0], bufs[i]) for i in outs}
    for b in bufs.values():
        ctx.release(b)
    ctx.release(k)
    ctx.release(prog)
    return res


@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


@pytest.mark.parametrize("n", [64, 512, 1024])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_matmul_bitexact_digest(ctx, queues, golden, n, P):
    a = O.gen_doubles(n * n, 42)
    b = O.gen_doubles(n * n, 43)
    out = run(ctx, "matmul", [a, b, ("out", n * n * 8), n, n, n], [2], queues[:P], global_rows=n,
              partitioned=P > 1)
    assert h(O.fnv1a(out[2])) == golden["digests"][f"matmul_{n}"]


def test_matmul_uneven_weights_still_bitexact(ctx, queues, golden):
    n = 512
    a = O.gen_doubles(n * n, 42)
    b = O.gen_doubles(n * n, 43)
    out = run(ctx, "matmul", [a, b, ("out", n * n * 8), n, n, n], [2], queues, global_rows=n, partitioned=True,
              weights=[5, 1, 3, 1])
    assert h(O.fnv1a(out[2])) == golden["digests"]["matmul_512"]


@pytest.mark.parametrize("n", [10**5, 10**7])
@pytest.mark.parametrize("P", [1, 4])
def test_vecadd_digest(ctx, queues, golden, n, P):
    a = O.gen_doubles(n, 42)
    b = O.gen_doubles(n, 43)
    out = run(ctx, "vecadd", [a, b, ("out", n * 8), n], [2], queues[:P], global_rows=n, partitioned=P > 1,
              weights=[2] * P)
    assert h(O.fnv1a(out[2])) == golden["digests"][f"vecadd_{n}"]


@pytest.mark.parametrize("V,E", [(1000, 10**4), (10**5, 10**6)])
def test_bfs_digest(ctx, queues, golden, V, E):
    """bfs (proj/src/kernels.cpp:154-193; whole range only, as bench.cpp:539-540):
    levels bit-identical to the reference digest, and to the oracle from
    another source (unreachable vertices stay -1)."""
    rp, ci = O.gen_graph(V, E, 42)
    hdr = np.array([V, V], np.int64)
    out = run(ctx, "bfs", [hdr, rp, ci, 0, ("out", V * 4)], [4], queues[:1])
    assert h(O.fnv1a(out[4])) == golden["digests"][f"bfs_{V}v{E}e"]
    out = run(ctx, "bfs", [hdr, rp, ci, V // 3, ("out", V * 4)], [4], queues[:1])
    assert (out[4].view(np.int32) == O.bfs(rp, ci, V // 3)).all()


def test_bfs_unreachable_and_errors(ctx, queues):
    # two components: 0-1-2 and 3-4; source 4 reaches only 3
    rp = np.array([0, 1, 3, 4, 5, 6], np.int64)
    ci = np.array([1, 0, 2, 1, 4, 3], np.int64)
    hdr = np.array([5, 5], np.int64)
    out = run(ctx, "bfs", [hdr, rp, ci, 4, ("out", 20)], [4], queues[:1])[4].view(np.int32)
    assert out.tolist() == [-1, -1, -1, 1, 0]
    with pytest.raises(HaoclError) as e:
        run(ctx, "bfs", [hdr, rp, ci, 5, ("out", 20)], [4], queues[:1])
    assert e.value.name == "argument"


@pytest.mark.parametrize("r,c,d", [(100, 100, 0.1), (10**4, 10**4, 1e-3), (10**5, 10**5, 1e-4)])
def test_spmv_two_stage_digest(ctx, queues, golden, r, c, d):
    """The reference bench's two-stage SpMV (proj/src/bench.cpp:210-321): stage 1
    spmv_partition on one device, stage 2 spmv_compute per part on rebased CSR
    slices, y reassembled at lo*8 — digest equal to the reference."""
    rp, ci, v = O.gen_csr(r, c, d, 42)
    x = O.gen_doubles(c, 43)
    hdr = np.array([r, c], np.int64)
    for P in (1, 2, 4):
        rng = run(ctx, "spmv_partition", [hdr, rp, P, ("out", (P + 1) * 8)], [3], queues[:1])[3].view(np.int64)
        assert (rng == O.spmv_partition_ranges(rp, P)).all()
        y = np.empty(r, np.float64)
        for p in range(P):
            lo, hi = int(rng[p]), int(rng[p + 1])
            first, last = rp[lo], rp[hi]
            part = [np.array([hi - lo, c], np.int64), (rp[lo:hi + 1] - first).astype(np.int64),
                    ci[first:last].copy(), v[first:last].copy(), x, 0, hi - lo, ("out", (hi - lo) * 8)]
            y[lo:hi] = run(ctx, "spmv_compute", part, [7], [queues[p]])[7].view(np.float64)
        assert h(O.fnv1a(y)) == golden["digests"][f"spmv_{r}x{c}@{d}"]


def test_spmv_compute_kats_and_errors(ctx, queues):
    # CSR identity gives y = x; empty range gives an empty slice
    n = 50
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int64)
    v = np.ones(n)
    x = O.gen_doubles(n, 1)
    hdr = np.array([n, n], np.int64)
    y = run(ctx, "spmv_compute", [hdr, rp, ci, v, x, 0, n, ("out", n * 8)], [7], queues[:1])[7].view(np.float64)
    assert (y == x).all()
    with pytest.raises(HaoclError) as e:
        run(ctx, "spmv_compute", [hdr, rp, ci, v, x, 5, 60, ("out", 8 * 8)], [7], queues[:1])
    assert e.value.name == "argument"
    bad = ci.copy()
    bad[7] = n + 3
    with pytest.raises(HaoclError) as e:
        run(ctx, "spmv_compute", [hdr, rp, bad, v, x, 0, n, ("out", n * 8)], [7], queues[:1])
    assert e.value.name == "argument" and "col_idx out of range" in str(e.value)


@pytest.mark.parametrize("R,Q,D,K", [(200, 20, 8, 5), (10**5, 10**3, 16, 10)])
@pytest.mark.parametrize("P", [1, 4])
def test_knn_digest(ctx, queues, golden, R, Q, D, K, P):
    rf = O.gen_doubles(R * D, 42)
    q = O.gen_doubles(Q * D, 43)
    out = run(ctx, "knn", [rf, q, R, Q, D, K, ("out", Q * K * 4), ("out", Q * K * 8)], [6, 7], queues[:P],
              global_rows=Q, partitioned=P > 1)
    assert h(O.fnv1a(out[7], O.fnv1a(out[6]))) == golden["digests"][f"knn_{R}x{Q}x{D}k{K}"]


def test_knn_tie_rule(ctx, queues, golden):
    k = golden["knn_kat"]
    out = run(ctx, "knn", [np.array(k["ref"]), np.array(k["query"]), 5, 2, 2, k["k"], ("out", 2 * 3 * 4),
                           ("out", 2 * 3 * 8)], [6, 7], queues[:1])
    assert out[6].view(np.int32).tolist() == k["idx"] and out[7].view(np.float64).tolist() == k["dist"]


def test_error_conventions(ctx, queues):
    prog = ctx.create_program("core")
    with pytest.raises(HaoclError) as e:
        ctx.create_kernel(prog, "nosuch")
    assert e.value.name == "name" and e.value.code == 10
    with pytest.raises(HaoclError) as e:
        ctx.create_program("nobundle")
    assert e.value.name == "name"
    k = ctx.create_kernel(prog, "vecadd")
    with pytest.raises(HaoclError) as e:
        ctx.enqueue_ndrange_kernel(queues[0], k)
    assert e.value.name == "argument" and "unbound" in str(e.value)
    a = ctx.create_buffer(32)
    ctx.set_kernel_arg(k, 0, a)
    ctx.set_kernel_arg(k, 1, a)
    ctx.set_kernel_arg(k, 2, ctx.create_buffer(32))
    ctx.set_kernel_arg(k, 3, 5)  # n=5 but 4-element buffers
    with pytest.raises(HaoclError) as e:
        ctx.enqueue_ndrange_kernel(queues[0], k)
    assert e.value.name == "argument"
    with pytest.raises(HaoclError) as e:
        ctx.enqueue_write_buffer(queues[0], a, np.zeros(5))
    assert e.value.name == "size"
    # never-written buffers read back as zeros; use after release is a handle error
    assert (ctx.enqueue_read_buffer(queues[0], a) == 0).all()
    ctx.release(a)
    with pytest.raises(HaoclError) as e:
        ctx.enqueue_read_buffer(queues[0], a, length=32)
    assert e.value.name == "handle"
    with pytest.raises(HaoclError) as e:
        ctx.release(a)
    assert e.value.name == "handle"


def test_buffer_migration_between_devices(ctx, queues):
    data = np.arange(1000, dtype=np.float64)
    b = ctx.create_buffer(data.nbytes)
    ctx.enqueue_write_buffer(queues[0], b, data)
    # a partial write on device 2 then a full read through device 3 gathers the pieces
    ctx.enqueue_write_buffer(queues[2], b, np.full(10, -1.0), offset=80)
    got = ctx.enqueue_read_buffer(queues[3], b).view(np.float64)
    want = data.copy()
    want[10:20] = -1.0
    assert (got == want).all()
    ctx.release(b)


def test_finish_reports_compute_and_profiles(ctx, queues):
    n = 256
    a = O.gen_doubles(n * n, 1)
    prog = ctx.create_program("core")
    k = ctx.create_kernel(prog, "matmul")
    ba, bb, bc = ctx.create_buffer(a.nbytes), ctx.create_buffer(a.nbytes), ctx.create_buffer(a.nbytes)
    ctx.enqueue_write_buffer(queues[1], ba, a)
    ctx.enqueue_write_buffer(queues[1], bb, a)
    for i, v in enumerate([ba, bb, bc, n, n, n]):
        ctx.set_kernel_arg(k, i, v)
    ctx.enqueue_ndrange_kernel(queues[1], k, (n, n, 1), 2)
    f = ctx.finish(queues[1])
    assert f.compute_ms > 0 and f.transfer_ms > 0 and f.modeled_ms > 0
    assert ctx.profiled_rate(1, "matmul") > 0
    assert ctx.finish(queues[1]).compute_ms == 0.0  # drained
    for x in (ba, bb, bc):
        ctx.release(x)


def test_kernel_launch_counter_advances(ctx, queues):
    before = N.lib().hcl_kernel_launch_count()
    run(ctx, "vecadd", [np.ones(64), np.ones(64), ("out", 64 * 8), 64], [2], queues[:1])
    assert N.lib().hcl_kernel_launch_count() > before


def test_async_copies_respect_raw_and_war(ctx, queues):
    """Non-blocking writes/reads on the copy streams overlap kernels on the
    compute stream; with two buffer sets reused every other iteration, each
    result must still match its own inputs (RAW for the kernel, WAR for the
    overwrite of a buffer the previous-but-one kernel read)."""
    n = 1 << 20
    q = queues[0]
    prog = ctx.create_program("core")
    sets = []
    for _ in range(2):
        k = ctx.create_kernel(prog, "vecadd")
        a, b, c = (ctx.create_buffer(n * 8) for _ in range(3))
        for i, v in enumerate([a, b, c, n]):
            ctx.set_kernel_arg(k, i, v)
        sets.append((k, a, b, c))
    ins = [O.gen_doubles(n, 100 + i) for i in range(8)]
    two = np.full(n, 2.0)
    outs = [np.empty(n, np.float64) for _ in range(8)]
    for i in range(8):
        k, a, b, c = sets[i % 2]
        ctx.enqueue_write_buffer(q, a, ins[i], blocking=False)
        ctx.enqueue_write_buffer(q, b, two, blocking=False)
        ctx.enqueue_ndrange_kernel(q, k)
        ctx.enqueue_read_buffer(q, c, out=outs[i], blocking=False)
    ctx.finish(q)
    for i in range(8):
        assert (outs[i] == ins[i] + 2.0).all(), i


def test_sm_budget_emulated_heterogeneity(ctx, queues):
    """A logical device with an SM budget sizes its grids to it (slower, same
    results) and the scheduler's model follows (relative_throughput)."""
    gids = ctx.get_device_ids()
    m = n = k = 2048
    a = O.gen_bf16(m * k, 42)
    b = O.gen_bf16(k * n, 43)
    outs = {}
    try:
        ctx.set_sm_budget(gids[1], 16)
        with pytest.raises(HaoclError) as e:
            ctx.set_sm_budget(gids[1], 100000)
        assert e.value.name == "argument"
        for qi in (0, 1):
            res = run(ctx, "gemm_bf16", [a, b, ("out", m * n * 4), m, k, n, 1], [2], [queues[qi]], bundle="b200")
            outs[qi] = res[2].tobytes()
    finally:
        ctx.set_sm_budget(gids[1], 0)
    assert outs[0] == outs[1]


def test_rate_driven_split(ctx, queues):
    """Partitioned launches without weights follow the EMA-profiled rates
    (Scheduler::partition_weights, proj/src/scheduler.cpp:136-149 generalised):
    a device with a quarter of the SMs ends up with well under half the rows,
    and the output equals the whole launch bit-for-bit."""
    gids = ctx.get_device_ids()
    m, n, k = 8192, 2048, 2048
    a = O.gen_bf16(m * k, 5)
    b = O.gen_bf16(k * n, 6)
    prog = ctx.create_program("b200")
    kh = ctx.create_kernel(prog, "gemm_bf16")
    ba, bb, bc = ctx.create_buffer(a.nbytes), ctx.create_buffer(b.nbytes), ctx.create_buffer(m * n * 4)
    qs = [queues[2], queues[3]]
    try:
        ctx.set_sm_budget(gids[2], 120)
        ctx.set_sm_budget(gids[3], 28)
        ctx.enqueue_write_buffer(qs[0], ba, a)
        ctx.enqueue_write_buffer(qs[0], bb, b)
        for i, v in enumerate([ba, bb, bc, m, k, n, 1]):
            ctx.set_kernel_arg(kh, i, v)
        plan0 = ctx.partition_plan(kh, (m, n, 1), qs)
        for _ in range(4):
            for _ in range(3):
                ctx.enqueue_ndrange_partitioned(kh, (m, n, 1), 2, qs)
            for q in qs:
                ctx.finish(q)
        plan = ctx.partition_plan(kh, (m, n, 1), qs)
        got = ctx.enqueue_read_buffer(qs[0], bc).tobytes()
        ctx.enqueue_ndrange_kernel(queues[0], kh, (m, n, 1), 2)
        ctx.finish(queues[0])
        whole = ctx.enqueue_read_buffer(queues[0], bc).tobytes()
    finally:
        ctx.set_sm_budget(gids[2], 0)
        ctx.set_sm_budget(gids[3], 0)
        for h in (ba, bb, bc, kh, prog):
            ctx.release(h)
    assert plan0[1] > m * 0.7  # model: 120 vs 28 SMs
    assert plan[1] > m * 0.65, plan  # profiled rates agree
    assert got == whole


def test_zero_weight_parts_are_skipped(ctx, queues, golden):
    """Parts with no rows launch nothing and leave the output intact."""
    n = 512
    a = O.gen_doubles(n * n, 42)
    b = O.gen_doubles(n * n, 43)
    out = run(ctx, "matmul", [a, b, ("out", n * n * 8), n, n, n], [2], queues, global_rows=n, partitioned=True,
              weights=[0, 1, 0, 3])
    assert h(O.fnv1a(out[2])) == golden["digests"]["matmul_512"]


def test_buffers_beyond_4gib(ctx, queues):
    """The reference caps a read at one 4 GiB frame (wire.cpp:337-338); here
    buffers, offsets, peer copies and partial reads are 64-bit: vecadd over
    4.8 GB operands split over four devices, read back at offsets > 4 GiB."""
    n = 600_000_000
    a = O.gen_doubles(n, 42)
    b = O.gen_doubles(n, 43)
    prog = ctx.create_program("core")
    k = ctx.create_kernel(prog, "vecadd")
    ba, bb, bc = (ctx.create_buffer(n * 8) for _ in range(3))
    try:
        ctx.enqueue_write_buffer(queues[0], ba, a)
        ctx.enqueue_write_buffer(queues[0], bb, b)
        for i, v in enumerate([ba, bb, bc, n]):
            ctx.set_kernel_arg(k, i, v)
        ctx.enqueue_ndrange_partitioned(k, (n, 1, 1), 1, queues, [1, 2, 3, 4])
        for q in queues:
            ctx.finish(q)
        for lo in (0, (1 << 32) // 8 - 3, n - 1000):  # straddles the 4 GiB offset and the part boundaries
            got = ctx.enqueue_read_buffer(queues[1], bc, offset=lo * 8, length=8000).view(np.float64)
            want = a[lo:lo + 1000] + b[lo:lo + 1000]
            assert got.tobytes() == want.tobytes(), lo
    finally:
        for hnd in (ba, bb, bc, k, prog):
            ctx.release(hnd)


def test_in_process_collective_c_abi(ctx, queues):
    """hcl_collective across the four logical devices of the
    session: allreduce in device order (bit-identical everywhere), allgather,
    broadcast; raw C-ABI calls on device-level buffer ids."""
    import ctypes as C

    from paper_2005_08466_b200 import _native as N

    L = N.lib()
    ndev, cnt = 4, 1000
    devs = (C.c_int * ndev)(0, 1, 2, 3)
    ids = (C.c_uint64 * ndev)(*[0x7700_0000 + i for i in range(ndev)])
    rng = np.random.default_rng(5)
    parts = [rng.standard_normal(cnt * ndev) * 10.0**rng.integers(-8, 17, cnt * ndev) for _ in range(ndev)]

    def put(arrs):
        for i, a in enumerate(arrs):
            assert L.hcl_buffer_alloc(i, ids[i], 0, a.nbytes) == 0
            assert L.hcl_buffer_write(i, ids[i], 0, a.ctypes.data, a.nbytes) == 0

    def get(i, nbytes, dt):
        out = np.empty(nbytes // np.dtype(dt).itemsize, dt)
        assert L.hcl_buffer_read(i, ids[i], 0, out.ctypes.data, nbytes) == 0
        return out

    try:
        put([p.astype(np.float64) for p in parts])
        assert L.hcl_collective(2, devs, ndev, ids, cnt * ndev, 1, 2) == 0  # allreduce f64, root 2
        want = ((parts[0] + parts[1]) + parts[2]) + parts[3]
        for i in range(ndev):
            assert get(i, cnt * ndev * 8, np.float64).tobytes() == want.tobytes()
        ints = [np.arange(cnt * ndev, dtype=np.int64) * (i + 1) for i in range(ndev)]
        put(ints)
        assert L.hcl_collective(1, devs, ndev, ids, cnt, 0, 0) == 0  # allgather: device i owns slice i
        want = np.concatenate([ints[i][i * cnt:(i + 1) * cnt] for i in range(ndev)])
        for i in range(ndev):
            assert (get(i, cnt * ndev * 8, np.int64) == want).all()
        fl = [np.full(cnt, i + 0.5, np.float32) for i in range(ndev)]
        put(fl)
        assert L.hcl_collective(0, devs, ndev, ids, cnt, 2, 3) == 0  # broadcast f32 from device 3
        for i in range(ndev):
            assert (get(i, cnt * 4, np.float32) == 3.5).all()
        rc = L.hcl_collective(2, devs, ndev, ids, cnt, 7, 0)
        assert rc == 1000 + 9  # argument
    finally:
        for i in range(ndev):
            L.hcl_buffer_release(i, ids[i])


def _launch_raw(L, dev, kernel, spec):
    """hcl_launch on device-level buffers: spec = list of int scalars or
    ('in', array) / ('out', nbytes). Returns (rc, work_units)."""
    import ctypes as C

    ids, args = [], (N.HclArg * max(1, len(spec)))()
    for i, a in enumerate(spec):
        if isinstance(a, tuple):
            bid = 0x7A00_0000 + i
            nbytes = a[1] if a[0] == "out" else a[1].nbytes
            assert L.hcl_buffer_alloc(dev, bid, 0, max(nbytes, 1)) == 0
            if a[0] == "in":
                arr = np.ascontiguousarray(a[1])
                assert L.hcl_buffer_write(dev, bid, 0, arr.ctypes.data, arr.nbytes) == 0
            ids.append(bid)
            args[i] = N.HclArg(1 if a[0] == "in" else 2, 0, 0, bid)
        else:
            args[i] = N.HclArg(0, 0, int(a), 0)
    work = C.c_uint64(0)
    rc = L.hcl_launch(dev, kernel.encode(), args, len(spec), None, None, 1, C.byref(work))
    assert L.hcl_finish(dev, None) == 0
    for b in ids:
        L.hcl_buffer_release(dev, b)
    return rc, work.value


def test_work_units_match_reference_work_estimate(ctx, golden):
    """hcl_launch reports the reference's work units (kernels::work_estimate,
    proj/src/kernels.cpp:285-298) -- the unit behind the scheduler's EMA rates
    (scheduler.cpp:136-149) and the roofline. Shapes of the golden fixture,
    tests/golden/make_golden.py (generated from the reference library)."""
    L = N.lib()
    we = golden["work_estimate"]
    _, w = _launch_raw(L, 0, "matmul", [("in", np.ones(3 * 5)), ("in", np.ones(5 * 7)), ("out", 3 * 7 * 8), 3, 5, 7])
    assert w == we["matmul"]  # 2 * 3 * 5 * 7
    rows = cols = 10  # values buffer of 800 bytes = 100 nnz
    hdr = np.array([rows, cols], np.int64)
    rp = (np.arange(rows + 1) * cols).astype(np.int64)
    ci = np.tile(np.arange(cols), rows).astype(np.int64)
    rc, w = _launch_raw(L, 0, "spmv_compute", [("in", hdr), ("in", rp), ("in", ci), ("in", np.ones(100)),
                                               ("in", np.ones(cols)), 0, rows, ("out", rows * 8)])
    assert rc == 0 and w == we["spmv_compute"]
    rc, w = _launch_raw(L, 0, "knn", [("in", np.ones(100 * 8)), ("in", np.ones(10 * 8)), 100, 10, 8, 3,
                                      ("out", 10 * 3 * 4), ("out", 10 * 3 * 8)])
    assert rc == 0 and w == we["knn"]
    rc, w = _launch_raw(L, 0, "vecadd", [("in", np.ones(1000)), ("in", np.ones(1000)), ("out", 8000), 1000])
    assert rc == 0 and w == we["vecadd"]
    if O.ref_available():  # and live against the reference library on the same shapes
        assert O.ref_work_estimate("matmul", [3, 5, 7], [0, 0, 0]) == we["matmul"]


def test_execute_error_codes_match_reference(ctx, golden):
    """kernels::execute's error codes (name = 10 for an unknown kernel,
    argument = 9 for arity and buffer-length violations), measured on the
    reference library (tests/golden/reference_golden.json "execute_errors"),
    come back from hcl_launch as 1000 + code."""
    L = N.lib()
    ee = golden["execute_errors"]
    assert _launch_raw(L, 0, "nosuch", [])[0] == 1000 + ee["unknown_kernel"]
    assert _launch_raw(L, 0, "vecadd", [1])[0] == 1000 + ee["arity"]
    rc, _ = _launch_raw(L, 0, "vecadd", [("in", np.ones(4)), ("in", np.ones(3)), ("out", 64), 4])
    assert rc == 1000 + ee["length"]
