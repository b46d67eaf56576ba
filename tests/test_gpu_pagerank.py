"""PageRank (config C3) parity.

* The graph format (product CSR builder) is bit-identical to the oracle's.
* SpMV: rows of <= 32 products are bit-identical to the reference-order
  (ascending) fp32 oracle; every row is bit-identical to the oracle's
  restatement of the kernel's fixed per-row order (ho_spmv_f32_b200), and the
  whole vector is within 1e-6 (relative to max|y|) of the ascending oracle.
* Ranks after 20 iterations: bit-identical to the restated-order oracle,
  within 1e-5 (normwise, L1 and max) of the ascending-order oracle, and
  bit-identical across partitions P in {1, 2, 4} (nnz-balanced ranges) and
  across row-block sizes."""
import numpy as np
import pytest

import oracle as O
from paper_2005_08466_b200 import datagen as G

SCALE, EDGES = 12, 16 * 4096


@pytest.fixture(scope="module")
def graph():
    return G.pagerank_csr(SCALE, EDGES, 42)


def test_product_csr_matches_oracle(graph):
    rp, ci, val, deg = graph
    rp2, ci2, val2, deg2 = O.pagerank_csr(SCALE, EDGES, 42)
    assert (rp == rp2).all() and (ci == ci2).all() and (deg == deg2).all()
    assert val.tobytes() == val2.tobytes()


def test_inv_outdeg_matches_csr_values(graph):
    """The fused step's precomputed reciprocals are the CSR's stored values
    (val[p] = fl(1/outdeg(col[p]))) bit for bit, 0 exactly for dangling vertices."""
    rp, ci, val, deg = graph
    inv = G.pagerank_inv_outdeg(deg)
    assert inv[ci].tobytes() == val.tobytes()
    assert ((inv == 0) == (deg == 0)).all()


def test_row_blocks_properties(graph):
    rp = graph[0]
    for mx in (1, 16, 300, 4096):
        b = G.csr_row_blocks(rp, mx)
        assert b[0] == 0 and b[-1] == len(rp) - 1 and (np.diff(b) >= 1).all()
        for s, e in zip(b[:-1], b[1:]):
            nnz = rp[e] - rp[s]
            assert nnz <= mx or e - s == 1


def test_restated_order_agrees_with_ascending_order(graph):
    rp, ci, val, deg = graph
    x = O.gen_doubles(len(rp) - 1, 7).astype(np.float32) + 1.5
    a = O.spmv_f32(rp, ci, val, x, 0, len(rp) - 1)
    b = O.spmv_f32_b200(rp, ci, val, x, 0, len(rp) - 1)
    short = np.diff(rp) <= 32
    assert (a[short] == b[short]).all()
    assert np.abs(a - b).max() <= 1e-6 * np.abs(a).max()


@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


def make_pr(ctx, queues, graph, P, max_nnz):
    from paper_2005_08466_b200.pagerank import PageRank

    return PageRank(ctx, queues[:P], *graph, max_nnz=max_nnz)


@pytest.mark.gpu
@pytest.mark.parametrize("max_nnz", [4096, 256, 32])
def test_spmv_matches_oracles(ctx, queues, graph, max_nnz):
    rp, ci, val, deg = graph
    x = O.gen_doubles(len(rp) - 1, 7).astype(np.float32) + 1.5
    pr = make_pr(ctx, queues, graph, 1, max_nnz)
    y = pr.spmv(x)
    pr.close()
    assert y.tobytes() == O.spmv_f32_b200(rp, ci, val, x, 0, len(rp) - 1).tobytes()
    asc = O.spmv_f32(rp, ci, val, x, 0, len(rp) - 1)
    short = np.diff(rp) <= 32
    assert (y[short] == asc[short]).all()
    assert np.abs(y - asc).max() <= 1e-6 * np.abs(asc).max()


@pytest.mark.gpu
@pytest.mark.parametrize("max_nnz", [4096, 64])
def test_pagerank_20_iterations(ctx, queues, graph, max_nnz):
    rp, ci, val, deg = graph
    pr = make_pr(ctx, queues, graph, 1, max_nnz)
    pr.reset()
    pr.iterate(20)
    x = pr.ranks()
    pr.close()
    assert x.tobytes() == O.pagerank(rp, ci, val, deg, 20, b200_order=True).tobytes()
    want = O.pagerank(rp, ci, val, deg, 20).astype(np.float64)
    x = x.astype(np.float64)
    assert np.abs(x - want).sum() / np.abs(want).sum() <= 1e-5
    assert np.abs(x - want).max() / want.max() <= 1e-5


@pytest.mark.gpu
def test_pagerank_partition_and_blocking_invariance(ctx, queues, graph):
    results = []
    for P, mx in ((1, 4096), (2, 4096), (4, 4096), (4, 128), (3, 32)):
        pr = make_pr(ctx, queues, graph, P, mx)
        pr.reset()
        pr.iterate(20)
        results.append(pr.ranks().tobytes())
        pr.close()
    assert all(r == results[0] for r in results)


@pytest.mark.gpu
def test_pagerank_uneven_weights(ctx, queues, graph):
    from paper_2005_08466_b200.pagerank import PageRank

    pr = PageRank(ctx, queues, *graph, max_nnz=1024, weights=[5, 1, 1, 3])
    pr.reset()
    pr.iterate(5)
    got = pr.ranks().tobytes()
    pr.close()
    rp, ci, val, deg = graph
    assert got == O.pagerank(rp, ci, val, deg, 5, b200_order=True).tobytes()


def test_relabel_preserves_results_cpu(graph):
    """Degree-ordered relabelling keeps every row's product sequence: the
    restated-order oracle on the relabelled graph equals the original, permuted."""
    rp, ci, val, deg = graph
    rp2, ci2, val2, deg2, perm = G.pagerank_relabel(rp, ci, val, deg)
    assert sorted(perm.tolist()) == list(range(len(rp) - 1))
    assert (np.diff(deg2) <= 0).all() and (deg2 == deg[perm]).all()
    r = O.pagerank(rp, ci, val, deg, 7, b200_order=True)
    r2 = O.pagerank(rp2, ci2, val2, deg2, 7, b200_order=True)
    assert r2.tobytes() == r[perm].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("P,weights", [(1, None), (4, [1, 2, 3, 4])])
def test_pagerank_relabelled(ctx, queues, graph, P, weights):
    from paper_2005_08466_b200.pagerank import PageRank

    rp, ci, val, deg = graph
    pr = PageRank(ctx, queues[:P], *graph, max_nnz=512, weights=weights, relabel=True)
    x = O.gen_doubles(len(rp) - 1, 7).astype(np.float32) + 1.5
    assert pr.spmv(x).tobytes() == O.spmv_f32_b200(rp, ci, val, x, 0, len(rp) - 1).tobytes()
    pr.reset()
    pr.iterate(20)
    got = pr.ranks().tobytes()
    pr.close()
    assert got == O.pagerank(rp, ci, val, deg, 20, b200_order=True).tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 3])
def test_implicit_values_bit_identical(ctx, queues, graph, P):
    """pagerank_prep + pagerank_step_implicit (values folded into xs = x/outdeg)
    equals the explicit-value step and the restated-order oracle bit-for-bit."""
    from paper_2005_08466_b200.pagerank import PageRank

    rp, ci, val, deg = graph
    out = []
    for implicit in (False, True):
        pr = PageRank(ctx, queues[:P], *graph, max_nnz=64, implicit=implicit)
        pr.reset()
        pr.iterate(20)
        out.append(pr.ranks().tobytes())
        pr.close()
    assert out[0] == out[1] == O.pagerank(rp, ci, val, deg, 20, b200_order=True).tobytes()


@pytest.mark.gpu
def test_step_rejects_short_col_buffer_and_revalidates(ctx, queues, graph):
    """The row_ptr coverage check (cached per row_ptr write version) still
    rejects a col/val slice that does not cover the rows, and a rewritten
    row_ptr is validated again."""
    from paper_2005_08466_b200 import HaoclError
    from paper_2005_08466_b200.datagen import pagerank_units

    rp, ci, val, deg = graph
    v, nnz = len(rp) - 1, int(rp[-1])
    units, long_rows, n_long = pagerank_units(rp, 64)
    prog = ctx.create_program("b200")
    k = ctx.create_kernel(prog, "pagerank_spmv")
    q = queues[0]
    mk = ctx.create_buffer
    b_rp, b_u, b_l = mk(rp.nbytes), mk(units.nbytes), mk(long_rows.nbytes)
    b_col, b_val = mk((nnz - 8) * 4), mk((nnz - 8) * 4)  # 8 non-zeros short
    b_x, b_y = mk(v * 4), mk(v * 4)
    for b, a in ((b_rp, rp), (b_u, units), (b_l, long_rows), (b_col, ci[: nnz - 8]), (b_val, val[: nnz - 8]),
                 (b_x, np.ones(v, np.float32))):
        ctx.enqueue_write_buffer(q, b, a)
    for j, a in enumerate([b_rp, b_col, b_val, b_u, b_l, b_x, b_y, v, 0, len(units), n_long, 64]):
        ctx.set_kernel_arg(k, j, a)
    with pytest.raises(HaoclError) as e:
        ctx.enqueue_ndrange_kernel(q, k, (v, 1, 1), 1)
    assert e.value.name == "argument"
    rp2 = rp.copy()
    rp2[1:] = np.minimum(rp2[1:], nnz - 8)  # now consistent with the short slice
    ctx.enqueue_write_buffer(q, b_rp, rp2)
    ctx.enqueue_ndrange_kernel(q, k, (v, 1, 1), 1)  # revalidated against the new contents: accepted
    ctx.finish(q)
    for b in (b_rp, b_u, b_l, b_col, b_val, b_x, b_y, k, prog):
        ctx.release(b)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 4])
def test_pagerank_vs_reference_spmv_scale20(ctx, queues, P):
    """20 GPU iterations (the default fused step, R-MAT scale 20, 2^24 edges)
    against PageRank iterated on the REFERENCE LIBRARY's spmv_compute in
    fp64/int64 (oracle/_ref, proj/src/kernels.cpp:132-152): normwise (L1)
    relative error <= 1e-5, elementwise <= 1e-4."""
    from paper_2005_08466_b200.pagerank import PageRank

    rp, ci, val, deg = G.pagerank_csr(20, 1 << 24, 42)
    pr = PageRank(ctx, queues[:P], rp, ci, val, deg, fused=True)
    pr.reset()
    pr.iterate(20)
    got = pr.ranks().astype(np.float64)
    pr.close()
    want = O.ref_pagerank(rp, ci, deg, 20)
    assert np.abs(got - want).sum() / np.abs(want).sum() <= 1e-5
    assert (np.abs(got - want) / want).max() <= 1e-4


@pytest.mark.gpu
def test_pagerank_full_c3(ctx, queues):
    """SURVEY.md §8(d) C3 at full size: R-MAT scale 24, 2^28 edges, seed 42,
    20 iterations with the default kernels (implicit values, 64-nnz warp units):
    ranks bit-identical to the restated-order oracle; the mass sums to 1."""
    from paper_2005_08466_b200.pagerank import PageRank

    rp, ci, val, deg = G.pagerank_csr(24, 1 << 28, 42)
    pr = PageRank(ctx, queues[:1], rp, ci, val, deg)
    pr.reset()
    pr.iterate(20)
    got = pr.ranks()
    pr.close()
    want = O.pagerank(rp, ci, val, deg, 20, b200_order=True)
    assert got.tobytes() == want.tobytes()
    assert abs(float(got.astype(np.float64).sum()) - 1.0) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4])
def test_step_exchange_fused(ctx, queues, graph, P):
    """pagerank_step_exchange: each device computes its nnz-balanced row range
    of x' and, for those rows, the next gather input xs' = fl(1/outdeg) x'
    (what pagerank_prep computes) into its own AND its peers' xs' (here logical
    devices of one process; across processes IPC-mapped peer buffers, bench.py),
    plus its dangling partial. The only collective is an allreduce of the
    dangling sums. After 20 iterations the rows are bit-identical to the
    restated-order oracle -- no prep pass, no allgather."""
    import ctypes as C

    from paper_2005_08466_b200 import _native as N
    from paper_2005_08466_b200.datagen import pagerank_units
    from paper_2005_08466_b200.runtime import spmv_partition_ranges

    L = N.lib()
    rp, ci, val, deg = graph
    v = len(rp) - 1
    units, long_rows, n_long = pagerank_units(rp, 64)
    bounds = [int(b) for b in spmv_partition_ranges(rp.astype(np.int64), P)]
    base = 0x7800_0000
    ids = {}

    def bid(dev, name):
        return ids.setdefault((dev, name), base + len(ids))

    def put(dev, name, arr):
        arr = np.ascontiguousarray(arr)
        i = bid(dev, name)
        N.check(L.hcl_buffer_alloc(dev, i, 0, arr.nbytes))
        N.check(L.hcl_buffer_write(dev, i, 0, arr.ctypes.data, arr.nbytes))

    def ptr(dev, name):
        p = C.c_void_p()
        N.check(L.hcl_buffer_device_ptr(dev, bid(dev, name), C.byref(p), None, None))
        return p.value

    def launch(dev, kernel, args, lo=None, rows=None):
        a = (N.HclArg * len(args))()
        for j, (kind, x) in enumerate(args):
            a[j].kind = kind
            if kind == 0:
                a[j].scalar = x
            else:
                a[j].buffer_id = x
        w = C.c_uint64()
        go, gs = ((C.c_uint64 * 3)(lo, 0, 0), (C.c_uint64 * 3)(rows, 1, 1)) if lo is not None else (None, None)
        N.check(L.hcl_launch(dev, kernel.encode(), a, len(args), go, gs, 1, C.byref(w)))

    I_, O_, S_ = 1, 2, 0
    x0 = np.full(v, np.float32(1.0 / v), np.float32)
    try:
        for d in range(P):
            for name, arr in (("rp", rp), ("col", ci), ("units", units), ("long", long_rows), ("deg", deg),
                              ("inv", G.pagerank_inv_outdeg(deg)),
                              ("x", x0), ("xs0", np.zeros(v, np.float32)), ("xs1", np.zeros(v, np.float32)),
                              ("dsum0", np.zeros(1, np.uint64)), ("dsum1", np.zeros(1, np.uint64))):
                put(d, name, arr)
        for d in range(P):  # peers' xs' for each parity
            for i in range(2):
                put(d, f"peers{i}", np.array([ptr(e, f"xs{i}") for e in range(P) if e != d] or [0], np.uint64))
            # iteration 0's gather input, once: xs0 = prep(x0), dsum0 = its dangling sum
            launch(d, "pagerank_prep", [(I_, bid(d, "x")), (I_, bid(d, "deg")), (O_, bid(d, "dsum0")),
                                        (O_, bid(d, "xs0")), (S_, v)])
        devs = (C.c_int * P)(*range(P))
        cur = 0
        for _ in range(20):
            nxt = 1 - cur
            for d in range(P):
                launch(d, "pagerank_step_exchange",
                       [(I_, bid(d, "rp")), (I_, bid(d, "col")), (I_, bid(d, "units")), (I_, bid(d, "long")),
                        (I_, bid(d, f"xs{cur}")), (I_, bid(d, f"dsum{cur}")), (O_, bid(d, "x")), (S_, v), (S_, 0),
                        (S_, len(units)), (S_, n_long), (S_, 64), (I_, bid(d, f"peers{nxt}")), (S_, P - 1),
                        (I_, bid(d, "inv")), (O_, bid(d, f"xs{nxt}")), (O_, bid(d, f"dsum{nxt}"))],
                       lo=bounds[d], rows=bounds[d + 1] - bounds[d])
            for d in range(P):  # every device's stores have landed
                N.check(L.hcl_finish(d, None))
            if P > 1:  # the one collective: allreduce of the dangling partials
                dids = (C.c_uint64 * P)(*[bid(d, f"dsum{nxt}") for d in range(P)])
                N.check(L.hcl_collective(2, devs, P, dids, 1, 0, 0))
            cur = nxt
        want = O.pagerank(rp, ci, val, deg, 20, b200_order=True)
        got = np.empty(v, np.float32)
        for d in range(P):
            part = np.empty(v, np.float32)
            N.check(L.hcl_buffer_read(d, bid(d, "x"), 0, part.ctypes.data, v * 4))
            got[bounds[d]:bounds[d + 1]] = part[bounds[d]:bounds[d + 1]]
        assert got.tobytes() == want.tobytes()
    finally:
        for (d, _), i in ids.items():
            L.hcl_buffer_release(d, i)


@pytest.mark.gpu
@pytest.mark.parametrize("P,weights", [(1, None), (2, None), (4, [1, 2, 3, 4])])
def test_pagerank_fused_partitioned(ctx, queues, graph, P, weights):
    """The fused step through the host API: one partitioned launch per iteration
    with the EXCHANGE output (xs' written into every device's copy), the
    runtime-filled PEERS list and the REDUCE_SUM dangling partials; ranks after
    20 iterations bit-identical to the restated-order oracle."""
    from paper_2005_08466_b200.pagerank import PageRank

    rp, ci, val, deg = graph
    pr = PageRank(ctx, queues[:P], *graph, max_nnz=64, weights=weights, fused=True)
    pr.reset()
    pr.iterate(20)
    got = pr.ranks().tobytes()
    pr.close()
    assert got == O.pagerank(rp, ci, val, deg, 20, b200_order=True).tobytes()
