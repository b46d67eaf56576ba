"""k-means (config C4) parity: assignments bit-exact vs the oracle (the
reference's knn k=1 semantics in fp32: diff = c - x, ascending d, rounded
multiply then add, ties to the smaller index), exact int64 sums, centroids
bit-exact after several iterations, and bit-identical for P in {1, 2, 4}."""
import numpy as np
import pytest

import oracle as O
from paper_2005_08466_b200 import HaoclError
from paper_2005_08466_b200 import datagen as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


def oracle_iterations(pts, n, d, k, cent, iters):
    for _ in range(iters):
        a = O.kmeans_assign(pts, n, d, cent, k)
        s, c = O.kmeans_accumulate(pts, n, d, a, k)
        cent = O.kmeans_finalize(s, c, k, d, cent)
    return a, s, c, cent


@pytest.mark.parametrize("n,d,k", [(20000, 32, 64), (5000, 32, 1030), (3000, 7, 33), (4099, 32, 1)])
def test_assign_and_update_bitexact(ctx, queues, n, d, k):
    from paper_2005_08466_b200.kmeans import KMeans

    pts = G.gen_kmeans_points(n, d, max(k, 2), 42)
    cent0 = pts[: k * d].copy()
    a_want, s_want, c_want, cent_want = oracle_iterations(pts, n, d, k, cent0, 3)
    km = KMeans(ctx, queues[:1], n, d, k)
    km.load_points(pts)
    km.set_centroids(cent0)
    km.iterate(2)
    km.assign_only()
    km.finish()
    # after 2 full iterations + assign: assignments of iteration 3
    got_a = km.assignments()
    km.iterate(1)
    s, c = km.sums()
    cent = km.centroids()
    km.close()
    assert (got_a == a_want).all()
    assert (s == s_want).all() and (c == c_want).all()
    assert cent.tobytes() == cent_want.reshape(k, d).tobytes()


def test_ties_go_to_smaller_index(ctx, queues):
    from paper_2005_08466_b200.kmeans import KMeans

    d, k, n = 32, 6, 64
    cent = np.zeros((k, d), np.float32)
    cent[1] = cent[3] = 1.0  # duplicates: equal distances
    cent[2] = cent[4] = -1.0
    cent[5] = 1.0
    pts = np.zeros((n, d), np.float32)
    pts[::2] = 1.0
    pts[1::2] = -1.0
    km = KMeans(ctx, queues[:1], n, d, k)
    km.load_points(pts)
    km.set_centroids(cent)
    km.assign_only()
    a = km.assignments()
    km.close()
    assert (a[::2] == 1).all() and (a[1::2] == 2).all()
    assert (a == O.kmeans_assign(pts.ravel(), n, d, cent.ravel(), k)).all()


@pytest.mark.parametrize("weights", [None, [3, 1, 2, 2]])
def test_partition_invariance(ctx, queues, weights):
    from paper_2005_08466_b200.kmeans import KMeans

    n, d, k = 30000, 32, 128
    pts = G.gen_kmeans_points(n, d, k, 43)
    cent0 = pts[: k * d].copy()
    outs = []
    for P in (1, 2, 4):
        km = KMeans(ctx, queues[:P], n, d, k, weights=weights[:P] if weights else None)
        km.load_points(pts)
        km.set_centroids(cent0)
        km.iterate(3)
        outs.append((km.centroids().tobytes(), km.assignments().tobytes()))
        km.close()
    assert outs[0] == outs[1] == outs[2]


def test_device_point_generator_matches_host(ctx, queues):
    from paper_2005_08466_b200.kmeans import KMeans

    n, d, k = 10000, 32, 16
    km = KMeans(ctx, queues[:3], n, d, k)
    km.generate_points(42, 1024)
    km.finish()
    got = ctx.enqueue_read_buffer(queues[0], km.b_pts).view(np.float32)
    km.close()
    assert (got == G.gen_kmeans_points(n, d, 1024, 42)).all()


# ---- tensor-filtered assignment (kmeans_assign_tc): identical results ----

@pytest.mark.parametrize("n,k,P", [(20000, 256, 1), (70001, 1024, 1), (33333, 512, 4), (9000, 768, 2)])
def test_tensor_filter_bitexact(ctx, queues, n, k, P):
    from paper_2005_08466_b200.kmeans import KMeans

    d = 32
    pts = G.gen_kmeans_points(n, d, k, 42)
    cent0 = pts[: k * d].copy()
    a_want, s_want, c_want, cent_want = oracle_iterations(pts, n, d, k, cent0, 3)
    km = KMeans(ctx, queues[:P], n, d, k, tensor_filter=True)
    km.load_points(pts)
    km.set_centroids(cent0)
    km.iterate(2)
    km.assign_only()
    got_a = km.assignments()
    km.iterate(1)
    s, c = km.sums()
    cent = km.centroids()
    km.close()
    assert (got_a == a_want).all()
    assert (s == s_want).all() and (c == c_want).all()
    assert cent.tobytes() == cent_want.reshape(k, d).tobytes()


def test_tensor_filter_ties_and_general_fp32(ctx, queues):
    """Exact ties (duplicate centroids) and points off the 2^-12 grid."""
    from paper_2005_08466_b200.kmeans import KMeans

    d, k, n = 32, 256, 4096
    rng = np.random.default_rng(3)
    cent = rng.standard_normal((k, d)).astype(np.float32) * 3
    cent[7] = cent[200]  # duplicates: ties must go to 7
    cent[9] = cent[10]
    pts = rng.standard_normal((n, d)).astype(np.float32) * 3
    pts[:50] = cent[200] + rng.standard_normal((50, d)).astype(np.float32) * 1e-3
    pts[50:100] = cent[10]
    want = O.kmeans_assign(pts.reshape(-1), n, d, cent.reshape(-1), k)
    km = KMeans(ctx, queues[:1], n, d, k, tensor_filter=True)
    km.load_points(pts, validate=False)  # assignment only: any fp32 data
    km.set_centroids(cent)
    km.assign_only()
    got = km.assignments()
    with pytest.raises(HaoclError) as e:  # the exact update needs grid points
        km.iterate(1)
    assert e.value.code == 9
    km.close()
    assert (got == want).all()
    assert (got[50:100] == 9).all()


@pytest.mark.parametrize("bad", [2.0**-13, 8.0, -8.0 - 2.0**-12, float("nan"), float("inf")])
def test_load_points_rejects_off_grid(ctx, queues, bad):
    """kmeans_accumulate's int32/int64 fixed-point tables are exact only
    for multiples of 2^-12 inside [-8, 8); anything else is an argument error at
    load time on the device that holds the row (here the last part's rows)."""
    from paper_2005_08466_b200.kmeans import KMeans

    n, d, k = 4096, 32, 16
    pts = G.gen_kmeans_points(n, d, k, 42).reshape(n, d)
    pts[n - 3, 17] = bad
    km = KMeans(ctx, queues[:2], n, d, k)
    with pytest.raises(HaoclError) as e:
        km.load_points(pts)
    assert e.value.code == 9 and "2^-12" in str(e.value)
    pts[n - 3, 17] = -8.0  # the smallest grid value is accepted
    km.load_points(pts)
    km.close()


def test_accumulate_many_points_one_cluster(ctx, queues):
    """Block-local int32 sums are flushed before they can overflow: 5M copies of
    the largest grid point in one cluster (int64 sums far beyond 2^31)."""
    from paper_2005_08466_b200.kmeans import KMeans

    n, d, k = 5_000_000, 32, 2
    pts = np.full((n, d), 8.0 - 2.0**-12, np.float32)
    pts[::2, ::2] = -8.0
    cent = np.stack([np.full(d, 7.0, np.float32), np.full(d, -100.0, np.float32)])
    a = O.kmeans_assign(pts.reshape(-1), n, d, cent.reshape(-1), k)
    s_want, c_want = O.kmeans_accumulate(pts.reshape(-1), n, d, a, k)
    km = KMeans(ctx, queues[:1], n, d, k)
    km.load_points(pts)
    km.set_centroids(cent)
    km.iterate(1)
    s, c = km.sums()
    km.close()
    assert (c == c_want).all() and (s == s_want).all()
    assert c_want[0] == n and abs(int(s_want[1])) > 2**31


def test_full_size_c4_sampled_parity(ctx, queues):
    """SURVEY.md §8(d) C4 at full size: 2^28 points generated in HBM, K = 1024,
    initial centroids = the first K points, one full iteration, then the
    tensor-filtered assignment of 2^16 sampled points (64 seeded blocks of 1024)
    recomputed by the oracle against the GPU's centroids, bit-exactly."""
    from paper_2005_08466_b200.kmeans import KMeans

    n, d, k = 1 << 28, 32, 1024
    km = KMeans(ctx, queues[:1], n, d, k, tensor_filter=True)
    try:
        km.generate_points(42, k)
        km.set_centroids(G.gen_kmeans_points(k, d, k, 42))
        km.iterate(1)
        cent = km.centroids().reshape(-1)
        _, counts = km.sums()
        assert int(counts.sum()) == n
        km.assign_only()
        got = km.assignments()
    finally:
        km.close()
    rng = np.random.default_rng(7)
    sample, sample_got = [], []
    for off in rng.choice(n // 1024, 64, replace=False) * 1024:
        pts = G.gen_kmeans_points(1024, d, k, 42, first=int(off))
        want = O.kmeans_assign(pts, 1024, d, cent, k)
        assert (got[off:off + 1024] == want).all(), off
        sample.append(pts)
        sample_got.append(got[off:off + 1024])
    # the same 2^16 assignments from the REFERENCE LIBRARY's knn with k = 1
    # (fp64, diff = ref - query, ties to the smaller index; kernels.cpp:195-233)
    import os

    q = 1 << 16
    rc, work, out = O.ref_execute("knn", [("in", cent.astype(np.float64)), ("in", np.concatenate(sample).astype(np.float64)),
                                         ("s", k), ("s", q), ("s", d), ("s", 1), ("out", None), ("out", None)],
                                  {6: q * 4, 7: q * 8}, threads=os.cpu_count() or 1)
    assert rc == 0 and work == d * k * q
    assert (out[6].view(np.int32) == np.concatenate(sample_got)).all()


@pytest.mark.parametrize("P,tc", [(1, True), (2, True), (3, False)])
def test_order_by_cluster_keeps_every_result(ctx, queues, P, tc):
    """order_by_cluster stores the points grouped by nearest centroid (per
    part); assignments map back to the caller's order and every result --
    assignments, int64 sums, centroids -- stays bit-identical to the oracle."""
    from paper_2005_08466_b200.kmeans import KMeans

    n, d, k = 30011, 32, 256
    pts = G.gen_kmeans_points(n, d, k, 44)
    cent0 = pts[: k * d].copy()
    a_want, s_want, c_want, cent_want = oracle_iterations(pts, n, d, k, cent0, 3)
    km = KMeans(ctx, queues[:P], n, d, k, tensor_filter=tc)
    km.load_points(pts)
    km.set_centroids(cent0)
    km.iterate(1)
    km.order_by_cluster()
    assert sorted(km.perm.tolist()) == list(range(n))
    km.iterate(1)
    km.assign_only()
    got_a = km.assignments()
    km.iterate(1)
    s, c = km.sums()
    cent = km.centroids()
    km.close()
    assert (got_a == a_want).all()
    assert (s == s_want).all() and (c == c_want).all()
    assert cent.tobytes() == cent_want.reshape(k, d).tobytes()


@pytest.mark.parametrize("n,k,P", [(672 * 7 + 5, 1024, 1), (100003, 64, 3), (671, 5, 1), (1 << 20, 1024, 2)])
def test_accumulate_q16_equals_fp32_path(ctx, queues, n, k, P):
    """kmeans_quantize_points + kmeans_accumulate_q16 (the update's int16 fixed-point
    stream) give the same int64 sums and counts as kmeans_accumulate over the fp32
    points and as the oracle -- bulk chunks, ragged tails and partitioned launches."""
    pts = G.gen_kmeans_points(n, 32, max(k, 2), 7)
    cent = pts[: k * 32].copy()
    a = O.kmeans_assign(pts, n, 32, cent, k)
    s_want, c_want = O.kmeans_accumulate(pts, n, 32, a, k)
    qs = queues[:P]
    mk = ctx.create_buffer
    b_p, b_q, b_a, b_s, b_c = mk(n * 128), mk(n * 64), mk(n * 4), mk(k * 256), mk(k * 8)
    ctx.enqueue_write_buffer(qs[0], b_p, pts)
    ctx.enqueue_write_buffer(qs[0], b_a, a.astype(np.int32))
    prog = ctx.create_program("b200")
    kq = ctx.create_kernel(prog, "kmeans_quantize_points")
    for j, v in enumerate([b_p, b_q, n, 32]):
        ctx.set_kernel_arg(kq, j, v)
    ctx.enqueue_ndrange_partitioned(kq, (n, 1, 1), 1, qs)
    q16 = ctx.enqueue_read_buffer(qs[0], b_q).view(np.int16)
    assert (q16 == np.round(pts * 4096).astype(np.int16)).all()
    for name, src in (("kmeans_accumulate_q16", b_q), ("kmeans_accumulate", b_p)):
        kk = ctx.create_kernel(prog, name)
        for j, v in enumerate([src, b_a, b_s, b_c, n, 32, k]):
            ctx.set_kernel_arg(kk, j, v)
        ctx.enqueue_ndrange_partitioned(kk, (n, 1, 1), 1, qs)
        for q in qs:
            ctx.finish(q)
        s = ctx.enqueue_read_buffer(qs[0], b_s).view(np.int64)
        c = ctx.enqueue_read_buffer(qs[0], b_c).view(np.int64)
        assert (s == s_want).all() and (c == c_want).all(), name
        ctx.release(kk)
    for b in (b_p, b_q, b_a, b_s, b_c):
        ctx.release(b)
