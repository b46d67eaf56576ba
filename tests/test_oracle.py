"""Pins the restated C oracle (oracle/haocl_oracle.c) to the HaoCL reference.

Checks against (a) tests/golden/reference_golden.json, produced by running the
reference library itself (tests/golden/make_golden.py), whose digests equal the
ones measured in SURVEY.md §8(c); and (b) the reference library directly
(oracle/_ref) where it is present. CPU only.
"""
import numpy as np
import pytest

import oracle as O

SURVEY_DIGESTS = {  # SURVEY.md §8(c), seed 42
    "matmul_64": "d6f917956c5bc4e2",
    "matmul_512": "d8bef020b109c5a9",
    "matmul_1024": "d0ec14e919c46d81",
    "spmv_100x100@0.1": "99903ad9f4a5ea25",
    "spmv_10000x10000@0.001": "36e5a0ede9bca61b",
    "spmv_100000x100000@0.0001": "d6e3bb9d7f59669f",
    "knn_200x20x8k5": "2ea1d52869135348",
    "knn_100000x1000x16k10": "f62259867e3dbb84",
    "bfs_1000v10000e": "d39a771194e63225",
    "bfs_100000v1000000e": "407ffea9dabcce06",
    "vecadd_100000": "e8d252c595d3a818",
    "vecadd_10000000": "dd08432e75686f10",
}


def h(x):
    return "%016x" % x


def test_golden_file_matches_survey(golden):
    assert golden["digests"] == SURVEY_DIGESTS


@pytest.mark.parametrize("n", [64, 512, 1024])
def test_matmul_digest(n):
    a = O.gen_doubles(n * n, 42)
    b = O.gen_doubles(n * n, 43)
    assert h(O.fnv1a(O.matmul_f64(a, b, n, n, n))) == SURVEY_DIGESTS[f"matmul_{n}"]


@pytest.mark.parametrize("r,c,d", [(100, 100, 0.1), (10**4, 10**4, 1e-3), (10**5, 10**5, 1e-4)])
def test_spmv_digest(r, c, d):
    rp, ci, v = O.gen_csr(r, c, d, 42)
    x = O.gen_doubles(c, 43)
    assert h(O.fnv1a(O.spmv_f64(rp, ci, v, x, 0, r))) == SURVEY_DIGESTS[f"spmv_{r}x{c}@{d}"]


@pytest.mark.parametrize("R,Q,D,K", [(200, 20, 8, 5), (10**5, 10**3, 16, 10)])
def test_knn_digest(R, Q, D, K):
    rf = O.gen_doubles(R * D, 42)
    q = O.gen_doubles(Q * D, 43)
    i, d = O.knn(rf, q, R, Q, D, K)
    assert h(O.fnv1a(d, O.fnv1a(i))) == SURVEY_DIGESTS[f"knn_{R}x{Q}x{D}k{K}"]


@pytest.mark.parametrize("V,E", [(1000, 10**4), (10**5, 10**6)])
def test_bfs_digest(V, E):
    rp, ci = O.gen_graph(V, E, 42)
    assert h(O.fnv1a(O.bfs(rp, ci, 0))) == SURVEY_DIGESTS[f"bfs_{V}v{E}e"]


@pytest.mark.parametrize("n", [10**5, 10**7])
def test_vecadd_digest(n):
    a = O.gen_doubles(n, 42)
    b = O.gen_doubles(n, 43)
    assert h(O.fnv1a(O.vecadd(a, b))) == SURVEY_DIGESTS[f"vecadd_{n}"]


def test_spmv_partition_matches_reference(golden):
    for key, case in golden["spmv_partition"].items():
        if key.startswith("gen_csr"):
            dims = key[len("gen_csr_"):].split("_P")[0]
            rc_, rest = dims.split("x")
            c_, d_ = rest.split("@")
            rp, _, _ = O.gen_csr(int(rc_), int(c_), float(d_), 42)
        else:
            rp = np.array(case["row_ptr"], np.int64)
        P = int(key.rsplit("_P", 1)[1])
        if case["rc"] != 0:
            with pytest.raises(ValueError):
                O.spmv_partition_ranges(rp, P)
        else:
            assert O.spmv_partition_ranges(rp, P).tolist() == case["ranges"], key


def test_spmv_partition_kats():
    # SPEC.md:490-492
    rp = np.arange(0, 17, 2, dtype=np.int64)
    assert O.spmv_partition_ranges(rp, 1).tolist() == [0, 8]
    assert O.spmv_partition_ranges(rp, 4).tolist() == [0, 2, 4, 6, 8]


def test_weighted_partition_reduces_to_reference():
    rng = np.random.default_rng(3)
    for _ in range(50):
        rows = int(rng.integers(2, 200))
        rp = np.concatenate([[0], np.cumsum(rng.integers(0, 30, rows) ** 2)]).astype(np.int64)
        P = int(rng.integers(1, min(rows, 9) + 1))
        assert (O.spmv_partition_ranges(rp, P, [5] * P) == O.spmv_partition_ranges(rp, P)).all()
        tot = int(rng.integers(0, 10**6))
        want = [tot * i // P for i in range(P + 1)]
        assert O.weighted_ranges(tot, [3] * P).tolist() == want  # block_range, bench.cpp:31-33


def test_knn_kat_and_merge(golden):
    k = golden["knn_kat"]
    i, d = O.knn(np.array(k["ref"]), np.array(k["query"]), 5, 2, 2, k["k"])
    assert i.tolist() == k["idx"] and d.tolist() == k["dist"]
    p1 = (2, np.array([1, 4, 0, 2], np.int32), np.array([0.5, 1.0, 0.25, 0.25]))
    p2 = (2, np.array([7, 9, 5, 6], np.int32), np.array([0.5, 2.0, 0.25, 3.0]))
    rc, mi, md = O.merge_topk([p1, p2], 2, 3)
    assert rc == golden["merge_topk"]["rc"]
    assert mi.tolist() == golden["merge_topk"]["idx"] and md.tolist() == golden["merge_topk"]["dist"]
    bad = (2, np.array([1, 4, 0, 2], np.int32), np.array([1.5, 1.0, 0.25, 0.25]))
    assert O.merge_topk([bad], 2, 2)[0] == golden["merge_topk_unsorted_rc"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_restatement_equals_reference_library_random():
    rng = np.random.default_rng(11)
    for _ in range(5):
        m, k, n = (int(x) for x in rng.integers(1, 40, 3))
        a = rng.standard_normal(m * k)
        b = rng.standard_normal(k * n)
        assert O.matmul_f64(a, b, m, k, n).tobytes() == O.ref_matmul(a, b, m, k, n).tobytes()
    for seed in (1, 2, 3):
        rp, ci, v = O.gen_csr(300, 200, 0.05, seed)
        rp2, ci2, v2 = O.ref_gen_csr(300, 200, 0.05, seed)
        assert (rp == rp2).all() and (ci == ci2).all() and v.tobytes() == v2.tobytes()
        rp, ci = O.gen_graph(500, 3000, seed)
        rp2, ci2 = O.ref_gen_graph(500, 3000, seed)
        assert (rp == rp2).all() and (ci == ci2).all()
        assert (O.bfs(rp, ci, 7) == O.ref_bfs(rp, ci, 7)).all()
    rf = rng.integers(0, 4, 300 * 3).astype(np.float64)  # many exact ties
    q = rng.integers(0, 4, 40 * 3).astype(np.float64)
    i1, d1 = O.knn(rf, q, 300, 40, 3, 7)
    i2, d2 = O.ref_knn(rf, q, 300, 40, 3, 7)
    assert (i1 == i2).all() and (d1 == d2).all()


def test_rmat_and_pagerank_restatement_properties():
    s, d = O.rmat_edges(10, 0, 5000, 42)
    s2, d2 = O.rmat_edges(10, 1000, 100, 42)  # counter based: any sub-range
    assert (s[1000:1100] == s2).all() and (d[1000:1100] == d2).all()
    assert s.max() < 1024 and d.max() < 1024
    rp, ci, val, outdeg = O.pagerank_csr(10, 16 * 1024, 42)
    assert rp[0] == 0 and rp[-1] == 16 * 1024 and (np.diff(rp) >= 0).all()
    for r in range(1024):  # columns sorted within each row
        assert (np.diff(ci[rp[r]:rp[r + 1]]) >= 0).all()
    x = O.pagerank(rp, ci, val, outdeg, 20)
    assert abs(float(x.astype(np.float64).sum()) - 1.0) < 1e-3
    # fp64 dense power iteration agrees to fp32 tolerance
    V = 1024
    A = np.zeros((V, V))
    for r in range(V):
        for p in range(rp[r], rp[r + 1]):
            A[r, ci[p]] += val[p]
    xd = np.full(V, 1.0 / V)
    dang = outdeg == 0
    for _ in range(20):
        xd = 0.15 / V + 0.85 * (A @ xd + xd[dang].sum() / V)
    assert np.abs(x - xd).max() / xd.max() < 1e-5


def test_kmeans_restatement_properties():
    pts = O.kmeans_points(42, 0, 2000, 8, 16)
    assert (np.abs(pts) <= 8).all()
    assert (pts * 4096 == np.round(pts * 4096)).all()  # multiples of 2^-12
    part = O.kmeans_points(42, 500, 10, 8, 16)
    assert (part == pts[500 * 8:510 * 8]).all()
    cent = pts[: 16 * 8].copy()
    a = O.kmeans_assign(pts, 2000, 8, cent, 16)
    # assignment = argmin of fp64 distance except for fp32 near-ties
    dd = ((pts.reshape(-1, 1, 8).astype(np.float64) - cent.reshape(1, -1, 8)) ** 2).sum(-1)
    assert (a == dd.argmin(1)).mean() > 0.999
    s, c = O.kmeans_accumulate(pts, 2000, 8, a, 16)
    assert c.sum() == 2000
    # accumulation is order free: permuted points give identical sums
    perm = np.random.default_rng(0).permutation(2000)
    s2, c2 = O.kmeans_accumulate(pts.reshape(-1, 8)[perm].ravel().copy(), 2000, 8, a[perm].copy(), 16)
    assert (s == s2).all() and (c == c2).all()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_pagerank_restatement_vs_reference_spmv():
    """The restated fp32 PageRank (both summation orders) stays within the
    SURVEY.md §8(c) tolerance of PageRank iterated on the reference library's
    own spmv_compute in fp64/int64: normwise (L1) <= 1e-5 after 20 iterations."""
    sc = 14
    rp, ci, val, deg = O.pagerank_csr(sc, 16 << sc, 42)
    want = O.ref_pagerank(rp, ci, deg, 20)
    for order in (False, True):
        got = O.pagerank(rp, ci, val, deg, 20, b200_order=order).astype(np.float64)
        assert np.abs(got - want).sum() / np.abs(want).sum() <= 1e-5
        assert (np.abs(got - want) / want).max() <= 1e-4
