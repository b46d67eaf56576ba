"""GPU parity of the knn reference-set split: the NDRange
is the reference set, each part computes every query's top-k over its rows
with global indices, and the runtime folds the MERGE_TOPK outputs with the
device merge (the reference's run_knn + merge_topk, proj/src/bench.cpp:367-447,
proj/src/kernels.cpp:323-361). Results must equal the reference's golden
digests bit-for-bit for every partition, including parts with fewer than k
reference rows."""
import numpy as np
import pytest

import oracle as O
from paper_2005_08466_b200 import HaoclError

from .test_gpu_core import h, run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


def knn_refsplit(ctx, queues, rf, q, R, Q, D, K, P, weights=None):
    out = run(ctx, "knn_refsplit", [rf, q, R, Q, D, K, ("out", Q * K * 4), ("out", Q * K * 8)], [6, 7],
              queues[:P], global_rows=R, partitioned=P > 1, weights=weights, bundle="b200")
    return out[6].view(np.int32), out[7].view(np.float64)


@pytest.mark.parametrize("R,Q,D,K", [(200, 20, 8, 5), (10**5, 10**3, 16, 10)])
@pytest.mark.parametrize("P,weights", [(1, None), (2, None), (4, None), (4, [5, 1, 3, 2])])
def test_knn_refsplit_digest(ctx, queues, golden, R, Q, D, K, P, weights):
    rf = O.gen_doubles(R * D, 42)
    q = O.gen_doubles(Q * D, 43)
    idx, dist = knn_refsplit(ctx, queues, rf, q, R, Q, D, K, P, weights)
    assert h(O.fnv1a(dist, O.fnv1a(idx))) == golden["digests"][f"knn_{R}x{Q}x{D}k{K}"]


@pytest.mark.parametrize("weights", [[1, 1, 1, 100], [100, 1, 1, 1], [1, 30, 1, 1]])
def test_knn_refsplit_small_parts(ctx, queues, weights):
    """Parts with fewer reference rows than k pad their lists; the merge still
    returns the reference's top-k (ties to the smaller index)."""
    R, Q, D, K = 120, 33, 4, 7
    rf = O.gen_doubles(R * D, 7)
    rf[40 * D:41 * D] = rf[3 * D:4 * D]  # duplicate point: equal distances, tie rule decides
    q = O.gen_doubles(Q * D, 8)
    q[:D] = rf[3 * D:4 * D]
    ei, ed = O.knn(rf, q, R, Q, D, K)
    idx, dist = knn_refsplit(ctx, queues, rf, q, R, Q, D, K, 4, weights)
    assert idx.tolist() == ei.tolist() and dist.tobytes() == ed.tobytes()
    assert idx[0] == 3 and idx[1] == 40


def test_knn_refsplit_whole_equals_core(ctx, queues):
    R, Q, D, K = 3000, 64, 12, 9
    rf = O.gen_doubles(R * D, 1)
    q = O.gen_doubles(Q * D, 2)
    core = run(ctx, "knn", [rf, q, R, Q, D, K, ("out", Q * K * 4), ("out", Q * K * 8)], [6, 7], queues[:1])
    idx, dist = knn_refsplit(ctx, queues, rf, q, R, Q, D, K, 1)
    assert core[6].tobytes() == idx.tobytes() and core[7].tobytes() == dist.tobytes()


def merge_direct(ctx, queues, a, b, Q, k):
    """Launch the merge companion directly on lists a, b = (idx[Q*k], dist[Q*k])."""
    out = run(ctx, "knn_refsplit_merge",
              [np.zeros(k, np.float64), np.zeros(Q, np.float64), k, Q, 1, k, a[0], a[1], b[0], b[1]],
              [6, 7], queues[:1], bundle="b200")
    return out[6].view(np.int32), out[7].view(np.float64)


def test_merge_topk_golden(ctx, queues, golden):
    """The reference's merge_topk KAT (tests/golden/make_golden.py): two k=2
    partials merged to k=3; partials padded to k with (+inf, INT32_MAX)."""
    inf, big = np.inf, np.iinfo(np.int32).max
    a = (np.array([1, 4, big, 0, 2, big], np.int32), np.array([0.5, 1.0, inf, 0.25, 0.25, inf]))
    b = (np.array([7, 9, big, 5, 6, big], np.int32), np.array([0.5, 2.0, inf, 0.25, 3.0, inf]))
    idx, dist = merge_direct(ctx, queues, a, b, 2, 3)
    g = golden["merge_topk"]
    assert idx.tolist() == g["idx"] and dist.tolist() == g["dist"]


def test_merge_topk_unsorted_is_contract_error(ctx, queues, golden):
    a = (np.array([1, 4, 0, 2], np.int32), np.array([1.5, 1.0, 0.25, 0.25]))  # query 0 not sorted
    b = (np.array([7, 9, 5, 6], np.int32), np.array([0.5, 2.0, 0.25, 3.0]))
    with pytest.raises(HaoclError) as e:
        merge_direct(ctx, queues, a, b, 2, 2)
    assert e.value.name == "contract" and golden["merge_topk_unsorted_rc"] == e.value.code


def test_knn_refsplit_errors(ctx, queues):
    rf = O.gen_doubles(10 * 2, 1)
    q = O.gen_doubles(3 * 2, 2)
    with pytest.raises(HaoclError) as e:  # k > R
        knn_refsplit(ctx, queues, rf, q, 10, 3, 2, 11, 1)
    assert e.value.name == "argument"
    with pytest.raises(HaoclError) as e:  # two parts on one device cannot hold full-size partials
        run(ctx, "knn_refsplit", [rf, q, 10, 3, 2, 2, ("out", 3 * 2 * 4), ("out", 3 * 2 * 8)], [6, 7],
            [queues[0], queues[0]], global_rows=10, partitioned=True, bundle="b200")
    assert e.value.name == "argument"


@pytest.mark.parametrize("R,Q,D,K", [(5000, 40, 16, 100), (700, 9, 5, 700), (3000, 17, 8, 33)])
@pytest.mark.parametrize("P,weights", [(1, None), (4, [3, 1, 2, 5])])
def test_knn_large_k(ctx, queues, R, Q, D, K, P, weights):
    """k > 32 (a block-wide sorted top-k; up to 4096): both the query-split core
    knn and the reference-set split equal the reference's ref::knn."""
    rf = O.gen_doubles(R * D, 11)
    rf[7 * D:8 * D] = rf[2 * D:3 * D]  # a tie
    q = O.gen_doubles(Q * D, 12)
    ei, ed = O.knn(rf, q, R, Q, D, K)
    idx, dist = knn_refsplit(ctx, queues, rf, q, R, Q, D, K, P, weights)
    assert idx.tolist() == ei.tolist() and dist.tobytes() == ed.tobytes()
    core = run(ctx, "knn", [rf, q, R, Q, D, K, ("out", Q * K * 4), ("out", Q * K * 8)], [6, 7], queues[:P],
               global_rows=Q, partitioned=P > 1)
    assert core[6].view(np.int32).tolist() == ei.tolist() and core[7].tobytes() == ed.tobytes()
