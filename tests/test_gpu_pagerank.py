"""PageRank (config C3) parity. The graph format (product CSR builder) must be
bit-identical to the oracle's; the GPU SpMV is bit-identical to the fp32
oracle (ascending per-row order) for every row that fits a row block, long rows
are within 1e-6 relative; ranks after 20 iterations are bit-identical to the
oracle when no row is long, within 1e-5 (normwise) otherwise, and always
bit-identical across partitions P in {1, 2, 4} (nnz-balanced ranges)."""
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


def test_row_blocks_properties(graph):
    rp = graph[0]
    for mx in (1, 16, 300, 4096):
        b = G.csr_row_blocks(rp, mx)
        assert b[0] == 0 and b[-1] == len(rp) - 1 and (np.diff(b) >= 1).all()
        for s, e in zip(b[:-1], b[1:]):
            nnz = rp[e] - rp[s]
            assert nnz <= mx or e - s == 1


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
@pytest.mark.parametrize("max_nnz", [4096, 64])
def test_spmv_matches_oracle(ctx, queues, graph, max_nnz):
    rp, ci, val, deg = graph
    x = O.gen_doubles(len(rp) - 1, 7).astype(np.float32) + 1.5
    want = O.spmv_f32(rp, ci, val, x, 0, len(rp) - 1)
    pr = make_pr(ctx, queues, graph, 1, max_nnz)
    y = pr.spmv(x)
    pr.close()
    lens = np.diff(rp)
    short = lens <= max_nnz
    assert y[short].tobytes() == want[short].tobytes()
    if (~short).any():
        assert np.abs(y[~short] - want[~short]).max() <= 1e-6 * np.abs(want[~short]).max()


@pytest.mark.gpu
def test_pagerank_bitexact_when_rows_fit(ctx, queues, graph):
    rp, ci, val, deg = graph
    assert np.diff(rp).max() <= 4096
    want = O.pagerank(rp, ci, val, deg, 20)
    pr = make_pr(ctx, queues, graph, 1, 4096)
    pr.reset()
    pr.iterate(20)
    x = pr.ranks()
    pr.close()
    assert x.tobytes() == want.tobytes()


@pytest.mark.gpu
def test_pagerank_long_rows_within_tolerance(ctx, queues, graph):
    rp, ci, val, deg = graph
    want = O.pagerank(rp, ci, val, deg, 20).astype(np.float64)
    pr = make_pr(ctx, queues, graph, 1, 32)  # forces the long-row path on hubs
    pr.reset()
    pr.iterate(20)
    x = pr.ranks().astype(np.float64)
    pr.close()
    assert np.abs(x - want).sum() / np.abs(want).sum() <= 1e-5
    assert np.abs(x - want).max() / want.max() <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("max_nnz", [4096, 32])
def test_pagerank_partition_invariance(ctx, queues, graph, max_nnz):
    results = []
    for P in (1, 2, 4):
        pr = make_pr(ctx, queues, graph, P, max_nnz)
        pr.reset()
        pr.iterate(20)
        results.append(pr.ranks().tobytes())
        pr.close()
    assert results[0] == results[1] == results[2]
