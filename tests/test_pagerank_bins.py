"""Binned (propagation-blocking) PageRank step, config C3.

CPU: the host-built layout (hcl_pagerank_bins_build) holds exactly the part's
edges: decoding chunks + src_local + gtab + dst16 gives back the multiset of
(source, destination) pairs of the pull CSR rows [lo, hi); units tile every
bin, split bins share an accumulator slot.

GPU: 20 iterations of pagerank_step_binned are bit-identical to the oracle's
order-free fixed-point restatement (ho_spmv_f32_fixed: each product rounded to
2^-56, exact integer row sums), for P in {1, 2, 4} parts and for layouts small
enough that every bin splits into several units; at scale 20 within 1e-5
(normwise) of PageRank iterated on the reference library's spmv_compute; at
full C3 size (scale 24, 2^28 edges) bit-identical to the oracle."""
import numpy as np
import pytest

import oracle as O
from paper_2005_08466_b200 import datagen as G

SCALE = 13


@pytest.fixture(scope="module")
def graph():
    return G.pagerank_csr(SCALE, 16 << SCALE, 42)


def decode(L, v):
    """(dst * v + src) of every layout entry, sorted; also checks the geometry."""
    S, gs, B, W = L["n_chunks"], L["gstride"], L["n_bins"], L["bin_rows"]
    ch = L["chunks"][:8 * S].reshape(-1, 8)
    g = L["gtab"].reshape(S + 1, gs)
    src = np.full(L["n_entries"], -1, np.int64)
    for s in range(S):
        u0, span, soff, n, doff, nseg = (int(x) for x in ch[s][:6])
        assert 1 <= span <= L["span_max"] and 0 < n <= L["chunk_edges"] and soff % 8 == 0
        lens = g[s + 1, :B].astype(np.int64) - g[s, :B]
        assert (lens >= 0).all() and lens.sum() == n
        loc = np.concatenate([[0], np.cumsum(lens)])
        sl = L["src_local"][soff:soff + n].astype(np.int64)
        assert (sl < span).all()
        for j in np.nonzero(lens)[0]:
            src[g[s, j]:g[s, j] + lens[j]] = u0 + sl[loc[j]:loc[j + 1]]
        # the scatter descriptor sends entry f to delta[k] + f (k: its non-empty segment)
        nwin = (n + 31) // 32
        ww = (2 * nwin + 3) // 4 * 4
        dsc = L["cdesc"][doff:doff + ww + nseg]
        bits, kb, delta = dsc[0:2 * nwin:2], dsc[1:2 * nwin:2], dsc[ww:].view(np.int32)
        assert nseg == np.count_nonzero(lens) and doff % 4 == 0
        f = np.arange(n)
        k = kb[f // 32].astype(np.int64) + np.array([bin(int(bits[x // 32]) & ((2 << (x % 32)) - 1)).count("1")
                                                      for x in f]) - 1
        dest = delta[k] + f
        jj = np.repeat(np.nonzero(lens)[0], lens[lens > 0])
        want = g[s, jj].astype(np.int64) + (f - loc[jj])
        assert (dest == want).all()
    dst = np.full(L["n_entries"], -1, np.int64)
    for j in range(B):
        assert g[0, j] % 8 == 0
        o = L["dst16"][g[0, j]:g[S, j]].astype(np.int64)
        o = o ^ ((o >> 5) & 31) ^ ((o >> 10) & 31)  # stored bank-folded (an involution)
        dst[g[0, j]:g[S, j]] = L["lo"] + j * W + o
    m = src >= 0
    assert ((dst >= 0) == m).all() and (dst[m] < L["hi"]).all()
    # units tile each bin's padded range; split bins carry a slot with their unit count
    u = L["units"][:4 * L["n_units"]].reshape(-1, 4)
    for j in range(B):
        uj = u[u[:, 0] == j]
        uj = uj[np.argsort(uj[:, 1])]
        assert uj[0, 1] == g[0, j] and uj[-1, 2] == (int(g[S, j]) + 7) // 8 * 8
        assert (uj[1:, 1] == uj[:-1, 2]).all() and (uj[:, 1] % 8 == 0).all()
        if len(uj) > 1:
            assert (uj[:, 3] == uj[0, 3]).all() and L["slot_units"][uj[0, 3]] == len(uj)
        else:
            assert uj[0, 3] == -1
    return np.sort(dst[m] * v + src[m])


@pytest.mark.parametrize("lo,hi,opts", [(0, None, {}), (1000, 5000, dict(bin_rows=512, chunk_edges=1024,
                                                                         span_max=256, unit_edges=800)),
                                        (17, 8191, dict(bin_rows=64, chunk_edges=64, span_max=64, unit_edges=64))])
def test_layout_holds_exactly_the_parts_edges(graph, lo, hi, opts):
    rp, ci, val, deg = graph
    v = len(rp) - 1
    hi = v if hi is None else hi
    L = G.pagerank_bins(rp, ci, lo, hi, **opts)
    assert L["n_edges"] == rp[hi] - rp[lo]
    rows = np.repeat(np.arange(lo, hi), np.diff(rp[lo:hi + 1])).astype(np.int64)
    want = np.sort(rows * v + ci[rp[lo]:rp[hi]])
    assert (decode(L, v) == want).all()


def test_layout_rejects_bad_geometry(graph):
    from paper_2005_08466_b200 import HaoclError

    rp, ci, _, _ = graph
    with pytest.raises(HaoclError):
        G.pagerank_bins(rp, ci, 0, len(rp) - 1, bin_rows=1 << 17)  # dst16 offsets are uint16


# ---- GPU ----------------------------------------------------------------------

@pytest.fixture(scope="module")
def queues(ctx):
    qs = [ctx.create_queue(g) for g in ctx.get_device_ids()[:4]]
    yield qs
    for q in qs:
        ctx.release(q)


def run_binned(ctx, queues, graph, P, iters=20, opts=None):
    from paper_2005_08466_b200.pagerank import PageRank

    pr = PageRank(ctx, queues[:P], *graph, binned=True, bin_options=opts)
    pr.reset()
    pr.iterate(iters)
    x = pr.ranks()
    pr.close()
    return x


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("opts", [None, dict(bin_rows=256, chunk_edges=512, span_max=128, unit_edges=64)])
def test_binned_step_bitexact_vs_fixed_oracle(ctx, queues, graph, P, opts):
    rp, ci, val, deg = graph
    x = run_binned(ctx, queues, graph, P, 20, opts)
    want = O.pagerank(rp, ci, val, deg, 20, b200_order="fixed")
    assert x.tobytes() == want.tobytes()
    asc = O.pagerank(rp, ci, val, deg, 20).astype(np.float64)
    assert np.abs(x - asc).sum() / np.abs(asc).sum() <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 4])
def test_binned_vs_reference_spmv_scale20(ctx, queues, P):
    """20 binned iterations at R-MAT scale 20 against PageRank iterated on the
    REFERENCE LIBRARY's spmv_compute (fp64/int64; proj/src/kernels.cpp:132-152)."""
    rp, ci, val, deg = G.pagerank_csr(20, 1 << 24, 42)
    x = run_binned(ctx, queues, (rp, ci, val, deg), P).astype(np.float64)
    want = O.ref_pagerank(rp, ci, deg, 20)
    assert np.abs(x - want).sum() / np.abs(want).sum() <= 1e-5
    assert (np.abs(x - want) / want).max() <= 1e-4
    assert x.astype(np.float32).tobytes() == O.pagerank(rp, ci, val, deg, 20, b200_order="fixed").tobytes()


@pytest.mark.gpu
def test_binned_full_c3(ctx, queues):
    """SURVEY.md §8(d) C3 at full size (scale 24, 2^28 edges, seed 42): 20
    binned iterations bit-identical to the fixed-point oracle; mass sums to 1."""
    rp, ci, val, deg = G.pagerank_csr(24, 1 << 28, 42)
    x = run_binned(ctx, queues, (rp, ci, val, deg), 1)
    want = O.pagerank(rp, ci, val, deg, 20, b200_order="fixed")
    assert x.tobytes() == want.tobytes()
    assert abs(float(x.astype(np.float64).sum()) - 1.0) <= 1e-3
