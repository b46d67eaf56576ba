"""World-size-2 and -8 `gloo` tests (CPU) of the multi-rank host logic: every
rank derives the same partition plan independently, the per-rank sub-ranges
tile the global NDRange exactly (GEMM row blocks, nnz-balanced and cost-model
PageRank rows), each rank's propagation-blocking layout covers exactly its
rows' edges, rank-local counter-based data generation concatenates to the
single-process stream, and the exchange helpers of bench.py (NCCL-id
broadcast, max/min/sum) agree on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import torch
    import torch.distributed as dist

    import bench
    from paper_2005_08466_b200 import datagen as G
    from paper_2005_08466_b200 import spmv_partition_ranges, split_ranges

    d = bench.Dist("gloo")
    try:
        out = {}
        # GEMM rows: block_range split (bench.cpp:31-33)
        b = split_ranges(16384, [1] * world)
        out["gemm"] = (b[rank], b[rank + 1])
        # PageRank rows: nnz-balanced split of the same graph on every rank
        rp, ci, val, deg = G.pagerank_csr(12, 16 * 4096, 42)
        r = spmv_partition_ranges(rp.astype(np.int64), world)
        out["pr"] = (int(r[rank]), int(r[rank + 1]), int(rp[r[rank]]), int(rp[r[rank + 1]]))
        # the bench's binned split (cost model nnz + 2.5 N per row) and this rank's layout
        cum = rp.astype(np.int64) + np.round(2.5 * world * np.arange(len(rp))).astype(np.int64)
        rb = [int(x) for x in spmv_partition_ranges(cum, world)]
        from paper_2005_08466_b200.pagerank import part_bin_options

        lo_r, hi_r = rb[rank], rb[rank + 1]
        L = G.pagerank_bins(rp, ci, lo_r, hi_r, **part_bin_options(int(rp[hi_r]) - int(rp[lo_r])))
        out["bins"] = (lo_r, hi_r, int(L["n_edges"]), int(rp[hi_r]) - int(rp[lo_r]))
        # rank-local slices of the counter-based streams
        lo, hi = b[rank] // 64, b[rank + 1] // 64
        out["bf16"] = G.gen_bf16((hi - lo) * 256, 42, first=lo * 256).tobytes()
        # exchange helpers
        out["uid"] = d.bcast_bytes(bytes(range(rank, rank + 128)) if rank == 0 else None)
        out["max"] = d.allmax(float(rank + 1))
        out["min"] = d.allmin(float(rank + 1))
        out["sum"] = d.allsum(float(rank + 1))
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            q.put(gathered)
    finally:
        d.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 8])
def test_rank_plans_and_data_agree(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # GEMM row blocks tile [0, 16384)
    assert res[0]["gemm"][0] == 0 and res[-1]["gemm"][1] == 16384
    assert all(res[i]["gemm"][1] == res[i + 1]["gemm"][0] for i in range(world - 1))
    # PageRank ranges tile rows and non-zeros
    from paper_2005_08466_b200 import datagen as G

    rp = G.pagerank_csr(12, 16 * 4096, 42)[0]
    assert res[0]["pr"][0] == 0 and res[-1]["pr"][1] == len(rp) - 1
    assert res[0]["pr"][2] == 0 and res[-1]["pr"][3] == rp[-1]
    assert all(res[i]["pr"][1] == res[i + 1]["pr"][0] for i in range(world - 1))
    # the binned split tiles the rows and each rank's layout holds exactly its rows' edges
    assert res[0]["bins"][0] == 0 and res[-1]["bins"][1] == len(rp) - 1
    assert all(res[i]["bins"][1] == res[i + 1]["bins"][0] for i in range(world - 1))
    assert all(r["bins"][2] == r["bins"][3] for r in res) and sum(r["bins"][2] for r in res) == rp[-1]
    # rank slices of the bf16 stream concatenate to the full stream
    full = G.gen_bf16(16384 // 64 * 256, 42).tobytes()
    assert b"".join(r["bf16"] for r in res) == full
    assert all(r["uid"] == bytes(range(0, 128)) for r in res)
    assert all(r["max"] == world and r["min"] == 1.0 and r["sum"] == world * (world + 1) / 2 for r in res)
