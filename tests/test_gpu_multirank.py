"""The N > 1 data plane of bench.py, one process per GPU over NCCL (the way
the driver launches `torchrun ... bench.py --gpus N`), checked against the
oracle. Skipped on a single-GPU box; run by `gpurun --gpus 2|4`.

* PageRank, binned step (default) and the pull fused step: rows split over the
  ranks, each rank's gather epilogue stores the next gather input into every
  rank's xs' -- one NVSwitch multicast store per row into symmetric memory
  (binned, default) or a store per peer into its IPC-mapped xs' (binned_ipc,
  pull) -- and an 8-byte NCCL allreduce of the dangling sums per step. 20 iterations, the ranks' rows gathered: bit-identical to the
  oracle's restatement (fixed-point order for binned, warp-unit order for pull).
* k-means: points split over the ranks, int64 NCCL allreduce of sums and
  counts; centroids after 2 iterations bit-identical to the oracle.
* GEMM: B enters as 1/N K-row slices per rank + the NCCL allgather (the e2e
  path, the rank's rows in chunks whose C streams back while later chunks
  compute); B complete and bit-identical on every rank, C rows within
  tolerance and identical on the host."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import sys

    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    try:
        import argparse

        import bench

        dist = bench.Dist("nccl")
        dist.torch.cuda.set_device(rank)
        args = argparse.Namespace(steps=3, warmup=3, workload=case)
        res = _CASES[case](bench, dist, args)
        out = dist.allgather_bytes(res)
        if rank == 0:
            q.put(("ok", out))
        dist.close()
    except Exception as e:  # reported to the parent, which fails the test
        import traceback

        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}\n{traceback.format_exc()}"))


def _pagerank(bench, dist, args, kernel, mcast="1"):
    os.environ["BENCH_PR_SCALE"] = "14"
    os.environ["BENCH_PR_KERNEL"] = kernel
    os.environ["BENCH_PR_MCAST"] = mcast
    wl = bench.PageRankW(args, dist)
    wl.setup()
    wl.reset()
    for _ in range(20):
        wl.step()
    wl.ctx.finish(wl.q)
    dist.barrier()
    x = wl.ctx.enqueue_read_buffer(wl.q, wl.b_x[0], offset=wl.lo * 4, length=wl.rows * 4).view(np.float32)
    return np.int64(wl.lo).tobytes() + x.tobytes()


def _kmeans(bench, dist, args):
    os.environ["BENCH_KM_N"] = str(1 << 16)
    wl = bench.KMeansW(args, dist)
    wl.setup()
    wl.step()
    wl.step()
    wl.ctx.finish(wl.q)
    return wl.ctx.enqueue_read_buffer(wl.q, wl.km.b_cent).tobytes()


def _gemm(bench, dist, args):
    class Small(bench.GemmBf16):
        S = 2048

    wl = Small(args, dist)
    wl.setup()
    wl.e2e_step()  # set 0: A rows + this rank's B slice from host, NCCL allgather of B, the GEMM
    wl.ctx.finish(wl.q)
    bB, chunks = wl.sets[0]  # B, then the rank's row chunks (kernel, A, C, rows)
    S = wl.S
    b = wl.ctx.enqueue_read_buffer(wl.q, bB).view(np.uint16)
    ok_b = b.tobytes() == wl.b_host.numpy().view(np.uint16).tobytes()
    c = np.concatenate([wl.ctx.enqueue_read_buffer(wl.q, bC).view(np.uint16) for _, _, bC, _ in chunks])
    ok_host = c.tobytes() == wl.c_hosts[0].numpy().view(np.uint16).tobytes()  # the e2e D2H landed
    assert ok_host, "e2e C rows on the host differ from the device's"
    return np.int64(wl.lo).tobytes() + np.int64(int(ok_b)).tobytes() + c.tobytes()


_CASES = {
    "pagerank_binned": lambda b, d, a: _pagerank(b, d, a, "binned"),
    "pagerank_binned_ipc": lambda b, d, a: _pagerank(b, d, a, "binned", mcast="0"),
    "pagerank_pull": lambda b, d, a: _pagerank(b, d, a, "pull"),
    "kmeans": _kmeans,
    "gemm": _gemm,
}


def _run(case):
    import torch
    import torch.multiprocessing as mp

    world = min(torch.cuda.device_count(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        status, payload = q.get(timeout=600)
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():  # a rank stuck in a collective after another rank failed
                p.kill()
    assert status == "ok", payload
    return world, payload


@pytest.mark.parametrize("kernel", ["binned", "binned_ipc", "pull"])
def test_pagerank_exchange_multirank(kernel):
    import oracle as O
    from paper_2005_08466_b200 import datagen as G

    world, parts = _run(f"pagerank_{kernel}")
    rp, ci, val, deg = G.pagerank_csr(14, 16 << 14, 42)
    x = np.empty(len(rp) - 1, np.float32)
    for p in parts:
        lo = int(np.frombuffer(p[:8], np.int64)[0])
        rows = np.frombuffer(p[8:], np.float32)
        x[lo:lo + len(rows)] = rows
    want = O.pagerank(rp, ci, val, deg, 20, b200_order="fixed" if kernel.startswith("binned") else True)
    assert x.tobytes() == want.tobytes(), f"{world} ranks"


def test_kmeans_allreduce_multirank():
    import oracle as O
    from paper_2005_08466_b200 import datagen as G

    world, parts = _run("kmeans")
    n, d, k = 1 << 16, 32, 1024
    pts = G.gen_kmeans_points(n, d, k, 42)
    cent = G.gen_kmeans_points(k, d, k, 42)
    for _ in range(2):
        a = O.kmeans_assign(pts, n, d, cent, k)
        s, c = O.kmeans_accumulate(pts, n, d, a, k)
        cent = O.kmeans_finalize(s, c, k, d, cent)
    for p in parts:  # every rank holds the same centroids
        assert p == cent.astype(np.float32).tobytes()


def test_gemm_b_allgather_multirank():
    import oracle as O

    world, parts = _run("gemm")
    S = 2048
    a = O.bf16_to_f32(O.gen_bf16(S * S, 42)).reshape(S, S).astype(np.float64)
    b = O.bf16_to_f32(O.gen_bf16(S * S, 43)).reshape(S, S).astype(np.float64)
    rows_seen = 0
    for p in parts:
        lo = int(np.frombuffer(p[:8], np.int64)[0])
        assert np.frombuffer(p[8:16], np.int64)[0] == 1, "B incomplete after the allgather"
        c = O.bf16_to_f32(np.frombuffer(p[16:], np.uint16)).reshape(-1, S).astype(np.float64)
        sel = np.arange(0, c.shape[0], 97)
        ref = a[lo + sel] @ b
        scale = np.abs(a[lo + sel]) @ np.abs(b)
        assert (np.abs(c[sel] - ref) <= 2.0**-10 * (1 + 2.0**-8) * scale + 2.0**-8 * np.abs(ref)).all()
        rows_seen += c.shape[0]
    assert rows_seen == S
