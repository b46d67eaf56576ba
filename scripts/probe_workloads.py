"""GPU probe: PageRank (scale 24) and k-means timing through the runtime."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402
from paper_2005_08466_b200.kmeans import KMeans  # noqa: E402
from paper_2005_08466_b200.pagerank import PageRank  # noqa: E402

ctx = HostContext([0])
q = ctx.create_queue(0)

scale = int(os.environ.get("PR_SCALE", "24"))
t = time.time()
g = G.pagerank_csr(scale, 16 << scale, 42)
print(f"csr build {time.time() - t:.1f}s maxrow {np.diff(g[0]).max()} dangling {(g[3] == 0).sum()}", flush=True)
for mx in (512, 1024, 2048):
    pr = PageRank(ctx, [q], *g, max_nnz=mx)
    pr.reset()
    pr.iterate(3)
    pr.finish()
    f = ctx.finish(q)
    t0 = time.time()
    pr.iterate(20)
    pr.finish()
    wall = time.time() - t0
    f = ctx.finish(q)
    v, e = 1 << scale, 16 << scale
    algo = e * 8 + (v + 1) * 4 + v * 4 + v * 4
    print(f"pagerank scale {scale} max_nnz {mx}: wall {wall * 1e3 / 20:.3f} ms/iter; "
          f"{algo / (wall / 20) / 1e9:.0f} GB/s algorithmic", flush=True)
    pr.close()

n = int(os.environ.get("KM_N", str(1 << 26)))
d, k = 32, 1024
t = time.time()
pts = G.gen_kmeans_points(n, d, k, 42)
print(f"kmeans gen {time.time() - t:.1f}s", flush=True)
km = KMeans(ctx, [q], n, d, k)
km.load_points(pts)
km.set_centroids(pts[: k * d])
km.iterate(1)
km.finish()
ctx.finish(q)
t0 = time.time()
km.assign_only()
km.finish()
ta = time.time() - t0
t0 = time.time()
km.iterate(2)
km.finish()
ti = (time.time() - t0) / 2
flop = 3.0 * n * k * d
print(f"kmeans n={n}: assign {ta * 1e3:.1f} ms = {flop / ta / 1e12:.1f} Tflop/s (3 flop/term); "
      f"iteration {ti * 1e3:.1f} ms", flush=True)
