"""PageRank scale-24 run for profiling: CSR build, then a few iterations."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402
from paper_2005_08466_b200.pagerank import PageRank  # noqa: E402

scale = int(os.environ.get("PR_SCALE", "24"))
iters = int(os.environ.get("PR_ITERS", "3"))
mx = int(os.environ.get("PR_MAXNNZ", "2048"))
ctx = HostContext([0])
q = ctx.create_queue(0)
g = G.pagerank_csr(scale, 16 << scale, 42)
pr = PageRank(ctx, [q], *g, max_nnz=mx)
pr.reset()
pr.iterate(iters)
pr.finish()
f = ctx.finish(q)
print(f"{iters} iterations: device {f.compute_ms:.3f} ms total", flush=True)
