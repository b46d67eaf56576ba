"""PageRank scale-24 run for timing/profiling: CSR build, then iterations; prints
device time per iteration (CUDA events of the runtime) per warp_nnz."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402
from paper_2005_08466_b200.pagerank import PageRank  # noqa: E402

scale = int(os.environ.get("PR_SCALE", "24"))
iters = int(os.environ.get("PR_ITERS", "10"))
mxs = [int(m) for m in os.environ.get("PR_MAXNNZ", "256,512,1024").split(",")]
ctx = HostContext([0])
q = ctx.create_queue(0)
g = G.pagerank_csr(scale, 16 << scale, 42)
v, e = 1 << scale, 16 << scale
algo = e * 8 + (v + 1) * 4 + v * 4 + v * 4
for mx in mxs:
    pr = PageRank(ctx, [q], *g, max_nnz=mx)
    pr.reset()
    pr.iterate(2)
    ctx.finish(q)
    t0 = time.time()
    pr.iterate(iters)
    f = ctx.finish(q)
    wall = (time.time() - t0) / iters
    dev = f.compute_ms / iters
    print(f"warp_nnz {mx}: device {dev:.3f} ms/iter ({algo / dev / 1e6:.0f} GB/s algorithmic), wall {wall * 1e3:.3f} ms",
          flush=True)
    pr.close()
