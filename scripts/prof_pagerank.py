"""PageRank scale-24 run for timing/profiling: CSR build (optionally degree-
ordered), then iterations; prints device time per iteration (CUDA events of
the runtime) per variant. PR_VARIANTS = "relabel:warp_nnz:threads:hot,..."
(hot -1 = all the shared memory left after the product staging)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402
from paper_2005_08466_b200.pagerank import PageRank  # noqa: E402

scale = int(os.environ.get("PR_SCALE", "24"))
iters = int(os.environ.get("PR_ITERS", "10"))
variants = [tuple(int(x) for x in v.split(":")) for v in
            os.environ.get("PR_VARIANTS", "0:512:256:0,1:512:256:0,1:512:1024:-1,1:256:1024:-1,1:512:256:8192").split(",")]
ctx = HostContext([0])
q = ctx.create_queue(0)
g = G.pagerank_csr(scale, 16 << scale, 42)
v, e = 1 << scale, 16 << scale
algo = e * 8 + (v + 1) * 4 + v * 4 + v * 4
ref = None
for rl, mx, nt, hot in variants:
    os.environ["HCL_PR_NT"] = str(nt)
    os.environ["HCL_PR_HOT"] = str(hot)
    pr = PageRank(ctx, [q], *g, max_nnz=mx, relabel=bool(rl))
    pr.reset()
    pr.iterate(2)
    ctx.finish(q)
    t0 = time.time()
    pr.iterate(iters)
    f = ctx.finish(q)
    wall = (time.time() - t0) / iters
    dev = f.compute_ms / iters
    r = pr.ranks()
    same = True if ref is None else bool(np.array_equal(r, ref))
    ref = r if ref is None else ref
    print(f"relabel {rl} warp_nnz {mx} threads {nt} hot {hot}: device {dev:.3f} ms/iter "
          f"({algo / dev / 1e6:.0f} GB/s algorithmic), wall {wall * 1e3:.3f} ms, ranks identical {same}", flush=True)
    pr.close()
