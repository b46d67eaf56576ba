"""k-means tensor-filtered assignment for profiling: N points generated in HBM,
split, then 2 assign launches (second one is the profiled one)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402
from paper_2005_08466_b200.kmeans import KMeans  # noqa: E402

n, d, k = int(os.environ.get("KM_N", str(1 << 22))), 32, 1024
tc = os.environ.get("KM_TC", "1") == "1"
ctx = HostContext([0])
q = ctx.create_queue(0)
km = KMeans(ctx, [q], n, d, k, tensor_filter=tc)
km.generate_points(42, k)
km.set_centroids(G.gen_kmeans_points(k, d, k, 42))
km.assign_only()
ctx.finish(q)
km.assign_only()
f = ctx.finish(q)
print(f"assign ({'tc' if tc else 'simt'}) n={n}: {f.compute_ms:.3f} ms")
