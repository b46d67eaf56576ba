"""Profiling driver: one k-means iteration + a tensor-filtered assignment of N
points (default 2^24) on GPU 0; a second argument 1 stores the points grouped
by cluster first (KMeans.order_by_cluster)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_2005_08466_b200 import HostContext
from paper_2005_08466_b200 import datagen as G
from paper_2005_08466_b200.kmeans import KMeans
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
order = len(sys.argv) > 2 and sys.argv[2] == "1"
ctx = HostContext([0]); q = ctx.create_queue(0)
km = KMeans(ctx, [q], n, 32, 1024, tensor_filter=True)
km.generate_points(42, 1024)
km.set_centroids(G.gen_kmeans_points(1024, 32, 1024, 42))
if order:
    km.order_by_cluster()
km.iterate(1)
km.assign_only(); km.finish()
t = time.perf_counter()
for _ in range(3):
    km.assign_only()
km.finish()
print("ok", "order" if order else "random", f"{(time.perf_counter() - t) / 3 * 1e3:.3f} ms per assign")
