"""Profiling driver: one k-means iteration + a tensor-filtered assignment of N points (default 2^24) on GPU 0."""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2005_08466_b200 import HostContext
from paper_2005_08466_b200 import datagen as G
from paper_2005_08466_b200.kmeans import KMeans
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
ctx = HostContext([0]); q = ctx.create_queue(0)
km = KMeans(ctx, [q], n, 32, 1024, tensor_filter=True)
km.generate_points(42, 1024)
km.set_centroids(G.gen_kmeans_points(1024, 32, 1024, 42))
km.iterate(1)
km.assign_only(); km.finish()
print("ok")
