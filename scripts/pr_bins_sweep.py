"""C3 PageRank binned step (scale 24) per layout option set (argv: dicts of bin options)."""
import ctypes, sys, time, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2005_08466_b200 import HostContext, _native as N
from paper_2005_08466_b200 import datagen as G
from paper_2005_08466_b200.pagerank import PageRank
sc = 24
rp, ci, val, deg = G.pagerank_csr(sc, 16 << sc, 42)
ctx = HostContext([0]); q = ctx.create_queue(0)
sp = ctypes.c_void_p(); N.check(N.lib().hcl_device_stream(0, ctypes.byref(sp)))
st = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
B = (16 << sc) * 8 + ((1 << sc) + 1) * 4 + (1 << sc) * 8
configs = [eval(a) for a in sys.argv[1:]] or [dict(bin_rows=16384, chunk_edges=65536), dict(bin_rows=8192, chunk_edges=65536),
                                              dict(bin_rows=8192, chunk_edges=32768)]
for opts in configs:
    pr = PageRank(ctx, [q], rp, ci, val, deg, binned=True, bin_options=opts)
    pr.reset(); pr.iterate(3); pr.finish()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); pr.iterate(20); e1.record(st); pr.finish()
    ms = e0.elapsed_time(e1) / 20
    print(f"{opts}: {ms:.4f} ms/iter -> {B / ms / 1e6:.1f} GB/s", flush=True)
    pr.close()
