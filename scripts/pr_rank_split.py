"""Per-part PageRank binned step times with the row ranges of an N-rank split emulated on one
GPU (argv: N, row cost, layout options): the data behind pagerank.part_bin_options."""
import ctypes, sys, time, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2005_08466_b200 import HostContext, spmv_partition_ranges, _native as N
from paper_2005_08466_b200 import datagen as G
from paper_2005_08466_b200.pagerank import BinnedLayout
sc = 24
W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rc = float(sys.argv[2]) if len(sys.argv) > 2 else 2.5
opts = eval(sys.argv[3]) if len(sys.argv) > 3 else None
rp, ci, val, deg = G.pagerank_csr(sc, 16 << sc, 42)
v = len(rp) - 1
cum = rp.astype(np.int64) + np.round(rc * W * np.arange(len(rp))).astype(np.int64)
bounds = [int(x) for x in spmv_partition_ranges(cum, W)]
ctx = HostContext([0]); q = ctx.create_queue(0)
sp = ctypes.c_void_p(); N.check(N.lib().hcl_device_stream(0, ctypes.byref(sp)))
st = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
mk = ctx.create_buffer
xs = mk(v * 4); xs2 = mk(v * 4); x = mk(v * 4); inv = mk(v * 4)
ctx.enqueue_write_buffer(q, xs, np.full(v, 1.0 / v, np.float32))
ctx.enqueue_write_buffer(q, inv, G.pagerank_inv_outdeg(deg))
ds = mk(8); ds2 = mk(8); peers = mk(8)
ctx.enqueue_write_buffer(q, ds, np.zeros(1, np.int64)); ctx.enqueue_write_buffer(q, peers, np.zeros(1, np.uint64))
for i in range(W):
    lo, hi = bounds[i], bounds[i + 1]
    bl = BinnedLayout(ctx, q, rp, ci, [lo, hi], opts)
    k = bl.kernel(v, xs, ds, x, peers, 0, inv, xs2, ds2)
    for _ in range(3): ctx.enqueue_ndrange_range(q, k, (v, 1, 1), 1, lo, hi - lo)
    ctx.finish(q)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20): ctx.enqueue_ndrange_range(q, k, (v, 1, 1), 1, lo, hi - lo)
    e1.record(st); ctx.finish(q)
    L = bl.layouts[0]
    print(f"part {i}: rows {hi-lo} nnz {int(rp[hi]-rp[lo])} chunks {L['n_chunks']} bins {L['n_bins']} units {L['n_units']} "
          f"slots {L['n_slots']} ent {L['n_entries']} desc {L['n_desc']} src {L['n_src']}: {e0.elapsed_time(e1)/20:.4f} ms", flush=True)
    ctx.release(k); bl.close()
