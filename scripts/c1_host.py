"""Host-side cost per C1 launch (fp32 GEMM 1024^3 through the host API): time N enqueues
without synchronising, then the device time of the same N launches."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_2005_08466_b200 import HostContext
from paper_2005_08466_b200 import _native as N

kern = os.environ.get("K", "gemm_f32x3")
S = 1024
ctx = HostContext([0]); q = ctx.create_queue(0)
a = O.gen_doubles(S * S, 42).astype(np.float32); b = O.gen_doubles(S * S, 43).astype(np.float32)
ba, bb, bc = ctx.create_buffer(a.nbytes), ctx.create_buffer(b.nbytes), ctx.create_buffer(S * S * 4)
ctx.enqueue_write_buffer(q, ba, a); ctx.enqueue_write_buffer(q, bb, b)
k = ctx.create_kernel(ctx.create_program("b200"), kern)
for i, v in enumerate([ba, bb, bc, S, S, S]): ctx.set_kernel_arg(k, i, v)
for _ in range(20): ctx.enqueue_ndrange_kernel(q, k, (S, S, 1), 2)
ctx.finish(q)
n = 200
t0 = time.perf_counter()
for _ in range(n): ctx.enqueue_ndrange_kernel(q, k, (S, S, 1), 2)
t1 = time.perf_counter()
f = ctx.finish(q)
t2 = time.perf_counter()
print(f"{kern}: host enqueue {1e6 * (t1 - t0) / n:.1f} us/launch; wall incl. drain {1e6 * (t2 - t0) / n:.1f} us/launch; device compute {1e3 * f.compute_ms / n:.1f} us/launch")
