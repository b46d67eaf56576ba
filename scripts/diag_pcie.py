"""PCIe H2D/D2H bandwidth through the runtime (blocking vs overlapped)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402

ctx = HostContext([0])
q = ctx.create_queue(0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
o = torch.empty(n // 2, dtype=torch.uint8, pin_memory=True)
b1, b2 = ctx.create_buffer(n), ctx.create_buffer(n // 2)
ctx.enqueue_write_buffer(q, b1, h)
ctx.enqueue_write_buffer(q, b2, o)
ctx.finish(q)
for name, fn in (("h2d 1GiB", lambda: ctx.enqueue_write_buffer(q, b1, h)),
                 ("d2h 0.5GiB", lambda: ctx.enqueue_read_buffer(q, b2, out=o)),
                 ("both async", lambda: (ctx.enqueue_write_buffer(q, b1, h, blocking=False),
                                         ctx.enqueue_read_buffer(q, b2, out=o, blocking=False)))):
    t = time.perf_counter()
    for _ in range(5):
        fn()
    ctx.finish(q)
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {dt * 1e3:.2f} ms", flush=True)
