"""One bf16 16384^3 gemm_bf16 launch after one warm-up (for ncu); knobs via HCL_GEMM_* env."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402

S = 16384
ctx = HostContext([0])
q = ctx.create_queue(0)
k = ctx.create_kernel(ctx.create_program("b200"), "gemm_bf16")
bufs = [ctx.create_buffer(S * S * 2) for _ in range(3)]
ctx.enqueue_write_buffer(q, bufs[0], G.gen_bf16(S * S, 42))
ctx.enqueue_write_buffer(q, bufs[1], G.gen_bf16(S * S, 43))
for i, v in enumerate([*bufs, S, S, S, 0]):
    ctx.set_kernel_arg(k, i, v)
for _ in range(2):
    ctx.enqueue_ndrange_kernel(q, k, (S, S, 1), 2)
f = ctx.finish(q)
print(f"2 launches: {f.compute_ms:.2f} ms")
