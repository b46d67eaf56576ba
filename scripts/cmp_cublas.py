"""Interleaved comparison at 16384^3 bf16: torch.matmul (cuBLAS) vs gemm_bf16, 20
back-to-back launches each, 3 rounds (same box, same thermal state)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402

S, REPS = 16384, 20
a = torch.randn(S, S, device="cuda", dtype=torch.bfloat16)
b = torch.randn(S, S, device="cuda", dtype=torch.bfloat16)
c = torch.empty(S, S, device="cuda", dtype=torch.bfloat16)
ctx = HostContext([0])
q = ctx.create_queue(0)
k = ctx.create_kernel(ctx.create_program("b200"), "gemm_bf16")
bufs = []
for t in (a, b, c):
    h = ctx.create_buffer(t.numel() * 2)
    bufs.append(h)
ctx.enqueue_write_buffer(q, bufs[0], a.view(torch.int16).cpu())
ctx.enqueue_write_buffer(q, bufs[1], b.view(torch.int16).cpu())
for i, v in enumerate([*bufs, S, S, S, 0]):
    ctx.set_kernel_arg(k, i, v)
for _ in range(3):
    torch.matmul(a, b, out=c)
    ctx.enqueue_ndrange_kernel(q, k, (S, S, 1), 2)
torch.cuda.synchronize()
ctx.finish(q)
def ours(persist, one=1, tmac=1):
    os.environ["HCL_GEMM_PERSIST"] = str(persist)
    os.environ["HCL_GEMM_ONE"] = str(one)
    os.environ["HCL_GEMM_TMAC"] = str(tmac)
    t = time.perf_counter()
    for _ in range(REPS):
        ctx.enqueue_ndrange_kernel(q, k, (S, S, 1), 2)
    ctx.finish(q)
    return (time.perf_counter() - t) / REPS


def cublas():
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(REPS):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / REPS


f = 2 * S**3
for rnd in range(int(os.environ.get("CMP_ROUNDS", "4"))):
    order = [("cuBLAS", cublas), ("2 pairs/SM + TMA C", lambda: ours(0, 1, 1)),
             ("2 pairs/SM, direct C", lambda: ours(0, 1, 0))]
    if rnd % 2:
        order.reverse()
    res = {name: fn() for name, fn in order}
    print(f"round {rnd}: " + "   ".join(f"{n} {f / v / 1e12:.1f} TF" for n, v in res.items()), flush=True)
