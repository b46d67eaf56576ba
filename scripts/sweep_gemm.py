"""GPU sweep: bf16 GEMM tile-raster group size (HCL_GEMM_GROUP) under sustained
back-to-back launches, plus the fp32 C1 kernels. Prints one line per variant."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402

ctx = HostContext([0])
q = ctx.create_queue(0)
prog = ctx.create_program("b200")
S = int(os.environ.get("SWEEP_S", "16384"))
REPS = int(os.environ.get("SWEEP_REPS", "20"))
groups = [int(x) for x in os.environ.get("SWEEP_GROUPS", "4,8,16,32").split(",")]

a = torch.empty(S * S, dtype=torch.int16)
b = torch.empty(S * S, dtype=torch.int16)
G.gen_bf16(S * S, 42, out=a)
G.gen_bf16(S * S, 43, out=b)
kh = ctx.create_kernel(prog, "gemm_bf16")
bA, bB, bC = (ctx.create_buffer(S * S * 2) for _ in range(3))
ctx.enqueue_write_buffer(q, bA, a)
ctx.enqueue_write_buffer(q, bB, b)
for i, v in enumerate([bA, bB, bC, S, S, S, 0]):
    ctx.set_kernel_arg(kh, i, v)
ref = None
for g in groups:
    os.environ["HCL_GEMM_GROUP"] = str(g)
    for _ in range(3):
        ctx.enqueue_ndrange_kernel(q, kh, (S, S, 1), 2)
    ctx.finish(q)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(REPS):
        ctx.enqueue_ndrange_kernel(q, kh, (S, S, 1), 2)
    f = ctx.finish(q)
    dt = (time.perf_counter() - t) / REPS
    out = ctx.enqueue_read_buffer(q, bC, length=1 << 20)
    same = True if ref is None else bool(np.array_equal(out, ref))
    ref = out if ref is None else ref
    print(f"group={g}: {dt * 1e3:.3f} ms/launch wall = {2 * S**3 / dt / 1e12:.1f} TFLOP/s "
          f"(compute_ms sum {f.compute_ms:.1f}) identical={same}", flush=True)
os.environ["HCL_GEMM_GROUP"] = "8"

# C1: fp32 1024^3
n = 1024
af = np.random.default_rng(1).standard_normal(n * n).astype(np.float32)
bf = np.random.default_rng(2).standard_normal(n * n).astype(np.float32)
ref64 = af.astype(np.float64).reshape(n, n) @ bf.astype(np.float64).reshape(n, n)
scale = np.abs(af.astype(np.float64).reshape(n, n)) @ np.abs(bf.astype(np.float64).reshape(n, n))
for name in ("gemm_f32", "gemm_tf32"):
    k2 = ctx.create_kernel(prog, name)
    x, y, z = (ctx.create_buffer(n * n * 4) for _ in range(3))
    ctx.enqueue_write_buffer(q, x, af)
    ctx.enqueue_write_buffer(q, y, bf)
    for i, v in enumerate([x, y, z, n, n, n]):
        ctx.set_kernel_arg(k2, i, v)
    ctx.enqueue_ndrange_kernel(q, k2, (n, n, 1), 2)
    ctx.finish(q)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    for _ in range(200):
        ctx.enqueue_ndrange_kernel(q, k2, (n, n, 1), 2)
    f = ctx.finish(q)
    dt = (time.perf_counter() - t) / 200
    c = ctx.enqueue_read_buffer(q, z).view(np.float32).reshape(n, n)
    err = float((np.abs(c - ref64) / scale).max())
    print(f"{name} {n}^3: wall {dt * 1e6:.1f} us/launch = {2 * n**3 / dt / 1e12:.2f} TFLOP/s; "
          f"compute {f.compute_ms / 200 * 1e3:.1f} us = {2 * n**3 / (f.compute_ms / 200 * 1e-3) / 1e12:.2f} TFLOP/s; "
          f"normwise err {err:.3g}", flush=True)
