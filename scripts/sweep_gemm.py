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
VARIANTS = [tuple(int(x) for x in v.split(":"))
            for v in os.environ.get("SWEEP_VARIANTS", "8:3,4:3,16:3,8:0,8:2").split(",")]  # group:promo
ROUNDS = int(os.environ.get("SWEEP_ROUNDS", "3"))

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
res = {v: [] for v in VARIANTS}
for rnd in range(ROUNDS):  # interleaved so thermal drift hits every variant alike
    for g, pr in VARIANTS:
        os.environ["HCL_GEMM_GROUP"] = str(g)
        os.environ["HCL_GEMM_PROMO"] = str(pr)
        ctx.enqueue_ndrange_kernel(q, kh, (S, S, 1), 2)
        ctx.finish(q)
        t = time.perf_counter()
        for _ in range(REPS):
            ctx.enqueue_ndrange_kernel(q, kh, (S, S, 1), 2)
        ctx.finish(q)
        dt = (time.perf_counter() - t) / REPS
        res[(g, pr)].append(2 * S**3 / dt / 1e12)
        out = ctx.enqueue_read_buffer(q, bC, length=1 << 20)
        assert ref is None or np.array_equal(out, ref), (g, pr)
        ref = out if ref is None else ref
for v, r in res.items():
    print(f"group={v[0]} promo={v[1]}: TFLOP/s per round {['%.1f' % x for x in r]} mean {np.mean(r):.1f}", flush=True)
os.environ["HCL_GEMM_GROUP"] = "8"
os.environ["HCL_GEMM_PROMO"] = "3"

# C1: fp32 1024^3
n = 1024
af = np.random.default_rng(1).standard_normal(n * n).astype(np.float32)
bf = np.random.default_rng(2).standard_normal(n * n).astype(np.float32)
ref64 = af.astype(np.float64).reshape(n, n) @ bf.astype(np.float64).reshape(n, n)
scale = np.abs(af.astype(np.float64).reshape(n, n)) @ np.abs(bf.astype(np.float64).reshape(n, n))
for name in ("gemm_f32", "gemm_tf32", "gemm_f32x3"):
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

# C2 fp32: 16384^3 (3xTF32 and 1xTF32), 2 guard rows
if os.environ.get("SWEEP_F32_BIG", "1") == "1":
    n = 16384
    af = torch.empty(n * n, dtype=torch.float32)
    bf = torch.empty(n * n, dtype=torch.float32)
    G.gen_f32(n * n, 42, out=af)
    G.gen_f32(n * n, 43, out=bf)
    b64 = bf.numpy().astype(np.float64).reshape(n, n)
    a64 = af.numpy()[: 2 * n].astype(np.float64).reshape(2, n)
    ref64, scale = a64 @ b64, np.abs(a64) @ np.abs(b64)
    for name in ("gemm_f32x3", "gemm_tf32", "gemm_f32"):
        k2 = ctx.create_kernel(prog, name)
        x, y, z = (ctx.create_buffer(n * n * 4) for _ in range(3))
        ctx.enqueue_write_buffer(q, x, af)
        ctx.enqueue_write_buffer(q, y, bf)
        for i, v in enumerate([x, y, z, n, n, n]):
            ctx.set_kernel_arg(k2, i, v)
        ctx.enqueue_ndrange_kernel(q, k2, (n, n, 1), 2)
        ctx.finish(q)
        reps = 5
        t = time.perf_counter()
        for _ in range(reps):
            ctx.enqueue_ndrange_kernel(q, k2, (n, n, 1), 2)
        ctx.finish(q)
        dt = (time.perf_counter() - t) / reps
        c = ctx.enqueue_read_buffer(q, z, length=2 * n * 4).view(np.float32).reshape(2, n)
        err = float((np.abs(c - ref64) / scale).max())
        print(f"{name} {n}^3: {dt * 1e3:.2f} ms = {2 * n**3 / dt / 1e12:.1f} TFLOP/s, 2-row normwise err {err:.3g}",
              flush=True)
        for h in (x, y, z, k2):
            ctx.release(h)
