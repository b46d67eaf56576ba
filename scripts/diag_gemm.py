"""GPU diagnostic: tf32 variants at small size and bf16 16384^3 timing per variant."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import _native as N  # noqa: E402

ctx = HostContext([0])
q = ctx.create_queue(0)
prog = ctx.create_program("b200")


def run(kernel, a, b, m, k, n, out_f32=True, reps=1):
    kh = ctx.create_kernel(prog, kernel)
    es = 4 if out_f32 else 2
    ba, bb, bc = ctx.create_buffer(a.nbytes), ctx.create_buffer(b.nbytes), ctx.create_buffer(m * n * es)
    ctx.enqueue_write_buffer(q, ba, a)
    ctx.enqueue_write_buffer(q, bb, b)
    args = [ba, bb, bc, m, k, n] + ([int(out_f32)] if kernel == "gemm_bf16" else [])
    for i, v in enumerate(args):
        ctx.set_kernel_arg(kh, i, v)
    ctx.enqueue_ndrange_kernel(q, kh, (m, n, 1), 2)
    ctx.finish(q)
    times = []
    for _ in range(reps):
        ctx.enqueue_ndrange_kernel(q, kh, (m, n, 1), 2)
        f = ctx.finish(q)
        times.append(f.compute_ms)
    out = ctx.enqueue_read_buffer(q, bc, length=min(m * n * es, 1 << 20))
    for x in (ba, bb, bc):
        ctx.release(x)
    ctx.release(kh)
    return out, times


m = n = k = 256
a = O.gen_doubles(m * k, 42).astype(np.float32)
b = O.gen_doubles(k * n, 43).astype(np.float32)
ref = a.astype(np.float64).reshape(m, k) @ b.astype(np.float64).reshape(k, n)
for cg in ("1", "2"):
    for km in ("0", "1"):
        os.environ["HCL_GEMM_CG"] = cg
        os.environ["HCL_GEMM_B_KMAJOR"] = km
        out, _ = run("gemm_tf32", a, b, m, k, n)
        c = out.view(np.float32).reshape(m, n)
        print(f"tf32 cg={cg} kmajor={km}: max|c|={np.abs(c).max():.4g} maxerr={np.abs(c - ref).max():.4g} "
              f"c[0,:4]={c[0, :4]} ref={ref[0, :4]}", flush=True)

# bf16 16384^3 timing
S = int(os.environ.get("DIAG_S", "16384"))
t = time.time()
a = O.gen_bf16(S * S, 42)
b = O.gen_bf16(S * S, 43)
print(f"gen {time.time() - t:.1f}s", flush=True)
for cg, km, of in (("2", "0", False), ("2", "0", True), ("2", "1", False), ("1", "0", False)):
    os.environ["HCL_GEMM_CG"] = cg
    os.environ["HCL_GEMM_B_KMAJOR"] = km
    _, times = run("gemm_bf16", a, b, S, S, S, out_f32=of, reps=5)
    best = min(times)
    print(f"bf16 {S}^3 cg={cg} kmajor={km} out_f32={of}: ms={['%.3f' % x for x in times]} "
          f"best {2 * S**3 / best / 1e9:.1f} TFLOP/s", flush=True)
print("launches", N.lib().hcl_kernel_launch_count())
