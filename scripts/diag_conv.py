"""GPU diagnostic: conv3x3 variants (HCL_CONV_MODE 0/1/2) correctness + timing."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200.conv import Conv3x3  # noqa: E402
from tests.test_gpu_conv import ref_conv  # noqa: E402

ctx = HostContext([0])
q = ctx.create_queue(0)
n, h, w, c, k = 2, 12, 30, 64, 128
xb = O.gen_bf16(n * h * w * c, 42).reshape(n, h, w, c)
wb = O.gen_bf16(k * 9 * c, 43).reshape(k, 3, 3, c)
ref, scale = ref_conv(O.bf16_to_f32(xb).astype(np.float64), O.bf16_to_f32(wb).astype(np.float64))
for mode in ("1", "2"):
    os.environ["HCL_CONV_MODE"] = mode
    cv = Conv3x3(ctx, [q], n, h, w, c, k, out_f32=True)
    cv.load(xb, wb)
    cv.run()
    got = cv.output()
    cv.close()
    print(f"mode {mode}: normwise err {(np.abs(got - ref) / scale).max():.3g}", flush=True)

N = 256
from paper_2005_08466_b200 import datagen as G  # noqa: E402
x = G.gen_bf16(N * 224 * 224 * 64, 42)
wt = G.gen_bf16(128 * 9 * 64, 43)
for mode in ("1", "2"):
    os.environ["HCL_CONV_MODE"] = mode
    cv = Conv3x3(ctx, [q], N, 224, 224, 64, 128)
    cv.load(x, wt)
    cv.run()
    ctx.finish(q)
    for _ in range(5):
        cv.run()
    f = ctx.finish(q)
    ms = f.compute_ms / 5
    print(f"mode {mode}: {ms:.3f} ms = {2 * N * 224 * 224 * 128 * 9 * 64 / ms / 1e9:.0f} TFLOP/s", flush=True)
    cv.close()
