"""conv3x3 C5 run for profiling (2 launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402
from paper_2005_08466_b200.conv import Conv3x3  # noqa: E402

N = int(os.environ.get("CONV_N", "256"))
ctx = HostContext([0])
q = ctx.create_queue(0)
cv = Conv3x3(ctx, [q], N, 224, 224, 64, 128)
cv.load(G.gen_bf16(N * 224 * 224 * 64, 42), G.gen_bf16(128 * 9 * 64, 43))
cv.run()
cv.run()
f = ctx.finish(q)
print(f"conv device ms (pad + 2 conv): {f.compute_ms:.3f}")
