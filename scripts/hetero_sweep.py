"""Heterogeneity-aware split on emulated heterogeneous devices (SURVEY.md §8(e)
C5 row, §8(f) 2): two logical devices on one B200 with different SM budgets
(hcl_device_set_sm_budget) run the C5 conv batch concurrently. Compares the
even split (the reference's block_range), the model split (SM-budget ratio),
the split from the runtime's EMA-profiled rates (weights=None ->
Scheduler::partition_weights) and a sweep of ratios. Makespan = wall time of
REPS partitioned launches with both queues drained, per launch."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_08466_b200 import HostContext  # noqa: E402
from paper_2005_08466_b200 import datagen as G  # noqa: E402
from paper_2005_08466_b200.conv import Conv3x3  # noqa: E402

N, H, W, C, K = (int(os.environ.get("HETERO_N", "256")), 224, 224, 64, 128)
SMS = [int(s) for s in os.environ.get("HETERO_SMS", "100,48").split(",")]
REPS = int(os.environ.get("HETERO_REPS", "10"))

ctx = HostContext([0] * len(SMS))
gids = ctx.get_device_ids()
for g, s in zip(gids, SMS):
    ctx.set_sm_budget(g, s)
queues = [ctx.create_queue(g) for g in gids]
conv = Conv3x3(ctx, queues, N, H, W, C, K)
x = G.gen_bf16(N * H * W * C, 42)
w = G.gen_bf16(K * 9 * C, 43)
conv.load(x, w, weights=[1] * len(SMS))
conv.finish()
flop = 2.0 * N * H * W * K * 9 * C


def sample():
    conv.finish()
    img = H * W * K * 2
    return b"".join(ctx.enqueue_read_buffer(queues[0], conv.b_out, offset=i * img, length=img).tobytes()
                    for i in (0, N // 2, N - 1))


def launch(weights):
    if weights is None:  # the runtime's own choice: Scheduler::partition_weights of the profiled rates
        ctx.enqueue_ndrange_partitioned(conv.k_conv, (N, 1, 1), 1, queues)
    else:
        conv.run(weights)


def timed(weights):
    launch(weights)  # warm: moves the SPLIT_ROWS pieces to the new split
    conv.finish()
    t = time.perf_counter()
    for _ in range(REPS):
        launch(weights)
    conv.finish()
    return (time.perf_counter() - t) / REPS * 1e3


rows = []
for label, wts in [("even (block_range)", [1] * len(SMS)), ("even", [1] * len(SMS))]:
    ms = timed(wts)
    rows.append((label, wts, ctx.partition_plan(conv.k_conv, (N, 1, 1), queues, wts), ms))
out_even = sample()
KNAME = "conv3x3" if conv.padded else "conv3x3_nhwc"  # the profiled kernel's registry name
ema_w = ctx.partition_weights(KNAME, gids)  # rates profiled by the runs above
for label, wts in [("model (SM budgets)", SMS), ("EMA-profiled rates", None)]:
    plan_w = wts if wts is not None else ctx.partition_weights(KNAME, gids)
    ms = timed(wts)
    rows.append((label, plan_w, ctx.partition_plan(conv.k_conv, (N, 1, 1), queues, plan_w), ms))
same = sample() == out_even
if len(SMS) == 2:
    for share in (0.5, 0.55, 0.6, 0.65, 0.7, 0.75, 0.8):
        wts = [int(share * 1000), 1000 - int(share * 1000)]
        ms = timed(wts)
        rows.append((f"sweep {share:.2f}", wts, ctx.partition_plan(conv.k_conv, (N, 1, 1), queues, wts), ms))
print(f"conv 3x3 ({KNAME}) {N}x{H}x{W}x{C}->{K} bf16 over {len(SMS)} logical devices on one B200, SM budgets {SMS}")
for label, wts, bounds, ms in rows[1:]:
    counts = [bounds[i + 1] - bounds[i] for i in range(len(bounds) - 1)]
    print(f"  {label:22s} images {counts}: {ms:7.3f} ms/launch = {flop / ms / 1e9:7.1f} TFLOP/s")
print("outputs identical across splits:", same)
best = min(rows[1:], key=lambda r: r[3])
print(json.dumps({"sm_budgets": SMS, "even_ms": rows[1][3], "ema_ms": rows[3][3], "model_ms": rows[2][3],
                  "best_sweep": best[0], "best_ms": best[3], "ema_weights": ema_w,
                  "ema_speedup_vs_even": rows[1][3] / rows[3][3]}))
