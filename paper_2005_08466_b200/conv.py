"""3x3 conv layer over the partitioned NDRange (config C5).

The NDRange is the batch: `conv3x3` runs as a partitioned launch over images
(SPLIT_ROWS input and output, REPLICATE weights), with weights from the
scheduler's measured rates or explicit ones (the heterogeneity-aware uneven
split sweep). With C == 64 the layer runs straight from plain NHWC
(`conv3x3_nhwc`: each tile's input halo is one TMA box whose out-of-image
part TMA zero-fills -- the padding is never materialised); other channel
counts (or padded=True) pad on the device first (`conv_pad_nhwc` + `conv3x3`).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .runtime import Handle, HostContext


class Conv3x3:
    def __init__(self, ctx: HostContext, queues: Sequence[Handle], n: int, h: int, w: int, c: int, k: int,
                 out_f32: bool = False, padded: Optional[bool] = None):
        self.ctx, self.queues = ctx, list(queues)
        self.n, self.h, self.w, self.c, self.k, self.out_f32 = n, h, w, c, k, out_f32
        self.padded = (c != 64) if padded is None else padded
        self.es_out = 4 if out_f32 else 2
        mk = ctx.create_buffer
        self.b_in = mk(n * h * w * c * 2)
        self.b_pad = mk(n * (h + 2) * (w + 2) * c * 2) if self.padded else None
        self.b_w = mk(k * 9 * c * 2)
        self.b_out = mk(n * h * w * k * self.es_out)
        prog = ctx.create_program("b200")
        self.k_conv = ctx.create_kernel(prog, "conv3x3" if self.padded else "conv3x3_nhwc")
        if self.padded:
            self.k_pad = ctx.create_kernel(prog, "conv_pad_nhwc")
            for j, a in enumerate([self.b_in, self.b_pad, n, h, w, c]):
                ctx.set_kernel_arg(self.k_pad, j, a)
        for j, a in enumerate([self.b_pad if self.padded else self.b_in, self.b_w, self.b_out, n, h, w, c, k,
                               int(out_f32)]):
            ctx.set_kernel_arg(self.k_conv, j, a)

    def plan(self, weights: Optional[Sequence[int]] = None):
        return self.ctx.partition_plan(self.k_conv, (self.n, 1, 1), self.queues, weights)

    def load(self, x_nhwc_bf16: np.ndarray, w_krsc_bf16: np.ndarray, weights: Optional[Sequence[int]] = None):
        """Scatter each queue's images (plain NHWC bf16 bits) to its device (padded
        there when the layer runs the padded kernel)."""
        flat = np.ascontiguousarray(x_nhwc_bf16).reshape(-1)
        img = self.h * self.w * self.c
        bounds = self.plan(weights)
        for i, q in enumerate(self.queues):
            lo, hi = bounds[i], bounds[i + 1]
            if hi > lo:
                self.ctx.enqueue_write_buffer(q, self.b_in, flat[lo * img:hi * img], offset=lo * img * 2)
        self.ctx.enqueue_write_buffer(self.queues[0], self.b_w, np.ascontiguousarray(w_krsc_bf16))
        if self.padded:
            self.ctx.enqueue_ndrange_partitioned(self.k_pad, (self.n, 1, 1), 1, self.queues, bounds=bounds)
        self.bounds = bounds

    def run(self, weights: Optional[Sequence[int]] = None) -> None:
        self.ctx.enqueue_ndrange_partitioned(self.k_conv, (self.n, 1, 1), 1, self.queues, weights,
                                             bounds=None if weights is not None else self.bounds)

    def finish(self) -> None:
        for q in self.queues:
            self.ctx.finish(q)

    def output(self) -> np.ndarray:
        self.finish()
        raw = self.ctx.enqueue_read_buffer(self.queues[0], self.b_out)
        if self.out_f32:
            return raw.view(np.float32).reshape(self.n, self.h, self.w, self.k)
        return ((raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32)).reshape(self.n, self.h, self.w, self.k)

    def close(self) -> None:
        for b in (self.b_in, self.b_pad, self.b_w, self.b_out):
            if b is not None:
                self.ctx.release(b)
