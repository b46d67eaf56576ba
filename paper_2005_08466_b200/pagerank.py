"""PageRank over the partitioned NDRange (config C3).

The caller side of the path: the graph lives in HBM as an int32/fp32 pull
CSR plus the SpMV's warp work units; each iteration runs `pagerank_dangling`
(exact fixed-point dangling mass) and `pagerank_step` (warp-unit SpMV fused
with the PageRank update) as a partitioned NDRange over the queues, split at
nnz-balanced row boundaries (`spmv_partition_ranges`, the reference's
kernels.cpp:300-321 generalised to weights). The rank vector is the step's
SPLIT_ROWS output; the next iteration's REPLICATE input gathers it onto every
device (peer-to-peer inside one process; NCCL allgather across processes).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .datagen import pagerank_bins, pagerank_inv_outdeg, pagerank_relabel, pagerank_units
from .runtime import Handle, HostContext, spmv_partition_ranges

DEFAULT_WARP_NNZ = 64  # measured best at scale 24 (profiles/r01_pagerank_experiments.txt)


class PageRank:
    def __init__(self, ctx: HostContext, queues: Sequence[Handle], row_ptr: np.ndarray, col_idx: np.ndarray,
                 val: np.ndarray, outdeg: np.ndarray, max_nnz: int = DEFAULT_WARP_NNZ,
                 weights: Optional[Sequence[int]] = None, relabel: bool = False, implicit: bool = True,
                 fused: bool = False, binned: bool = False, bounds: Optional[Sequence[int]] = None,
                 bin_options: Optional[dict] = None):
        """relabel: store the graph degree-ordered (hcl_pagerank_relabel) so the
        hot ranks form a dense prefix of x; per-row sums are unchanged, and
        ranks()/spmv() map results back to the caller's vertex ids. implicit: the
        iteration uses pagerank_prep + pagerank_step_implicit (values folded into
        xs = x/outdeg, bit-identical products, no value stream)."""
        self.implicit = implicit
        # fused: one partitioned pagerank_step_exchange per iteration -- each part writes its
        # rows of x', the next gather input xs' into EVERY device's copy (EXCHANGE output,
        # NVLink stores through the runtime-filled PEERS list) and its dangling partial
        # (REDUCE_SUM); no prep pass and no copies of the rank vector between iterations
        self.fused = fused and implicit
        # binned: one partitioned pagerank_step_binned per iteration (propagation blocking:
        # a scatter pass streams each edge's value into its destination bin, a gather pass
        # accumulates each bin in shared memory -- no random gathers; order-free 2^-56
        # fixed-point row sums) with the same exchange epilogue as the fused step
        self.binned = binned
        if binned:
            self.fused = False
        self.ctx, self.queues = ctx, list(queues)
        self.perm = None
        if relabel:
            row_ptr, col_idx, val, outdeg, self.perm = pagerank_relabel(row_ptr, col_idx, val, outdeg)
        self.v = len(row_ptr) - 1
        self.nnz = int(row_ptr[-1])
        self.warp_nnz = max_nnz
        units, long_rows, n_long = pagerank_units(row_ptr, max_nnz)
        self.n_units, self.n_long = len(units), n_long
        rp64 = np.ascontiguousarray(row_ptr, np.int64)
        self.bounds = [int(b) for b in (bounds if bounds is not None else
                                        spmv_partition_ranges(rp64, len(self.queues), weights))]
        q0 = self.queues[0]
        mk = ctx.create_buffer
        self.b_rp, self.b_units, self.b_long = mk(row_ptr.nbytes), mk(units.nbytes), mk(long_rows.nbytes)
        self.b_col, self.b_val, self.b_deg = mk(col_idx.nbytes), mk(val.nbytes), mk(outdeg.nbytes)
        self.b_x = [mk(self.v * 4), mk(self.v * 4)]
        self.b_dsum = mk(8)
        for b, a in ((self.b_rp, row_ptr), (self.b_units, units), (self.b_long, long_rows), (self.b_col, col_idx),
                     (self.b_val, val), (self.b_deg, outdeg)):
            ctx.enqueue_write_buffer(q0, b, np.ascontiguousarray(a))
        prog = ctx.create_program("b200")
        self.k_dang = ctx.create_kernel(prog, "pagerank_dangling")
        self.k_step = [ctx.create_kernel(prog, "pagerank_step") for _ in range(2)]
        self.k_spmv = ctx.create_kernel(prog, "pagerank_spmv")
        self.tail = [self.v, 0, self.n_units, self.n_long, max_nnz]
        for i, kk in enumerate(self.k_step):  # step i reads x[i], writes x[1-i]
            for j, a in enumerate([self.b_rp, self.b_col, self.b_val, self.b_units, self.b_long, self.b_x[i],
                                   self.b_dsum, self.b_x[1 - i]] + self.tail):
                ctx.set_kernel_arg(kk, j, a)
        for j, a in enumerate([self.b_deg, self.b_dsum, self.v]):
            ctx.set_kernel_arg(self.k_dang, j + 1, a)
        if implicit:
            self.b_xs = mk(self.v * 4)
            self.k_prep = ctx.create_kernel(prog, "pagerank_prep")
            self.k_stepi = [ctx.create_kernel(prog, "pagerank_step_implicit") for _ in range(2)]
            for i, kk in enumerate(self.k_stepi):  # reads xs (from x[i]), writes x[1-i]
                for j, a in enumerate([self.b_rp, self.b_col, self.b_units, self.b_long, self.b_xs, self.b_dsum,
                                       self.b_x[1 - i]] + self.tail):
                    ctx.set_kernel_arg(kk, j, a)
            for j, a in enumerate([self.b_deg, self.b_dsum, self.b_xs, self.v]):
                ctx.set_kernel_arg(self.k_prep, j + 1, a)
        if self.fused:
            P = len(self.queues)
            self.b_xs2, self.b_dsum2 = [mk(self.v * 4), mk(self.v * 4)], [mk(8), mk(8)]
            self.b_inv = mk(self.v * 4)
            ctx.enqueue_write_buffer(q0, self.b_inv, pagerank_inv_outdeg(outdeg))
            self.b_peers = mk(8 * max(1, P - 1))
            self.k_prep0 = ctx.create_kernel(prog, "pagerank_prep")
            for j, a in enumerate([self.b_x[0], self.b_deg, self.b_dsum2[0], self.b_xs2[0], self.v]):
                ctx.set_kernel_arg(self.k_prep0, j, a)
            self.k_stepx = [ctx.create_kernel(prog, "pagerank_step_exchange") for _ in range(2)]
            for i, kk in enumerate(self.k_stepx):  # reads xs[i], dsum[i]; writes x rows, xs[1-i], dsum[1-i]
                for j, a in enumerate([self.b_rp, self.b_col, self.b_units, self.b_long, self.b_xs2[i],
                                       self.b_dsum2[i], self.b_x[0]] + self.tail +
                                      [self.b_peers, P - 1, self.b_inv, self.b_xs2[1 - i], self.b_dsum2[1 - i]]):
                    ctx.set_kernel_arg(kk, j, a)
        if self.binned:
            self._setup_binned(row_ptr, col_idx, outdeg, bin_options or {})
        self.cur = 0

    def _setup_binned(self, row_ptr, col_idx, outdeg, opts) -> None:
        ctx, q0, mk = self.ctx, self.queues[0], self.ctx.create_buffer
        self.bl = BinnedLayout(ctx, q0, row_ptr, col_idx, self.bounds, opts)
        n_parts = self.bl.n_parts
        self.b_xs2, self.b_dsum2 = [mk(self.v * 4), mk(self.v * 4)], [mk(8), mk(8)]
        self.b_inv = mk(self.v * 4)
        ctx.enqueue_write_buffer(q0, self.b_inv, pagerank_inv_outdeg(outdeg))
        self.b_peers = mk(8 * max(1, n_parts - 1))
        prog = ctx.create_program("b200")
        # the binned step's gather input is xs scaled by 2^56 (its fixed-point grid)
        self.k_prep0 = ctx.create_kernel(prog, "pagerank_prep_fixed")
        for j, a in enumerate([self.b_x[0], self.b_deg, self.b_dsum2[0], self.b_xs2[0], self.v]):
            ctx.set_kernel_arg(self.k_prep0, j, a)
        self.k_bin = [self.bl.kernel(self.v, self.b_xs2[i], self.b_dsum2[i], self.b_x[0], self.b_peers, n_parts - 1,
                                     self.b_inv, self.b_xs2[1 - i], self.b_dsum2[1 - i]) for i in range(2)]

    def reset(self) -> None:
        x0 = np.full(self.v, np.float32(1.0 / self.v), np.float32)
        self.ctx.enqueue_write_buffer(self.queues[0], self.b_x[0], x0)
        self.cur = 0
        if self.fused or self.binned:  # iteration 0's gather input and dangling sum
            self.ctx.enqueue_ndrange_kernel(self.queues[0], self.k_prep0)

    def iterate(self, iterations: int) -> None:
        ctx = self.ctx
        for _ in range(iterations):
            if self.binned:
                ctx.enqueue_ndrange_partitioned(self.k_bin[self.cur], (self.v, 1, 1), 1, self.queues,
                                                bounds=self.bounds)
                self.cur = 1 - self.cur
                continue
            if self.fused:
                ctx.enqueue_ndrange_partitioned(self.k_stepx[self.cur], (self.v, 1, 1), 1, self.queues,
                                                bounds=self.bounds)
                self.cur = 1 - self.cur
                continue
            if self.implicit:
                ctx.set_kernel_arg(self.k_prep, 0, self.b_x[self.cur])
                ctx.enqueue_ndrange_kernel(self.queues[0], self.k_prep)
                step = self.k_stepi[self.cur]
            else:
                ctx.set_kernel_arg(self.k_dang, 0, self.b_x[self.cur])
                ctx.enqueue_ndrange_kernel(self.queues[0], self.k_dang)
                step = self.k_step[self.cur]
            ctx.enqueue_ndrange_partitioned(step, (self.v, 1, 1), 1, self.queues, bounds=self.bounds)
            self.cur = 1 - self.cur

    def finish(self) -> None:
        for q in self.queues:
            self.ctx.finish(q)

    def ranks(self) -> np.ndarray:
        self.finish()
        bx = self.b_x[0] if (self.fused or self.binned) else self.b_x[self.cur]
        return self._to_caller(self.ctx.enqueue_read_buffer(self.queues[0], bx).view(np.float32))

    def _to_caller(self, r: np.ndarray) -> np.ndarray:
        if self.perm is None:
            return r
        out = np.empty_like(r)
        out[self.perm] = r
        return out

    def spmv(self, x: np.ndarray) -> np.ndarray:
        """One y = A x through the partitioned pagerank_spmv kernel."""
        ctx = self.ctx
        bx, by = ctx.create_buffer(self.v * 4), ctx.create_buffer(self.v * 4)
        x = np.ascontiguousarray(x, np.float32)
        ctx.enqueue_write_buffer(self.queues[0], bx, x if self.perm is None else x[self.perm])
        for j, a in enumerate([self.b_rp, self.b_col, self.b_val, self.b_units, self.b_long, bx, by] + self.tail):
            ctx.set_kernel_arg(self.k_spmv, j, a)
        ctx.enqueue_ndrange_partitioned(self.k_spmv, (self.v, 1, 1), 1, self.queues, bounds=self.bounds)
        self.finish()
        y = self._to_caller(ctx.enqueue_read_buffer(self.queues[0], by).view(np.float32).copy())
        ctx.release(bx)
        ctx.release(by)
        return y

    def close(self) -> None:
        for b in (self.b_rp, self.b_units, self.b_long, self.b_col, self.b_val, self.b_deg, self.b_dsum, *self.b_x):
            self.ctx.release(b)
        if self.implicit:
            self.ctx.release(self.b_xs)
        if self.fused or self.binned:
            for b in (*self.b_xs2, *self.b_dsum2, self.b_peers, self.b_inv):
                self.ctx.release(b)
        if self.binned:
            self.bl.close()


def part_bin_options(n_edges: int, sm_count: int = 148) -> dict:
    """Chunking of one part's layout: ~16 chunks per scatter CTA (two per SM), so the
    static chunk-to-CTA assignment stays balanced when a part holds a fraction of
    the edges (one rank of N). chunk_edges = the power of two nearest to
    n_edges / (32 * SMs), in [16384, 65536]; spans of up to 16384 sources (the
    largest with 65536-edge chunks in one shared-memory stage; longer spans mean
    fewer, fuller chunks). Measured at C3 (rank row ranges emulated on one GPU,
    scripts/pr_rank_split.py; slowest part): N=1 65536/16384 0.967 ms vs 65536/8192
    0.993 (12288: 0.980); N=2 32768/16384 0.51 vs 0.56 ms; N=4 16384/16384 0.32 vs
    0.38 ms; N=8 16384/16384 0.23 vs 0.28 ms."""
    import math

    raw = max(1.0, n_edges / (32.0 * sm_count))
    ce = int(min(65536, max(16384, 2 ** round(math.log2(raw)))))
    return dict(chunk_edges=ce, span_max=16384)


class BinnedLayout:
    """Device copy of the propagation-blocking layout (hcl_pagerank_bins_build)
    of every part [bounds[i], bounds[i+1]) with rows, concatenated into one
    buffer per array with a parts table; pagerank_step_binned finds its part by
    the row range of the launch. One part per process under torchrun (bench.py),
    several logical devices in one process (tests)."""

    ARRAYS = ("chunks", "src_local", "cdesc", "dst16", "units", "slot_units")

    def __init__(self, ctx: HostContext, q0: Handle, row_ptr, col_idx, bounds: Sequence[int], opts=None):
        self.ctx = ctx
        mk = ctx.create_buffer
        parts, arrays = [], {k: [] for k in self.ARRAYS}
        base = dict(chunk=0, src=0, desc=0, ent=0, unit=0, slot=0)
        self.layouts = []
        for i in range(len(bounds) - 1):
            lo, hi = int(bounds[i]), int(bounds[i + 1])
            if hi <= lo:
                continue
            L = pagerank_bins(row_ptr, col_idx, lo, hi,
                              **(opts if opts is not None else part_bin_options(int(row_ptr[hi]) - int(row_ptr[lo]))))
            self.layouts.append({k: v for k, v in L.items() if not isinstance(v, np.ndarray)})
            parts.append([lo, hi, base["chunk"], L["n_chunks"], L["n_bins"], L["gstride"], base["desc"], base["src"],
                          base["ent"], base["unit"], L["n_units"], base["slot"], L["n_slots"], L["bin_rows"],
                          L["span_max"], L["n_edges"], L["chunk_edges"], 0, 0, 0])
            arrays["chunks"].append(L["chunks"][:8 * L["n_chunks"]])
            arrays["src_local"].append(L["src_local"][:L["n_src"]])
            arrays["cdesc"].append(L["cdesc"][:L["n_desc"]])
            arrays["dst16"].append(L["dst16"][:L["n_entries"]])
            arrays["units"].append(L["units"][:4 * L["n_units"]])
            arrays["slot_units"].append(L["slot_units"][:L["n_slots"]])
            base["chunk"] += L["n_chunks"]
            base["src"] += L["n_src"]
            base["desc"] += L["n_desc"]
            base["ent"] += L["n_entries"]
            base["unit"] += L["n_units"]
            base["slot"] += L["n_slots"]
        self.n_parts = len(parts)
        self.n_edges = sum(L["n_edges"] for L in self.layouts)
        self.bin_rows = self.layouts[0]["bin_rows"]
        table = np.array(parts, np.int64).reshape(-1)
        cat = {k: np.concatenate(v) if sum(len(x) for x in v) else np.zeros(8, v[0].dtype)
               for k, v in arrays.items()}
        cat["dst16"] = np.concatenate([cat["dst16"], np.zeros(8, np.uint16)])  # >= 8 entries
        self.b_parts = mk(table.nbytes)
        ctx.enqueue_write_buffer(q0, self.b_parts, table)
        self.b = {}
        for k, a in cat.items():
            self.b[k] = mk(a.nbytes)
            ctx.enqueue_write_buffer(q0, self.b[k], np.ascontiguousarray(a))
        self.b_vals = mk(4 * len(cat["dst16"]))  # LOCAL: zero-filled per device (padding entries stay 0)
        self.b_slot_acc = mk(max(1, base["slot"]) * (self.bin_rows * 8 + 4))

    def kernel(self, v, xs, dsum, x_out, peers, n_peers, inv, xs_next, dsum_next) -> Handle:
        """A pagerank_step_binned kernel bound to this layout: reads xs, dsum;
        writes the part's rows of x_out, xs_next (here and through peers) and
        the dangling partial dsum_next."""
        ctx, B = self.ctx, self.b
        k = ctx.create_kernel(ctx.create_program("b200"), "pagerank_step_binned")
        for j, a in enumerate([self.b_parts, B["chunks"], B["src_local"], B["cdesc"], B["dst16"], B["units"],
                               B["slot_units"], xs, dsum, x_out, v, self.n_parts, peers, n_peers, inv, xs_next,
                               dsum_next, self.b_vals, self.b_slot_acc]):
            ctx.set_kernel_arg(k, j, a)
        return k

    def close(self) -> None:
        for b in (self.b_parts, *self.b.values(), self.b_vals, self.b_slot_acc):
            self.ctx.release(b)
