#!/usr/bin/env python
"""Benchmark of the B200 partitioned-NDRange hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...   (one process per GPU)

Workload (BASELINE.json configs[1]): C = A * B with A, B
16384 x 16384 bf16 (SplitMix64 seeds 42 / 43, U[-1,1) rounded to bf16), fp32
accumulation, bf16 C. The NDRange's 16384 rows are split row-block over the N
ranks (cumulative-floor split = the reference's block_range); each rank runs its
sub-range through HostContext.enqueue_ndrange_range on its GPU with B
replicated. A step is one partitioned launch over the whole 16384^3 problem, so
total work is fixed as N grows ("scaling": "strong").

value : total flop / max-over-ranks device time (CUDA events on the runtime's
        stream), inputs resident in HBM (1 GiB of inputs > 126 MB L2, no flush).
e2e   : the same metric through the public API with host buffers: per step each
        rank writes its A slice and B from pinned memory, launches, and reads its C
        slice back (wall clock, max over ranks).
--impl reference : the reference's own CPU matmul (haocl::kernels::execute,
        compiled from /root/reference into oracle/_ref) on the host cores, on a
        bounded row sample of the same GEMM, in the reference's fp64 encoding.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Per-kernel GFLOP/s or GB/s at 1/2/4/8 B200 (% roofline); scaling efficiency"
S = 16384
FLOP_STEP = 2.0 * S * S * S


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    p = {"hbm_gbs": 6535.1, "bf16_tflops": 1684.4, "bf16_tflops_sustained": 1420.9, "src": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        p.update({k: j[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in j})
        p["src"] = "measured"
    return p


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", ",".join(str(g) for g in gpus),
                                       "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference library itself)


def reference_sample(threads: int, rows: int, cols: int):
    """One bounded sample of the GEMM on the reference engine: rows x K=16384 of
    A times a 16384 x cols block of B through haocl::kernels::execute("matmul")
    (proj/src/kernels.cpp:96-119), fp64 as the reference encodes it."""
    import numpy as np

    import oracle as O

    a = O.ref_gen_doubles(rows * S, 42)
    b = O.ref_gen_doubles(S * cols, 43)
    args = [("in", a), ("in", b), ("out", None), ("s", rows), ("s", S), ("s", cols)]

    def step():
        t = time.perf_counter()
        rc, work, _ = O.ref_execute("matmul", args, {2: rows * cols * 8}, threads=threads)
        dt = time.perf_counter() - t
        assert rc == 0
        return work, dt

    return step, np.nan


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    rows = max(64, 2 * threads)
    cols = 512
    step, _ = reference_sample(threads, rows, cols)
    for _ in range(args.warmup):
        step()
    tot_w = tot_t = 0.0
    for _ in range(args.steps):
        w, dt = step()
        tot_w += w
        tot_t += dt
    gflops = tot_w / tot_t / 1e9
    sample = (f"haocl::kernels::execute('matmul') fp64 (reference encoding) on {rows} rows x K={S} x {cols} "
              f"cols of the {S}^3 GEMM per step, {threads} OpenMP threads, oracle/_ref built from /root/reference")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_t / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 seeds 42/43, U[-1,1))",
        "config": {"workload": f"gemm {S}x{S}x{S} row-block (C2), reference CPU engine on a row sample",
                   "sample": {"rows": rows, "k": S, "cols": cols}},
        "cpu_baseline": {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(gflops, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg():
    threads = os.cpu_count() or 1
    rows = max(64, 2 * threads)
    cols = 512
    step, _ = reference_sample(threads, rows, cols)
    step()  # warm
    tot_w = tot_t = 0.0
    while tot_t < 10.0 and tot_w < 2e13:
        w, dt = step()
        tot_w += w
        tot_t += dt
    return {"value": round(tot_w / tot_t / 1e9, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
            "sample": f"reference matmul fp64 via oracle/_ref, {rows}x{S}x{cols} per call, "
                      f"{tot_w / 1e9:.0f} GFLOP in {tot_t:.1f} s on {threads} threads"}


# ---------------------------------------------------------------------------
# B200 arm


def run_b200(args):
    import numpy as np
    import torch

    from paper_2005_08466_b200 import HostContext, split_ranges
    from paper_2005_08466_b200 import _native as N
    from paper_2005_08466_b200 import datagen as G

    rank, world, local = env_rank()
    if world != args.gpus:
        print(f"warning: WORLD_SIZE {world} != --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    ctx = HostContext([local])
    q = ctx.create_queue(0)
    bounds = split_ranges(S, [1] * world)  # == block_range (proj/src/bench.cpp:31-33)
    lo, hi = bounds[rank], bounds[rank + 1]
    rows = hi - lo

    # pinned host inputs from the product's counter-based SplitMix64 generator
    t0 = time.perf_counter()
    a_host = torch.empty(rows * S, dtype=torch.int16, pin_memory=True)
    b_host = torch.empty(S * S, dtype=torch.int16, pin_memory=True)
    c_host = torch.empty(rows * S, dtype=torch.int16, pin_memory=True)
    G.gen_bf16(rows * S, 42, first=lo * S, out=a_host)
    G.gen_bf16(S * S, 43, out=b_host)
    ctx.add_data_creation_ms((time.perf_counter() - t0) * 1e3)

    prog = ctx.create_program("b200")
    k = ctx.create_kernel(prog, "gemm_bf16")
    bA, bB, bC = ctx.create_buffer(S * S * 2), ctx.create_buffer(S * S * 2), ctx.create_buffer(S * S * 2)
    ctx.enqueue_write_buffer(q, bA, a_host, offset=lo * S * 2)
    ctx.enqueue_write_buffer(q, bB, b_host)
    for i, v in enumerate([bA, bB, bC, S, S, S, 0]):
        ctx.set_kernel_arg(k, i, v)
    glob = (S, S, 1)

    stream_ptr = __import__("ctypes").c_void_p()
    N.check(N.lib().hcl_device_stream(0, __import__("ctypes").byref(stream_ptr)))
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=torch.device("cuda", local))

    for _ in range(args.warmup):
        ctx.enqueue_ndrange_range(q, k, glob, 2, lo, rows)
    ctx.finish(q)

    # parity guard on two output rows (fp64 numpy of the same bf16 inputs)
    c2 = ctx.enqueue_read_buffer(q, bC, offset=lo * S * 2, length=2 * S * 2).view(np.uint16)
    a2 = (a_host[: 2 * S].numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64).reshape(2, S)
    bf = (b_host.numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32).reshape(S, S)
    ref = a2 @ bf.astype(np.float64)
    scale = np.abs(a2) @ np.abs(bf).astype(np.float64)
    got = (c2.astype(np.uint32) << 16).view(np.float32).astype(np.float64).reshape(2, S)
    check_err = float((np.abs(got - ref) / scale).max())
    del bf

    sampler = ClockSampler(list(range(world))) if rank == 0 else None
    barrier()
    launches0 = N.lib().hcl_kernel_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ctx.enqueue_ndrange_range(q, k, glob, 2, lo, rows)
    e1.record(stream)
    ctx.finish(q)
    barrier()
    launches = N.lib().hcl_kernel_launch_count() - launches0
    dev_ms = e0.elapsed_time(e1)
    ms_max = allmax(dev_ms)
    launches_total = int(allsum(launches))

    # end to end through the public API with host buffers
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.enqueue_write_buffer(q, bA, a_host, offset=lo * S * 2)
        ctx.enqueue_write_buffer(q, bB, b_host)
        ctx.enqueue_ndrange_range(q, k, glob, 2, lo, rows)
        ctx.enqueue_read_buffer(q, bC, offset=lo * S * 2, length=rows * S * 2, out=c_host)
    ctx.finish(q)
    e2e_ms = allmax((time.perf_counter() - t0) * 1e3)
    barrier()
    clocks = sampler.stop() if sampler else None

    if rank != 0:
        return 0
    pk = peaks()
    per_launch_ms = dev_ms / args.steps
    achieved = 2.0 * rows * S * S / (per_launch_ms / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "gemm_bf16_ncu.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    value = FLOP_STEP * args.steps / (ms_max / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (SplitMix64 seeds 42/43, U[-1,1) -> bf16; product datagen)",
        "config": {"workload": f"gemm_bf16 {S}x{S}x{S} (C2), NDRange rows split row-block over {world} rank(s), "
                               "B replicated, fp32 accumulate, bf16 C",
                   "rows_per_rank": rows, "kernel": "gemm_bf16 tcgen05 cta_group::2 256x256 tiles, TMA, TMEM",
                   "l2": "inputs 1 GiB > 126 MB L2; no flush", "parity_rows_normwise_err": check_err},
        "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": pk["bf16_tflops"],
                     "unit": "TFLOP/s", "frac": round(achieved / pk["bf16_tflops"], 4), "traffic": traffic,
                     "peak_src": f"MEASURED_PEAKS.json bf16_tflops (burst), {pk['src']}",
                     "per_launch_flop": 2.0 * rows * S * S, "per_launch_ms": round(per_launch_ms, 4)},
        "e2e": {"value": round(FLOP_STEP * args.steps / (e2e_ms / 1e3) / 1e9, 1), "unit": "GFLOP/s",
                "h2d_bytes_per_step": S * S * 2 + world * S * S * 2, "d2h_bytes_per_step": S * S * 2},
        "gpu_launches": launches_total,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_leg()
        except Exception as e:  # the baseline is reported, never the measured path
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
