#!/usr/bin/env python
"""Benchmark of the B200 partitioned-NDRange hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload W]
    torchrun --nproc-per-node N ... bench.py --gpus N ...   (one process per GPU)

Default workload (BASELINE.json configs[1]): C = A * B, A and
B 16384 x 16384 bf16 (SplitMix64 seeds 42/43, U[-1,1) -> bf16), fp32 accumulate,
bf16 C. The NDRange rows are split row-block over the N ranks (cumulative floor
= the reference's block_range); each rank runs its sub-range through
HostContext.enqueue_ndrange_range, B replicated. One step = the whole 16384^3
product, so total work is fixed as N grows ("scaling": "strong").

Other workloads (same JSON contract, not run by the driver): gemm_f32 (C1,
1024^3 fp32 through the host API on one device), pagerank (C3, R-MAT scale 24,
rank allgather per iteration), kmeans (C4, 2^28 x 32, K=1024, sums allreduce per
iteration), conv (C5, 256 x 224^2 x 64 -> 128, batch split).

value : work / max-over-ranks device time (CUDA events on the runtime's stream),
        inputs resident in HBM (inputs larger than L2; no flush).
e2e   : the same metric through the public API with pinned host buffers (host ->
        device copies of the step's inputs and device -> host of its result inside
        the timed region), wall clock, max over ranks.
--impl reference : the reference's own CPU implementation (oracle/_ref, compiled
        from /root/reference) on a bounded sample of the workload, all host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Per-kernel GFLOP/s or GB/s at 1/2/4/8 B200 (% roofline); scaling efficiency"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    p = {"hbm_gbs": 6535.1, "bf16_tflops": 1684.4, "bf16_tflops_sustained": 1420.9, "src": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        p.update({k: j[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained", "sm_max_mhz") if k in j})
        p["src"] = "measured"
    return p


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region.

    A reader thread timestamps each 100 ms sample on arrival; the constructor
    returns once sampling is live, and stop() keeps the samples from mark()
    on. Timed regions shorter than a few samples are followed by a hold loop
    of the same steps (run_b200), whose samples are reported with it."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        import threading

        self.lines, self.t_mark, self.t_end = [], 0.0, float("inf")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", ",".join(str(g) for g in gpus),
                                       "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
            return

        def reader():
            for line in self.p.stdout:
                self.lines.append((time.time(), line))

        self.t = threading.Thread(target=reader, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.lines and time.time() - t0 < 3.0 and self.p.poll() is None:
            time.sleep(0.01)

    def mark(self):
        self.t_mark = time.time()

    def end(self):
        self.t_end = time.time()

    def count(self):
        return sum(1 for t, _ in self.lines if t >= self.t_mark)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=10)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.t.join(timeout=5)
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, line in self.lines:
            if t < self.t_mark or t > self.t_end + 0.15:  # one sample period of slack
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [x for x, pw in zip(sm, power) if pw > 300] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


class Dist:
    def __init__(self, backend: str | None):
        import torch

        self.rank, self.world, self.local = env_rank()
        self.torch = torch
        self.d = None
        if self.world > 1 and backend:
            import torch.distributed as d

            import datetime

            # a rank that diverges should fail the run in minutes, not hold every GPU for NCCL's default 10
            timeout = datetime.timedelta(seconds=int(os.environ.get("BENCH_PG_TIMEOUT_S", "240")))
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                d.init_process_group("nccl", device_id=torch.device("cuda", self.local), timeout=timeout)
            else:
                d.init_process_group("gloo", timeout=timeout)
            self.d = d
        self.dev = "cuda" if backend == "nccl" else "cpu"

    def barrier(self):
        if self.d is not None:
            self.d.barrier()
        if self.dev == "cuda":
            self.torch.cuda.synchronize()

    def _red(self, x, op):
        if self.d is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.d.all_reduce(t, op=op)
        return float(t.item())

    def allmax(self, x):
        return self._red(x, self.d.ReduceOp.MAX if self.d else None)

    def allmin(self, x):
        return self._red(x, self.d.ReduceOp.MIN if self.d else None)

    def allsum(self, x):
        return self._red(x, self.d.ReduceOp.SUM if self.d else None)

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if self.d is None:
            return b
        obj = [b]
        self.d.broadcast_object_list(obj, src=0)
        return obj[0]

    def allgather_bytes(self, b: bytes) -> list:
        if self.d is None:
            return [b]
        out = [None] * self.world
        self.d.all_gather_object(out, b)
        return out

    def close(self):
        if self.d is not None:
            self.d.destroy_process_group()


# ---------------------------------------------------------------------------
# workloads


class Workload:
    name = ""
    unit = "GFLOP/s"
    dtype = "bf16"
    scaling = "strong"

    def __init__(self, args, dist: Dist):
        self.args, self.dist = args, dist

    # dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel from one
    # `ncu --set full` capture of this workload at N=1 (profiles/ncu_traffic.json);
    # per-launch traffic at other N (or other kernels) is not measured -> null
    traffic_key = None

    def l2_flush_bytes(self):
        """Bytes to write between timed steps when the inputs fit in L2 (0: inputs > L2)."""
        return 0

    def traffic(self):
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if self.dist.world != 1 or not self.traffic_key or not os.path.exists(prof):
            return None
        with open(prof) as f:
            e = json.load(f).get(self.traffic_key)
        return e.get("dram_bytes_per_launch") if e else None

    # device handles of the runtime (set in setup)
    def stream(self):
        from paper_2005_08466_b200 import _native as N

        sp = ctypes.c_void_p()
        N.check(N.lib().hcl_device_stream(0, ctypes.byref(sp)))
        return self.dist.torch.cuda.ExternalStream(sp.value, device=self.dist.torch.device("cuda", self.dist.local))


class GemmBf16(Workload):
    name = "gemm_bf16"
    S = 16384

    def setup(self):
        import numpy as np
        import torch

        from paper_2005_08466_b200 import HostContext, split_ranges
        from paper_2005_08466_b200 import datagen as G

        S, d = self.S, self.dist
        self.ctx = ctx = HostContext([d.local])
        self.q = q = ctx.create_queue(0)
        b = split_ranges(S, [1] * d.world)  # == block_range (proj/src/bench.cpp:31-33)
        self.lo, self.rows = b[d.rank], b[d.rank + 1] - b[d.rank]
        t0 = time.perf_counter()
        self.a_host = torch.empty(self.rows * S, dtype=torch.int16, pin_memory=True)
        self.b_host = torch.empty(S * S, dtype=torch.int16, pin_memory=True)
        self.c_host = torch.empty(self.rows * S, dtype=torch.int16, pin_memory=True)
        G.gen_bf16(self.rows * S, 42, first=self.lo * S, out=self.a_host)
        G.gen_bf16(S * S, 43, out=self.b_host)
        ctx.add_data_creation_ms((time.perf_counter() - t0) * 1e3)
        prog = ctx.create_program("b200")
        self.k = ctx.create_kernel(prog, "gemm_bf16")
        self.bA, self.bB, self.bC = (ctx.create_buffer(S * S * 2) for _ in range(3))
        ctx.enqueue_write_buffer(q, self.bA, self.a_host, offset=self.lo * S * 2)
        ctx.enqueue_write_buffer(q, self.bB, self.b_host)
        for i, v in enumerate([self.bA, self.bB, self.bC, S, S, S, 0]):
            ctx.set_kernel_arg(self.k, i, v)
        self.step()
        ctx.finish(q)
        # parity guard: two output rows vs fp64 of the same bf16 inputs
        c2 = ctx.enqueue_read_buffer(q, self.bC, offset=self.lo * S * 2, length=2 * S * 2).view(np.uint16)
        a2 = (self.a_host[: 2 * S].numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32)
        bf = (self.b_host.numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32).reshape(S, S)
        a2 = a2.astype(np.float64).reshape(2, S)
        ref = a2 @ bf.astype(np.float64)
        scale = np.abs(a2) @ np.abs(bf).astype(np.float64)
        got = (c2.astype(np.uint32) << 16).view(np.float32).astype(np.float64).reshape(2, S)
        self.check = float((np.abs(got - ref) / scale).max())
        assert self.check <= 2.0**-8, f"gemm parity guard failed: {self.check}"
        if d.world > 1:  # B reaches the GPUs as 1/N slices over each rank's PCIe + an NVLink allgather
            from paper_2005_08466_b200 import HostContext as HC

            uid = d.bcast_bytes(HC.nccl_unique_id() if d.rank == 0 else None)
            ctx.init_collectives(q, d.rank, d.world, uid)
            self.kb = split_ranges(S, [1] * d.world)
        self.e2e_setup()

    def step(self):
        self.ctx.enqueue_ndrange_range(self.q, self.k, (self.S, self.S, 1), 2, self.lo, self.rows)

    def dominant(self):
        return self.step  # the step is one tcgen05 GEMM launch

    def dominant_work(self):
        return 2.0 * self.rows * self.S * self.S

    E2E_CHUNKS = 4

    def e2e_setup(self):
        """The e2e step's buffers: two sets (step i uses set i % 2, so step i's
        copies overlap step i-1's work), each holding B and the rank's rows in
        E2E_CHUNKS row chunks with their own A and C buffers and GEMM kernel. A
        chunk's D2H then depends only on its own GEMM, and the next chunk's GEMM
        only on its own A -- the C rows stream back while later chunks compute,
        and the next step's H2D streams in meanwhile (copies in both directions
        on two copy streams each)."""
        import torch

        ctx, S = self.ctx, self.S
        prog = ctx.create_program("b200")
        nc = max(1, min(self.E2E_CHUNKS, self.rows // 256))
        cb = [self.rows * i // nc for i in range(nc + 1)]
        self.chunk_bounds = cb
        self.sets = []
        for _ in range(2):
            bB = ctx.create_buffer(S * S * 2)
            chunks = []
            for c in range(nc):
                rc = cb[c + 1] - cb[c]
                bA, bC = ctx.create_buffer(rc * S * 2), ctx.create_buffer(rc * S * 2)
                k = ctx.create_kernel(prog, "gemm_bf16")
                for i, v in enumerate([bA, bB, bC, rc, S, S, 0]):
                    ctx.set_kernel_arg(k, i, v)
                chunks.append((k, bA, bC, rc))
            self.sets.append((bB, chunks))
        self.c_hosts = [self.c_host, torch.empty(self.rows * S, dtype=torch.int16, pin_memory=True)]
        # allocate and touch both sets on the device now (outside any timed region)
        for bB, chunks in self.sets:
            ctx.enqueue_write_buffer(self.q, bB, self.b_host)
            for c, (k, bA, bC, rc) in enumerate(chunks):
                ctx.enqueue_write_buffer(self.q, bA, self.a_host[cb[c] * S:cb[c + 1] * S])
                ctx.enqueue_ndrange_kernel(self.q, k, (rc, S, 1), 2)
        ctx.finish(self.q)
        self.e2e_i = 0

    def _e2e_b(self, bB, blocking=False):
        ctx, q, S = self.ctx, self.q, self.S
        if self.dist.world == 1:
            ctx.enqueue_write_buffer(q, bB, self.b_host, blocking=blocking)
        else:  # this rank's K-rows of B from host, the rest from the peers over NVLink
            r, kb = self.dist.rank, self.kb
            ctx.enqueue_write_buffer(q, bB, self.b_host[kb[r] * S:kb[r + 1] * S], offset=kb[r] * S * 2,
                                     blocking=blocking)

    def e2e_step(self):
        ctx, q, S, cb = self.ctx, self.q, self.S, self.chunk_bounds
        s = self.e2e_i % 2
        self.e2e_i += 1
        bB, chunks = self.sets[s]
        self._e2e_b(bB)  # B first: the allgather (N > 1) needs every rank's slice
        if self.dist.world > 1:
            ctx.enqueue_allgather(q, bB, [x * S * 2 for x in self.kb])
        for c, (k, bA, bC, rc) in enumerate(chunks):
            ctx.enqueue_write_buffer(q, bA, self.a_host[cb[c] * S:cb[c + 1] * S], blocking=False)
            ctx.enqueue_ndrange_kernel(q, k, (rc, S, 1), 2)
            ctx.enqueue_read_buffer(q, bC, out=self.c_hosts[s][cb[c] * S:cb[c + 1] * S], blocking=False)

    def work_per_step(self):
        return 2.0 * self.S**3

    def e2e_phases(self):
        """One e2e step with a device sync after each phase (wall ms on this rank):
        A rows + this rank's B slice H2D, the B allgather, the GEMM, C rows D2H."""
        ctx, q, S, d, cb = self.ctx, self.q, self.S, self.dist, self.chunk_bounds
        bB, chunks = self.sets[0]
        out = {}

        def phase(name, fn):
            d.barrier()
            t = time.perf_counter()
            fn()
            ctx.finish(q)
            out[name] = (time.perf_counter() - t) * 1e3

        def h2d():
            self._e2e_b(bB)
            for c, (k, bA, bC, rc) in enumerate(chunks):
                ctx.enqueue_write_buffer(q, bA, self.a_host[cb[c] * S:cb[c + 1] * S], blocking=False)

        phase("h2d", h2d)
        if d.world > 1:
            phase("allgather", lambda: ctx.enqueue_allgather(q, bB, [x * S * 2 for x in self.kb]))
        phase("gemm", lambda: [ctx.enqueue_ndrange_kernel(q, k, (rc, S, 1), 2) for k, _, _, rc in chunks])
        phase("d2h", lambda: [ctx.enqueue_read_buffer(q, bC, out=self.c_hosts[0][cb[c] * S:cb[c + 1] * S],
                                                      blocking=False) for c, (_, _, bC, _) in enumerate(chunks)])
        return out

    def e2e_bytes(self):
        S = self.S  # all ranks together: A once, B once (sliced + NVLink allgather), C once
        return 2 * S * S * 2, S * S * 2

    def roofline(self, pk):
        return "tensor", pk["bf16_tflops"], "TFLOP/s", 1e12, "MEASURED_PEAKS.json bf16_tflops (burst)"

    def config(self):
        return {"workload": f"gemm_bf16 {self.S}^3 (C2), NDRange rows split row-block over {self.dist.world} rank(s), "
                            "B replicated, fp32 accumulate, bf16 C",
                "rows_per_rank": self.rows, "kernel": "tcgen05 cta_group::2 256x256 tiles, TMA, 2 TMEM accumulators",
                "l2": "inputs 1 GiB > 126 MB L2; no flush", "parity_rows_normwise_err": self.check,
                "e2e_inputs": "per step: A rows per rank H2D; B as 1/N K-row slices H2D per rank + NCCL allgather "
                              "over NVLink (N>1); C rows D2H; double-buffered, non-blocking copies"}

    def traffic(self):
        prof = os.path.join(ROOT, "profiles", "gemm_bf16_ncu.json")
        if os.path.exists(prof):
            with open(prof) as f:
                return json.load(f).get("dram_bytes_per_launch")
        return None

    # reference arm: haocl::kernels::execute("matmul") fp64 on a row sample
    @staticmethod
    def reference_sampler():
        import oracle as O

        threads = os.cpu_count() or 1
        rows, cols, S = max(64, 2 * threads), 512, GemmBf16.S
        a = O.ref_gen_doubles(rows * S, 42)
        b = O.ref_gen_doubles(S * cols, 43)
        args = [("in", a), ("in", b), ("out", None), ("s", rows), ("s", S), ("s", cols)]

        def step():
            t = time.perf_counter()
            rc, work, _ = O.ref_execute("matmul", args, {2: rows * cols * 8}, threads=threads)
            assert rc == 0
            return float(work), time.perf_counter() - t

        desc = (f"haocl::kernels::execute('matmul') fp64 (reference encoding) on {rows} rows x K={S} x {cols} cols "
                f"of the {S}^3 GEMM per call, {threads} OpenMP threads, oracle/_ref built from /root/reference")
        return step, desc, threads, "reference", "f64", 1e9


class GemmF32(Workload):
    name = "gemm_f32"
    KERNEL = "gemm_f32"  # exact fp32 SIMT (k-ascending FFMA chains)
    dtype = "f32"
    scaling = "weak"
    S = 1024

    def setup(self):
        from paper_2005_08466_b200 import HostContext
        from paper_2005_08466_b200 import datagen as G
        import numpy as np
        import torch

        self.S = S = int(os.environ.get("BENCH_GEMM_F32_S", self.S))
        self.kernel = os.environ.get("BENCH_GEMM_F32_KERNEL", self.KERNEL)
        self.traffic_key = f"{self.kernel}_{S}"
        self.ctx = ctx = HostContext([self.dist.local])
        self.q = q = ctx.create_queue(0)
        self.a_host = torch.empty(S * S, dtype=torch.float32, pin_memory=True)
        self.b_host = torch.empty(S * S, dtype=torch.float32, pin_memory=True)
        self.c_host = torch.empty(S * S, dtype=torch.float32, pin_memory=True)
        G.gen_f32(S * S, 42, out=self.a_host)
        G.gen_f32(S * S, 43, out=self.b_host)
        prog = ctx.create_program("b200")
        self.k = ctx.create_kernel(prog, self.kernel)
        self.bA, self.bB, self.bC = (ctx.create_buffer(S * S * 4) for _ in range(3))
        ctx.enqueue_write_buffer(q, self.bA, self.a_host)
        ctx.enqueue_write_buffer(q, self.bB, self.b_host)
        for i, v in enumerate([self.bA, self.bB, self.bC, S, S, S]):
            ctx.set_kernel_arg(self.k, i, v)
        self.step()
        ctx.finish(q)
        R = S if S <= 2048 else 2  # parity guard rows (all of C1; 2 rows at C2 size)
        c = ctx.enqueue_read_buffer(q, self.bC, length=R * S * 4).view(np.float32).reshape(R, S).astype(np.float64)
        a = self.a_host.numpy()[: R * S].astype(np.float64).reshape(R, S)
        b = self.b_host.numpy().astype(np.float64).reshape(S, S)
        self.check = float((np.abs(c - a @ b) / (np.abs(a) @ np.abs(b))).max())
        tol = {"gemm_tf32": 2.0**-10, "gemm_f32x3": 2.0**-16 if S > 1024 else 2.0**-20}.get(self.kernel, 2.0**-20)
        assert self.check <= tol, f"{self.kernel} parity guard failed: {self.check}"

    def step(self):
        self.ctx.enqueue_ndrange_kernel(self.q, self.k, (self.S, self.S, 1), 2)

    def dominant(self):
        return self.step

    def dominant_work(self):
        return 2.0 * self.S**3

    def e2e_step(self):
        ctx, q = self.ctx, self.q
        ctx.enqueue_write_buffer(q, self.bA, self.a_host)
        ctx.enqueue_write_buffer(q, self.bB, self.b_host)
        self.step()
        ctx.enqueue_read_buffer(q, self.bC, out=self.c_host)

    def work_per_step(self):
        return 2.0 * self.S**3 * self.dist.world  # replicas

    def e2e_bytes(self):
        return 2 * self.S * self.S * 4 * self.dist.world, self.S * self.S * 4 * self.dist.world

    def roofline(self, pk):
        if self.kernel == "gemm_tf32":
            return "tensor", pk["bf16_tflops"] / 2, "TFLOP/s", 1e12, "TF32 tensor peak = MEASURED_PEAKS bf16 / 2"
        if self.kernel == "gemm_f32x3":
            return ("tensor", pk["bf16_tflops"] / 6, "TFLOP/s", 1e12,
                    "3xTF32 effective fp32 peak = MEASURED_PEAKS bf16 / 2 (tf32) / 3 (products)")
        # fp32 FFMA peak: 148 SM x 128 lanes x 2 flop x max clock
        sm = pk.get("sm_max_mhz", 1965.0)
        return "fp32_simt", 148 * 128 * 2 * sm * 1e6 / 1e12, "TFLOP/s", 1e12, "derived FFMA peak at max SM clock"

    def l2_flush_bytes(self):
        # A, B and C (3 * S^2 * 4 bytes) fit in the 126 MB L2 up to S ~ 3000
        return 256 << 20 if 3 * self.S * self.S * 4 < (126 << 20) else 0

    def config(self):
        cfg = "C1" if self.S == 1024 else "C2 fp32"
        return {"workload": f"fp32 GEMM {self.S}^3 ({cfg}) via the host API on one device ({self.kernel})",
                "replicas": self.dist.world, "normwise_err": self.check,
                "l2": ("inputs fit in L2: 256 MB flush write + 256 MB read (write-backs drained) before every timed step, per-step CUDA events"
                       if self.l2_flush_bytes() else f"inputs {3 * self.S * self.S * 4 >> 20} MB > L2; no flush")}

    @staticmethod
    def reference_sampler():
        import oracle as O

        threads = os.cpu_count() or 1
        S = GemmF32.S
        a = O.ref_gen_doubles(S * S, 42)
        b = O.ref_gen_doubles(S * S, 43)
        args = [("in", a), ("in", b), ("out", None), ("s", S), ("s", S), ("s", S)]

        def step():
            t = time.perf_counter()
            rc, work, _ = O.ref_execute("matmul", args, {2: S * S * 8}, threads=threads)
            assert rc == 0
            return float(work), time.perf_counter() - t

        return step, f"reference matmul {S}^3 fp64 (full problem), {threads} threads", threads, "reference", "f64", 1e9


class GemmF32x3(GemmF32):
    """C1 on the tensor cores: 3xTF32 split products, K split into 4 slices summed
    in order (2^-20 normwise at 1024^3, SURVEY.md §8(c)'s fp32 bound)."""
    name = "gemm_f32x3"
    KERNEL = "gemm_f32x3"


class PageRankW(Workload):
    name = "pagerank"
    unit = "GB/s"
    dtype = "f32"
    scale = 24

    def setup(self):
        import numpy as np

        from paper_2005_08466_b200 import HostContext, HaoclError, spmv_partition_ranges
        from paper_2005_08466_b200 import datagen as G

        d = self.dist
        self.scale = int(os.environ.get("BENCH_PR_SCALE", self.scale))
        self.v, self.e = 1 << self.scale, 16 << self.scale
        self.ctx = ctx = HostContext([d.local])
        self.q = q = ctx.create_queue(0)
        t0 = time.perf_counter()
        rp, ci, val, deg = G.pagerank_csr(self.scale, self.e, 42)
        # default step: the binned (propagation-blocking) kernel; BENCH_PR_KERNEL=pull
        # selects the warp-unit pull SpMV (fused exchange step) of round 1
        self.binned = os.environ.get("BENCH_PR_KERNEL", "binned") == "binned"
        if self.binned:
            return self.setup_binned(rp, ci, val, deg, t0)
        # degree-ordered vertex ids (per-row sums unchanged; tests/test_gpu_pagerank.py)
        self.relabel = os.environ.get("BENCH_PR_RELABEL", "0") == "1"
        if self.relabel:
            rp, ci, val, deg, _ = G.pagerank_relabel(rp, ci, val, deg)
        ctx.add_data_creation_ms((time.perf_counter() - t0) * 1e3)
        self.wn = wn = int(os.environ.get("BENCH_PR_WARP_NNZ", "64"))
        units, long_rows, n_long = G.pagerank_units(rp, wn)
        # rows balanced on a cost model, not on nnz alone: with the fused step every row also
        # costs its x'/xs' stores (one per rank). Measured per rank at N=4 (BENCH_PR_RANK_TIMES=1):
        # nnz-balanced ranges take 0.40 / 0.43 / 0.49 / 0.61 ms (0.45M .. 9.4M rows of equal nnz);
        # cost(row) = nnz + BENCH_PR_ROW_COST * N gives 3.59 (0) / 3.81 (1.0) / 4.02 (1.5) /
        # 4.22 (2.2) / 4.25 (2.8) TB/s at N=4 and 2.81 (1.0) / 2.98 (2.2) TB/s at N=2. A
        # least-squares refit from the ranks' measured times (t = a*nnz + b*rows) landed on
        # ~10 nnz per row at N=4 and no faster split: the residual imbalance is not linear
        # in (nnz, rows) -- gather locality differs between the hub rows and the tail
        fused_step = (os.environ.get("BENCH_PR_IMPLICIT", "1") == "1"
                      and os.environ.get("BENCH_PR_EXCHANGE", "1") == "1")
        self.row_cost = row_cost = float(os.environ.get("BENCH_PR_ROW_COST", "2.5")) * (d.world if fused_step else 0)
        cum = rp.astype(np.int64) + np.round(row_cost * np.arange(len(rp))).astype(np.int64)
        self.bounds = [int(x) for x in spmv_partition_ranges(cum, d.world)]
        lo, hi = self.bounds[d.rank], self.bounds[d.rank + 1]
        self.lo, self.rows = lo, hi - lo
        p0, p1 = int(rp[lo]), int(rp[hi])
        self.col_slice, self.val_slice = ci[p0:p1].copy(), val[p0:p1].copy()
        self.nnz_local = p1 - p0
        mk = ctx.create_buffer
        self.b_rp, self.b_u, self.b_l = mk(rp.nbytes), mk(units.nbytes), mk(long_rows.nbytes)
        self.b_col, self.b_val, self.b_deg = mk(self.col_slice.nbytes), mk(self.val_slice.nbytes), mk(deg.nbytes)
        self.b_x = [mk(self.v * 4), mk(self.v * 4)]
        self.b_dsum = mk(8)
        for b, a in ((self.b_rp, rp), (self.b_u, units), (self.b_l, long_rows), (self.b_col, self.col_slice),
                     (self.b_val, self.val_slice), (self.b_deg, deg)):
            ctx.enqueue_write_buffer(q, b, a)
        prog = ctx.create_program("b200")
        self.k_dang = ctx.create_kernel(prog, "pagerank_dangling")
        self.k_step = [ctx.create_kernel(prog, "pagerank_step") for _ in range(2)]
        for i in range(2):
            for j, a in enumerate([self.b_rp, self.b_col, self.b_val, self.b_u, self.b_l, self.b_x[i], self.b_dsum,
                                   self.b_x[1 - i], self.v, p0, len(units), n_long, wn]):
                ctx.set_kernel_arg(self.k_step[i], j, a)
        for j, a in enumerate([self.b_deg, self.b_dsum, self.v]):
            ctx.set_kernel_arg(self.k_dang, j + 1, a)
        # implicit values (default): pagerank_prep folds val = 1/outdeg into xs, the
        # step gathers xs (bit-identical products, no 1 GB value stream per iteration)
        self.implicit = os.environ.get("BENCH_PR_IMPLICIT", "1") == "1"
        if self.implicit:
            self.b_xs = mk(self.v * 4)
            self.k_prep = ctx.create_kernel(prog, "pagerank_prep")
            self.k_stepi = [ctx.create_kernel(prog, "pagerank_step_implicit") for _ in range(2)]
            for i in range(2):
                for j, a in enumerate([self.b_rp, self.b_col, self.b_u, self.b_l, self.b_xs, self.b_dsum,
                                       self.b_x[1 - i], self.v, p0, len(units), n_long, wn]):
                    ctx.set_kernel_arg(self.k_stepi[i], j, a)
            for j, a in enumerate([self.b_deg, self.b_dsum, self.b_xs, self.v]):
                ctx.set_kernel_arg(self.k_prep, j + 1, a)
        if d.world > 1:
            uid = d.bcast_bytes(HostContext.nccl_unique_id() if d.rank == 0 else None)
            ctx.init_collectives(q, d.rank, d.world, uid)
        self.byte_bounds = [4 * b for b in self.bounds]
        # fused step (default with implicit values, any N): pagerank_step_exchange writes
        # the rank's rows of x', the next gather input xs' = fl(1/outdeg) x' for those rows
        # into this rank's AND every peer's xs' (IPC-mapped peer buffers, NVLink stores)
        # and its dangling partial; an allreduce of the dangling sums is the only
        # collective (and the step barrier). No prep pass, no rank-vector allgather.
        # BENCH_PR_EXCHANGE=0: prep + step + NCCL allgather (the unfused baseline).
        self.fused = self.implicit and os.environ.get("BENCH_PR_EXCHANGE", "1") == "1"
        self.traffic_key = f"pagerank_step_exchange_scale{self.scale}" if self.fused and not self.relabel else None
        if self.fused:
            self.b_xs2 = [mk(self.v * 4), mk(self.v * 4)]
            handles = d.allgather_bytes(b"".join(ctx.share_buffer(q, b) for b in self.b_xs2)) if d.world > 1 else None
            self.b_dsum2 = [mk(8), mk(8)]
            self.b_peers, self.k_stepx = [], [ctx.create_kernel(prog, "pagerank_step_exchange") for _ in range(2)]
            for i in range(2):
                addrs = [ctx.open_shared_buffer(q, handles[r][64 * i:64 * (i + 1)], self.v * 4)
                         for r in range(d.world) if r != d.rank] if d.world > 1 else []
                arr = np.array(addrs or [0], np.uint64)
                bp = mk(arr.nbytes)
                ctx.enqueue_write_buffer(q, bp, arr)
                self.b_peers.append(bp)
            self.b_inv = mk(self.v * 4)  # fl(1/outdeg), computed once per graph
            ctx.enqueue_write_buffer(q, self.b_inv, G.pagerank_inv_outdeg(deg))
            for i in range(2):  # reads xs[i], dsum[i]; writes x rows, xs[1-i] (here + peers), dsum[1-i]
                for j, a in enumerate([self.b_rp, self.b_col, self.b_u, self.b_l, self.b_xs2[i], self.b_dsum2[i],
                                       self.b_x[0], self.v, p0, len(units), n_long, wn, self.b_peers[1 - i],
                                       d.world - 1, self.b_inv, self.b_xs2[1 - i], self.b_dsum2[1 - i]]):
                    ctx.set_kernel_arg(self.k_stepx[i], j, a)
            self.k_prep0 = ctx.create_kernel(prog, "pagerank_prep")  # x0 -> xs[0], dsum[0]
            for j, a in enumerate([self.b_x[0], self.b_deg, self.b_dsum2[0], self.b_xs2[0], self.v]):
                ctx.set_kernel_arg(self.k_prep0, j, a)
        import torch

        self.x0 = torch.full((self.v,), 1.0 / self.v, dtype=torch.float32).pin_memory()
        self.r_host = torch.empty(self.rows, dtype=torch.float32, pin_memory=True)
        # parity guard (the full 20-iteration oracle check is in tests/): one step's rows
        # sum to 1 over the ranks; the fused step equals prep + step + allgather bit for bit
        fused = self.fused
        self.fused = False
        self.reset()
        self.step()
        ctx.finish(q)
        ref = ctx.enqueue_read_buffer(q, self.b_x[self.cur]).view(np.float32).copy()
        self.check = float(abs(d.allsum(float(ref[lo:hi].astype(np.float64).sum())) - 1.0))
        self.fused = fused
        if self.fused:
            d.barrier()
            self.reset()
            self.step()
            ctx.finish(q)
            d.barrier()
            x = ctx.enqueue_read_buffer(q, self.b_x[0], offset=lo * 4, length=self.rows * 4).view(np.float32)
            assert x.tobytes() == ref[lo:hi].tobytes(), "pagerank_step_exchange rows differ from step + allgather"
            # its xs' must be prep(x') over all rows (the peers' stores included)
            xs_f = ctx.enqueue_read_buffer(q, self.b_xs2[self.cur]).view(np.float32).copy()
            ctx.enqueue_write_buffer(q, self.b_x[1], ref)
            ctx.set_kernel_arg(self.k_prep, 0, self.b_x[1])
            ctx.enqueue_ndrange_kernel(q, self.k_prep)
            ctx.finish(q)
            xs_r = ctx.enqueue_read_buffer(q, self.b_xs).view(np.float32)
            assert xs_r.tobytes() == xs_f.tobytes(), "pagerank_step_exchange xs' differs from prep(allgathered x')"
            d.barrier()
        self.reset()
        if os.environ.get("BENCH_PR_RANK_TIMES") == "1" and self.fused:  # diagnostics: per-rank kernel time
            print(f"rank {d.rank}: rows {self.rows} nnz {self.nnz_local} fused kernel "
                  f"{self.rank_kernel_ms():.4f} ms", file=sys.stderr, flush=True)
            self.reset()

    def setup_binned(self, rp, ci, val, deg, t0):
        """The rank's rows [lo, hi) (cost-balanced: nnz + row_cost * N per row)
        as one propagation-blocking part; the gather epilogue stores the next
        gather input xs' of its rows into every rank's xs' (IPC-mapped peer
        buffers over NVLink) and an 8-byte allreduce of the dangling sums is the
        only collective per step."""
        import numpy as np
        import torch

        from paper_2005_08466_b200 import HostContext, spmv_partition_ranges
        from paper_2005_08466_b200 import datagen as G
        from paper_2005_08466_b200.pagerank import BinnedLayout

        d, ctx, q, mk = self.dist, self.ctx, self.q, self.ctx.create_buffer
        self.relabel, self.implicit, self.fused, self.wn = False, True, True, 0
        self.row_cost = row_cost = float(os.environ.get("BENCH_PR_ROW_COST", "2.5")) * d.world
        cum = rp.astype(np.int64) + np.round(row_cost * np.arange(len(rp))).astype(np.int64)
        self.bounds = [int(x) for x in spmv_partition_ranges(cum, d.world)]
        lo, hi = self.bounds[d.rank], self.bounds[d.rank + 1]
        self.lo, self.rows = lo, hi - lo
        self.nnz_local = int(rp[hi]) - int(rp[lo])
        t1 = time.perf_counter()
        self.bl = BinnedLayout(ctx, q, rp, ci, [lo, hi])
        self.layout_s = time.perf_counter() - t1
        ctx.add_data_creation_ms((time.perf_counter() - t0) * 1e3)
        self.b_deg, self.b_inv, self.b_x = mk(deg.nbytes), mk(self.v * 4), [mk(self.v * 4)]
        ctx.enqueue_write_buffer(q, self.b_deg, deg)
        ctx.enqueue_write_buffer(q, self.b_inv, G.pagerank_inv_outdeg(deg))
        if d.world > 1:
            uid = d.bcast_bytes(HostContext.nccl_unique_id() if d.rank == 0 else None)
            ctx.init_collectives(q, d.rank, d.world, uid)
        self.b_xs2 = [mk(self.v * 4), mk(self.v * 4)]
        self.b_dsum2 = [mk(8), mk(8)]
        self.b_peers = []
        # xs' reaches the other ranks either through one NVSwitch multicast store per row
        # (BENCH_PR_MCAST=1, default: symmetric-memory xs' buffers, egress 4 B/row) or
        # through a store per peer into its IPC-mapped xs' (egress 4 (N-1) B/row)
        self.mcast = d.world > 1 and os.environ.get("BENCH_PR_MCAST", "1") == "1" and self.bind_multicast()
        if self.mcast:
            n_peers = -1
        else:
            n_peers = d.world - 1
            handles = d.allgather_bytes(b"".join(ctx.share_buffer(q, b) for b in self.b_xs2)) if d.world > 1 else None
            for i in range(2):  # b_peers[i]: the peers' copies of xs2[i]
                addrs = [ctx.open_shared_buffer(q, handles[r][64 * i:64 * (i + 1)], self.v * 4)
                         for r in range(d.world) if r != d.rank] if d.world > 1 else []
                arr = np.array(addrs or [0], np.uint64)
                bp = mk(arr.nbytes)
                ctx.enqueue_write_buffer(q, bp, arr)
                self.b_peers.append(bp)
        # kernel i reads xs[i], dsum[i]; writes x rows, xs[1-i] (here + peers), dsum[1-i]
        self.k_stepx = [self.bl.kernel(self.v, self.b_xs2[i], self.b_dsum2[i], self.b_x[0], self.b_peers[1 - i],
                                       n_peers, self.b_inv, self.b_xs2[1 - i], self.b_dsum2[1 - i])
                        for i in range(2)]
        prog = ctx.create_program("b200")
        # x0 -> xs[0] (scaled by 2^56: the binned step's fixed-point gather input), dsum[0]
        self.k_prep0 = ctx.create_kernel(prog, "pagerank_prep_fixed")
        for j, a in enumerate([self.b_x[0], self.b_deg, self.b_dsum2[0], self.b_xs2[0], self.v]):
            ctx.set_kernel_arg(self.k_prep0, j, a)
        self.traffic_key = f"pagerank_step_binned_scale{self.scale}"
        self.x0 = torch.full((self.v,), 1.0 / self.v, dtype=torch.float32).pin_memory()
        self.r_host = torch.empty(self.rows, dtype=torch.float32, pin_memory=True)
        # parity guard (bit-exact 20-iteration checks are in tests/test_pagerank_bins.py):
        # after one step the rows of all ranks carry the whole mass
        self.reset()
        self.step()
        ctx.finish(q)
        d.barrier()
        x = ctx.enqueue_read_buffer(q, self.b_x[0], offset=lo * 4, length=self.rows * 4).view(np.float32)
        self.check = float(abs(d.allsum(float(x.astype(np.float64).sum())) - 1.0))
        assert self.check <= 1e-3, f"pagerank binned parity guard: mass {self.check}"
        self.reset()
        if os.environ.get("BENCH_PR_RANK_TIMES") == "1":  # diagnostics: per-rank kernel time
            print(f"rank {d.rank}: rows {self.rows} nnz {self.nnz_local} binned step "
                  f"{self.rank_kernel_ms():.4f} ms", file=sys.stderr, flush=True)
            self.reset()

    def bind_multicast(self):
        """Back xs'[0], xs'[1] with torch symmetric memory (one allocation per rank,
        mapped into an NVSwitch multicast object) and hand the kernels the multicast
        addresses; False (IPC peer stores instead) when the fabric has no multicast."""
        import numpy as np
        import torch
        import torch.distributed._symmetric_memory as symm_mem

        d, ctx, q = self.dist, self.ctx, self.q
        self.symm = []
        try:
            for i in range(2):
                t = symm_mem.empty(self.v, dtype=torch.float32, device=torch.device("cuda", d.local))
                t.zero_()
                h = symm_mem.rendezvous(t, d.d.group.WORLD.group_name)
                self.symm.append((t, h))
            ok = all(h.multicast_ptr for _, h in self.symm)
        except Exception as e:  # no symmetric-memory support here: every rank falls back together
            print(f"rank {d.rank}: no NVSwitch multicast ({type(e).__name__}: {e}); IPC peer stores",
                  file=sys.stderr, flush=True)
            ok = False
        if not d.allmin(float(ok)):
            self.symm = []
            return False
        torch.cuda.synchronize()
        for i, (t, h) in enumerate(self.symm):
            ctx.bind_external(q, self.b_xs2[i], t.data_ptr())
            bp = ctx.create_buffer(8)
            ctx.enqueue_write_buffer(q, bp, np.array([h.multicast_ptr], np.uint64))
            self.b_peers.append(bp)
        return True

    def reset(self):
        ctx, q = self.ctx, self.q
        if self.fused and self.dist.world > 1:
            ctx.finish(q)  # the previous step's collective: no peer store is still landing
            self.dist.barrier()
        ctx.enqueue_write_buffer(q, self.b_x[0], self.x0)
        self.cur = 0
        if self.fused:
            ctx.enqueue_ndrange_kernel(q, self.k_prep0)

    def spmv(self):
        k = self.k_stepi[self.cur] if self.implicit else self.k_step[self.cur]
        self.ctx.enqueue_ndrange_range(self.q, k, (self.v, 1, 1), 1, self.lo, self.rows)

    def step(self):
        ctx, q = self.ctx, self.q
        if self.fused:
            ctx.enqueue_ndrange_range(q, self.k_stepx[self.cur], (self.v, 1, 1), 1, self.lo, self.rows)
            if self.dist.world > 1:  # the one collective; the next step's kernel waits on it (reads dsum')
                ctx.enqueue_allreduce_sum_i64(q, self.b_dsum2[1 - self.cur])
            self.cur = 1 - self.cur
            return
        if self.implicit:
            ctx.set_kernel_arg(self.k_prep, 0, self.b_x[self.cur])
            ctx.enqueue_ndrange_kernel(q, self.k_prep)
        else:
            ctx.set_kernel_arg(self.k_dang, 0, self.b_x[self.cur])
            ctx.enqueue_ndrange_kernel(q, self.k_dang)
        self.spmv()
        if self.dist.world > 1:
            ctx.enqueue_allgather(q, self.b_x[1 - self.cur], self.byte_bounds)
        self.cur = 1 - self.cur

    def rank_kernel_ms(self, n=10):
        """This rank's fused-kernel time (CUDA events, n launches after a reset)."""
        import torch

        self.reset()
        st = self.stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(n):
            self.step_kernel()
        e1.record(st)
        self.ctx.finish(self.q)
        self.dist.barrier()
        return e0.elapsed_time(e1) / n

    def step_kernel(self):  # the fused step's kernel alone (no collective): the dominant launch
        self.ctx.enqueue_ndrange_range(self.q, self.k_stepx[self.cur], (self.v, 1, 1), 1, self.lo, self.rows)

    def dominant(self):
        return self.step_kernel if self.fused else self.spmv

    def dominant_work(self):
        # SURVEY.md §8(d) algorithmic bytes of the CSR formulation (nnz*8 + (V+1)*4 + 2*V*4), for
        # every kernel variant (the binned step moves ~12 bytes per edge for the same work)
        return self.nnz_local * 8.0 + (self.rows + 1) * 4 + self.rows * 4 * 2

    def e2e_step(self):
        # one iteration with the rank vector from host and the rank's slice back
        ctx, q = self.ctx, self.q
        if self.fused:
            self.reset()  # x0 from host (+ its gather input)
            self.step()
            ctx.enqueue_read_buffer(q, self.b_x[0], offset=self.lo * 4, length=self.rows * 4, out=self.r_host)
            return
        ctx.enqueue_write_buffer(q, self.b_x[self.cur], self.x0)
        self.step()
        ctx.enqueue_read_buffer(q, self.b_x[self.cur], offset=self.lo * 4, length=self.rows * 4, out=self.r_host)

    def work_per_step(self):
        return float(self.e * 8 + (self.v + 1) * 4 + self.v * 4 * 2)

    def e2e_bytes(self):
        return self.v * 4 * self.dist.world, self.v * 4

    def roofline(self, pk):
        return "hbm", pk["hbm_gbs"], "GB/s", 1e9, "MEASURED_PEAKS.json hbm_gbs"

    def config(self):
        if self.binned:
            L = self.bl.layouts[0]
            return {"workload": f"PageRank iteration (C3): R-MAT scale {self.scale}, {self.e} edges, rows split over "
                                f"{self.dist.world} rank(s) (cost-balanced), binned step: propagation blocking "
                                "(scatter edge values into destination bins, shared-memory fixed-point gather), "
                                "next gather input stored to every rank over NVLink, dangling-sum allreduce",
                    "kernel": "pagerank_step_binned (pr_bin_scatter + pr_bin_gather)",
                    "row_sums": "order-free: values rounded to 2^-56, exact uint64 sums (oracle ho_spmv_f32_fixed)",
                    "layout": {k: L[k] for k in ("bin_rows", "chunk_edges", "span_max", "n_chunks", "n_bins",
                                                 "n_units", "n_slots")},
                    "layout_build_s": round(self.layout_s, 2),
                    "algorithmic_bytes_per_iteration": self.work_per_step(), "rank_sum_err": self.check,
                    "row_cost_nnz_per_row": self.row_cost,
                    "xs_exchange": ("NVSwitch multicast store (symmetric memory)" if self.mcast else
                                    "IPC peer stores" if self.dist.world > 1 else "none (one rank)"),
                    "l2": "2.35 GB algorithmic (~3.6 GB moved) per iteration > L2"}
        return {"workload": f"PageRank iteration (C3): R-MAT scale {self.scale}, {self.e} edges, int32/fp32 pull CSR, "
                            f"nnz-balanced rows over {self.dist.world} rank(s), " + (
                                "fused step: x' rows + next gather input xs' stored to every rank over NVLink, "
                                "dangling-sum allreduce" if self.fused else "prep + step + rank allgather"),
                "values": "implicit: val = 1/outdeg(src) folded into xs by pagerank_prep (bit-identical products); "
                          "bytes are counted per the CSR definition (nnz*8 + ...)" if self.implicit
                else "explicit fp32 value stream",
                "vertex_ids": "out-degree ordered (hcl_pagerank_relabel; per-row sums unchanged)" if self.relabel
                else "R-MAT ids", "warp_nnz": self.wn,
                "algorithmic_bytes_per_iteration": self.work_per_step(), "rank_sum_err": self.check,
                "row_cost_nnz_per_row": self.row_cost,
                "l2": "2.35 GB streamed per iteration > L2"}

    @staticmethod
    def reference_sampler():
        import numpy as np

        import oracle as O

        threads = os.cpu_count() or 1
        sc = 20
        rp, ci, val, deg = O.pagerank_csr(sc, 16 << sc, 42)
        v = 1 << sc
        hdr = np.array([v, v], np.int64)
        args = [("in", hdr), ("in", rp.astype(np.int64)), ("in", ci.astype(np.int64)), ("in", val.astype(np.float64)),
                ("in", np.full(v, 1.0 / v)), ("s", 0), ("s", v), ("out", None)]
        nbytes = (16 << sc) * 16 + (v + 1) * 8 + v * 8 * 2

        def step():
            t = time.perf_counter()
            rc, _, _ = O.ref_execute("spmv_compute", args, {7: v * 8}, threads=threads)
            assert rc == 0
            return float(nbytes), time.perf_counter() - t

        return (step, f"reference spmv_compute (fp64/int64 encoding) on an R-MAT scale-{sc} graph, one iteration "
                      f"per call, {threads} threads", threads, "reference", "f64", 1e9)


class KMeansW(Workload):
    name = "kmeans"
    dtype = "f32"
    N, D, K = 1 << 28, 32, 1024

    def setup(self):
        import numpy as np

        from paper_2005_08466_b200 import HostContext, split_ranges
        from paper_2005_08466_b200.kmeans import KMeans

        d = self.dist
        self.N = int(os.environ.get("BENCH_KM_N", self.N))
        self.ctx = ctx = HostContext([d.local])
        self.q = q = ctx.create_queue(0)
        b = split_ranges(self.N, [1] * d.world)
        self.lo, self.rows = b[d.rank], b[d.rank + 1] - b[d.rank]
        # tensor-filtered assignment (kmeans_assign_tc: tcgen05 split-bf16 scores + exact fp32
        # verification, identical assignments); BENCH_KM_TC=0 selects the exact SIMT kernel
        self.tc = os.environ.get("BENCH_KM_TC", "1") == "1"
        self.traffic_key = f"kmeans_assign_tc_n{self.N}" if self.tc else None
        self.km = km = KMeans(ctx, [q], self.N, self.D, self.K, tensor_filter=self.tc)
        # this rank's rows of the point set, generated in HBM (counter-based SplitMix64)
        kg = ctx.create_kernel(ctx.create_program("b200"), "gen_kmeans_points")
        for j, a in enumerate([km.b_pts, self.N, self.D, self.K, 42]):
            ctx.set_kernel_arg(kg, j, a)
        ctx.enqueue_ndrange_range(q, kg, (self.N, 1, 1), 1, self.lo, self.rows)
        if self.tc:  # bf16 split rows + |x|^2 of the resident points, once
            ctx.enqueue_ndrange_range(q, km.k_split, (self.N, 1, 1), 1, self.lo, self.rows)
        km.on_grid = True  # generated on the 2^-12 grid by construction
        if km.q16:  # the update's int16 fixed-point copy, once
            ctx.enqueue_ndrange_range(q, km.k_quant, (self.N, 1, 1), 1, self.lo, self.rows)
        ctx.finish(q)
        from paper_2005_08466_b200 import datagen as G

        self.cent0 = G.gen_kmeans_points(self.K, self.D, self.K, 42)  # first K points = initial centroids
        km.set_centroids(self.cent0)
        # store the rank's points grouped by their nearest initial centroid (a layout transform,
        # results unchanged): a warp's points then share candidate centroids and the tensor
        # assignment skips its candidate-mask pass warp-wide where none has one
        self.ordered = self.tc and os.environ.get("BENCH_KM_ORDER", "1") == "1"
        if self.ordered:
            km.order_by_cluster(parts=[(q, self.lo, self.lo + self.rows)])
            km.set_centroids(self.cent0)
        if d.world > 1:
            uid = d.bcast_bytes(HostContext.nccl_unique_id() if d.rank == 0 else None)
            ctx.init_collectives(q, d.rank, d.world, uid)
        self.check = None

    def _assign(self):
        c = self.ctx
        k = self.km.k_assign_tc if self.tc else self.km.k_assign
        c.enqueue_ndrange_range(self.q, k, (self.N, 1, 1), 1, self.lo, self.rows)

    def step(self):
        c, q, km = self.ctx, self.q, self.km
        self._assign()
        c.enqueue_ndrange_range(q, km.acc_kernel, (self.N, 1, 1), 1, self.lo, self.rows)
        if self.dist.world > 1:
            c.enqueue_allreduce_sum_i64(q, km.b_sums)
            c.enqueue_allreduce_sum_i64(q, km.b_counts)
        c.enqueue_ndrange_kernel(q, km.k_fin)

    def dominant(self):
        return self._assign

    def dominant_work(self):
        if self.tc:  # the assignment as one bf16 GEMM, 2 N K D flop (10.4 ms at C4 at the
            return 2.0 * self.rows * self.K * self.D  # bf16 peak) -- not the split-operand MMAs actually issued
        return 3.0 * self.rows * self.K * self.D

    def e2e_step(self):
        # centroids from host, new centroids back (the points are the resident data set)
        self.km.set_centroids(self.cent0)
        self.step()
        self.ctx.enqueue_read_buffer(self.q, self.km.b_cent)

    def work_per_step(self):
        return 3.0 * self.N * self.K * self.D

    def e2e_bytes(self):
        return self.K * self.D * 4 * self.dist.world, self.K * self.D * 4 * self.dist.world

    def roofline(self, pk):
        if self.tc:
            return ("tensor", pk["bf16_tflops"], "TFLOP/s", 1e12,
                    "MEASURED_PEAKS.json bf16_tflops; achieved = 2 N K D / assign time: the assignment's "
                    "algorithmic bf16-GEMM bound (SURVEY.md §8(d) C4), frac = that GEMM's time / assign time")
        sm = pk.get("sm_max_mhz", 1965.0)
        # exact (non-FMA) fp32: one add or multiply per lane per clock (FADD2 issues
        # two lanes' worth but occupies the FP32 pipe twice, measured)
        return ("fp32_simt", 148 * 128 * sm * 1e6 / 1e12, "TFLOP/s", 1e12,
                "derived non-FMA fp32 rate (148 SM x 128 lanes x max SM clock)")

    def config(self):
        return {"workload": f"k-means iteration (C4): {self.N} points x {self.D} dims, K={self.K}, exact fp32 "
                            f"assignment (3 flop/term), int64 sums, points split over {self.dist.world} rank(s)",
                "assign_kernel": "kmeans_assign_tc (tcgen05 split-bf16 filter + exact fp32 verify)" if self.tc
                else "kmeans_assign (exact fp32 SIMT)",
                "points": "SplitMix64 blobs, multiples of 2^-12, generated in HBM" +
                          ("; stored grouped by nearest initial centroid (KMeans.order_by_cluster)" if self.ordered
                           else ""),
                "l2": f"points {self.N * self.D * 4 >> 30} GiB > L2; no flush"}

    @staticmethod
    def reference_sampler():
        import oracle as O

        threads = os.cpu_count() or 1
        q, r, dd = 8192, KMeansW.K, KMeansW.D
        pts = O.kmeans_points(42, 0, q, dd, r).astype("float64")
        cent = O.kmeans_points(42, 0, r, dd, r).astype("float64")
        args = [("in", cent), ("in", pts), ("s", r), ("s", q), ("s", dd), ("s", 1), ("out", None), ("out", None)]

        def step():
            t = time.perf_counter()
            rc, work, _ = O.ref_execute("knn", args, {6: q * 4, 7: q * 8}, threads=threads)
            assert rc == 0
            return 3.0 * work, time.perf_counter() - t

        return (step, f"reference knn k=1 (assignment semantics, fp64) {q} points x {r} centroids x {dd} dims per "
                      f"call, {threads} threads", threads, "reference", "f64", 1e9)


class ConvW(Workload):
    name = "conv"
    N, H, W, C, K = 256, 224, 224, 64, 128

    def setup(self):
        import numpy as np
        import torch

        from paper_2005_08466_b200 import HostContext, split_ranges
        from paper_2005_08466_b200 import datagen as G

        d = self.dist
        self.N = int(os.environ.get("BENCH_CONV_N", self.N))
        self.traffic_key = f"conv3x3_n{self.N}"
        self.ctx = ctx = HostContext([d.local])
        self.q = q = ctx.create_queue(0)
        b = split_ranges(self.N, [1] * d.world)
        self.lo, self.cnt = b[d.rank], b[d.rank + 1] - b[d.rank]
        img_in, img_out = self.H * self.W * self.C, self.H * self.W * self.K
        self.x_host = torch.empty(self.cnt * img_in, dtype=torch.int16, pin_memory=True)
        self.o_host = torch.empty(self.cnt * img_out, dtype=torch.int16, pin_memory=True)
        G.gen_bf16(self.cnt * img_in, 42, first=self.lo * img_in, out=self.x_host)
        w = G.gen_bf16(self.K * 9 * self.C, 43)
        mk = ctx.create_buffer
        self.b_in = mk(self.N * img_in * 2)
        self.b_w = mk(w.nbytes)
        self.b_out = mk(self.N * img_out * 2)
        ctx.enqueue_write_buffer(q, self.b_in, self.x_host, offset=self.lo * img_in * 2)
        ctx.enqueue_write_buffer(q, self.b_w, w)
        prog = ctx.create_program("b200")
        # the whole layer from plain NHWC (conv3x3_nhwc): no padded copy of the input
        self.k_conv = ctx.create_kernel(prog, "conv3x3_nhwc")
        for j, a in enumerate([self.b_in, self.b_w, self.b_out, self.N, self.H, self.W, self.C, self.K, 0]):
            ctx.set_kernel_arg(self.k_conv, j, a)
        self.conv()
        ctx.finish(q)
        self.img_in, self.img_out = img_in, img_out
        self.check = None

    def conv(self):
        self.ctx.enqueue_ndrange_range(self.q, self.k_conv, (self.N, 1, 1), 1, self.lo, self.cnt)

    def step(self):
        self.conv()

    def dominant(self):
        return self.step  # the step is one conv3x3 launch

    def dominant_work(self):
        return 2.0 * self.cnt * self.H * self.W * self.K * 9 * self.C

    def e2e_step(self):
        ctx, q = self.ctx, self.q
        ctx.enqueue_write_buffer(q, self.b_in, self.x_host, offset=self.lo * self.img_in * 2)
        self.conv()
        ctx.enqueue_read_buffer(q, self.b_out, offset=self.lo * self.img_out * 2, length=self.cnt * self.img_out * 2,
                                out=self.o_host)

    def work_per_step(self):
        return 2.0 * self.N * self.H * self.W * self.K * 9 * self.C

    def e2e_bytes(self):
        return self.N * self.img_in * 2, self.N * self.img_out * 2

    def roofline(self, pk):
        return "tensor", pk["bf16_tflops"], "TFLOP/s", 1e12, "MEASURED_PEAKS.json bf16_tflops (burst)"

    def config(self):
        return {"workload": f"conv3x3 (C5): batch {self.N}, {self.H}x{self.W}x{self.C} -> {self.K}, stride 1 pad 1, "
                            f"bf16 in/out, fp32 accumulate, batch split over {self.dist.world} rank(s)",
                "kernel": "conv3x3_nhwc: 16x16-pixel pair tiles, one 4D TMA halo box per CTA tile (zero fill = "
                          "padding), 9 taps from shifted descriptors, tcgen05 cta_group::2, resident weights",
                "layout": "NHWC input (unpadded), KRSC weights, NHWK output",
                "l2": f"input {self.N * self.H * self.W * self.C * 2 >> 20} MB and output "
                      f"{self.N * self.H * self.W * self.K * 2 >> 20} MB > L2; no flush"}

    @staticmethod
    def reference_sampler():
        import numpy as np

        import oracle as O

        h, w, c, k = ConvW.H, ConvW.W, ConvW.C, ConvW.K
        x = O.gen_bf16(h * w * c, 42)
        wt = O.gen_bf16(k * 9 * c, 43)
        rows = 4

        def step():
            t = time.perf_counter()
            O.conv3x3_rows(x, wt, h, w, c, k, 0, 0, rows)
            return 2.0 * 9 * c * rows * w * k, time.perf_counter() - t

        return (step, f"restated direct conv (oracle port, no reference conv exists): {rows} output rows x {w} x {k} "
                      "of image 0 per call, fp64, 1 thread", 1, "port", "f64", 1e9)


WORKLOADS = {w.name: w for w in (GemmBf16, GemmF32, GemmF32x3, PageRankW, KMeansW, ConvW)}


# ---------------------------------------------------------------------------


def cpu_leg(wl_cls, seconds=10.0, steps=None, warmup=1):
    step, desc, threads, kind, dtype, scale = wl_cls.reference_sampler()
    for _ in range(warmup):
        step()
    tot_w = tot_t = 0.0
    n = 0
    while (steps is None and tot_t < seconds) or (steps is not None and n < steps):
        w, dt = step()
        tot_w += w
        tot_t += dt
        n += 1
    return tot_w / tot_t / scale, tot_t / max(n, 1), desc, threads, kind, dtype


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    wl_cls = WORKLOADS[args.workload]
    value, per_step, desc, threads, kind, dtype = cpu_leg(wl_cls, steps=args.steps, warmup=args.warmup)
    unit = wl_cls.unit
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per_step * 1e3, 3), "higher_is_better": True,
        "scaling": wl_cls.scaling, "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (SplitMix64 seeds 42/43)",
        "config": {"workload": f"{wl_cls.name}: the reference CPU path on a bounded sample", "sample": desc},
        "cpu_baseline": {"value": round(value, 3), "unit": unit, "cores": threads, "kind": kind, "sample": desc},
        "e2e": {"value": round(value, 3), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def measure(wl, args, dist, sampler=None, cpu_seconds=10.0, hold=True):
    """W warm-up steps, then K timed steps (CUDA events on the runtime's
    stream, max over ranks), the dominant kernel alone, and the e2e loop through
    the public API with host buffers. Returns the JSON line (rank 0) or None."""
    from paper_2005_08466_b200 import _native as N

    torch = dist.torch
    wl.setup()
    for _ in range(args.warmup):
        wl.step()
    wl.ctx.finish(wl.q)
    stream = wl.stream()

    # value: K steps, inputs resident, device time (CUDA events on the runtime's stream)
    dist.barrier()
    if sampler:
        sampler.mark()
    launches0 = N.lib().hcl_kernel_launch_count()
    flush = wl.l2_flush_bytes()
    if flush:
        # inputs smaller than L2: every timed step starts from a flushed L2 (a write
        # larger than L2 on the same stream, outside the per-step event pairs), then a
        # read of another buffer larger than L2, so the flush's dirty lines are written
        # back before the step starts instead of competing with its loads (a write-only
        # flush leaves ~126 MB of write-back inside the next timed step)
        flush = int(os.environ.get("BENCH_FLUSH_MB", flush >> 20)) << 20
        fbuf = torch.empty(flush // 4, dtype=torch.float32, device=torch.device("cuda", dist.local))
        rbuf = torch.ones(flush // 4, dtype=torch.float32, device=torch.device("cuda", dist.local))
        rsum = torch.empty(1, dtype=torch.float32, device=torch.device("cuda", dist.local))
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a, b in evs:
            with torch.cuda.stream(stream):
                fbuf.zero_()
                torch.sum(rbuf, dim=0, keepdim=True, out=rsum)
            a.record(stream)
            wl.step()
            b.record(stream)
    else:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            wl.step()
        e1.record(stream)
    wl.ctx.finish(wl.q)
    dist.barrier()
    launches = N.lib().hcl_kernel_launch_count() - launches0
    # clock hold: a timed region shorter than ~3 nvidia-smi samples is followed by
    # the same steps, untimed, until the sampler has seen them under load
    hold_ms, t_hold = 0.0, time.time()
    # (every rank takes part in these reductions; only rank 0 samples)
    need_hold = hold and dist.allmax(1.0 if sampler and sampler.count() < 3 else 0.0) > 0
    while need_hold:
        for _ in range(max(1, args.steps)):
            wl.step()
        wl.ctx.finish(wl.q)
        hold_ms = (time.time() - t_hold) * 1e3
        need_hold = dist.allmax(1.0 if (sampler and sampler.count() < 3 and hold_ms < 3000) else 0.0) > 0
    if sampler:
        sampler.end()
    dev_ms = sum(a.elapsed_time(b) for a, b in evs) if flush else e0.elapsed_time(e1)
    ms_max = dist.allmax(dev_ms)
    launches_total = int(dist.allsum(launches))

    # dominant kernel alone, same stream, averaged over K launches (when the step
    # is that one kernel, the value loop above already is this measurement)
    dom = wl.dominant()
    if dom == wl.step:
        dom_ms = dev_ms / args.steps
    else:
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for _ in range(args.steps):
            dom()
        d1.record(stream)
        wl.ctx.finish(wl.q)
        dom_ms = d0.elapsed_time(d1) / args.steps

    # e2e through the public API with host buffers (untimed warm-up first: the
    # first collectives set up NCCL's peer channels)
    for _ in range(min(args.warmup, 2)):
        wl.e2e_step()
    wl.ctx.finish(wl.q)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.e2e_step()
    wl.ctx.finish(wl.q)
    e2e_ms = dist.allmax((time.perf_counter() - t0) * 1e3)
    dist.barrier()
    # the e2e step's phases one after the other (the reference's per-phase report,
    # bench.cpp:179-200), max over ranks; untimed for the line
    phases = {k: round(dist.allmax(v), 3) for k, v in wl.e2e_phases().items()} if hasattr(wl, "e2e_phases") else None
    clocks = sampler.stop() if sampler else None
    if clocks is not None:
        clocks["hold_ms"] = round(hold_ms, 1)  # untimed repeat of the steps while sampling (short regions)
    line = None
    if dist.rank == 0:
        pk = peaks()
        bound, peak, runit, rscale, psrc = wl.roofline(pk)
        achieved = wl.dominant_work() / (dom_ms / 1e3) / rscale
        scale = 1e9
        value = wl.work_per_step() * args.steps / (ms_max / 1e3) / scale
        h2d, d2h = wl.e2e_bytes()
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": wl.unit, "n_gpus": dist.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": wl.scaling, "vs_baseline": None, "dtype": wl.dtype,
            "data": "synthetic (SplitMix64, product datagen)", "config": wl.config(),
            "roofline": {"bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": runit,
                         "frac": round(achieved / peak, 4), "traffic": wl.traffic(), "peak_src": psrc,
                         "kernel_ms": round(dom_ms, 4), "kernel_work": wl.dominant_work()},
            "e2e": {"value": round(wl.work_per_step() * args.steps / (e2e_ms / 1e3) / scale, 1), "unit": wl.unit,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches_total,
            **({"e2e_phases_ms": phases} if phases else {}),
        }
        if clocks is not None:
            line["clocks"] = clocks
        if wl.name == "gemm_bf16":
            line["roofline"]["frac_of_sustained_peak"] = round(achieved / pk["bf16_tflops_sustained"], 4)
        if dist.world == 1 and not args.no_cpu_baseline:
            try:
                v, _, desc, threads, kind, _ = cpu_leg(type(wl), seconds=cpu_seconds)
                line["cpu_baseline"] = {"value": round(v, 3), "unit": wl.unit, "cores": threads, "kind": kind,
                                        "sample": desc}
            except Exception as e:  # reported baseline only, never the measured path
                line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    return line


# the other BASELINE configs, measured in the same default run
SECONDARY = (("C1", "gemm_f32"), ("C1-3xTF32", "gemm_f32x3"), ("C3", "pagerank"), ("C4", "kmeans"), ("C5", "conv"))


def run_b200(args):
    dist = Dist("nccl")
    torch = dist.torch
    torch.cuda.set_device(dist.local)
    if dist.world != args.gpus and dist.rank == 0:
        print(f"warning: WORLD_SIZE {dist.world} != --gpus {args.gpus}", file=sys.stderr)
    sampler = ClockSampler(list(range(dist.world))) if dist.rank == 0 else None
    wl = WORKLOADS[args.workload](args, dist)
    line = measure(wl, args, dist, sampler)
    wl.ctx.close()
    del wl
    if args.workload == "gemm_bf16" and not args.no_secondary:
        # every other config of BASELINE.json through the same contract, so the
        # driver's run records them too: a shorter timed loop each, CPU leg 3 s
        sub = argparse.Namespace(**vars(args))
        sub.steps, sub.warmup = max(3, min(args.steps, 10)), max(3, min(args.warmup, 3))
        secondary = {}
        for tag, name in SECONDARY:
            t0 = time.perf_counter()
            try:
                w = WORKLOADS[name](sub, dist)
                r = measure(w, sub, dist, None, cpu_seconds=3.0, hold=False)
                w.ctx.close()
                del w
                torch.cuda.empty_cache()
            except Exception as e:  # one failing config must not hide the others
                r = {"error": f"{type(e).__name__}: {str(e)[:300]}"} if dist.rank == 0 else None
            if dist.rank == 0:
                r = {k: v for k, v in r.items() if k not in ("metric", "higher_is_better", "vs_baseline")}
                r["wall_s"] = round(time.perf_counter() - t0, 1)
                secondary[tag] = r
        if dist.rank == 0:
            line["workloads"] = secondary
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="gemm_bf16")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="headline config only (default: also C1, C3, C4, C5 under 'workloads')")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
