"""Remote-node path, measured: the reference's own host runtime + bench layer
(oracle/_ref/ref_bench_remote) against (a) the reference's own CPU node daemon
(oracle/_ref/ref_node, all host threads per device) and (b) this repo's B200
node daemon (python -m paper_2005_08466_b200.node). Same host program, same TCP
protocol, same inputs; only the node changes. Prints one row per run and writes
gpurun_out/remote_compare.json.

    python scripts/remote_compare.py [--parts 1,2] [--devices 2]
"""
import argparse
import json
import os
import random
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests import hcl1_client as W  # noqa: E402

REMOTE = os.path.join(ROOT, "oracle", "_ref", "ref_bench_remote")
REF_NODE = os.path.join(ROOT, "oracle", "_ref", "ref_node")
WORKLOADS = [
    ("matmul", ["m=1024", "k=1024", "n=1024"]),
    ("spmv", ["rows=100000", "cols=100000", "density=0.0001"]),
    ("knn", ["knn_r=100000", "knn_q=1000", "knn_d=16", "knn_k=10"]),
    ("bfs", ["vertices=100000", "edges=1000000"]),
    ("vecadd", ["length=10000000"]),
]


def start(cmd, marker):
    for _ in range(10):
        port = random.randint(20000, 60000)
        p = subprocess.Popen([c.replace("PORT", str(port)) for c in cmd], cwd=ROOT, stdout=subprocess.PIPE,
                             stderr=subprocess.STDOUT, text=True)
        if marker in p.stdout.readline():
            return p, port
        p.wait(timeout=30)
    raise RuntimeError(f"could not start {cmd}")


def stop(p, port):
    c = W.Conn(port)
    c.send(W.frame(W.SHUTDOWN, 1))
    c.close()
    p.wait(timeout=120)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", default="1,2")
    ap.add_argument("--devices", type=int, default=2)
    ap.add_argument("--repeat", type=int, default=2, help="runs per case; rows carry the run index")
    a = ap.parse_args()
    threads = os.cpu_count()
    arms = {
        "reference_cpu_node": ([REF_NODE, "PORT", str(a.devices), str(threads)], "ref node serving", "cpu"),
        "b200_node": ([sys.executable, "-m", "paper_2005_08466_b200.node", "--port", "PORT", "--devices",
                       ",".join(["0"] * a.devices)], "serving", "gpu"),
    }
    rows = []
    for arm, (cmd, marker, typ) in arms.items():
        proc, port = start(cmd, marker)
        try:
            for bench, args in WORKLOADS:
                for parts, rep_i in [(int(x), i) for x in a.parts.split(",") for i in range(a.repeat)]:
                    if bench == "bfs" and parts > 1:
                        continue
                    t0 = time.time()
                    r = subprocess.run([REMOTE, str(port), str(a.devices), bench, str(parts)] + args + [f"type={typ}"],
                                       capture_output=True, text=True, timeout=3600)
                    wall = time.time() - t0
                    if r.returncode != 0:
                        rows.append({"arm": arm, "bench": bench, "parts": parts, "error": r.stderr[-300:]})
                        print(arm, bench, parts, "ERROR", r.stderr[-300:], flush=True)
                        continue
                    rep = json.loads(r.stdout)
                    t = rep["timing"]
                    row = {"arm": arm, "run": rep_i, "bench": bench, "size": rep["size"], "parts": parts,
                           "verify": rep["verify"],
                           "digest": rep["result_digest"], "compute_ms": round(t["compute_ms"], 3),
                           "transfer_ms": round(t["transfer_ms"], 3), "total_ms": round(t["total_ms"], 3),
                           "wall_s": round(wall, 2), "node_threads": threads if typ == "cpu" else None}
                    rows.append(row)
                    print(json.dumps(row), flush=True)
        finally:
            stop(proc, port)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "remote_compare.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
