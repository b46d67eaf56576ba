"""Remote-node path end to end: the reference's own host
runtime and bench layer (compiled in place into oracle/_ref/ref_bench_remote)
drive this repo's node daemon (python -m paper_2005_08466_b200.node) over TCP
with the HCL1 protocol. The daemon runs the reference's core kernels on the
B200; the reference's in-process oracle must pass and the result digests must
equal the reference's own (tests/golden/reference_golden.json), for one and two
parts (block_range row splits over two logical devices)."""
import json
import os
import random
import subprocess
import sys

import pytest

from tests import hcl1_client as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REMOTE = os.path.join(ROOT, "oracle", "_ref", "ref_bench_remote")

CASES = [
    ("matmul", ["m=64", "k=64", "n=64"], "matmul_64"),
    ("matmul", ["m=512", "k=512", "n=512"], "matmul_512"),
    ("spmv", ["rows=100", "cols=100", "density=0.1"], "spmv_100x100@0.1"),
    ("spmv", ["rows=10000", "cols=10000", "density=0.001"], "spmv_10000x10000@0.001"),
    ("knn", ["knn_r=200", "knn_q=20", "knn_d=8", "knn_k=5"], "knn_200x20x8k5"),
    ("bfs", ["vertices=1000", "edges=10000"], "bfs_1000v10000e"),
    ("vecadd", ["length=100000"], "vecadd_100000"),
]


@pytest.fixture(scope="module")
def node():
    if not os.path.exists(REMOTE):
        pytest.fail(f"{REMOTE} missing: build it with `make -C oracle ref` where /root/reference exists")
    for _ in range(10):
        port = random.randint(20000, 60000)
        proc = subprocess.Popen([sys.executable, "-m", "paper_2005_08466_b200.node", "--port", str(port),
                                 "--devices", "0,0"], cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                text=True)
        line = proc.stdout.readline()
        if "serving" in line:
            break
        proc.wait(timeout=30)
    else:
        pytest.fail("node daemon did not start")
    yield port, 2
    c = W.Conn(port)
    c.send(W.frame(W.SHUTDOWN, 1))
    c.close()
    assert proc.wait(timeout=60) == 0


@pytest.mark.parametrize("bench,args,key", CASES, ids=[c[2] for c in CASES])
@pytest.mark.parametrize("parts", [1, 2])
def test_reference_host_drives_b200_node(node, golden, bench, args, key, parts):
    if bench == "bfs" and parts > 1:
        pytest.skip("the reference runs bfs whole (bench.cpp:539-540)")
    port, ndev = node
    r = subprocess.run([REMOTE, str(port), str(ndev), bench, str(parts)] + args, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    report = json.loads(r.stdout)
    assert report["verify"] == "pass"
    assert report["result_digest"].lower() == golden["digests"][key]
    assert report["partition"] == parts and len(report["devices"]) == ndev
    assert all(d.endswith(":gpu") for d in report["devices"])


def _vecadd(c, call_id, dev, a, b, out, n):
    return c.call(call_id, "launch_kernel",
                  [(W.STRING, "vecadd"), (W.STRING, "default"), (W.I32, 1), (W.I32, dev), (W.I32, 1),
                   (W.I64, n), (W.I64, 1), (W.I64, 1), (W.I32, 4),
                   (W.HANDLE, a), (W.HANDLE, b), (W.HANDLE, out), (W.I64, n)])


def test_residency_peer_staging_and_invalidation(node):
    """HBM residency of the daemon's buffers: an output feeds a launch on the
    other device (peer copy, never read back), a rewritten input invalidates
    the resident copies, and read_buffer returns the newest bytes."""
    import numpy as np

    port, _ = node
    n = 1 << 16
    rng = np.random.default_rng(1)
    a, b, a2 = (rng.standard_normal(n) for _ in range(3))
    m, d = W.Conn(port), W.Conn(port + 1)

    def put(cid, bid, arr):
        m.call(cid, "alloc_buffer", [(W.HANDLE, bid), (W.I64, arr.nbytes)])
        raw = arr.tobytes()
        for off in range(0, len(raw), 1 << 18):  # 256 KiB chunks, last one acknowledged
            d.send(W.frame(W.DATA, cid * 100 + off // (1 << 18), W.data_chunk(bid, off, len(raw), raw[off:off + (1 << 18)])))
        kind, _, body = d.recv_frame()
        assert kind == W.ACK

    put(1, 101, a)
    put(2, 102, b)
    for bid in (103, 104):
        m.call(3, "alloc_buffer", [(W.HANDLE, bid), (W.I64, n * 8)])
    res = _vecadd(m, 4, 0, 101, 102, 103, n)  # c = a + b on device 0
    assert res[2] == n  # work units = n (kernels.cpp:296)
    _vecadd(m, 5, 1, 103, 101, 104, n)         # e = c + a on device 1: c staged by peer copy
    e = np.frombuffer(d.call(6, "read_buffer", [(W.HANDLE, 104)])[0], np.float64)
    assert (e == (a + b) + a).all()
    put(7, 101, a2)                             # rewrite a: device copies are stale now
    _vecadd(m, 8, 0, 101, 102, 103, n)
    c = np.frombuffer(d.call(9, "read_buffer", [(W.HANDLE, 103)])[0], np.float64)
    assert (c == a2 + b).all()
    for bid in (101, 102, 103, 104):
        m.call(10, "release_object", [(W.HANDLE, bid)])
    m.close(), d.close()
