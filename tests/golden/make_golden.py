"""Regenerate tests/golden/*.json from the HaoCL reference itself.

Runs the reference library compiled in place from /root/reference
(oracle/_ref/libhaocl_ref.so, see oracle/Makefile) — never the restatement —
so the committed fixtures pin the restated oracle and the CUDA path to the
reference's own outputs. Only runnable where /root/reference exists:

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def h(x):
    return "%016x" % x


def main():
    assert O.ref_available(), "oracle/_ref/libhaocl_ref.so missing (needs /root/reference)"
    out = {"source": "oracle/_ref/libhaocl_ref.so built from /root/reference/proj/src "
                     "(kernels, reference, datagen, error .cpp)"}

    # FNV-1a digests of the reference's own outputs (bench.cpp:35-41 convention)
    dig = {}
    for n in (64, 512, 1024):
        a = O.ref_gen_doubles(n * n, 42)
        b = O.ref_gen_doubles(n * n, 43)
        dig[f"matmul_{n}"] = h(O.fnv1a(O.ref_matmul(a, b, n, n, n)))
    for r, c, d in ((100, 100, 0.1), (10**4, 10**4, 1e-3), (10**5, 10**5, 1e-4)):
        rp, ci, v = O.ref_gen_csr(r, c, d, 42)
        x = O.ref_gen_doubles(c, 43)
        dig[f"spmv_{r}x{c}@{d}"] = h(O.fnv1a(O.ref_spmv(rp, ci, v, x, 0, r)))
    for R, Q, D, K in ((200, 20, 8, 5), (10**5, 10**3, 16, 10)):
        rf = O.ref_gen_doubles(R * D, 42)
        q = O.ref_gen_doubles(Q * D, 43)
        i, dd = O.ref_knn(rf, q, R, Q, D, K)
        dig[f"knn_{R}x{Q}x{D}k{K}"] = h(O.fnv1a(dd, O.fnv1a(i)))
    for V, E in ((1000, 10**4), (10**5, 10**6)):
        rp, ci = O.ref_gen_graph(V, E, 42)
        dig[f"bfs_{V}v{E}e"] = h(O.fnv1a(O.ref_bfs(rp, ci, 0)))
    for n in (10**5, 10**7):
        a = O.ref_gen_doubles(n, 42)
        b = O.ref_gen_doubles(n, 43)
        dig[f"vecadd_{n}"] = h(O.fnv1a(O.ref_vecadd(a, b)))
    out["digests"] = dig

    # spmv_partition ranges (kernels.cpp:300-321) on uniform and skewed CSRs
    parts = {}
    for r, c, d in ((100, 100, 0.1), (10**4, 10**4, 1e-3)):
        rp, _, _ = O.ref_gen_csr(r, c, d, 42)
        for P in (1, 2, 3, 4, 7, 8):
            rc, rg = O.ref_spmv_partition_ranges(rp, P)
            parts[f"gen_csr_{r}x{c}@{d}_P{P}"] = {"rc": rc, "ranges": rg.tolist()}
    rng = np.random.default_rng(7)
    for t in range(6):
        rows = int(rng.integers(1, 40))
        lens = rng.integers(0, 50, rows) ** (1 + t % 3)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        for P in (1, 2, 3, 5, 8, 41):
            rc, rg = O.ref_spmv_partition_ranges(rp, P)
            parts[f"skew{t}_P{P}"] = {"row_ptr": rp.tolist(), "rc": rc,
                                      "ranges": rg.tolist() if rc == 0 else None}
    out["spmv_partition"] = parts

    # knn ties and identity KATs
    ref_pts = np.array([0, 0, 1, 0, 0, 1, 3, 4, 1, 1], np.float64)
    query = np.array([3, 4, 0.5, 0.5], np.float64)
    i, dd = O.ref_knn(ref_pts, query, 5, 2, 2, 3)
    out["knn_kat"] = {"ref": ref_pts.tolist(), "query": query.tolist(), "k": 3,
                      "idx": i.tolist(), "dist": dd.tolist()}

    # merge_topk (kernels.cpp:323-361)
    p1 = (2, np.array([1, 4, 0, 2], np.int32), np.array([0.5, 1.0, 0.25, 0.25]))
    p2 = (2, np.array([7, 9, 5, 6], np.int32), np.array([0.5, 2.0, 0.25, 3.0]))
    rc, mi, md = O.ref_merge_topk([p1, p2], 2, 3)
    out["merge_topk"] = {"rc": rc, "idx": mi.tolist(), "dist": md.tolist()}
    bad = (2, np.array([1, 4, 0, 2], np.int32), np.array([1.5, 1.0, 0.25, 0.25]))
    out["merge_topk_unsorted_rc"] = O.ref_merge_topk([bad], 2, 2)[0]

    # work_estimate (kernels.cpp:285-298)
    out["work_estimate"] = {
        "matmul": O.ref_work_estimate("matmul", [3, 5, 7], [0, 0, 0]),
        "spmv_compute": O.ref_work_estimate("spmv_compute", [0, 10], [16, 88, 800, 800, 80, 80]),
        "knn": O.ref_work_estimate("knn", [100, 10, 8, 3], [6400, 640, 120, 240]),
        "vecadd": O.ref_work_estimate("vecadd", [1000], [8000, 8000, 8000]),
    }

    # kernels::execute error codes (argument=9, name=10)
    rc_name, _, _ = O.ref_execute("nosuch", [], {})
    rc_arity, _, _ = O.ref_execute("vecadd", [("s", 1)], {})
    a = np.ones(4)
    rc_len, _, _ = O.ref_execute("vecadd", [("in", a), ("in", np.ones(3)), ("out", None), ("s", 4)],
                                 {2: 64})
    out["execute_errors"] = {"unknown_kernel": rc_name, "arity": rc_arity, "length": rc_len}

    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
