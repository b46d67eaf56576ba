"""TEST INFRASTRUCTURE ONLY — CPU oracle for the partitioned-NDRange hot path.

Python (numpy + ctypes) front end over two checker libraries built by
``oracle/Makefile``:

* ``_build/liboracle.so`` — the plain-C restatement ``haocl_oracle.c``;
* ``_ref/libhaocl_ref.so`` — the HaoCL reference library itself, compiled in
  place from ``/root/reference/proj/src/{kernels,reference,datagen,error}.cpp``
  with the ``ref_shim.cpp`` C shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product package
``paper_2005_08466_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhaocl_ref.so")

_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)
_f32p = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_u16p = C.POINTER(C.c_uint16)


def build(force: bool = False) -> None:
    """Compile the checker libraries (no-op when present)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.isdir("/root/reference/proj/src") and not os.path.exists(REF_SO)
    ):
        subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(ORACLE_SO)
        L.ho_splitmix_at.restype = C.c_uint64
        L.ho_splitmix_at.argtypes = [C.c_uint64, C.c_uint64]
        L.ho_gen_doubles.argtypes = [_f64p, C.c_size_t, C.c_uint64]
        L.ho_gen_bf16.argtypes = [_u16p, C.c_size_t, C.c_uint64]
        L.ho_gen_csr_per_row.restype = C.c_int64
        L.ho_gen_csr_per_row.argtypes = [C.c_int64, C.c_double]
        L.ho_gen_csr.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, _i64p, _i64p, _f64p]
        L.ho_gen_graph.restype = C.c_int64
        L.ho_gen_graph.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _i64p, _i64p]
        L.ho_matmul_f64.argtypes = [_f64p, _f64p, _f64p, C.c_int64, C.c_int64, C.c_int64]
        L.ho_spmv_f64.argtypes = [_i64p, _i64p, _f64p, _f64p, C.c_int64, C.c_int64, _f64p]
        L.ho_spmv_partition_ranges.argtypes = [C.c_int64, _i64p, C.c_int64, _i64p]
        L.ho_spmv_partition_ranges_weighted.argtypes = [C.c_int64, _i64p, C.c_int64, _u64p, _i64p]
        L.ho_bfs.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, _i32p]
        L.ho_knn.argtypes = [_f64p, _f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i32p, _f64p]
        L.ho_vecadd.argtypes = [_f64p, _f64p, _f64p, C.c_int64]
        L.ho_merge_topk.argtypes = [C.c_int64, _i64p, C.POINTER(_i32p), C.POINTER(_f64p),
                                    C.c_int64, C.c_int64, _i32p, _f64p]
        L.ho_fnv1a.restype = C.c_uint64
        L.ho_fnv1a.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.ho_weighted_ranges.argtypes = [C.c_int64, C.c_int64, _u64p, _i64p]
        L.ho_rmat_edges.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64, _u32p, _u32p]
        L.ho_pagerank_csr.argtypes = [C.c_int, C.c_int64, C.c_uint64, _i32p, _i32p, _f32p, _i32p]
        L.ho_spmv_f32.argtypes = [_i32p, _i32p, _f32p, _f32p, C.c_int64, C.c_int64, _f32p]
        L.ho_pagerank.argtypes = [C.c_int64, _i32p, _i32p, _f32p, _i32p, C.c_int, C.c_int, _f32p]
        L.ho_spmv_f32_b200.argtypes = [_i32p, _i32p, _f32p, _f32p, C.c_int64, C.c_int64, _f32p]
        L.ho_kmeans_points.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.ho_kmeans_assign.argtypes = [_f32p, C.c_int64, C.c_int64, _f32p, C.c_int64, _i32p]
        L.ho_kmeans_accumulate.argtypes = [_f32p, C.c_int64, C.c_int64, _i32p, C.c_int64, _i64p, _i64p]
        L.ho_kmeans_finalize.argtypes = [_i64p, _i64p, C.c_int64, C.c_int64, _f32p]
        L.ho_conv3x3_point.argtypes = [_u16p, _u16p] + [C.c_int64] * 8 + [_f64p]
        L.ho_conv3x3_rows.argtypes = [_u16p, _u16p] + [C.c_int64] * 7 + [_f64p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference library compiled from /root/reference (oracle/_ref)."""
    global _ref
    if _ref is None:
        build()
        R = C.CDLL(REF_SO)
        R.href_last_error.restype = C.c_char_p
        R.href_matmul.argtypes = [_f64p, _f64p, _f64p, C.c_int64, C.c_int64, C.c_int64]
        R.href_spmv.argtypes = [_i64p, _i64p, _f64p, _f64p, C.c_int64, C.c_int64, _f64p]
        R.href_bfs.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, _i32p]
        R.href_knn.argtypes = [_f64p, _f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i32p, _f64p]
        R.href_vecadd.argtypes = [_f64p, _f64p, _f64p, C.c_int64]
        R.href_spmv_partition_ranges.argtypes = [C.c_int64, _i64p, C.c_int64, _i64p]
        R.href_merge_topk.argtypes = [C.c_int64, _i64p, C.POINTER(_i32p), C.POINTER(_f64p),
                                      C.c_int64, C.c_int64, _i32p, _f64p]
        R.href_work_estimate.restype = C.c_uint64
        R.href_work_estimate.argtypes = [C.c_char_p, C.c_int, _i64p, C.c_int, _u64p]
        R.href_gen_doubles.argtypes = [_f64p, C.c_uint64, C.c_uint64]
        R.href_gen_csr.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, _i64p, _i64p,
                                   _f64p, _i64p]
        R.href_gen_graph.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _i64p, _i64p, _i64p]
        R.href_execute.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int), _i64p,
                                   C.POINTER(C.c_void_p), _u64p, C.POINTER(C.c_void_p), _u64p,
                                   _u64p, C.c_int, _u64p]
        _ref = R
    return _ref


# --------------------------------------------------------------------------
# restatement front end


def fnv1a(arr, h: int = 0xCBF29CE484222325) -> int:
    a = np.ascontiguousarray(arr)
    return int(lib().ho_fnv1a(a.ctypes.data, a.nbytes, C.c_uint64(h)))


def splitmix_at(seed: int, index: int) -> int:
    return int(lib().ho_splitmix_at(seed, index))


def gen_doubles(count: int, seed: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    lib().ho_gen_doubles(_ptr(out, _f64p), count, seed)
    return out


def gen_bf16(count: int, seed: int) -> np.ndarray:
    """bf16 bit patterns (uint16) of gen_doubles rounded double->f32->bf16 (RN)."""
    out = np.empty(count, np.uint16)
    lib().ho_gen_bf16(_ptr(out, _u16p), count, seed)
    return out


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def gen_csr(rows: int, cols: int, density: float, seed: int):
    per_row = int(lib().ho_gen_csr_per_row(cols, density))
    row_ptr = np.empty(rows + 1, np.int64)
    col_idx = np.empty(rows * per_row, np.int64)
    values = np.empty(rows * per_row, np.float64)
    rc = lib().ho_gen_csr(rows, cols, density, seed, _ptr(row_ptr, _i64p), _ptr(col_idx, _i64p),
                          _ptr(values, _f64p))
    assert rc == 0
    return row_ptr, col_idx, values


def gen_graph(vertices: int, edges: int, seed: int):
    row_ptr = np.empty(vertices + 1, np.int64)
    col_idx = np.empty(2 * edges + 1, np.int64)
    m = lib().ho_gen_graph(vertices, edges, seed, _ptr(row_ptr, _i64p), _ptr(col_idx, _i64p))
    return row_ptr, col_idx[:m].copy()


def matmul_f64(a: np.ndarray, b: np.ndarray, m: int, k: int, n: int) -> np.ndarray:
    c = np.empty(m * n, np.float64)
    lib().ho_matmul_f64(_ptr(np.ascontiguousarray(a), _f64p), _ptr(np.ascontiguousarray(b), _f64p),
                        _ptr(c, _f64p), m, k, n)
    return c


def spmv_f64(row_ptr, col_idx, values, x, lo: int, hi: int) -> np.ndarray:
    y = np.empty(hi - lo, np.float64)
    lib().ho_spmv_f64(_ptr(row_ptr, _i64p), _ptr(col_idx, _i64p), _ptr(values, _f64p),
                      _ptr(x, _f64p), lo, hi, _ptr(y, _f64p))
    return y


def spmv_partition_ranges(row_ptr: np.ndarray, parts: int, weights=None) -> np.ndarray:
    rows = len(row_ptr) - 1
    out = np.empty(parts + 1, np.int64)
    if weights is None:
        rc = lib().ho_spmv_partition_ranges(rows, _ptr(row_ptr, _i64p), parts, _ptr(out, _i64p))
    else:
        w = np.ascontiguousarray(weights, np.uint64)
        rc = lib().ho_spmv_partition_ranges_weighted(rows, _ptr(row_ptr, _i64p), parts,
                                                     _ptr(w, _u64p), _ptr(out, _i64p))
    if rc:
        raise ValueError(f"partition error {rc}")
    return out


def weighted_ranges(total: int, weights) -> np.ndarray:
    w = np.ascontiguousarray(weights, np.uint64)
    out = np.empty(len(w) + 1, np.int64)
    lib().ho_weighted_ranges(total, len(w), _ptr(w, _u64p), _ptr(out, _i64p))
    return out


def bfs(row_ptr, col_idx, source: int) -> np.ndarray:
    v = len(row_ptr) - 1
    out = np.empty(v, np.int32)
    lib().ho_bfs(v, _ptr(row_ptr, _i64p), _ptr(col_idx, _i64p), source, _ptr(out, _i32p))
    return out


def knn(ref_pts, query_pts, r: int, q: int, d: int, k: int):
    idx = np.empty(q * k, np.int32)
    dist = np.empty(q * k, np.float64)
    lib().ho_knn(_ptr(ref_pts, _f64p), _ptr(query_pts, _f64p), r, q, d, k, _ptr(idx, _i32p),
                 _ptr(dist, _f64p))
    return idx, dist


def vecadd(a, b) -> np.ndarray:
    c = np.empty(len(a), np.float64)
    lib().ho_vecadd(_ptr(a, _f64p), _ptr(b, _f64p), _ptr(c, _f64p), len(a))
    return c


def _merge_args(partials):
    n = len(partials)
    ks = np.array([p[0] for p in partials], np.int64)
    idx_arrs = [np.ascontiguousarray(p[1], np.int32) for p in partials]
    dist_arrs = [np.ascontiguousarray(p[2], np.float64) for p in partials]
    ip = (_i32p * n)(*[_ptr(a, _i32p) for a in idx_arrs])
    dp = (_f64p * n)(*[_ptr(a, _f64p) for a in dist_arrs])
    return n, ks, ip, dp, (idx_arrs, dist_arrs)


def merge_topk(partials, queries: int, k: int):
    """partials: list of (k_i, idx[q*k_i], dist[q*k_i]). Returns (rc, idx, dist)."""
    n, ks, ip, dp, keep = _merge_args(partials)
    oi = np.empty(queries * k, np.int32)
    od = np.empty(queries * k, np.float64)
    rc = lib().ho_merge_topk(n, _ptr(ks, _i64p), ip, dp, queries, k, _ptr(oi, _i32p), _ptr(od, _f64p))
    return rc, oi, od


def rmat_edges(scale: int, first: int, count: int, seed: int):
    s = np.empty(count, np.uint32)
    d = np.empty(count, np.uint32)
    lib().ho_rmat_edges(scale, first, count, seed, _ptr(s, _u32p), _ptr(d, _u32p))
    return s, d


def pagerank_csr(scale: int, edges: int, seed: int):
    v = 1 << scale
    row_ptr = np.empty(v + 1, np.int32)
    col_idx = np.empty(edges, np.int32)
    val = np.empty(edges, np.float32)
    outdeg = np.empty(v, np.int32)
    rc = lib().ho_pagerank_csr(scale, edges, seed, _ptr(row_ptr, _i32p), _ptr(col_idx, _i32p),
                               _ptr(val, _f32p), _ptr(outdeg, _i32p))
    assert rc == 0
    return row_ptr, col_idx, val, outdeg


def spmv_f32(row_ptr, col_idx, val, x, lo: int, hi: int) -> np.ndarray:
    y = np.empty(hi - lo, np.float32)
    lib().ho_spmv_f32(_ptr(row_ptr, _i32p), _ptr(col_idx, _i32p), _ptr(val, _f32p),
                      _ptr(x, _f32p), lo, hi, _ptr(y, _f32p))
    return y


def spmv_f32_b200(row_ptr, col_idx, val, x, lo: int, hi: int) -> np.ndarray:
    """fp32 SpMV in the GPU kernel's fixed per-row order (see haocl_oracle.c)."""
    y = np.empty(hi - lo, np.float32)
    lib().ho_spmv_f32_b200(_ptr(row_ptr, _i32p), _ptr(col_idx, _i32p), _ptr(val, _f32p),
                           _ptr(x, _f32p), lo, hi, _ptr(y, _f32p))
    return y


def pagerank(row_ptr, col_idx, val, outdeg, iterations: int, b200_order=False) -> np.ndarray:
    """PageRank; b200_order=False sums rows in the reference's ascending order,
    True in the warp-unit kernel's restated order, "fixed" in the binned step's
    order-free 2^-56 fixed-point sums (bit-exact checks)."""
    b200_order = 2 if b200_order == "fixed" else int(bool(b200_order))
    v = len(row_ptr) - 1
    x = np.empty(v, np.float32)
    lib().ho_pagerank(v, _ptr(row_ptr, _i32p), _ptr(col_idx, _i32p), _ptr(val, _f32p),
                      _ptr(outdeg, _i32p), iterations, int(b200_order), _ptr(x, _f32p))
    return x


def kmeans_points(seed: int, first: int, count: int, d: int, blobs: int) -> np.ndarray:
    out = np.empty(count * d, np.float32)
    lib().ho_kmeans_points(seed, first, count, d, blobs, _ptr(out, _f32p))
    return out


def kmeans_assign(pts, n: int, d: int, cent, k: int) -> np.ndarray:
    out = np.empty(n, np.int32)
    lib().ho_kmeans_assign(_ptr(pts, _f32p), n, d, _ptr(cent, _f32p), k, _ptr(out, _i32p))
    return out


def kmeans_accumulate(pts, n: int, d: int, assign, k: int):
    sums = np.zeros(k * d, np.int64)
    counts = np.zeros(k, np.int64)
    lib().ho_kmeans_accumulate(_ptr(pts, _f32p), n, d, _ptr(assign, _i32p), k, _ptr(sums, _i64p),
                               _ptr(counts, _i64p))
    return sums, counts


def kmeans_finalize(sums, counts, k: int, d: int, cent) -> np.ndarray:
    out = np.array(cent, np.float32, copy=True)
    lib().ho_kmeans_finalize(_ptr(sums, _i64p), _ptr(counts, _i64p), k, d, _ptr(out, _f32p))
    return out


def conv3x3_point(inp, w, h: int, wd: int, c: int, kout: int, n: int, y: int, x: int, ko: int) -> float:
    out = C.c_double()
    lib().ho_conv3x3_point(_ptr(inp, _u16p), _ptr(w, _u16p), h, wd, c, kout, n, y, x, ko,
                           C.byref(out))
    return out.value


def conv3x3_rows(inp, w, h: int, wd: int, c: int, kout: int, n: int, y0: int, y1: int) -> np.ndarray:
    """fp64 direct conv of output rows [y0, y1) of image n: [y1-y0][wd][kout]."""
    out = np.empty((y1 - y0) * wd * kout, np.float64)
    lib().ho_conv3x3_rows(_ptr(inp, _u16p), _ptr(w, _u16p), h, wd, c, kout, n, y0, y1, _ptr(out, _f64p))
    return out.reshape(y1 - y0, wd, kout)


# --------------------------------------------------------------------------
# the reference library itself


def ref_matmul(a, b, m, k, n) -> np.ndarray:
    c = np.empty(m * n, np.float64)
    ref().href_matmul(_ptr(a, _f64p), _ptr(b, _f64p), _ptr(c, _f64p), m, k, n)
    return c


def ref_gen_doubles(count: int, seed: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    ref().href_gen_doubles(_ptr(out, _f64p), count, seed)
    return out


def ref_gen_csr(rows: int, cols: int, density: float, seed: int):
    nnz = C.c_int64()
    rc = ref().href_gen_csr(rows, cols, density, seed, None, None, None, C.byref(nnz))
    assert rc == 0
    row_ptr = np.empty(rows + 1, np.int64)
    col_idx = np.empty(nnz.value, np.int64)
    values = np.empty(nnz.value, np.float64)
    rc = ref().href_gen_csr(rows, cols, density, seed, _ptr(row_ptr, _i64p), _ptr(col_idx, _i64p),
                            _ptr(values, _f64p), C.byref(nnz))
    assert rc == 0
    return row_ptr, col_idx, values


def ref_gen_graph(vertices: int, edges: int, seed: int):
    nnz = C.c_int64()
    rc = ref().href_gen_graph(vertices, edges, seed, None, None, C.byref(nnz))
    assert rc == 0
    row_ptr = np.empty(vertices + 1, np.int64)
    col_idx = np.empty(nnz.value, np.int64)
    rc = ref().href_gen_graph(vertices, edges, seed, _ptr(row_ptr, _i64p), _ptr(col_idx, _i64p),
                              C.byref(nnz))
    assert rc == 0
    return row_ptr, col_idx


def ref_spmv(row_ptr, col_idx, values, x, lo, hi) -> np.ndarray:
    y = np.empty(hi - lo, np.float64)
    ref().href_spmv(_ptr(row_ptr, _i64p), _ptr(col_idx, _i64p), _ptr(values, _f64p),
                    _ptr(x, _f64p), lo, hi, _ptr(y, _f64p))
    return y


def ref_spmv_partition_ranges(row_ptr, parts: int):
    out = np.empty(parts + 1, np.int64)
    rc = ref().href_spmv_partition_ranges(len(row_ptr) - 1, _ptr(row_ptr, _i64p), parts,
                                          _ptr(out, _i64p))
    return rc, out


def ref_bfs(row_ptr, col_idx, source: int) -> np.ndarray:
    v = len(row_ptr) - 1
    out = np.empty(v, np.int32)
    ref().href_bfs(v, _ptr(row_ptr, _i64p), _ptr(col_idx, _i64p), source, _ptr(out, _i32p))
    return out


def ref_knn(ref_pts, query_pts, r, q, d, k):
    idx = np.empty(q * k, np.int32)
    dist = np.empty(q * k, np.float64)
    ref().href_knn(_ptr(ref_pts, _f64p), _ptr(query_pts, _f64p), r, q, d, k, _ptr(idx, _i32p),
                   _ptr(dist, _f64p))
    return idx, dist


def ref_vecadd(a, b) -> np.ndarray:
    c = np.empty(len(a), np.float64)
    ref().href_vecadd(_ptr(a, _f64p), _ptr(b, _f64p), _ptr(c, _f64p), len(a))
    return c


def ref_merge_topk(partials, queries: int, k: int):
    n, ks, ip, dp, keep = _merge_args(partials)
    oi = np.empty(queries * k, np.int32)
    od = np.empty(queries * k, np.float64)
    rc = ref().href_merge_topk(n, _ptr(ks, _i64p), ip, dp, queries, k, _ptr(oi, _i32p),
                               _ptr(od, _f64p))
    return rc, oi, od


def ref_work_estimate(kernel: str, scalars, sizes) -> int:
    s = np.ascontiguousarray(scalars, np.int64)
    z = np.ascontiguousarray(sizes, np.uint64)
    return int(ref().href_work_estimate(kernel.encode(), len(s), _ptr(s, _i64p), len(z),
                                        _ptr(z, _u64p)))


def ref_execute(kernel: str, args, out_caps, threads: int = 1):
    """Run kernels::execute. args: list of ("s", int) | ("in", ndarray) | ("out", None).
    out_caps: byte capacity per output arg (dict index->bytes). Returns (rc, work, outs)."""
    n = len(args)
    kinds = (C.c_int * n)()
    scalars = np.zeros(n, np.int64)
    in_ptrs = (C.c_void_p * n)()
    in_lens = np.zeros(n, np.uint64)
    out_ptrs = (C.c_void_p * n)()
    caps = np.zeros(n, np.uint64)
    lens = np.zeros(n, np.uint64)
    keep = []
    outs = {}
    for i, (kind, val) in enumerate(args):
        if kind == "s":
            kinds[i] = 0
            scalars[i] = val
        elif kind == "in":
            kinds[i] = 1
            arr = np.ascontiguousarray(val)
            keep.append(arr)
            in_ptrs[i] = arr.ctypes.data
            in_lens[i] = arr.nbytes
        else:
            kinds[i] = 2
            buf = np.zeros(max(1, out_caps[i]), np.uint8)
            outs[i] = buf
            out_ptrs[i] = buf.ctypes.data
            caps[i] = out_caps[i]
    work = C.c_uint64()
    rc = ref().href_execute(kernel.encode(), n, kinds, _ptr(scalars, _i64p), in_ptrs,
                            _ptr(in_lens, _u64p), out_ptrs, _ptr(caps, _u64p), _ptr(lens, _u64p),
                            threads, C.byref(work))
    res = {i: outs[i][: int(lens[i])] for i in outs}
    return rc, int(work.value), res


def ref_pagerank(row_ptr, col_idx, outdeg, iterations: int, d: float = 0.85, threads: int = 0) -> np.ndarray:
    """PageRank iterated on the REFERENCE LIBRARY's spmv_compute (fp64 values,
    int64 CSR: proj/src/kernels.cpp:132-152 through kernels::execute), with the
    damping, teleport and dangling mass applied here in fp64:
    x' = (1-d)/V + d (A x + dangling(x)/V), A_vu = 1/outdeg(u), x0 = 1/V."""
    import os

    v = len(row_ptr) - 1
    hdr = np.array([v, v], np.int64)
    rp64 = np.ascontiguousarray(row_ptr, np.int64)
    ci64 = np.ascontiguousarray(col_idx, np.int64)
    deg = np.asarray(outdeg)
    val64 = 1.0 / deg[col_idx].astype(np.float64)
    x = np.full(v, 1.0 / v)
    for _ in range(iterations):
        dang = float(x[deg == 0].sum())
        rc, _, out = ref_execute("spmv_compute", [("in", hdr), ("in", rp64), ("in", ci64), ("in", val64), ("in", x),
                                                  ("s", 0), ("s", v), ("out", None)], {7: v * 8},
                                 threads=threads or os.cpu_count() or 1)
        if rc != 0:
            raise RuntimeError(f"reference spmv_compute failed: {rc}")
        x = (1.0 - d) / v + d * (out[7].view(np.float64) + dang / v)
    return x
