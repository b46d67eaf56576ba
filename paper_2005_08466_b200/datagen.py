"""Synthetic inputs (include/hcl_datagen.h): the reference's SplitMix64
streams, counter based so any row block of any rank is generated directly,
multithreaded on the host. `out` may be a numpy array or a (pinned) torch CPU
tensor of the right dtype and size."""
from __future__ import annotations

import numpy as np

from . import _native as N


def _ptr(out):
    if isinstance(out, np.ndarray):
        return out.ctypes.data
    return int(out.data_ptr())


def splitmix_at(seed: int, index: int) -> int:
    return int(N.lib().hcl_gen_splitmix_at(seed, index))


def gen_doubles(count: int, seed: int, first: int = 0, out=None, threads: int = 0):
    out = np.empty(count, np.float64) if out is None else out
    N.lib().hcl_gen_doubles(_ptr(out), first, count, seed, threads)
    return out


def gen_f32(count: int, seed: int, first: int = 0, out=None, threads: int = 0):
    out = np.empty(count, np.float32) if out is None else out
    N.lib().hcl_gen_f32(_ptr(out), first, count, seed, threads)
    return out


def gen_bf16(count: int, seed: int, first: int = 0, out=None, threads: int = 0):
    """bf16 bit patterns (uint16) of gen_doubles rounded double->f32->bf16."""
    out = np.empty(count, np.uint16) if out is None else out
    N.lib().hcl_gen_bf16(_ptr(out), first, count, seed, threads)
    return out


def gen_rmat_edges(scale: int, count: int, seed: int, first: int = 0, threads: int = 0):
    src = np.empty(count, np.uint32)
    dst = np.empty(count, np.uint32)
    N.lib().hcl_gen_rmat_edges(scale, first, count, seed, src.ctypes.data, dst.ctypes.data, threads)
    return src, dst


def gen_kmeans_points(count: int, d: int, blobs: int, seed: int, first: int = 0, out=None, threads: int = 0):
    out = np.empty(count * d, np.float32) if out is None else out
    N.lib().hcl_gen_kmeans_points(seed, first, count, d, blobs, _ptr(out), threads)
    return out


def pagerank_csr(scale: int, edges: int, seed: int, threads: int = 0):
    """Pull CSR of the R-MAT graph: (row_ptr int32[V+1], col_idx int32[E],
    val fp32[E] = 1/outdeg(src), outdeg int32[V])."""
    v = 1 << scale
    row_ptr = np.empty(v + 1, np.int32)
    col_idx = np.empty(edges, np.int32)
    val = np.empty(edges, np.float32)
    outdeg = np.empty(v, np.int32)
    rc = N.lib().hcl_pagerank_csr(scale, edges, seed, row_ptr.ctypes.data, col_idx.ctypes.data, val.ctypes.data,
                                  outdeg.ctypes.data, threads)
    if rc:
        raise N.HaoclError(rc - N.HCL_ERR_BASE, "pagerank_csr: bad arguments")
    return row_ptr, col_idx, val, outdeg


def pagerank_units(row_ptr: np.ndarray, warp_nnz: int):
    """Warp work units of the PageRank SpMV: (units int32[n,4] {row0,row1,p0,p1},
    long_rows int32[max(m,1),3] {row, first_unit, nchunks}, m)."""
    import ctypes as C

    rp = np.ascontiguousarray(row_ptr, np.int32)
    nu, nl = C.c_int64(), C.c_int64()
    rc = N.lib().hcl_pagerank_units(rp.ctypes.data, len(rp) - 1, warp_nnz, None, None, C.byref(nu), C.byref(nl))
    if rc:
        raise N.HaoclError(rc - N.HCL_ERR_BASE, "pagerank_units: warp_nnz must be in [1, 4096]")
    units = np.empty((nu.value, 4), np.int32)
    long_rows = np.empty((max(1, nl.value), 3), np.int32)
    N.lib().hcl_pagerank_units(rp.ctypes.data, len(rp) - 1, warp_nnz, units.ctypes.data, long_rows.ctypes.data,
                               C.byref(nu), C.byref(nl))
    return units, long_rows, nl.value


def pagerank_relabel(row_ptr, col_idx, val, outdeg, threads: int = 0):
    """Degree-ordered relabelling (hcl_pagerank_relabel): returns
    (row_ptr, col_idx, val, outdeg, perm) of the relabelled graph, perm[i] =
    old id of new vertex i. Ranks map back as old[perm] = new."""
    v = len(row_ptr) - 1
    rp = np.ascontiguousarray(row_ptr, np.int32)
    ci = np.ascontiguousarray(col_idx, np.int32)
    va = np.ascontiguousarray(val, np.float32)
    od = np.ascontiguousarray(outdeg, np.int32)
    out = (np.empty_like(rp), np.empty_like(ci), np.empty_like(va), np.empty_like(od), np.empty(v, np.int32))
    rc = N.lib().hcl_pagerank_relabel(rp.ctypes.data, ci.ctypes.data, va.ctypes.data, od.ctypes.data, v,
                                      *(a.ctypes.data for a in out), threads)
    if rc:
        raise N.HaoclError(rc - N.HCL_ERR_BASE, "pagerank_relabel: bad arguments")
    return out


def csr_row_blocks(row_ptr: np.ndarray, max_nnz: int) -> np.ndarray:
    """CSR-adaptive row blocks: start rows of blocks of <= max_nnz non-zeros
    (a longer row is its own block); last entry = rows."""
    rp = np.ascontiguousarray(row_ptr, np.int32)
    n = int(N.lib().hcl_csr_row_blocks(rp.ctypes.data, len(rp) - 1, max_nnz, None))
    out = np.empty(n + 1, np.int32)
    N.lib().hcl_csr_row_blocks(rp.ctypes.data, len(rp) - 1, max_nnz, out.ctypes.data)
    return out


def pagerank_inv_outdeg(outdeg: np.ndarray) -> np.ndarray:
    """fp32 fl(1/outdeg) per vertex, 0 for dangling vertices: the reciprocal the CSR
    builder stores as val (IEEE round-to-nearest division, as __fdiv_rn), computed
    once per graph for pagerank_step_exchange."""
    d = np.asarray(outdeg, np.int32)
    inv = np.zeros(len(d), np.float32)
    nz = d > 0
    inv[nz] = np.float32(1.0) / d[nz].astype(np.float32)
    return inv
