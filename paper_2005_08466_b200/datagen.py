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


# binned (propagation-blocking) PageRank layout defaults: 8192-row bins (the
# gather's shared-memory accumulator is bin_rows x 8 bytes: two gather CTAs per
# SM; dst16 offsets need bin_rows <= 65536), chunks of <= 65536 edges spanning
# <= 16384 sources (the scatter stages a chunk's descriptor, src_local and gather
# inputs in shared memory: 216 KB at these limits). Measured at C3 on B200 (ms
# per iteration): 8192-row bins 0.977, 16384-row 1.002; 65536-edge chunks 1.00,
# 32768 1.12-1.15, 16384 1.25-1.27 -- the per-chunk cost dominates; spans of
# 16384 sources 0.967 vs 8192 0.993 (fewer, fuller chunks)
PR_BIN_ROWS, PR_CHUNK_EDGES, PR_SPAN_MAX = 8192, 65536, 16384


def pagerank_bins(row_ptr: np.ndarray, col_idx: np.ndarray, lo: int = 0, hi: int | None = None,
                  bin_rows: int = PR_BIN_ROWS, chunk_edges: int = PR_CHUNK_EDGES, span_max: int = PR_SPAN_MAX,
                  unit_edges: int = 0) -> dict:
    """Propagation-blocking layout of rows [lo, hi) (hcl_pagerank_bins_build):
    a dict of numpy arrays (chunks, src_local, gtab, dst16, units, slot_units, cdesc)
    plus the sizes. unit_edges = 0 sizes the gather units for ~4 per SM of a
    148-SM B200 (heavy bins split, the rest one unit per bin)."""
    import ctypes as C

    rp = np.ascontiguousarray(row_ptr, np.int32)
    ci = np.ascontiguousarray(col_idx, np.int32)
    v = len(rp) - 1
    hi = v if hi is None else hi
    if unit_edges <= 0:
        unit_edges = max(4096, int(rp[hi]) - int(rp[lo])) // (148 * 4) + 8
    info = N.PrBinsInfo()
    h = N.lib().hcl_pagerank_bins_build(rp.ctypes.data, ci.ctypes.data, v, lo, hi, bin_rows, chunk_edges, span_max,
                                        unit_edges, C.byref(info))
    if not h:
        raise N.HaoclError(9, "pagerank_bins: bad arguments")
    try:
        out = {f: int(getattr(info, f)) for f, _ in N.PrBinsInfo._fields_}
        out["chunks"] = np.empty(8 * info.n_chunks, np.int32)
        out["src_local"] = np.empty(max(1, info.n_src), np.uint16)
        out["gtab"] = np.empty((info.n_chunks + 1) * info.gstride, np.uint32)
        out["dst16"] = np.empty(max(8, info.n_entries), np.uint16)
        out["units"] = np.empty(max(4, 4 * info.n_units), np.int32)
        out["slot_units"] = np.empty(max(1, info.n_slots), np.int32)
        out["cdesc"] = np.empty(max(4, info.n_desc), np.uint32)
        N.lib().hcl_pagerank_bins_export(h, *(out[k].ctypes.data for k in
                                              ("chunks", "src_local", "gtab", "dst16", "units", "slot_units",
                                               "cdesc")))
    finally:
        N.lib().hcl_pagerank_bins_free(h)
    return out


def counting_order(keys: np.ndarray, k: int) -> np.ndarray:
    """Stable order of keys in [0, k) (hcl_counting_order): int32 indices."""
    keys = np.ascontiguousarray(keys, np.int32)
    perm = np.empty(len(keys), np.int32)
    rc = N.lib().hcl_counting_order(keys.ctypes.data, len(keys), k, perm.ctypes.data)
    if rc != 0:
        raise N.HaoclError(rc - N.HCL_ERR_BASE, "counting_order: keys outside [0, k)")
    return perm
