/*
 * hcl_datagen.h — synthetic input generators of the product (host side,
 * multithreaded). Replace haocl::gen_doubles / SplitMix64
 * (proj/include/haocl/datagen.hpp:13-62, proj/src/datagen.cpp:11-16) and add
 * the restated generators of the B200 configs. Every generator is counter
 * based: element i of a stream depends only on (seed, i), so `first` selects
 * any sub-range (one rank's row block) bit-identically. threads <= 0: all cores.
 */
#ifndef HCL_DATAGEN_H
#define HCL_DATAGEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t hcl_gen_splitmix_at(uint64_t seed, uint64_t index);
/* U[-1,1) doubles: element i = gen_doubles(seed)[first + i] (datagen.cpp:11-16) */
void hcl_gen_doubles(double* out, uint64_t first, uint64_t count, uint64_t seed, int threads);
/* the same values rounded to fp32 (RN) */
void hcl_gen_f32(float* out, uint64_t first, uint64_t count, uint64_t seed, int threads);
/* the same values rounded double -> fp32 -> bf16 (RN-even), bf16 bit patterns */
void hcl_gen_bf16(uint16_t* out, uint64_t first, uint64_t count, uint64_t seed, int threads);
/* R-MAT (.57,.19,.19,.05) edges [first_edge, first_edge+count) of a 2^scale graph */
void hcl_gen_rmat_edges(int scale, uint64_t first_edge, uint64_t count, uint64_t seed, uint32_t* src, uint32_t* dst,
                        int threads);
/* k-means points [first, first+count) x d, multiples of 2^-12 in [-8, 8) */
void hcl_gen_kmeans_points(uint64_t seed, uint64_t first, uint64_t count, int64_t d, int64_t blobs, float* out,
                           int threads);

/* Pull CSR (rows = dst, cols = src ascending, val = 1/outdeg(src)) of the R-MAT
 * graph with 2^scale vertices and `edges` edges; int32 indices, fp32 values.
 * row_ptr: 2^scale+1, col_idx/val: edges, outdeg: 2^scale. Returns 0. */
int hcl_pagerank_csr(int scale, uint64_t edges, uint64_t seed, int32_t* row_ptr, int32_t* col_idx, float* val,
                     int32_t* outdeg, int threads);
/* Warp work units of the PageRank SpMV: int32x4 {row0,row1,p0,p1} per unit and
 * {row, first_unit, nchunks} per long row (> warp_nnz). Pass NULL arrays to count. */
int hcl_pagerank_units(const int32_t* row_ptr, int64_t rows, int64_t warp_nnz, int32_t* units, int32_t* long_rows,
                       int64_t* n_units, int64_t* n_long);
/* Degree-ordered relabelling of a pull CSR: perm[i] = old id of new vertex i
 * (out-degree descending, ties by id); rows keep their column order (columns
 * renamed), so per-row SpMV sums are unchanged and results are permuted.
 * Outputs have the input sizes. Returns 0 or 1000+argument. */
int hcl_pagerank_relabel(const int32_t* row_ptr, const int32_t* col_idx, const float* val, const int32_t* outdeg,
                         int64_t v, int32_t* new_row_ptr, int32_t* new_col, float* new_val, int32_t* new_outdeg,
                         int32_t* perm, int threads);
/* Propagation-blocking layout of one part's rows [lo, hi) for the binned
 * PageRank step (pagerank_step_binned, csrc/host/pagerank_bins.cpp): chunks of
 * the part's edges in source order regrouped by destination bin, and the
 * bin-major destination stream. build returns an opaque handle (NULL on bad
 * arguments) and fills the sizes; export copies the arrays (any may be NULL):
 * chunks int32[8*n_chunks] {u0, span, src_off, n_edges, desc_off, n_seg, 0, 0},
 * src_local uint16[n_src], gtab uint32[(n_chunks+1)*gstride], dst16
 * uint16[n_entries], units int32[4*n_units] {bin, e0, e1, slot}, slot_units
 * int32[n_slots], cdesc uint32[n_desc] (per chunk: {bitmap, k_base} per
 * 32-entry window, then one delta per non-empty segment). */
typedef struct hcl_pr_bins_info {
  int64_t lo, hi, bin_rows, chunk_edges, span_max, unit_edges;
  int64_t n_edges, n_chunks, n_bins, gstride, n_entries, n_src, n_units, n_slots, n_desc;
} hcl_pr_bins_info;
void* hcl_pagerank_bins_build(const int32_t* row_ptr, const int32_t* col_idx, int64_t v, int64_t lo, int64_t hi,
                              int64_t bin_rows, int64_t chunk_edges, int64_t span_max, int64_t unit_edges,
                              hcl_pr_bins_info* info);
int hcl_pagerank_bins_export(void* h, int32_t* chunks, uint16_t* src_local, uint32_t* gtab, uint16_t* dst16,
                             int32_t* units, int32_t* slot_units, uint32_t* cdesc);
void hcl_pagerank_bins_free(void* h);

/* Stable counting order of n keys in [0, k): perm[i] = index of the i-th key
 * in ascending order (ties by index). Returns 0 or 1000+argument. */
int hcl_counting_order(const int32_t* keys, int64_t n, int32_t k, int32_t* perm);

/* CSR-adaptive row blocks (<= max_nnz per multi-row block); out may be NULL to
 * count. Returns the number of blocks; out[0..n] are block start rows. */
int64_t hcl_csr_row_blocks(const int32_t* row_ptr, int64_t rows, int64_t max_nnz, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
