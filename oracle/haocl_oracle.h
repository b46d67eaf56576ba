/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the partitioned-NDRange hot path.
 *
 * This is a plain-C restatement of the HaoCL reference algorithms (and of the
 * restated B200 workloads that follow the reference's conventions). It is the
 * CHECKER: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product path
 * (paper_2005_08466_b200/) never links or calls it.
 *
 * Parity pinning: every reference-covered function is checked by
 * tests/test_oracle.py against (1) the FNV-1a golden digests measured from the
 * reference itself, and (2) the reference library compiled
 * from /root/reference sources into oracle/_ref/ (oracle/Makefile), via the
 * committed fixtures in tests/golden/.
 *
 * Conventions copied from the reference (cited per function in the .c):
 *   - ascending summation order, separate multiply and add (no FP contraction,
 *     proj/src/CMakeLists.txt:22-24 builds with -ffp-contract=off);
 *   - (value, index) lexicographic order, ties to the smaller index
 *     (proj/src/kernels.cpp:224-225);
 *   - SplitMix64 streams with seed / seed+1 (proj/include/haocl/datagen.hpp:13-31,
 *     proj/src/bench.cpp:149-150).
 */
#ifndef HAOCL_ORACLE_H
#define HAOCL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- datagen (proj/include/haocl/datagen.hpp, proj/src/datagen.cpp) ---- */
uint64_t ho_splitmix_next(uint64_t* state);
uint64_t ho_splitmix_at(uint64_t seed, uint64_t index); /* index-th output, 0-based */
void ho_gen_doubles(double* out, size_t count, uint64_t seed);
int64_t ho_gen_csr_per_row(int64_t cols, double density);
int ho_gen_csr(int64_t rows, int64_t cols, double density, uint64_t seed, int64_t* row_ptr,
               int64_t* col_idx, double* values);
/* col_idx must hold 2*edges entries; returns nnz, or -1 on error */
int64_t ho_gen_graph(int64_t vertices, int64_t edges, uint64_t seed, int64_t* row_ptr,
                     int64_t* col_idx);

/* ---- reference kernels (proj/src/reference.cpp, proj/src/kernels.cpp) ---- */
void ho_matmul_f64(const double* a, const double* b, double* c, int64_t m, int64_t k, int64_t n);
void ho_spmv_f64(const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                 const double* x, int64_t lo, int64_t hi, double* y);
int ho_spmv_partition_ranges(int64_t rows, const int64_t* row_ptr, int64_t parts, int64_t* out);
int ho_spmv_partition_ranges_weighted(int64_t rows, const int64_t* row_ptr, int64_t parts,
                                      const uint64_t* weights, int64_t* out);
void ho_bfs(int64_t vertices, const int64_t* row_ptr, const int64_t* col_idx, int64_t source,
            int32_t* levels);
void ho_knn(const double* ref_pts, const double* query_pts, int64_t r, int64_t q, int64_t d,
            int64_t k, int32_t* idx, double* dist);
void ho_vecadd(const double* a, const double* b, double* c, int64_t n);
int ho_merge_topk(int64_t nparts, const int64_t* part_k, const int32_t* const* part_idx,
                  const double* const* part_dist, int64_t queries, int64_t k, int32_t* out_idx,
                  double* out_dist);
uint64_t ho_fnv1a(const void* bytes, size_t len, uint64_t h);
void ho_block_range(int64_t total, int64_t parts, int64_t index, int64_t* lo, int64_t* hi);
void ho_weighted_ranges(int64_t total, int64_t parts, const uint64_t* weights, int64_t* out);

/* ---- restated B200 workloads (not in the reference; follow its conventions) ---- */
void ho_rmat_edges(int scale, int64_t first_edge, int64_t count, uint64_t seed, uint32_t* src,
                   uint32_t* dst);
int ho_pagerank_csr(int scale, int64_t edges, uint64_t seed, int32_t* row_ptr, int32_t* col_idx,
                    float* val, int32_t* outdeg);
void ho_spmv_f32(const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                 const float* x, int64_t lo, int64_t hi, float* y);
void ho_spmv_f32_b200(const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                      const float* x, int64_t lo, int64_t hi, float* y);
void ho_spmv_f32_fixed(const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                       const float* x, int64_t lo, int64_t hi, float* y);
void ho_pagerank(int64_t v, const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                 const int32_t* outdeg, int iterations, int b200_order, float* x);
void ho_kmeans_points(uint64_t seed, int64_t first, int64_t count, int64_t d, int64_t blobs,
                      float* out);
void ho_kmeans_assign(const float* pts, int64_t n, int64_t d, const float* cent, int64_t k,
                      int32_t* assign);
void ho_kmeans_accumulate(const float* pts, int64_t n, int64_t d, const int32_t* assign,
                          int64_t k, int64_t* sums, int64_t* counts);
void ho_kmeans_finalize(const int64_t* sums, const int64_t* counts, int64_t k, int64_t d,
                        float* cent);
void ho_conv3x3_point(const uint16_t* in_bf16, const uint16_t* w_bf16, int64_t h, int64_t w,
                      int64_t c, int64_t kout, int64_t n_img, int64_t y, int64_t x, int64_t ko,
                      double* out);
void ho_conv3x3_rows(const uint16_t* in_bf16, const uint16_t* w_bf16, int64_t h, int64_t w, int64_t c,
                     int64_t kout, int64_t n_img, int64_t y0, int64_t y1, double* out);
void ho_gen_bf16(uint16_t* out, size_t count, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
