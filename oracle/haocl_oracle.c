/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (checker) for the partitioned-NDRange
 * hot path. See haocl_oracle.h for the contract. Compiled by oracle/Makefile
 * with -O2 -ffp-contract=off (the reference's own flag,
 * proj/src/CMakeLists.txt:22-24), so every a*b+c below is a rounded multiply
 * followed by a rounded add, exactly as in the reference.
 */
#include "haocl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* SplitMix64 — proj/include/haocl/datagen.hpp:13-31                          */

#define SM_GAMMA 0x9e3779b97f4a7c15ULL

static inline uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t ho_splitmix_next(uint64_t* state) { return sm_mix(*state += SM_GAMMA); }

/* The generator is counter based: the i-th output (0-based) of a stream seeded
 * with `seed` is mix(seed + (i+1)*gamma). Used by the restated generators so
 * that any sub-range can be produced independently (and on the GPU). */
uint64_t ho_splitmix_at(uint64_t seed, uint64_t index) {
  return sm_mix(seed + (index + 1) * SM_GAMMA);
}

static inline double sm_double(uint64_t* s) {
  return (double)(ho_splitmix_next(s) >> 11) * 0x1.0p-53;
}

/* gen_doubles: U[-1,1) — proj/src/datagen.cpp:11-16 */
void ho_gen_doubles(double* out, size_t count, uint64_t seed) {
  uint64_t s = seed;
  for (size_t i = 0; i < count; ++i) out[i] = sm_double(&s) * 2.0 - 1.0;
}

/* bf16 of gen_doubles: double -> float (RN) -> bf16 (RNE). Restated input
 * encoding for the bf16 GEMM / conv configs. */
static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

void ho_gen_bf16(uint16_t* out, size_t count, uint64_t seed) {
  uint64_t s = seed;
  for (size_t i = 0; i < count; ++i) {
    double x = sm_double(&s) * 2.0 - 1.0;
    out[i] = f32_to_bf16_rne((float)x);
  }
}

/* gen_csr — proj/src/datagen.cpp:18-40: per row, draw next_below(cols) until
 * per_row distinct columns are collected (std::set), then one value per column
 * in ascending column order. */
int64_t ho_gen_csr_per_row(int64_t cols, double density) {
  int64_t per_row = 0;
  if (density > 0.0) {
    per_row = (int64_t)(density * (double)cols + 0.5);
    if (per_row < 1) per_row = 1;
  }
  if (per_row > cols) per_row = cols;
  return per_row;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

int ho_gen_csr(int64_t rows, int64_t cols, double density, uint64_t seed, int64_t* row_ptr,
               int64_t* col_idx, double* values) {
  if (rows < 1 || cols < 1 || density < 0.0 || density > 1.0) return 9;
  int64_t per_row = ho_gen_csr_per_row(cols, density);
  uint8_t* seen = (uint8_t*)calloc((size_t)cols, 1);
  if (!seen) return 0;
  uint64_t s = seed;
  int64_t nnz = 0;
  row_ptr[0] = 0;
  for (int64_t i = 0; i < rows; ++i) {
    int64_t* row = col_idx + nnz;
    int64_t have = 0;
    while (have < per_row) {
      uint64_t r = ho_splitmix_next(&s);
      int64_t c = (int64_t)(r % (uint64_t)cols);
      if (!seen[c]) {
        seen[c] = 1;
        row[have++] = c;
      }
    }
    qsort(row, (size_t)have, sizeof(int64_t), cmp_i64);
    for (int64_t j = 0; j < have; ++j) {
      seen[row[j]] = 0;
      values[nnz + j] = sm_double(&s) * 2.0 - 1.0;
    }
    nnz += have;
    row_ptr[i + 1] = nnz;
  }
  free(seen);
  return 0;
}

/* gen_graph — proj/src/datagen.cpp:42-68: G(n,m), both directions, sorted,
 * duplicates and self loops removed. */
typedef struct {
  int64_t u, v;
} arc_t;

static int cmp_arc(const void* a, const void* b) {
  const arc_t* x = (const arc_t*)a;
  const arc_t* y = (const arc_t*)b;
  if (x->u != y->u) return (x->u > y->u) - (x->u < y->u);
  return (x->v > y->v) - (x->v < y->v);
}

int64_t ho_gen_graph(int64_t vertices, int64_t edges, uint64_t seed, int64_t* row_ptr,
                     int64_t* col_idx) {
  if (vertices < 1) return -1;
  arc_t* arcs = (arc_t*)malloc(sizeof(arc_t) * (size_t)(2 * edges + 1));
  if (!arcs) return -1;
  uint64_t s = seed;
  int64_t n = 0;
  for (int64_t e = 0; e < edges; ++e) {
    int64_t u = (int64_t)(ho_splitmix_next(&s) % (uint64_t)vertices);
    int64_t v = (int64_t)(ho_splitmix_next(&s) % (uint64_t)vertices);
    if (u == v) continue;
    arcs[n].u = u; arcs[n].v = v; ++n;
    arcs[n].u = v; arcs[n].v = u; ++n;
  }
  qsort(arcs, (size_t)n, sizeof(arc_t), cmp_arc);
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (m == 0 || arcs[i].u != arcs[m - 1].u || arcs[i].v != arcs[m - 1].v) arcs[m++] = arcs[i];
  memset(row_ptr, 0, sizeof(int64_t) * (size_t)(vertices + 1));
  for (int64_t i = 0; i < m; ++i) {
    row_ptr[arcs[i].u + 1]++;
    col_idx[i] = arcs[i].v;
  }
  for (int64_t i = 0; i < vertices; ++i) row_ptr[i + 1] += row_ptr[i];
  free(arcs);
  return m;
}

/* ------------------------------------------------------------------------- */
/* Reference kernels                                                          */

/* matmul — proj/src/reference.cpp:8-17 (naive i-j-k, k ascending). Restated in
 * i-k-j order with a zero-initialised row accumulator, which performs the same
 * per-element sequence 0 + a0*b0 + a1*b1 + ... (proj/src/kernels.cpp:107-117). */
void ho_matmul_f64(const double* a, const double* b, double* c, int64_t m, int64_t k,
                   int64_t n) {
  for (int64_t i = 0; i < m; ++i) {
    double* crow = c + i * n;
    for (int64_t j = 0; j < n; ++j) crow[j] = 0.0;
    for (int64_t p = 0; p < k; ++p) {
      double aik = a[i * k + p];
      const double* brow = b + p * n;
      for (int64_t j = 0; j < n; ++j) crow[j] += aik * brow[j];
    }
  }
}

/* spmv — proj/src/reference.cpp:19-27 */
void ho_spmv_f64(const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                 const double* x, int64_t lo, int64_t hi, double* y) {
  for (int64_t i = lo; i < hi; ++i) {
    double sum = 0.0;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) sum += values[p] * x[col_idx[p]];
    y[i - lo] = sum;
  }
}

/* spmv_partition_ranges — proj/src/kernels.cpp:300-321. Greedy sweep toward
 * ceil(nnz/P); every part takes >= 1 row and leaves >= 1 row per later part. */
int ho_spmv_partition_ranges(int64_t rows, const int64_t* row_ptr, int64_t parts, int64_t* out) {
  if (parts < 1 || parts > rows) return 9;
  int64_t nnz_total = row_ptr[rows];
  int64_t target = (nnz_total + parts - 1) / parts;
  out[0] = 0;
  int64_t row = 0;
  for (int64_t p = 0; p + 1 < parts; ++p) {
    int64_t max_end = rows - (parts - 1 - p);
    int64_t end = row, acc = 0;
    do {
      acc += row_ptr[end + 1] - row_ptr[end];
      ++end;
    } while (end < max_end && acc < target);
    out[p + 1] = end;
    row = end;
  }
  out[parts] = rows;
  return 0;
}

/* Weighted generalisation: part p targets
 * ceil(nnz * w_p / W); equal weights reduce exactly to the function above. */
int ho_spmv_partition_ranges_weighted(int64_t rows, const int64_t* row_ptr, int64_t parts,
                                      const uint64_t* weights, int64_t* out) {
  if (parts < 1 || parts > rows) return 9;
  unsigned __int128 wsum = 0;
  for (int64_t p = 0; p < parts; ++p) wsum += weights[p];
  if (wsum == 0) return 9;
  int64_t nnz_total = row_ptr[rows];
  out[0] = 0;
  int64_t row = 0;
  for (int64_t p = 0; p + 1 < parts; ++p) {
    unsigned __int128 num = (unsigned __int128)(uint64_t)nnz_total * weights[p];
    int64_t target = (int64_t)((num + wsum - 1) / wsum);
    int64_t max_end = rows - (parts - 1 - p);
    int64_t end = row, acc = 0;
    do {
      acc += row_ptr[end + 1] - row_ptr[end];
      ++end;
    } while (end < max_end && acc < target);
    out[p + 1] = end;
    row = end;
  }
  out[parts] = rows;
  return 0;
}

/* bfs — proj/src/reference.cpp:29-47 (queue BFS) */
void ho_bfs(int64_t vertices, const int64_t* row_ptr, const int64_t* col_idx, int64_t source,
            int32_t* levels) {
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)(vertices > 0 ? vertices : 1));
  for (int64_t i = 0; i < vertices; ++i) levels[i] = -1;
  levels[source] = 0;
  int64_t head = 0, tail = 0;
  queue[tail++] = source;
  while (head < tail) {
    int64_t u = queue[head++];
    for (int64_t p = row_ptr[u]; p < row_ptr[u + 1]; ++p) {
      int64_t v = col_idx[p];
      if (levels[v] == -1) {
        levels[v] = levels[u] + 1;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
}

/* knn — proj/src/reference.cpp:49-69: squared distance with diff = ref - query,
 * ascending d, then the k smallest (dist, idx) pairs in lexicographic order.
 * Selection of the k smallest under a strict total order equals the full sort's
 * prefix. */
static inline int pair_less(double da, int32_t ia, double db, int32_t ib) {
  return da < db || (da == db && ia < ib);
}

void ho_knn(const double* ref_pts, const double* query_pts, int64_t r, int64_t q, int64_t d,
            int64_t k, int32_t* idx, double* dist) {
  double* bd = (double*)malloc(sizeof(double) * (size_t)k);
  int32_t* bi = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  for (int64_t qi = 0; qi < q; ++qi) {
    const double* query = query_pts + qi * d;
    int64_t have = 0;
    for (int64_t ri = 0; ri < r; ++ri) {
      const double* point = ref_pts + ri * d;
      double sum = 0.0;
      for (int64_t di = 0; di < d; ++di) {
        double diff = point[di] - query[di];
        sum += diff * diff;
      }
      int32_t id = (int32_t)ri;
      if (have < k) {
        int64_t pos = have++;
        while (pos > 0 && pair_less(sum, id, bd[pos - 1], bi[pos - 1])) {
          bd[pos] = bd[pos - 1]; bi[pos] = bi[pos - 1]; --pos;
        }
        bd[pos] = sum; bi[pos] = id;
      } else if (pair_less(sum, id, bd[k - 1], bi[k - 1])) {
        int64_t pos = k - 1;
        while (pos > 0 && pair_less(sum, id, bd[pos - 1], bi[pos - 1])) {
          bd[pos] = bd[pos - 1]; bi[pos] = bi[pos - 1]; --pos;
        }
        bd[pos] = sum; bi[pos] = id;
      }
    }
    for (int64_t ki = 0; ki < k; ++ki) {
      idx[qi * k + ki] = bi[ki];
      dist[qi * k + ki] = bd[ki];
    }
  }
  free(bd);
  free(bi);
}

/* vecadd — proj/src/reference.cpp:71-73 */
void ho_vecadd(const double* a, const double* b, double* c, int64_t n) {
  for (int64_t i = 0; i < n; ++i) c[i] = a[i] + b[i];
}

/* merge_topk — proj/src/kernels.cpp:323-361. Returns 0, 9 (argument) or
 * 22 (contract) like the reference's ErrorCode values. */
int ho_merge_topk(int64_t nparts, const int64_t* part_k, const int32_t* const* part_idx,
                  const double* const* part_dist, int64_t queries, int64_t k, int32_t* out_idx,
                  double* out_dist) {
  if (k < 1) return 9;
  int64_t total = 0;
  for (int64_t p = 0; p < nparts; ++p) {
    total += part_k[p];
    for (int64_t qi = 0; qi < queries; ++qi)
      for (int64_t i = 1; i < part_k[p]; ++i) {
        int64_t at = qi * part_k[p] + i;
        if (pair_less(part_dist[p][at], part_idx[p][at], part_dist[p][at - 1],
                      part_idx[p][at - 1]))
          return 22;
      }
  }
  if (total < k) return 22;
  /* gather all candidates per query and selection-sort the k smallest pairs:
   * the same prefix std::partial_sort yields under the strict pair order */
  double* pd = (double*)malloc(sizeof(double) * (size_t)total);
  int32_t* pi = (int32_t*)malloc(sizeof(int32_t) * (size_t)total);
  for (int64_t qi = 0; qi < queries; ++qi) {
    int64_t n = 0;
    for (int64_t p = 0; p < nparts; ++p)
      for (int64_t i = 0; i < part_k[p]; ++i) {
        pd[n] = part_dist[p][qi * part_k[p] + i];
        pi[n] = part_idx[p][qi * part_k[p] + i];
        ++n;
      }
    for (int64_t i = 0; i < k; ++i) {
      int64_t best = i;
      for (int64_t j = i + 1; j < n; ++j)
        if (pair_less(pd[j], pi[j], pd[best], pi[best])) best = j;
      double td = pd[i]; pd[i] = pd[best]; pd[best] = td;
      int32_t ti = pi[i]; pi[i] = pi[best]; pi[best] = ti;
      out_dist[qi * k + i] = pd[i];
      out_idx[qi * k + i] = pi[i];
    }
  }
  free(pd);
  free(pi);
  return 0;
}

/* FNV-1a-64 — proj/src/bench.cpp:35-41 */
uint64_t ho_fnv1a(const void* bytes, size_t len, uint64_t h) {
  const uint8_t* p = (const uint8_t*)bytes;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* block_range — proj/src/bench.cpp:31-33 */
void ho_block_range(int64_t total, int64_t parts, int64_t index, int64_t* lo, int64_t* hi) {
  *lo = total * index / parts;
  *hi = total * (index + 1) / parts;
}

/* Cumulative-floor weighted split:
 * boundary_i = floor(T * W_{<i} / W) in 128-bit arithmetic. Equal weights give
 * block_range exactly. out holds parts+1 boundaries. */
void ho_weighted_ranges(int64_t total, int64_t parts, const uint64_t* weights, int64_t* out) {
  unsigned __int128 wsum = 0;
  for (int64_t p = 0; p < parts; ++p) wsum += weights[p];
  unsigned __int128 acc = 0;
  out[0] = 0;
  for (int64_t p = 0; p < parts; ++p) {
    acc += weights[p];
    out[p + 1] = (int64_t)(((unsigned __int128)(uint64_t)total * acc) / wsum);
  }
}

/* ------------------------------------------------------------------------- */
/* Restated workloads                                                         */

/* R-MAT (a,b,c,d) = (.57,.19,.19,.05) as exact 32-bit thresholds. Edge e,
 * level l consumes SplitMix64 output e*scale + l of the stream `seed`; the
 * upper 32 bits select the quadrant. Fully counter based. */
#define RMAT_T1 2448131358u
#define RMAT_T2 3264175144u
#define RMAT_T3 4080218930u

void ho_rmat_edges(int scale, int64_t first_edge, int64_t count, uint64_t seed, uint32_t* src,
                   uint32_t* dst) {
  for (int64_t i = 0; i < count; ++i) {
    uint64_t e = (uint64_t)(first_edge + i);
    uint32_t s = 0, d = 0;
    for (int l = 0; l < scale; ++l) {
      uint32_t u = (uint32_t)(ho_splitmix_at(seed, e * (uint64_t)scale + (uint64_t)l) >> 32);
      uint32_t bs = u >= RMAT_T2;               /* quadrants c, d */
      uint32_t bd = (u >= RMAT_T1 && u < RMAT_T2) || u >= RMAT_T3; /* b, d */
      s = (s << 1) | bs;
      d = (d << 1) | bd;
    }
    src[i] = s;
    dst[i] = d;
  }
}

/* Pull CSR by destination: row = dst, columns = src sorted ascending (multi
 * edges kept), val = 1.0f / outdeg(src). Counting sort by src then a stable
 * counting sort by dst gives the (dst, src) order. */
int ho_pagerank_csr(int scale, int64_t edges, uint64_t seed, int32_t* row_ptr, int32_t* col_idx,
                    float* val, int32_t* outdeg) {
  int64_t v = (int64_t)1 << scale;
  uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)edges);
  uint32_t* dst = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)edges);
  uint32_t* tmp_src = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)edges);
  uint32_t* tmp_dst = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)edges);
  int64_t* cnt = (int64_t*)calloc((size_t)v + 1, sizeof(int64_t));
  if (!src || !dst || !tmp_src || !tmp_dst || !cnt) return 1;
  ho_rmat_edges(scale, 0, edges, seed, src, dst);
  /* stable counting sort by src */
  for (int64_t i = 0; i < edges; ++i) cnt[src[i] + 1]++;
  for (int64_t i = 0; i < v; ++i) cnt[i + 1] += cnt[i];
  for (int64_t i = 0; i < v; ++i) outdeg[i] = (int32_t)(cnt[i + 1] - cnt[i]);
  for (int64_t i = 0; i < edges; ++i) {
    int64_t at = cnt[src[i]]++;
    tmp_src[at] = src[i];
    tmp_dst[at] = dst[i];
  }
  /* stable counting sort by dst */
  memset(cnt, 0, sizeof(int64_t) * ((size_t)v + 1));
  for (int64_t i = 0; i < edges; ++i) cnt[tmp_dst[i] + 1]++;
  for (int64_t i = 0; i < v; ++i) cnt[i + 1] += cnt[i];
  for (int64_t i = 0; i <= v; ++i) row_ptr[i] = (int32_t)cnt[i];
  for (int64_t i = 0; i < edges; ++i) {
    int64_t at = cnt[tmp_dst[i]]++;
    col_idx[at] = (int32_t)tmp_src[i];
    val[at] = 1.0f / (float)outdeg[tmp_src[i]];
  }
  free(src); free(dst); free(tmp_src); free(tmp_dst); free(cnt);
  return 0;
}

/* spmv fp32 — the reference spmv (proj/src/reference.cpp:19-27) in fp32 with
 * int32 indices: ascending storage order, separate multiply and add. */
void ho_spmv_f32(const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                 const float* x, int64_t lo, int64_t hi, float* y) {
  for (int64_t i = lo; i < hi; ++i) {
    float sum = 0.0f;
    for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) sum += val[p] * x[col_idx[p]];
    y[i - lo] = sum;
  }
}

/* The GPU kernel's fixed per-row summation order (csrc/k_graph.cu), restated
 * so the CUDA path can be checked bit-for-bit; it depends only on the row's
 * length, never on the partition. Rows of <= 32 products: ascending (the
 * reference's order, reference.cpp:22-25). Longer rows: 4096-element chunks;
 * in a chunk, lane l (0..31) sums elements l, l+32, ... sequentially, then an
 * xor butterfly (offsets 16, 8, 4, 2, 1) combines the lanes (lane 0's value);
 * chunk totals are added in chunk order. */
static float row_sum_b200(const int32_t* col_idx, const float* val, const float* x, int64_t p0, int64_t n) {
  if (n <= 32) {
    float s = 0.0f;
    for (int64_t q = 0; q < n; ++q) s += val[p0 + q] * x[col_idx[p0 + q]];
    return s;
  }
  float total = 0.0f;
  int first = 1;
  for (int64_t c0 = 0; c0 < n; c0 += 4096) {
    int64_t cl = n - c0 < 4096 ? n - c0 : 4096;
    float v[32], w[32];
    for (int l = 0; l < 32; ++l) {
      float s = 0.0f;
      for (int64_t q = l; q < cl; q += 32) s += val[p0 + c0 + q] * x[col_idx[p0 + c0 + q]];
      v[l] = s;
    }
    for (int o = 16; o > 0; o >>= 1) {
      for (int l = 0; l < 32; ++l) w[l] = v[l] + v[l ^ o];
      for (int l = 0; l < 32; ++l) v[l] = w[l];
    }
    total = first ? v[0] : total + v[0];
    first = 0;
  }
  return total;
}

void ho_spmv_f32_b200(const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                      const float* x, int64_t lo, int64_t hi, float* y) {
  for (int64_t i = lo; i < hi; ++i)
    y[i - lo] = row_sum_b200(col_idx, val, x, row_ptr[i], (int64_t)row_ptr[i + 1] - row_ptr[i]);
}

/* Order-free row sums of the binned (propagation-blocking) step
 * (csrc/k_graph.cu, pagerank_step_binned): every product val[p] * x[col[p]]
 * (= fl32(fl32(1/outdeg) * x), the gather input c of the source) is rounded
 * to the 2^-56 fixed-point grid (round to nearest even; the scaled product is
 * exact in fp64, so llrint rounds once), the row sum is the exact integer sum
 * in any order (mass <= 1 < 2^7), and y = fl32(fl64(sum) * 2^-56). 2^-56 is
 * also the dangling sum's grid. */
void ho_spmv_f32_fixed(const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                       const float* x, int64_t lo, int64_t hi, float* y) {
  for (int64_t i = lo; i < hi; ++i) {
    int64_t sum = 0;
    for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      float c = val[p] * x[col_idx[p]];
      sum += llrint((double)c * 0x1p56);
    }
    y[i - lo] = (float)((double)sum * 0x1p-56);
  }
}

/* PageRank (restated; not in the reference). d = 0.85, x0 = 1/V, dangling mass
 * summed exactly in 2^-56 fixed point (order free), then
 *   x_new[i] = base + d * (y[i] + dangling * invV)
 * with every operation individually rounded in fp32. Row sums y: order 0 =
 * ascending (the reference's), 1 = the warp-unit kernel's restated order,
 * 2 = the binned step's order-free fixed-point sums. */
void ho_pagerank(int64_t v, const int32_t* row_ptr, const int32_t* col_idx, const float* val,
                 const int32_t* outdeg, int iterations, int b200_order, float* x) {
  const float d = 0.85f;
  const float base = (float)((1.0 - 0.85) / (double)v);
  const float inv_v = (float)(1.0 / (double)v);
  float* y = (float*)malloc(sizeof(float) * (size_t)v);
  for (int64_t i = 0; i < v; ++i) x[i] = inv_v;
  for (int it = 0; it < iterations; ++it) {
    int64_t dsum = 0;
    for (int64_t j = 0; j < v; ++j)
      if (outdeg[j] == 0) dsum += (int64_t)(x[j] * 0x1p56f);
    float dangling = (float)((double)dsum * 0x1p-56);
    float t = dangling * inv_v;
    if (b200_order == 2)
      ho_spmv_f32_fixed(row_ptr, col_idx, val, x, 0, v, y);
    else if (b200_order)
      ho_spmv_f32_b200(row_ptr, col_idx, val, x, 0, v, y);
    else
      ho_spmv_f32(row_ptr, col_idx, val, x, 0, v, y);
    for (int64_t i = 0; i < v; ++i) {
      float s = y[i] + t;
      float m = d * s;
      x[i] = base + m;
    }
  }
  free(y);
}

/* k-means points (restated): `blobs` centres with coordinates in [-4,4), each
 * point = centre[b] + Irwin-Hall(4) noise, everything an integer multiple of
 * 2^-12 clamped to [-8, 8). Point i uses stream outputs at fixed indices:
 * blob id = out(seed^0xB10B, i) % blobs; centre coord = out(seed^0xCE47E2,
 * b*d+j) >> 49 (15 bits) - 2^14; noise = sum of the four 16-bit lanes of
 * out(seed, i*d+j), centred, >> 5. */
void ho_kmeans_points(uint64_t seed, int64_t first, int64_t count, int64_t d, int64_t blobs,
                      float* out) {
  for (int64_t ii = 0; ii < count; ++ii) {
    uint64_t i = (uint64_t)(first + ii);
    uint64_t b = ho_splitmix_at(seed ^ 0xB10BULL, i) % (uint64_t)blobs;
    for (int64_t j = 0; j < d; ++j) {
      int64_t c = (int64_t)(ho_splitmix_at(seed ^ 0xCE47E2ULL, b * (uint64_t)d + (uint64_t)j) >> 49) -
                  16384;
      uint64_t r = ho_splitmix_at(seed, i * (uint64_t)d + (uint64_t)j);
      int64_t nsum = (int64_t)(r & 0xffff) + (int64_t)((r >> 16) & 0xffff) +
                     (int64_t)((r >> 32) & 0xffff) + (int64_t)(r >> 48) - 131070;
      int64_t q = c + (nsum >> 5);
      if (q < -32768) q = -32768;
      if (q > 32767) q = 32767;
      out[ii * d + j] = (float)q * 0x1p-12f;
    }
  }
}

/* k-means assignment = knn with k=1 (proj/src/kernels.cpp:195-233) in fp32:
 * diff = centroid - point, ascending d, rounded mul then add; strict < keeps
 * the smaller centroid index on ties (proj/src/kernels.cpp:224-225). */
void ho_kmeans_assign(const float* pts, int64_t n, int64_t d, const float* cent, int64_t k,
                      int32_t* assign) {
  for (int64_t i = 0; i < n; ++i) {
    const float* x = pts + i * d;
    float best = 0.0f;
    int32_t bi = 0;
    for (int64_t c = 0; c < k; ++c) {
      const float* m = cent + c * d;
      float sum = 0.0f;
      for (int64_t j = 0; j < d; ++j) {
        float diff = m[j] - x[j];
        sum += diff * diff;
      }
      if (c == 0 || sum < best) {
        best = sum;
        bi = (int32_t)c;
      }
    }
    assign[i] = bi;
  }
}

/* Exact update: points are multiples of 2^-12, so per-cluster sums are exact
 * int64 in 2^-12 units and independent of order and partitioning. */
void ho_kmeans_accumulate(const float* pts, int64_t n, int64_t d, const int32_t* assign,
                          int64_t k, int64_t* sums, int64_t* counts) {
  (void)k;
  for (int64_t i = 0; i < n; ++i) {
    int32_t c = assign[i];
    counts[c]++;
    for (int64_t j = 0; j < d; ++j) sums[c * d + j] += (int64_t)(pts[i * d + j] * 4096.0f);
  }
}

void ho_kmeans_finalize(const int64_t* sums, const int64_t* counts, int64_t k, int64_t d,
                        float* cent) {
  for (int64_t c = 0; c < k; ++c) {
    if (counts[c] == 0) continue; /* empty cluster keeps its centroid */
    for (int64_t j = 0; j < d; ++j)
      cent[c * d + j] = (float)(((double)sums[c * d + j] * 0x1p-12) / (double)counts[c]);
  }
}

/* Direct 3x3 conv, stride 1, pad 1, NHWC input, KRSC weights, fp64 accumulate
 * of exact bf16 products in fixed c -> r -> s order. One output element. */

static inline double bf16_to_f64(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* Output rows [y0, y1) of image n_img, all K channels, into out[(y - y0)][x][k]
 * (same fixed c -> r -> s order as ho_conv3x3_point). */
void ho_conv3x3_rows(const uint16_t* in_bf16, const uint16_t* w_bf16, int64_t h, int64_t w, int64_t c,
                     int64_t kout, int64_t n_img, int64_t y0, int64_t y1, double* out) {
  for (int64_t y = y0; y < y1; ++y)
    for (int64_t x = 0; x < w; ++x)
      for (int64_t ko = 0; ko < kout; ++ko) {
        double acc = 0.0;
        for (int64_t ci = 0; ci < c; ++ci)
          for (int64_t r = 0; r < 3; ++r)
            for (int64_t s = 0; s < 3; ++s) {
              int64_t yy = y + r - 1, xx = x + s - 1;
              if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
              acc += bf16_to_f64(in_bf16[((n_img * h + yy) * w + xx) * c + ci]) *
                     bf16_to_f64(w_bf16[((ko * 3 + r) * 3 + s) * c + ci]);
            }
        out[((y - y0) * w + x) * kout + ko] = acc;
      }
}

void ho_conv3x3_point(const uint16_t* in_bf16, const uint16_t* w_bf16, int64_t h, int64_t w,
                      int64_t c, int64_t kout, int64_t n_img, int64_t y, int64_t x, int64_t ko,
                      double* out) {
  (void)kout;
  double acc = 0.0;
  for (int64_t ci = 0; ci < c; ++ci)
    for (int64_t r = 0; r < 3; ++r)
      for (int64_t s = 0; s < 3; ++s) {
        int64_t yy = y + r - 1, xx = x + s - 1;
        if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
        double a = bf16_to_f64(in_bf16[((n_img * h + yy) * w + xx) * c + ci]);
        double b = bf16_to_f64(w_bf16[((ko * 3 + r) * 3 + s) * c + ci]);
        acc += a * b;
      }
  *out = acc;
}
