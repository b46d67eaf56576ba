// Product-side synthetic data generation: the
// reference's SplitMix64 streams (proj/include/haocl/datagen.hpp:13-31,
// proj/src/datagen.cpp:11-16) plus the restated generators of the B200
// configs. SplitMix64 is counter based — output i of the stream seeded with s
// is mix(s + (i+1)*gamma) — so any sub-range (one rank's row block) is
// generated independently and in parallel, bit-identical to the serial stream.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "hcl_datagen.h"

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

inline uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline uint64_t at(uint64_t seed, uint64_t i) { return mix(seed + (i + 1) * kGamma); }
inline double unit_sym(uint64_t r) { return static_cast<double>(r >> 11) * 0x1.0p-53 * 2.0 - 1.0; }

inline uint16_t bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

template <typename F>
void parallel_for(uint64_t n, int threads, F&& f) {
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  if (n < (1u << 16) || threads == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  uint64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    uint64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    ts.emplace_back([&, lo, hi] { f(lo, hi); });
  }
  for (auto& t : ts) t.join();
}

// R-MAT quadrant thresholds (a, b, c) = (.57, .19, .19) as 32-bit integers.
constexpr uint32_t kT1 = 2448131358u, kT2 = 3264175144u, kT3 = 4080218930u;

}  // namespace

extern "C" {

uint64_t hcl_gen_splitmix_at(uint64_t seed, uint64_t index) { return at(seed, index); }

void hcl_gen_doubles(double* out, uint64_t first, uint64_t count, uint64_t seed, int threads) {
  parallel_for(count, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) out[i] = unit_sym(at(seed, first + i));
  });
}

void hcl_gen_f32(float* out, uint64_t first, uint64_t count, uint64_t seed, int threads) {
  parallel_for(count, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) out[i] = static_cast<float>(unit_sym(at(seed, first + i)));
  });
}

void hcl_gen_bf16(uint16_t* out, uint64_t first, uint64_t count, uint64_t seed, int threads) {
  parallel_for(count, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) out[i] = bf16_rne(static_cast<float>(unit_sym(at(seed, first + i))));
  });
}

void hcl_gen_rmat_edges(int scale, uint64_t first_edge, uint64_t count, uint64_t seed, uint32_t* src,
                        uint32_t* dst, int threads) {
  parallel_for(count, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      uint64_t e = first_edge + i;
      uint32_t s = 0, d = 0;
      for (int l = 0; l < scale; ++l) {
        uint32_t u = static_cast<uint32_t>(at(seed, e * static_cast<uint64_t>(scale) + l) >> 32);
        uint32_t bs = u >= kT2;
        uint32_t bd = (u >= kT1 && u < kT2) || u >= kT3;
        s = (s << 1) | bs;
        d = (d << 1) | bd;
      }
      src[i] = s;
      dst[i] = d;
    }
  });
}

void hcl_gen_kmeans_points(uint64_t seed, uint64_t first, uint64_t count, int64_t d, int64_t blobs, float* out,
                           int threads) {
  parallel_for(count, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t ii = lo; ii < hi; ++ii) {
      uint64_t i = first + ii;
      uint64_t b = at(seed ^ 0xB10BULL, i) % static_cast<uint64_t>(blobs);
      for (int64_t j = 0; j < d; ++j) {
        int64_t c = static_cast<int64_t>(at(seed ^ 0xCE47E2ULL, b * d + j) >> 49) - 16384;
        uint64_t r = at(seed, i * d + j);
        int64_t nsum = static_cast<int64_t>(r & 0xffff) + static_cast<int64_t>((r >> 16) & 0xffff) +
                       static_cast<int64_t>((r >> 32) & 0xffff) + static_cast<int64_t>(r >> 48) - 131070;
        int64_t q = c + (nsum >> 5);
        q = q < -32768 ? -32768 : (q > 32767 ? 32767 : q);
        out[ii * d + j] = static_cast<float>(q) * 0x1p-12f;
      }
    }
  });
}

// Pull CSR of the R-MAT graph by destination (rows = dst, columns = src
// ascending, multi-edges kept, val = 1/outdeg(src) in fp32): identical to the
// oracle's serial counting sorts (oracle/haocl_oracle.c ho_pagerank_csr). Built
// with a parallel LSD radix sort of 48-bit (dst, src) keys.
int hcl_pagerank_csr(int scale, uint64_t edges, uint64_t seed, int32_t* row_ptr, int32_t* col_idx, float* val,
                     int32_t* outdeg, int threads) {
  if (scale < 1 || scale > 30 || edges >= (1ull << 31)) return 1009;
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const uint64_t v = 1ull << scale;
  std::vector<uint64_t> keys(edges), tmp(edges);
  {
    std::vector<uint32_t> s(edges), d(edges);
    hcl_gen_rmat_edges(scale, 0, edges, seed, s.data(), d.data(), threads);
    std::vector<std::atomic<int32_t>> deg(v);
    parallel_for(v, threads, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i) deg[i].store(0, std::memory_order_relaxed);
    });
    parallel_for(edges, threads, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i) {
        keys[i] = (static_cast<uint64_t>(d[i]) << 32) | s[i];
        deg[s[i]].fetch_add(1, std::memory_order_relaxed);
      }
    });
    parallel_for(v, threads, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i) outdeg[i] = deg[i].load(std::memory_order_relaxed);
    });
  }
  // LSD radix sort on src (bits 0..scale) then dst (bits 32..32+scale), 16-bit digits
  std::vector<int> shifts;
  for (int b = 0; b < scale; b += 16) shifts.push_back(b);
  for (int b = 0; b < scale; b += 16) shifts.push_back(32 + b);
  const int T = threads;
  const uint64_t chunk = (edges + T - 1) / T;
  std::vector<uint64_t> hist(static_cast<size_t>(T) * 65536);
  for (int sh : shifts) {
    std::fill(hist.begin(), hist.end(), 0);
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        uint64_t lo = t * chunk, hi = std::min(edges, lo + chunk);
        uint64_t* h = &hist[static_cast<size_t>(t) * 65536];
        for (uint64_t i = lo; i < hi; ++i) h[(keys[i] >> sh) & 0xffff]++;
      });
    for (auto& x : ts) x.join();
    ts.clear();
    uint64_t run = 0;  // digit-major, thread-minor exclusive scan -> stable
    for (int dg = 0; dg < 65536; ++dg)
      for (int t = 0; t < T; ++t) {
        uint64_t c = hist[static_cast<size_t>(t) * 65536 + dg];
        hist[static_cast<size_t>(t) * 65536 + dg] = run;
        run += c;
      }
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        uint64_t lo = t * chunk, hi = std::min(edges, lo + chunk);
        uint64_t* h = &hist[static_cast<size_t>(t) * 65536];
        for (uint64_t i = lo; i < hi; ++i) tmp[h[(keys[i] >> sh) & 0xffff]++] = keys[i];
      });
    for (auto& x : ts) x.join();
    keys.swap(tmp);
  }
  // row_ptr by dst
  std::vector<int64_t> cnt(v + 1, 0);
  for (uint64_t i = 0; i < edges; ++i) cnt[(keys[i] >> 32) + 1]++;
  for (uint64_t i = 0; i < v; ++i) cnt[i + 1] += cnt[i];
  for (uint64_t i = 0; i <= v; ++i) row_ptr[i] = static_cast<int32_t>(cnt[i]);
  parallel_for(edges, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      uint32_t src = static_cast<uint32_t>(keys[i] & 0xffffffffu);
      col_idx[i] = static_cast<int32_t>(src);
      val[i] = 1.0f / static_cast<float>(outdeg[src]);
    }
  });
  return 0;
}

// Warp work units of the PageRank SpMV (csrc/k_graph.cu). A unit is
// {row0, row1, p0, p1}: either consecutive rows with <= warp_nnz products in
// total (one warp), or one 4096-product chunk of a longer row (row1 = row0+1,
// [p0,p1) the chunk). Long rows get a fixup entry {row, first_unit, nchunks}:
// a second pass folds the chunk totals in chunk order. Units are sorted by row
// and depend only on row_ptr (so every partition sees the same units).
int hcl_pagerank_units(const int32_t* row_ptr, int64_t rows, int64_t warp_nnz, int32_t* units, int32_t* long_rows,
                       int64_t* n_units, int64_t* n_long) {
  if (warp_nnz < 1 || warp_nnz > 4096) return 1009;
  int64_t nu = 0, nl = 0, r = 0;
  while (r < rows) {
    int64_t start = row_ptr[r];
    int64_t len = row_ptr[r + 1] - start;
    if (len > warp_nnz) {
      int64_t nch = (len + 4095) / 4096;
      if (long_rows) {
        long_rows[3 * nl] = static_cast<int32_t>(r);
        long_rows[3 * nl + 1] = static_cast<int32_t>(nu);
        long_rows[3 * nl + 2] = static_cast<int32_t>(nch);
      }
      for (int64_t c = 0; c < nch; ++c) {
        if (units) {
          int32_t* u = units + 4 * (nu + c);
          u[0] = static_cast<int32_t>(r);
          u[1] = static_cast<int32_t>(r + 1);
          u[2] = static_cast<int32_t>(start + c * 4096);
          u[3] = static_cast<int32_t>(std::min<int64_t>(start + (c + 1) * 4096, start + len));
        }
      }
      nu += nch;
      ++nl;
      ++r;
      continue;
    }
    int64_t e = r + 1;
    while (e < rows && row_ptr[e + 1] - start <= warp_nnz) ++e;
    if (units) {
      int32_t* u = units + 4 * nu;
      u[0] = static_cast<int32_t>(r);
      u[1] = static_cast<int32_t>(e);
      u[2] = static_cast<int32_t>(start);
      u[3] = row_ptr[e];
    }
    ++nu;
    r = e;
  }
  *n_units = nu;
  *n_long = nl;
  return 0;
}

// Row blocks of a CSR for the PageRank SpMV (CSR-adaptive): consecutive rows
// grouped while their nnz total stays <= max_nnz; a row longer than max_nnz
// is a block by itself. out[0..count] are block start rows (out[count] = rows).
// Depends only on row_ptr, so a partitioned launch gives P-invariant results.
int64_t hcl_csr_row_blocks(const int32_t* row_ptr, int64_t rows, int64_t max_nnz, int32_t* out) {
  int64_t n = 0;
  int64_t r = 0;
  while (r < rows) {
    if (out) out[n] = static_cast<int32_t>(r);
    ++n;
    int64_t start = row_ptr[r];
    int64_t e = r + 1;
    if (row_ptr[e] - start <= max_nnz)
      while (e < rows && row_ptr[e + 1] - start <= max_nnz) ++e;
    r = e;
  }
  if (out) out[n] = static_cast<int32_t>(rows);
  return n;
}

// Degree-ordered relabelling of a pull CSR (vertices = rows = columns): new id
// i is the vertex with the i-th largest out-degree (= how often its rank is
// gathered), ties by old id. Rows move with their vertex and keep their column
// ORDER (each old column c becomes inv[c]), so every row's product sequence,
// and hence the SpMV's per-row summation, is unchanged: results are the old
// ones permuted (rank_old[perm[i]] = rank_new[i]). The hot sources become one
// dense prefix of x, which the gathers then find in L1/L2.
int hcl_pagerank_relabel(const int32_t* row_ptr, const int32_t* col_idx, const float* val, const int32_t* outdeg,
                         int64_t v, int32_t* new_row_ptr, int32_t* new_col, float* new_val, int32_t* new_outdeg,
                         int32_t* perm, int threads) {
  if (v < 1 || v > INT32_MAX) return 1000 + 9;
  // perm = vertices sorted by (outdeg desc, id asc): counting sort on degree
  int32_t maxd = 0;
  for (int64_t i = 0; i < v; ++i) maxd = std::max(maxd, outdeg[i]);
  std::vector<int64_t> start(static_cast<size_t>(maxd) + 2, 0);
  for (int64_t i = 0; i < v; ++i) ++start[static_cast<size_t>(maxd - outdeg[i]) + 1];
  for (size_t d = 1; d < start.size(); ++d) start[d] += start[d - 1];
  for (int64_t i = 0; i < v; ++i) perm[start[static_cast<size_t>(maxd - outdeg[i])]++] = static_cast<int32_t>(i);
  std::vector<int32_t> inv(static_cast<size_t>(v));
  parallel_for(static_cast<uint64_t>(v), threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) inv[perm[i]] = static_cast<int32_t>(i);
  });
  new_row_ptr[0] = 0;
  for (int64_t i = 0; i < v; ++i) {
    const int32_t o = perm[i];
    new_row_ptr[i + 1] = new_row_ptr[i] + (row_ptr[o + 1] - row_ptr[o]);
    new_outdeg[i] = outdeg[o];
  }
  parallel_for(static_cast<uint64_t>(v), threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      const int32_t o = perm[i];
      int64_t q = new_row_ptr[i];
      for (int64_t p = row_ptr[o]; p < row_ptr[o + 1]; ++p, ++q) {
        new_col[q] = inv[col_idx[p]];
        new_val[q] = val[p];
      }
    }
  });
  return 0;
}

// Stable counting order: perm[i] = the index of the i-th key in ascending key
// order (ties by index). keys in [0, k); returns 0 or 1000+argument.
int hcl_counting_order(const int32_t* keys, int64_t n, int32_t k, int32_t* perm) {
  if (n < 0 || k < 1 || (n && (!keys || !perm))) return 1000 + 9;
  std::vector<int64_t> start(static_cast<size_t>(k) + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (keys[i] < 0 || keys[i] >= k) return 1000 + 9;
    ++start[static_cast<size_t>(keys[i]) + 1];
  }
  for (int32_t j = 0; j < k; ++j) start[j + 1] += start[j];
  for (int64_t i = 0; i < n; ++i) perm[start[keys[i]]++] = static_cast<int32_t>(i);
  return 0;
}

}  // extern "C"
