// TEST INFRASTRUCTURE ONLY — extern "C" shim over the HaoCL reference library.
//
// Compiled by oracle/Makefile together with the UNMODIFIED reference sources
// /root/reference/proj/src/{kernels,reference,datagen,error}.cpp (read in place,
// never copied) into oracle/_ref/libhaocl_ref.so. Used to validate the C
// restatement (oracle/haocl_oracle.c) and, in bench.py --impl reference and the
// cpu_baseline leg, as the reference CPU implementation timed on host cores.
//
// Every entry point returns 0 on success or the reference haocl::ErrorCode
// value (proj/include/haocl/error.hpp:11-36) of the thrown haocl::Error.

#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "haocl/datagen.hpp"
#include "haocl/error.hpp"
#include "haocl/kernels.hpp"
#include "haocl/reference.hpp"

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const haocl::Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1000;
  }
}

std::vector<uint8_t> bytes_of(const void* p, size_t n) {
  std::vector<uint8_t> v(n);
  if (n) std::memcpy(v.data(), p, n);
  return v;
}

}  // namespace

extern "C" {

const char* href_last_error() { return g_last_error.c_str(); }

// kernels::execute through the reference's own engine (proj/src/kernels.cpp:268-283).
// kinds[i]: 0 scalar, 1 buffer_in, 2 buffer_out. For outputs, out_ptrs[i] receives
// the produced bytes (caller sizes out_caps[i]); out_lens[i] returns the length.
int href_execute(const char* kernel, int nargs, const int* kinds, const int64_t* scalars,
                 const void* const* in_ptrs, const uint64_t* in_lens, void* const* out_ptrs,
                 const uint64_t* out_caps, uint64_t* out_lens, int threads, uint64_t* work) {
  return guarded([&] {
    std::vector<std::vector<uint8_t>> store(static_cast<size_t>(nargs));
    std::vector<haocl::kernels::BoundArg> args(static_cast<size_t>(nargs));
    for (int i = 0; i < nargs; ++i) {
      if (kinds[i] == 0) {
        args[i] = haocl::kernels::BoundArg::of_scalar(scalars[i]);
      } else {
        if (kinds[i] == 1) store[i] = bytes_of(in_ptrs[i], in_lens[i]);
        args[i] = haocl::kernels::BoundArg::of_buffer(&store[i]);
      }
    }
    uint64_t w = haocl::kernels::execute(kernel, args, threads);
    if (work) *work = w;
    for (int i = 0; i < nargs; ++i) {
      if (kinds[i] != 2) continue;
      out_lens[i] = store[i].size();
      if (store[i].size() > out_caps[i]) haocl::fail(haocl::ErrorCode::size, "output capacity");
      if (!store[i].empty()) std::memcpy(out_ptrs[i], store[i].data(), store[i].size());
    }
  });
}

// Serial oracles (proj/src/reference.cpp).
void href_matmul(const double* a, const double* b, double* c, int64_t m, int64_t k, int64_t n) {
  haocl::ref::matmul(a, b, c, m, k, n);
}
void href_spmv(const int64_t* rp, const int64_t* ci, const double* v, const double* x, int64_t lo,
               int64_t hi, double* y) {
  haocl::ref::spmv(rp, ci, v, x, lo, hi, y);
}
void href_bfs(int64_t vertices, const int64_t* rp, const int64_t* ci, int64_t source,
              int32_t* levels) {
  auto out = haocl::ref::bfs(vertices, rp, ci, source);
  std::memcpy(levels, out.data(), out.size() * sizeof(int32_t));
}
void href_knn(const double* r, const double* q, int64_t nr, int64_t nq, int64_t d, int64_t k,
              int32_t* idx, double* dist) {
  haocl::ref::knn(r, q, nr, nq, d, k, idx, dist);
}
void href_vecadd(const double* a, const double* b, double* c, int64_t n) {
  haocl::ref::vecadd(a, b, c, n);
}

int href_spmv_partition_ranges(int64_t rows, const int64_t* row_ptr, int64_t parts,
                               int64_t* out) {
  return guarded([&] {
    auto r = haocl::kernels::spmv_partition_ranges(rows, row_ptr, parts);
    std::memcpy(out, r.data(), r.size() * sizeof(int64_t));
  });
}

int href_merge_topk(int64_t nparts, const int64_t* part_k, const int32_t* const* part_idx,
                    const double* const* part_dist, int64_t queries, int64_t k, int32_t* out_idx,
                    double* out_dist) {
  return guarded([&] {
    std::vector<haocl::kernels::KnnPartial> parts(static_cast<size_t>(nparts));
    for (int64_t p = 0; p < nparts; ++p) {
      parts[p].k = part_k[p];
      size_t n = static_cast<size_t>(part_k[p] * queries);
      parts[p].idx.assign(part_idx[p], part_idx[p] + n);
      parts[p].dist.assign(part_dist[p], part_dist[p] + n);
    }
    auto m = haocl::kernels::merge_topk(parts, queries, k);
    std::memcpy(out_idx, m.idx.data(), m.idx.size() * sizeof(int32_t));
    std::memcpy(out_dist, m.dist.data(), m.dist.size() * sizeof(double));
  });
}

uint64_t href_work_estimate(const char* kernel, int nscalars, const int64_t* scalars,
                            int nbuffers, const uint64_t* sizes) {
  uint64_t w = 0;
  guarded([&] {
    w = haocl::kernels::work_estimate(kernel, std::span<const int64_t>(scalars, nscalars),
                                      std::span<const uint64_t>(sizes, nbuffers));
  });
  return w;
}

// Datagen (proj/src/datagen.cpp).
void href_gen_doubles(double* out, uint64_t count, uint64_t seed) {
  auto v = haocl::gen_doubles(count, seed);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}

// gen_csr: call with col_idx/values == nullptr to get nnz in *nnz first.
int href_gen_csr(int64_t rows, int64_t cols, double density, uint64_t seed, int64_t* row_ptr,
                 int64_t* col_idx, double* values, int64_t* nnz) {
  return guarded([&] {
    auto c = haocl::gen_csr(rows, cols, density, seed);
    *nnz = c.nnz();
    if (row_ptr) std::memcpy(row_ptr, c.row_ptr.data(), c.row_ptr.size() * 8);
    if (col_idx) std::memcpy(col_idx, c.col_idx.data(), c.col_idx.size() * 8);
    if (values) std::memcpy(values, c.values.data(), c.values.size() * 8);
  });
}

int href_gen_graph(int64_t vertices, int64_t edges, uint64_t seed, int64_t* row_ptr,
                   int64_t* col_idx, int64_t* nnz) {
  return guarded([&] {
    auto c = haocl::gen_graph(vertices, edges, seed);
    *nnz = static_cast<int64_t>(c.col_idx.size());
    if (row_ptr) std::memcpy(row_ptr, c.row_ptr.data(), c.row_ptr.size() * 8);
    if (col_idx) std::memcpy(col_idx, c.col_idx.data(), c.col_idx.size() * 8);
  });
}

}  // extern "C"
