// sm_100a kernels for the reference's own "core" bundle
// (proj/src/kernels.cpp:13-33): matmul, spmv_partition, spmv_compute, knn,
// vecadd, in the reference's buffer encodings (fp64 values, int64 indices,
// int32 knn indices). Every floating-point reduction keeps the reference's
// ascending order with a separately rounded multiply and add (__dmul_rn /
// __dadd_rn: the reference is built with -ffp-contract=off,
// proj/src/CMakeLists.txt:22-24), so outputs are bit-identical to the
// reference for any partition of the NDRange.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "common.hpp"
#include "../../include/hcl_cabi.h"

namespace hcl {
namespace {

// ---------------------------------------------------------------------------
// vecadd — proj/src/kernels.cpp:235-246. Streaming, 128-bit accesses.

__global__ void __launch_bounds__(256) vecadd_f64_kernel(const double* __restrict__ a,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ c, int64_t n) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t n2 = n / 2;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double2* c2 = reinterpret_cast<double2*>(c);
  for (int64_t i = tid; i < n2; i += stride) {
    double2 x = __ldcs(a2 + i), y = __ldcs(b2 + i);
    __stcs(c2 + i, make_double2(__dadd_rn(x.x, y.x), __dadd_rn(x.y, y.y)));
  }
  if (tid == 0 && (n & 1)) c[n - 1] = __dadd_rn(a[n - 1], b[n - 1]);
}

uint64_t launch_vecadd(LaunchCtx& c) {
  int64_t n = scalar_arg(c, 3, "vecadd n");
  if (n < 0) fail(ErrorCode::argument, "vecadd: n must be >= 0");
  // NDRange sub-range over elements
  uint64_t lo, cnt;
  sub_range(c, static_cast<uint64_t>(n), lo, cnt, "vecadd");
  const BufView& A = buffer_arg(c, 0, "vecadd a");
  const BufView& B = buffer_arg(c, 1, "vecadd b");
  const BufView& C = buffer_arg(c, 2, "vecadd c");
  if (c.whole && A.bytes != static_cast<uint64_t>(n) * 8)
    fail(ErrorCode::argument, "vecadd: input length mismatch");
  if (c.whole && B.bytes != static_cast<uint64_t>(n) * 8)
    fail(ErrorCode::argument, "vecadd: input length mismatch");
  const double* a = at_byte<const double>(A, lo * 8, cnt * 8, "vecadd a");
  const double* b = at_byte<const double>(B, lo * 8, cnt * 8, "vecadd b");
  double* cc = at_byte<double>(C, lo * 8, cnt * 8, "vecadd c");
  if (cnt == 0) return 0;
  bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                   reinterpret_cast<uintptr_t>(cc)) & 15) == 0;
  if (!aligned) fail(ErrorCode::argument, "vecadd: sub-range must start on an even element");
  int blocks = static_cast<int>(std::min<uint64_t>(ceil_div(cnt / 2 + 1, 256), c.sm_count * 8));
  vecadd_f64_kernel<<<blocks, 256, 0, c.stream>>>(a, b, cc, static_cast<int64_t>(cnt));
  HCL_LAUNCHED();
  return cnt;
}

// ---------------------------------------------------------------------------
// matmul — proj/src/kernels.cpp:96-119, oracle reference.cpp:8-17.
// C[i][j] = ((0 + a_i0*b_0j) + a_i1*b_1j) + ... in ascending k, each product
// and sum rounded separately. 64x64 output tile per 256-thread block, 4x4 per
// thread, K staged through shared memory in 16-wide panels.

constexpr int MM_T = 64, MM_K = 16;

__global__ void __launch_bounds__(256) matmul_f64_exact_kernel(const double* __restrict__ A,
                                                               const double* __restrict__ B,
                                                               double* __restrict__ C, int64_t M,
                                                               int64_t K, int64_t N) {
  __shared__ double sa[MM_K][MM_T + 1];
  __shared__ double sb[MM_K][MM_T];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t row0 = blockIdx.y * (int64_t)MM_T, col0 = blockIdx.x * (int64_t)MM_T;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t k0 = 0; k0 < K; k0 += MM_K) {
    for (int e = threadIdx.x; e < MM_T * MM_K; e += 256) {
      int r = e / MM_K, kk = e % MM_K;
      int64_t gr = row0 + r, gk = k0 + kk;
      sa[kk][r] = (gr < M && gk < K) ? A[gr * K + gk] : 0.0;
      int kb = e / MM_T, cb = e % MM_T;
      int64_t gkb = k0 + kb, gc = col0 + cb;
      sb[kb][cb] = (gkb < K && gc < N) ? B[gkb * N + gc] : 0.0;
    }
    __syncthreads();
    int kmax = static_cast<int>(K - k0 < MM_K ? K - k0 : MM_K);
    for (int kk = 0; kk < kmax; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = sa[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = sb[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(av[i], bv[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t r = row0 + ty + 16 * i, cc = col0 + tx + 16 * j;
      if (r < M && cc < N) C[r * N + cc] = acc[i][j];
    }
}

uint64_t launch_matmul(LaunchCtx& c) {
  int64_t m = scalar_arg(c, 3, "matmul M");
  int64_t k = scalar_arg(c, 4, "matmul K");
  int64_t n = scalar_arg(c, 5, "matmul N");
  if (m < 1 || k < 1 || n < 1) fail(ErrorCode::argument, "matmul: dimensions must be >= 1");
  const BufView& A = buffer_arg(c, 0, "matmul A");
  const BufView& B = buffer_arg(c, 1, "matmul B");
  const BufView& Cb = buffer_arg(c, 2, "matmul C");
  if (c.whole && A.bytes != static_cast<uint64_t>(m * k) * 8)
    fail(ErrorCode::argument, "matmul: A size != M*K");
  if (B.first_byte != 0 || B.bytes != static_cast<uint64_t>(k * n) * 8)
    fail(ErrorCode::argument, "matmul: B size != K*N");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(m), lo, rows, "matmul");
  const double* a = at_byte<const double>(A, lo * k * 8, rows * k * 8, "matmul A");
  const double* b = at_byte<const double>(B, 0, static_cast<uint64_t>(k * n) * 8, "matmul B");
  double* cc = at_byte<double>(Cb, lo * n * 8, rows * n * 8, "matmul C");
  if (rows == 0) return 0;
  dim3 grid(static_cast<unsigned>(ceil_div(n, MM_T)), static_cast<unsigned>(ceil_div(rows, MM_T)));
  matmul_f64_exact_kernel<<<grid, 256, 0, c.stream>>>(a, b, cc, static_cast<int64_t>(rows), k, n);
  HCL_LAUNCHED();
  return 2ull * rows * n * k;
}

// ---------------------------------------------------------------------------
// CSR validation — csr_view, proj/src/kernels.cpp:55-94. Run on the device;
// the error flag is read back so violations surface synchronously with the
// reference's error code and message.

__global__ void csr_validate_kernel(const int64_t* __restrict__ row_ptr, int64_t rows,
                                    const int64_t* __restrict__ col_idx, int64_t nnz, int64_t cols,
                                    int* __restrict__ flags) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < rows; i += stride)
    if (row_ptr[i + 1] < row_ptr[i]) atomicOr(flags, 1);
  if (col_idx)
    for (int64_t p = tid; p < nnz; p += stride) {
      int64_t v = col_idx[p];
      if (v < 0 || v >= cols) atomicOr(flags, 2);
    }
}

struct Csr64 {
  int64_t rows = 0, cols = 0, nnz = 0;
  const int64_t* row_ptr = nullptr;
  const int64_t* col_idx = nullptr;
  const double* values = nullptr;
};

Csr64 csr_view(LaunchCtx& c, uint32_t hdr_i, uint32_t rp_i, int ci_i, int val_i, const char* what) {
  Csr64 s;
  const BufView& H = buffer_arg(c, hdr_i, what);
  if (H.first_byte != 0 || H.bytes != 16)
    fail(ErrorCode::argument, std::string(what) + ": header must hold [rows, cols]");
  int64_t hdr[2];
  HCL_CUDA(cudaMemcpyAsync(hdr, H.ptr, 16, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  s.rows = hdr[0];
  s.cols = hdr[1];
  if (s.rows < 0 || s.cols < 0) fail(ErrorCode::argument, std::string(what) + ": negative dimension");
  const BufView& R = buffer_arg(c, rp_i, what);
  if (R.first_byte != 0 || R.bytes != static_cast<uint64_t>(s.rows + 1) * 8)
    fail(ErrorCode::argument, std::string(what) + ": row_ptr must hold rows+1 entries");
  s.row_ptr = reinterpret_cast<const int64_t*>(R.ptr);
  int64_t ends[2];
  HCL_CUDA(cudaMemcpyAsync(&ends[0], s.row_ptr, 8, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaMemcpyAsync(&ends[1], s.row_ptr + s.rows, 8, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  if (ends[0] != 0) fail(ErrorCode::argument, std::string(what) + ": row_ptr[0] != 0");
  s.nnz = ends[1];
  if (ci_i >= 0) {
    const BufView& CI = buffer_arg(c, ci_i, what);
    if (CI.first_byte != 0 || CI.bytes % 8 || CI.bytes / 8 != static_cast<uint64_t>(s.nnz < 0 ? 0 : s.nnz))
      fail(ErrorCode::argument, std::string(what) + ": col_idx size != nnz");
    s.col_idx = reinterpret_cast<const int64_t*>(CI.ptr);
  }
  int* flags = static_cast<int*>(c.scratch(c.dev, 64));
  HCL_CUDA(cudaMemsetAsync(flags, 0, 4, c.stream));
  int blocks = static_cast<int>(std::min<uint64_t>(ceil_div(std::max(s.rows, s.nnz) + 1, 256), c.sm_count * 4));
  csr_validate_kernel<<<blocks, 256, 0, c.stream>>>(s.row_ptr, s.rows, s.col_idx, s.nnz, s.cols, flags);
  HCL_LAUNCHED();
  int hflags = 0;
  HCL_CUDA(cudaMemcpyAsync(&hflags, flags, 4, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  if (hflags & 1) fail(ErrorCode::argument, std::string(what) + ": row_ptr not nondecreasing");
  if (hflags & 2) fail(ErrorCode::argument, std::string(what) + ": col_idx out of range");
  if (val_i >= 0) {
    const BufView& V = buffer_arg(c, val_i, what);
    if (V.first_byte != 0 || V.bytes % 8 || V.bytes / 8 != static_cast<uint64_t>(s.nnz))
      fail(ErrorCode::argument, std::string(what) + ": values size != nnz");
    s.values = reinterpret_cast<const double*>(V.ptr);
  }
  return s;
}

// ---------------------------------------------------------------------------
// spmv_partition — proj/src/kernels.cpp:121-130 / 300-321. The greedy sweep
// "extend part p while acc < ceil(nnz/P)" stops at the first row end e with
// row_ptr[e] - row_ptr[start] >= target (or at the cap that leaves one row for
// each later part), so each boundary is one binary search: P searches instead
// of an O(rows) scan, bit-identical boundaries.

__global__ void spmv_partition_kernel(const int64_t* __restrict__ row_ptr, int64_t rows,
                                      int64_t parts, int64_t* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t nnz_total = row_ptr[rows];
  int64_t target = (nnz_total + parts - 1) / parts;
  out[0] = 0;
  int64_t row = 0;
  for (int64_t p = 0; p + 1 < parts; ++p) {
    int64_t max_end = rows - (parts - 1 - p);
    int64_t want = row_ptr[row] + target;
    // first e in [row+1, max_end] with row_ptr[e] >= want, else max_end
    int64_t lo = row + 1, hi = max_end;
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (row_ptr[mid] >= want) hi = mid; else lo = mid + 1;
    }
    out[p + 1] = lo;
    row = lo;
  }
  out[parts] = rows;
}

uint64_t launch_spmv_partition(LaunchCtx& c) {
  Csr64 s = csr_view(c, 0, 1, -1, -1, "spmv_partition");
  int64_t parts = scalar_arg(c, 2, "spmv_partition P");
  if (parts < 1) fail(ErrorCode::argument, "spmv_partition: P must be >= 1");
  if (parts > s.rows) fail(ErrorCode::argument, "spmv_partition: P exceeds row count");
  const BufView& O = buffer_arg(c, 3, "spmv_partition ranges");
  int64_t* out = at_byte<int64_t>(O, 0, static_cast<uint64_t>(parts + 1) * 8, "spmv_partition ranges");
  spmv_partition_kernel<<<1, 32, 0, c.stream>>>(s.row_ptr, s.rows, parts, out);
  HCL_LAUNCHED();
  return static_cast<uint64_t>(s.rows);
}

// ---------------------------------------------------------------------------
// spmv_compute — proj/src/kernels.cpp:132-152. One thread per row, the row's
// products summed in ascending storage order (bit-exact with ref::spmv).

__global__ void __launch_bounds__(256) spmv_f64_exact_kernel(const int64_t* __restrict__ row_ptr,
                                                             const int64_t* __restrict__ col_idx,
                                                             const double* __restrict__ values,
                                                             const double* __restrict__ x,
                                                             int64_t lo, int64_t hi,
                                                             double* __restrict__ y) {
  int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= hi) return;
  int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
  double sum = 0.0;
  for (int64_t p = p0; p < p1; ++p) sum = __dadd_rn(sum, __dmul_rn(__ldg(values + p), __ldg(x + __ldg(col_idx + p))));
  y[i - lo] = sum;
}

uint64_t launch_spmv_compute(LaunchCtx& c) {
  Csr64 s = csr_view(c, 0, 1, 2, 3, "spmv_compute");
  const BufView& X = buffer_arg(c, 4, "spmv_compute x");
  if (X.first_byte != 0 || X.bytes != static_cast<uint64_t>(s.cols) * 8)
    fail(ErrorCode::argument, "spmv_compute: x size != cols");
  int64_t lo = scalar_arg(c, 5, "spmv_compute lo");
  int64_t hi = scalar_arg(c, 6, "spmv_compute hi");
  if (lo < 0 || hi < lo || hi > s.rows) fail(ErrorCode::argument, "spmv_compute: bad row range");
  const BufView& Y = buffer_arg(c, 7, "spmv_compute y");
  double* y = at_byte<double>(Y, 0, static_cast<uint64_t>(hi - lo) * 8, "spmv_compute y");
  if (hi > lo) {
    unsigned blocks = static_cast<unsigned>(ceil_div(hi - lo, 256));
    spmv_f64_exact_kernel<<<blocks, 256, 0, c.stream>>>(s.row_ptr, s.col_idx, s.values,
                                                        reinterpret_cast<const double*>(X.ptr), lo, hi, y);
    HCL_LAUNCHED();
  }
  int64_t nz[2] = {0, 0};
  HCL_CUDA(cudaMemcpyAsync(&nz[0], s.row_ptr + lo, 8, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaMemcpyAsync(&nz[1], s.row_ptr + hi, 8, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  return 2ull * static_cast<uint64_t>(nz[1] - nz[0]);
}

// ---------------------------------------------------------------------------
// bfs — proj/src/kernels.cpp:154-193. Level-synchronous: pass L visits every
// vertex of level L-1 and claims each unseen neighbour with a CAS, so every
// vertex gets its unique BFS level (-1 when unreachable) under any schedule --
// the same levels as the reference's CAS frontier loop. One pass per level;
// the host stops after a pass that claims nothing.

__global__ void __launch_bounds__(256) bfs_level_kernel(const int64_t* __restrict__ row_ptr,
                                                        const int64_t* __restrict__ col_idx, int64_t vertices,
                                                        int32_t level, int32_t* __restrict__ levels,
                                                        int* __restrict__ claimed) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int any = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < vertices; u += stride) {
    if (levels[u] != level - 1) continue;
    for (int64_t p = row_ptr[u], e = row_ptr[u + 1]; p < e; ++p) {
      const int64_t v = __ldg(col_idx + p);
      if (levels[v] == -1 && atomicCAS(levels + v, -1, level) == -1) any = 1;
    }
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(claimed, 1);
}

uint64_t launch_bfs(LaunchCtx& c) {
  Csr64 s = csr_view(c, 0, 1, 2, -1, "bfs");
  const int64_t source = scalar_arg(c, 3, "bfs source");
  if (source < 0 || source >= s.rows) fail(ErrorCode::argument, "bfs: source out of range");
  const BufView& L = buffer_arg(c, 4, "bfs levels");
  int32_t* levels = at_byte<int32_t>(L, 0, static_cast<uint64_t>(s.rows) * 4, "bfs levels");
  HCL_CUDA(cudaMemsetAsync(levels, 0xff, static_cast<size_t>(s.rows) * 4, c.stream));
  const int32_t zero = 0;
  HCL_CUDA(cudaMemcpyAsync(levels + source, &zero, 4, cudaMemcpyHostToDevice, c.stream));
  int* claimed = static_cast<int*>(c.scratch(c.dev, 64));
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(s.rows, 256), static_cast<int64_t>(c.sm_count) * 8)));
  for (int32_t level = 1;; ++level) {
    HCL_CUDA(cudaMemsetAsync(claimed, 0, 4, c.stream));
    bfs_level_kernel<<<blocks, 256, 0, c.stream>>>(s.row_ptr, s.col_idx, s.rows, level, levels, claimed);
    HCL_LAUNCHED();
    int h = 0;
    HCL_CUDA(cudaMemcpyAsync(&h, claimed, 4, cudaMemcpyDeviceToHost, c.stream));
    HCL_CUDA(cudaStreamSynchronize(c.stream));
    if (!h) break;
  }
  return static_cast<uint64_t>(s.nnz);
}

// ---------------------------------------------------------------------------
// knn — proj/src/kernels.cpp:195-233. One 128-thread block per query; each
// thread keeps a sorted top-k of its strided reference subset under the
// (dist, idx) order, then the block merges the 128 lists k times by a
// shared-memory argmin. Distances use diff = ref - query, ascending d, rounded
// multiply then add, so results equal the reference bit-for-bit.

constexpr int KNN_MAXK = 32, KNN_T = 128;

__device__ __forceinline__ bool pair_lt(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

// `refp` holds reference rows [idx_base, idx_base + R) of the whole set; the
// emitted indices are global. Fewer than k candidates (a reference-set part
// with R < k) pad the list with (+inf, INT32_MAX), which sorts after every
// real candidate.
__global__ void __launch_bounds__(KNN_T) knn_f64_kernel(const double* __restrict__ refp,
                                                        const double* __restrict__ query, int64_t R,
                                                        int64_t D, int k, int64_t idx_base,
                                                        int32_t* __restrict__ out_idx,
                                                        double* __restrict__ out_dist) {
  extern __shared__ double sq[];  // D query coords
  __shared__ double hd[KNN_T];
  __shared__ int hi[KNN_T];
  __shared__ int hw[KNN_T];
  const int64_t q = blockIdx.x;
  for (int64_t d = threadIdx.x; d < D; d += KNN_T) sq[d] = query[q * D + d];
  __syncthreads();
  double bd[KNN_MAXK];
  int bi[KNN_MAXK];
  int have = 0;
  for (int64_t r = threadIdx.x; r < R; r += KNN_T) {
    const double* p = refp + r * D;
    double sum = 0.0;
    for (int64_t d = 0; d < D; ++d) {
      double diff = __dsub_rn(p[d], sq[d]);
      sum = __dadd_rn(sum, __dmul_rn(diff, diff));
    }
    int id = static_cast<int>(idx_base + r);
    if (have < k || pair_lt(sum, id, bd[k - 1], bi[k - 1])) {
      int pos = have < k ? have++ : k - 1;
      while (pos > 0 && pair_lt(sum, id, bd[pos - 1], bi[pos - 1])) {
        bd[pos] = bd[pos - 1];
        bi[pos] = bi[pos - 1];
        --pos;
      }
      bd[pos] = sum;
      bi[pos] = id;
    }
  }
  int head = 0;
  for (int out = 0; out < k; ++out) {
    hd[threadIdx.x] = head < have ? bd[head] : __longlong_as_double(0x7ff0000000000000LL);
    hi[threadIdx.x] = head < have ? bi[head] : 0x7fffffff;
    hw[threadIdx.x] = threadIdx.x;
    __syncthreads();
    for (int s = KNN_T / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        int o = threadIdx.x + s;
        if (pair_lt(hd[o], hi[o], hd[threadIdx.x], hi[threadIdx.x])) {
          hd[threadIdx.x] = hd[o];
          hi[threadIdx.x] = hi[o];
          hw[threadIdx.x] = hw[o];
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      out_idx[q * k + out] = hi[0];
      out_dist[q * k + out] = hd[0];
    }
    if (threadIdx.x == hw[0]) ++head;
    __syncthreads();
  }
}

// k > 32 (up to KNN_LARGE_MAXK): one 256-thread block per query keeps the
// running top-k sorted in shared memory. Each tile of 256 references is
// scored (same exact order), the candidates below the current k-th pair are
// compacted and bitonic-sorted, and the two sorted runs are merged by rank
// (pairs are distinct: indices are unique), so the result is the k smallest
// under (dist, idx) exactly as the reference's partial_sort.
constexpr int KNN_LT = 256, KNN_LARGE_MAXK = 4096;

__device__ __forceinline__ int rank_lt(const double* d, const int* ix, int n, double vd, int vi) {
  int lo = 0, hi = n;  // number of elements < (vd, vi)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pair_lt(d[mid], ix[mid], vd, vi)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(KNN_LT) knn_large_kernel(const double* __restrict__ refp,
                                                          const double* __restrict__ query, int64_t R, int64_t D,
                                                          int k, int64_t idx_base, int32_t* __restrict__ out_idx,
                                                          double* __restrict__ out_dist) {
  extern __shared__ __align__(16) uint8_t kl_smem[];
  double* bd = reinterpret_cast<double*>(kl_smem);          // k
  double* od = bd + k;                                       // k
  double* cd = od + k;                                       // KNN_LT
  double* sq = cd + KNN_LT;                                  // D
  int* bi = reinterpret_cast<int*>(sq + D);                  // k
  int* oi = bi + k;                                          // k
  int* ci = oi + k;                                          // KNN_LT
  __shared__ int n_cand;
  const int64_t q = blockIdx.x;
  const int t = threadIdx.x;
  for (int64_t d = t; d < D; d += KNN_LT) sq[d] = query[q * D + d];
  int cur = 0;
  __syncthreads();
  for (int64_t r0 = 0; r0 < R; r0 += KNN_LT) {
    const int64_t r = r0 + t;
    double dist = __longlong_as_double(0x7ff0000000000000LL);
    int id = 0x7fffffff;
    if (r < R) {
      const double* p = refp + r * D;
      double sum = 0.0;
      for (int64_t d = 0; d < D; ++d) {
        const double diff = __dsub_rn(p[d], sq[d]);
        sum = __dadd_rn(sum, __dmul_rn(diff, diff));
      }
      dist = sum;
      id = static_cast<int>(idx_base + r);
    }
    const bool pass = r < R && (cur < k || pair_lt(dist, id, bd[k - 1], bi[k - 1]));
    if (t == 0) n_cand = 0;
    __syncthreads();
    if (pass) {
      const int slot = atomicAdd(&n_cand, 1);
      cd[slot] = dist;
      ci[slot] = id;
    }
    __syncthreads();
    const int nc = n_cand;
    __syncthreads();        // every thread has read n_cand before thread 0 resets it
    if (nc == 0) continue;  // uniform
    // bitonic sort of the candidates (padded to a power of two with +inf)
    int np = 1;
    while (np < nc) np <<= 1;
    for (int i = nc + t; i < np; i += KNN_LT) {
      cd[i] = __longlong_as_double(0x7ff0000000000000LL);
      ci[i] = 0x7fffffff;
    }
    __syncthreads();
    for (int size = 2; size <= np; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = t; i < np; i += KNN_LT) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            if (pair_lt(cd[j], ci[j], cd[i], ci[i]) == up) {
              const double td = cd[i];
              const int ti = ci[i];
              cd[i] = cd[j];
              ci[i] = ci[j];
              cd[j] = td;
              ci[j] = ti;
            }
          }
        }
        __syncthreads();
      }
    // merge the sorted runs by rank into od/oi, keep the first k
    for (int i = t; i < cur; i += KNN_LT) {
      const int pos = i + rank_lt(cd, ci, nc, bd[i], bi[i]);
      if (pos < k) {
        od[pos] = bd[i];
        oi[pos] = bi[i];
      }
    }
    for (int j = t; j < nc; j += KNN_LT) {
      const int pos = j + rank_lt(bd, bi, cur, cd[j], ci[j]);
      if (pos < k) {
        od[pos] = cd[j];
        oi[pos] = ci[j];
      }
    }
    __syncthreads();
    cur = min(k, cur + nc);
    for (int i = t; i < cur; i += KNN_LT) {
      bd[i] = od[i];
      bi[i] = oi[i];
    }
    __syncthreads();
  }
  for (int i = t; i < k; i += KNN_LT) {
    out_dist[q * k + i] = i < cur ? bd[i] : __longlong_as_double(0x7ff0000000000000LL);
    out_idx[q * k + i] = i < cur ? bi[i] : 0x7fffffff;
  }
}

void launch_knn_large(LaunchCtx& c, const double* refp, const double* qp, int64_t r, int64_t d, int64_t k,
                      int64_t idx_base, int64_t nq, int32_t* oi, double* od) {
  if (k > KNN_LARGE_MAXK)
    fail(ErrorCode::argument, "knn: the GPU path supports k <= " + std::to_string(KNN_LARGE_MAXK));
  const size_t smem = static_cast<size_t>(2 * k + KNN_LT + d) * 8 + static_cast<size_t>(2 * k + KNN_LT) * 4;
  if (smem > 220 * 1024) fail(ErrorCode::argument, "knn: k and D too large for the GPU path");
  if (smem > 48 * 1024)
    HCL_CUDA(cudaFuncSetAttribute(knn_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  knn_large_kernel<<<static_cast<unsigned>(nq), KNN_LT, smem, c.stream>>>(refp, qp, r, d, static_cast<int>(k),
                                                                          idx_base, oi, od);
  HCL_LAUNCHED();
}

uint64_t launch_knn(LaunchCtx& c) {
  int64_t r = scalar_arg(c, 2, "knn R");
  int64_t q = scalar_arg(c, 3, "knn Q");
  int64_t d = scalar_arg(c, 4, "knn D");
  int64_t k = scalar_arg(c, 5, "knn k");
  if (r < 1 || q < 1 || d < 1) fail(ErrorCode::argument, "knn: R, Q, D must be >= 1");
  if (k < 1 || k > r) fail(ErrorCode::argument, "knn: need 1 <= k <= R");
  if (r > INT32_MAX) fail(ErrorCode::argument, "knn: R exceeds int32 indices");
  const BufView& Rf = buffer_arg(c, 0, "knn ref");
  const BufView& Qb = buffer_arg(c, 1, "knn query");
  if (Rf.first_byte != 0 || Rf.bytes != static_cast<uint64_t>(r * d) * 8)
    fail(ErrorCode::argument, "knn: ref size != R*D");
  if (c.whole && Qb.bytes != static_cast<uint64_t>(q * d) * 8)
    fail(ErrorCode::argument, "knn: query size != Q*D");
  // NDRange over queries
  uint64_t lo, cnt;
  sub_range(c, static_cast<uint64_t>(q), lo, cnt, "knn");
  const double* qp = at_byte<const double>(Qb, lo * d * 8, cnt * d * 8, "knn query");
  int32_t* oi = at_byte<int32_t>(buffer_arg(c, 6, "knn idx"), lo * k * 4, cnt * k * 4, "knn idx");
  double* od = at_byte<double>(buffer_arg(c, 7, "knn dist"), lo * k * 8, cnt * k * 8, "knn dist");
  if (k > KNN_MAXK) {
    if (cnt) launch_knn_large(c, reinterpret_cast<const double*>(Rf.ptr), qp, r, d, k, 0, cnt, oi, od);
    return static_cast<uint64_t>(d) * r * cnt;
  }
  size_t smem = static_cast<size_t>(d) * 8;
  if (smem > 200 * 1024) fail(ErrorCode::argument, "knn: D too large for the GPU path");
  if (smem > 48 * 1024)
    HCL_CUDA(cudaFuncSetAttribute(knn_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  if (cnt) {
    knn_f64_kernel<<<static_cast<unsigned>(cnt), KNN_T, smem, c.stream>>>(
        reinterpret_cast<const double*>(Rf.ptr), qp, r, d, static_cast<int>(k), 0, oi, od);
    HCL_LAUNCHED();
  }
  return static_cast<uint64_t>(d) * r * cnt;
}

// knn_refsplit(ref, query, R, Q, D, k, idx, dist): the reference's knn
// partitioning (proj/src/bench.cpp:367-447): the NDRange is the REFERENCE set
// (dim 0 = R), each part computes every query's top-k over its reference rows
// [lo, hi) with global indices (the reference adds `lo` on the host, 417-418),
// and the MERGE_TOPK outputs are folded by knn_refsplit_merge. Launched whole
// it equals core knn bit-for-bit.
uint64_t launch_knn_refsplit(LaunchCtx& c) {
  int64_t r = scalar_arg(c, 2, "knn_refsplit R");
  int64_t q = scalar_arg(c, 3, "knn_refsplit Q");
  int64_t d = scalar_arg(c, 4, "knn_refsplit D");
  int64_t k = scalar_arg(c, 5, "knn_refsplit k");
  if (r < 1 || q < 1 || d < 1) fail(ErrorCode::argument, "knn_refsplit: R, Q, D must be >= 1");
  if (k < 1 || k > r) fail(ErrorCode::argument, "knn_refsplit: need 1 <= k <= R");
  if (r > INT32_MAX) fail(ErrorCode::argument, "knn_refsplit: R exceeds int32 indices");
  const BufView& Rf = buffer_arg(c, 0, "knn_refsplit ref");
  const BufView& Qb = buffer_arg(c, 1, "knn_refsplit query");
  if (c.whole && Rf.bytes != static_cast<uint64_t>(r * d) * 8) fail(ErrorCode::argument, "knn_refsplit: ref size != R*D");
  if (Qb.first_byte != 0 || Qb.bytes != static_cast<uint64_t>(q * d) * 8)
    fail(ErrorCode::argument, "knn_refsplit: query size != Q*D");
  uint64_t lo, cnt;
  sub_range(c, static_cast<uint64_t>(r), lo, cnt, "knn_refsplit");
  const double* rp = at_byte<const double>(Rf, lo * d * 8, cnt * d * 8, "knn_refsplit ref");
  int32_t* oi = at_byte<int32_t>(buffer_arg(c, 6, "knn_refsplit idx"), 0, q * k * 4, "knn_refsplit idx");
  double* od = at_byte<double>(buffer_arg(c, 7, "knn_refsplit dist"), 0, q * k * 8, "knn_refsplit dist");
  if (k > KNN_MAXK) {
    if (cnt) launch_knn_large(c, rp, reinterpret_cast<const double*>(Qb.ptr), static_cast<int64_t>(cnt), d, k,
                              static_cast<int64_t>(lo), q, oi, od);
    return static_cast<uint64_t>(d) * cnt * q;
  }
  size_t smem = static_cast<size_t>(d) * 8;
  if (smem > 200 * 1024) fail(ErrorCode::argument, "knn_refsplit: D too large for the GPU path");
  if (smem > 48 * 1024)
    HCL_CUDA(cudaFuncSetAttribute(knn_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (cnt) {
    knn_f64_kernel<<<static_cast<unsigned>(q), KNN_T, smem, c.stream>>>(rp, reinterpret_cast<const double*>(Qb.ptr),
                                                                      static_cast<int64_t>(cnt), d, static_cast<int>(k),
                                                                      static_cast<int64_t>(lo), oi, od);
    HCL_LAUNCHED();
  }
  return static_cast<uint64_t>(d) * cnt * q;
}

// Fold two per-query sorted top-k lists into the first: the k smallest of the
// union under the (dist, idx) order -- merge_topk's partial_sort of the pool
// (proj/src/kernels.cpp:347-358) restricted to two partials, which is
// associative, so folding parts in order equals the P-way merge. A list that
// is not sorted raises the reference's contract error (333-340).
__global__ void knn_merge2_kernel(int32_t* __restrict__ ia, double* __restrict__ da, const int32_t* __restrict__ ib,
                                  const double* __restrict__ db, int64_t Q, int k, int* __restrict__ bad) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= Q) return;
  int32_t oi[KNN_MAXK];
  double od[KNN_MAXK];
  const int32_t* pa = ia + q * k;
  const double* qa = da + q * k;
  const int32_t* pb = ib + q * k;
  const double* qb = db + q * k;
  for (int i = 1; i < k; ++i)
    if (pair_lt(qa[i], pa[i], qa[i - 1], pa[i - 1]) || pair_lt(qb[i], pb[i], qb[i - 1], pb[i - 1])) atomicOr(bad, 1);
  int x = 0, y = 0;
  for (int o = 0; o < k; ++o) {
    if (pair_lt(qb[y], pb[y], qa[x], pa[x])) {
      od[o] = qb[y];
      oi[o] = pb[y];
      ++y;
    } else {
      od[o] = qa[x];
      oi[o] = pa[x];
      ++x;
    }
  }
  for (int o = 0; o < k; ++o) {
    ia[q * k + o] = oi[o];
    da[q * k + o] = od[o];
  }
}

// k > 32: one block per query merges the two sorted lists by rank in shared memory
__global__ void __launch_bounds__(KNN_LT) knn_merge2_large_kernel(int32_t* __restrict__ ia, double* __restrict__ da,
                                                                 const int32_t* __restrict__ ib,
                                                                 const double* __restrict__ db, int k,
                                                                 int* __restrict__ bad) {
  extern __shared__ __align__(16) uint8_t km_smem[];
  double* ad = reinterpret_cast<double*>(km_smem);
  double* bdd = ad + k;
  int* ai = reinterpret_cast<int*>(bdd + k);
  int* bii = ai + k;
  const int64_t q = blockIdx.x;
  const int t = threadIdx.x;
  for (int i = t; i < k; i += KNN_LT) {
    ad[i] = da[q * k + i];
    ai[i] = ia[q * k + i];
    bdd[i] = db[q * k + i];
    bii[i] = ib[q * k + i];
  }
  __syncthreads();
  for (int i = t + 1; i < k; i += KNN_LT)
    if (pair_lt(ad[i], ai[i], ad[i - 1], ai[i - 1]) || pair_lt(bdd[i], bii[i], bdd[i - 1], bii[i - 1])) atomicOr(bad, 1);
  // equal pairs (padding) rank a before b; distinct real pairs have distinct ranks
  for (int i = t; i < k; i += KNN_LT) {
    int lo = 0, hi = k;  // b elements strictly below a[i]
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pair_lt(bdd[mid], bii[mid], ad[i], ai[i])) lo = mid + 1; else hi = mid;
    }
    const int pos = i + lo;
    if (pos < k) {
      da[q * k + pos] = ad[i];
      ia[q * k + pos] = ai[i];
    }
  }
  for (int j = t; j < k; j += KNN_LT) {
    int lo = 0, hi = k;  // a elements at or below b[j]
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (!pair_lt(bdd[j], bii[j], ad[mid], ai[mid])) lo = mid + 1; else hi = mid;
    }
    const int pos = j + lo;
    if (pos < k) {
      da[q * k + pos] = bdd[j];
      ia[q * k + pos] = bii[j];
    }
  }
}

// knn_refsplit_merge(ref, query, R, Q, D, k, idx, dist, idx2, dist2): the
// MERGE_TOPK companion (same arguments + the other part's lists).
uint64_t launch_knn_refsplit_merge(LaunchCtx& c) {
  int64_t q = scalar_arg(c, 3, "knn merge Q");
  int64_t k = scalar_arg(c, 5, "knn merge k");
  if (q < 1 || k < 1 || k > KNN_LARGE_MAXK) fail(ErrorCode::argument, "knn merge: bad Q or k");
  int32_t* ia = at_byte<int32_t>(buffer_arg(c, 6, "knn merge idx"), 0, q * k * 4, "knn merge idx");
  double* da = at_byte<double>(buffer_arg(c, 7, "knn merge dist"), 0, q * k * 8, "knn merge dist");
  const int32_t* ib = at_byte<const int32_t>(buffer_arg(c, 8, "knn merge idx2"), 0, q * k * 4, "knn merge idx2");
  const double* db = at_byte<const double>(buffer_arg(c, 9, "knn merge dist2"), 0, q * k * 8, "knn merge dist2");
  int* bad = static_cast<int*>(c.scratch(c.dev, sizeof(int)));
  HCL_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
  if (k <= KNN_MAXK) {
    knn_merge2_kernel<<<static_cast<unsigned>(ceil_div(q, 128)), 128, 0, c.stream>>>(ia, da, ib, db, q,
                                                                                   static_cast<int>(k), bad);
  } else {
    const size_t smem = static_cast<size_t>(k) * 24;
    if (smem > 48 * 1024)
      HCL_CUDA(cudaFuncSetAttribute(knn_merge2_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    knn_merge2_large_kernel<<<static_cast<unsigned>(q), KNN_LT, smem, c.stream>>>(ia, da, ib, db,
                                                                                 static_cast<int>(k), bad);
  }
  HCL_LAUNCHED();
  int h = 0;
  HCL_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  if (h) fail(ErrorCode::contract, "merge_topk: partial not sorted");
  return static_cast<uint64_t>(q * k);
}

uint64_t rows_knn_refsplit(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[2]); }
uint64_t rowbytes_knn_refsplit(const int64_t* s, uint32_t, uint32_t) { return static_cast<uint64_t>(s[4]) * 8; }

uint64_t rows_matmul(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[3]); }
uint64_t rowbytes_matmul(const int64_t* s, uint32_t, uint32_t i) {
  return static_cast<uint64_t>(i == 0 ? s[4] : s[5]) * 8;  // A: K*8, C: N*8
}
uint64_t rows_vecadd(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[3]); }
uint64_t rowbytes_vecadd(const int64_t*, uint32_t, uint32_t) { return 8; }
uint64_t rows_knn(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[3]); }
uint64_t rowbytes_knn(const int64_t* s, uint32_t, uint32_t i) {
  if (i == 1) return static_cast<uint64_t>(s[4]) * 8;  // query: D*8
  if (i == 6) return static_cast<uint64_t>(s[5]) * 4;  // idx: k*4
  return static_cast<uint64_t>(s[5]) * 8;              // dist: k*8
}

}  // namespace

// Registry entries of the reference bundle "core" (proj/src/kernels.cpp:13-33).
void register_core(std::vector<KernelDef>& r) {
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS;
  r.push_back({"core", "matmul", {I, I, O, S, S, S}, {X, P, X, N, N, N}, launch_matmul,
               rowbytes_matmul, rows_matmul});
  r.push_back({"core", "spmv_partition", {I, I, S, O}, {P, P, N, P}, launch_spmv_partition, nullptr,
               nullptr});
  r.push_back({"core", "spmv_compute", {I, I, I, I, I, S, S, O}, {P, P, P, P, P, N, N, P},
               launch_spmv_compute, nullptr, nullptr});
  r.push_back({"core", "bfs", {I, I, I, S, O}, {P, P, P, N, P}, launch_bfs, nullptr, nullptr});
  r.push_back({"core", "knn", {I, I, S, S, S, S, O, O}, {P, X, N, N, N, N, X, X}, launch_knn,
               rowbytes_knn, rows_knn});
  r.push_back({"core", "vecadd", {I, I, O, S}, {X, X, X, N}, launch_vecadd, rowbytes_vecadd,
               rows_vecadd});
  // the reference-set split of knn (§8(f) 3) and its MERGE_TOPK companion
  constexpr uint8_t M = HCL_PART_MERGE_TOPK, IO = HCL_ARG_INOUT;
  r.push_back({"b200", "knn_refsplit", {I, I, S, S, S, S, O, O}, {X, P, N, N, N, N, M, M}, launch_knn_refsplit,
               rowbytes_knn_refsplit, rows_knn_refsplit});
  r.push_back({"b200", "knn_refsplit_merge", {I, I, S, S, S, S, IO, IO, I, I}, {P, P, N, N, N, N, P, P, P, P},
               launch_knn_refsplit_merge, nullptr, nullptr});
}

}  // namespace hcl
