// PageRank SpMV on the pull CSR of an R-MAT graph (config C3; SURVEY.md §8(a)
// a13 spmv_compute iterated, proj/src/kernels.cpp:132-152), int32 indices and
// fp32 values, HBM-bound.
//
// CSR-adaptive schedule: the row-block array (hcl_csr_row_blocks) groups
// consecutive rows into blocks of <= max_nnz non-zeros; a longer row is a block
// of its own. A CTA takes one row block at a time:
//   * multi-row block: the block's products val[p]*x[col[p]] are streamed with
//     coalesced loads into shared memory, then each thread sums ONE row in
//     ascending storage order — the reference's order, so these rows are
//     bit-identical to the fp32 oracle;
//   * single long row: thread-strided partial sums and a fixed shuffle tree.
// Row blocks depend only on row_ptr, and a partitioned launch clips them to
// its row range [lo,hi), so results are bit-identical for every partition P.
// The PageRank update x' = base + d*(y + dangling/V) is fused into the store,
// every operation separately rounded (matches oracle ho_pagerank).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "common.hpp"
#include "../../include/hcl_cabi.h"

namespace hcl {
namespace {

constexpr int PR_T = 256;

__global__ void __launch_bounds__(256) pr_dangling_kernel(const float* __restrict__ x, const int* __restrict__ outdeg,
                                                          int64_t v, unsigned long long* __restrict__ out) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0;
  for (int64_t i = tid; i < v; i += stride)
    if (outdeg[i] == 0) s += static_cast<unsigned long long>(__float2ll_rz(__fmul_rn(x[i], 0x1p56f)));
  // integer sums: any order gives the same bits
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

__device__ __forceinline__ int first_block_ending_after(const int* __restrict__ blocks, int n, int row) {
  // smallest b in [0,n) with blocks[b+1] > row
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (blocks[mid + 1] > row) hi = mid; else lo = mid + 1;
  }
  return lo;
}

template <bool UPDATE>
__global__ void __launch_bounds__(PR_T) pr_spmv_kernel(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                       const float* __restrict__ val, int64_t nnz_off,
                                                       const int* __restrict__ blocks, int nblocks,
                                                       const float* __restrict__ x,
                                                       const unsigned long long* __restrict__ dsum,
                                                       float* __restrict__ y, int lo, int hi, float base, float damp,
                                                       float inv_v, int max_nnz) {
  extern __shared__ float prod[];
  __shared__ float wsum[PR_T / 32];
  const int tid = threadIdx.x;
  float t = 0.f;
  if constexpr (UPDATE) {
    float dangling = static_cast<float>(static_cast<double>(*dsum) * 0x1p-56);
    t = __fmul_rn(dangling, inv_v);
  }
  auto store = [&](int r, float s) {
    if constexpr (UPDATE)
      y[r - lo] = __fadd_rn(base, __fmul_rn(damp, __fadd_rn(s, t)));
    else
      y[r - lo] = s;
  };
  const int b_first = first_block_ending_after(blocks, nblocks, lo);
  const int b_last = first_block_ending_after(blocks, nblocks, hi - 1) + 1;
  const int* colp = col - nnz_off;
  const float* valp = val - nnz_off;
  for (int b = b_first + blockIdx.x; b < b_last; b += gridDim.x) {
    const int br0 = blocks[b], br1 = blocks[b + 1];
    const int r0 = max(br0, lo), r1 = min(br1, hi);
    const int p0 = row_ptr[r0], p1 = row_ptr[r1];
    const int n = p1 - p0;
    if (br1 - br0 == 1 && n > max_nnz) {
      // long row
      float s = 0.f;
      int p = p0 + tid;
      for (; p + 3 * PR_T < p1; p += 4 * PR_T) {
        int c0 = __ldg(colp + p), c1 = __ldg(colp + p + PR_T), c2 = __ldg(colp + p + 2 * PR_T), c3 = __ldg(colp + p + 3 * PR_T);
        float v0 = __ldg(valp + p), v1 = __ldg(valp + p + PR_T), v2 = __ldg(valp + p + 2 * PR_T), v3 = __ldg(valp + p + 3 * PR_T);
        s = __fadd_rn(s, __fmul_rn(v0, __ldg(x + c0)));
        s = __fadd_rn(s, __fmul_rn(v1, __ldg(x + c1)));
        s = __fadd_rn(s, __fmul_rn(v2, __ldg(x + c2)));
        s = __fadd_rn(s, __fmul_rn(v3, __ldg(x + c3)));
      }
      for (; p < p1; p += PR_T) s = __fadd_rn(s, __fmul_rn(__ldg(valp + p), __ldg(x + __ldg(colp + p))));
      for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
      if ((tid & 31) == 0) wsum[tid >> 5] = s;
      __syncthreads();
      if (tid == 0) {
        float tot = wsum[0];
        for (int w = 1; w < PR_T / 32; ++w) tot = __fadd_rn(tot, wsum[w]);
        store(r0, tot);
      }
      __syncthreads();
    } else {
      int i = tid;
      for (; i + 3 * PR_T < n; i += 4 * PR_T) {
        int c0 = __ldg(colp + p0 + i), c1 = __ldg(colp + p0 + i + PR_T), c2 = __ldg(colp + p0 + i + 2 * PR_T),
            c3 = __ldg(colp + p0 + i + 3 * PR_T);
        float v0 = __ldg(valp + p0 + i), v1 = __ldg(valp + p0 + i + PR_T), v2 = __ldg(valp + p0 + i + 2 * PR_T),
              v3 = __ldg(valp + p0 + i + 3 * PR_T);
        prod[i] = __fmul_rn(v0, __ldg(x + c0));
        prod[i + PR_T] = __fmul_rn(v1, __ldg(x + c1));
        prod[i + 2 * PR_T] = __fmul_rn(v2, __ldg(x + c2));
        prod[i + 3 * PR_T] = __fmul_rn(v3, __ldg(x + c3));
      }
      for (; i < n; i += PR_T) prod[i] = __fmul_rn(__ldg(valp + p0 + i), __ldg(x + __ldg(colp + p0 + i)));
      __syncthreads();
      for (int r = r0 + tid; r < r1; r += PR_T) {
        const int q0 = row_ptr[r] - p0, q1 = row_ptr[r + 1] - p0;
        float s = 0.f;
        for (int q = q0; q < q1; ++q) s = __fadd_rn(s, prod[q]);
        store(r, s);
      }
      __syncthreads();
    }
  }
}

struct Graph {
  const int* row_ptr;
  const int* col;
  const float* val;
  const int* blocks;
  int64_t v, nnz_off, nblocks, max_nnz;
};

// args: row_ptr, col, val, blocks, x, ... ; scalars at the end: V, nnz_off, nblocks, max_nnz
Graph graph_args(LaunchCtx& c, uint32_t s0, const char* what) {
  Graph g;
  g.v = scalar_arg(c, s0, what);
  g.nnz_off = scalar_arg(c, s0 + 1, what);
  g.nblocks = scalar_arg(c, s0 + 2, what);
  g.max_nnz = scalar_arg(c, s0 + 3, what);
  if (g.v < 1 || g.v > INT32_MAX - 1) fail(ErrorCode::argument, std::string(what) + ": V out of range");
  if (g.max_nnz < 1 || g.max_nnz > 12288) fail(ErrorCode::argument, std::string(what) + ": max_nnz must be in [1, 12288]");
  const BufView& R = buffer_arg(c, 0, what);
  if (R.first_byte != 0 || R.bytes != static_cast<uint64_t>(g.v + 1) * 4)
    fail(ErrorCode::argument, std::string(what) + ": row_ptr must hold V+1 int32");
  const BufView& B = buffer_arg(c, 3, what);
  if (B.first_byte != 0 || B.bytes != static_cast<uint64_t>(g.nblocks + 1) * 4)
    fail(ErrorCode::argument, std::string(what) + ": blocks must hold nblocks+1 int32");
  const BufView& C = buffer_arg(c, 1, what);
  const BufView& V = buffer_arg(c, 2, what);
  if (C.bytes != V.bytes) fail(ErrorCode::argument, std::string(what) + ": col_idx and values differ in size");
  g.row_ptr = reinterpret_cast<const int*>(R.ptr);
  g.blocks = reinterpret_cast<const int*>(B.ptr);
  g.col = reinterpret_cast<const int*>(C.ptr);
  g.val = reinterpret_cast<const float*>(V.ptr);
  if (C.first_byte != 0 || V.first_byte != 0)
    fail(ErrorCode::argument, std::string(what) + ": col_idx/values must be whole buffers (use nnz_off for slices)");
  return g;
}

template <bool UPDATE>
uint64_t launch_pr(LaunchCtx& c) {
  const char* what = UPDATE ? "pagerank_step" : "pagerank_spmv";
  // UPDATE: row_ptr col val blocks x dsum xnew | V nnz_off nblocks max_nnz
  // SPMV  : row_ptr col val blocks x y         | V nnz_off nblocks max_nnz
  const uint32_t s0 = UPDATE ? 7 : 6;
  Graph g = graph_args(c, s0, what);
  const BufView& X = buffer_arg(c, 4, what);
  if (X.first_byte != 0 || X.bytes != static_cast<uint64_t>(g.v) * 4)
    fail(ErrorCode::argument, std::string(what) + ": x must hold V floats");
  const unsigned long long* dsum = nullptr;
  if (UPDATE) {
    const BufView& D = buffer_arg(c, 5, what);
    if (D.bytes != 8) fail(ErrorCode::argument, std::string(what) + ": dangling sum is one uint64");
    dsum = reinterpret_cast<const unsigned long long*>(D.ptr);
  }
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(g.v), lo, rows, what);
  const BufView& Y = buffer_arg(c, UPDATE ? 6 : 5, what);
  float* y = at_byte<float>(Y, lo * 4, rows * 4, what);
  if (!rows) return 0;
  // host-side checks need the nnz range of [lo, hi): two int32 reads
  int rp[2];
  HCL_CUDA(cudaMemcpyAsync(&rp[0], g.row_ptr + lo, 4, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaMemcpyAsync(&rp[1], g.row_ptr + lo + rows, 4, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  const BufView& C = buffer_arg(c, 1, what);
  if (rp[0] < g.nnz_off || static_cast<uint64_t>(rp[1] - g.nnz_off) * 4 > C.bytes)
    fail(ErrorCode::argument, std::string(what) + ": col_idx/values do not cover the rows' non-zeros");
  const size_t smem = static_cast<size_t>(g.max_nnz) * 4;
  auto kern = pr_spmv_kernel<UPDATE>;
  HCL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  HCL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PR_T, smem));
  const int grid = std::max(1, per_sm) * c.sm_count;
  kern<<<grid, PR_T, smem, c.stream>>>(g.row_ptr, g.col, g.val, g.nnz_off, g.blocks, static_cast<int>(g.nblocks),
                                       reinterpret_cast<const float*>(X.ptr), dsum, y, static_cast<int>(lo),
                                       static_cast<int>(lo + rows), static_cast<float>((1.0 - 0.85) / g.v), 0.85f,
                                       static_cast<float>(1.0 / g.v), static_cast<int>(g.max_nnz));
  HCL_LAUNCHED();
  return 2ull * static_cast<uint64_t>(rp[1] - rp[0]);
}

// pagerank_dangling(x, outdeg, dsum, V): dsum = sum over outdeg==0 of x in 2^-56 fixed point
uint64_t launch_pr_dangling(LaunchCtx& c) {
  int64_t v = scalar_arg(c, 3, "pagerank_dangling V");
  const BufView& X = buffer_arg(c, 0, "pagerank_dangling x");
  const BufView& O = buffer_arg(c, 1, "pagerank_dangling outdeg");
  const BufView& D = buffer_arg(c, 2, "pagerank_dangling dsum");
  if (X.first_byte != 0 || X.bytes != static_cast<uint64_t>(v) * 4 || O.first_byte != 0 ||
      O.bytes != static_cast<uint64_t>(v) * 4 || D.bytes != 8)
    fail(ErrorCode::argument, "pagerank_dangling: x, outdeg must hold V elements, dsum one uint64");
  HCL_CUDA(cudaMemsetAsync(D.ptr, 0, 8, c.stream));
  int grid = c.sm_count * 4;
  pr_dangling_kernel<<<grid, 256, 0, c.stream>>>(reinterpret_cast<const float*>(X.ptr),
                                                 reinterpret_cast<const int*>(O.ptr), v,
                                                 reinterpret_cast<unsigned long long*>(D.ptr));
  HCL_LAUNCHED();
  return static_cast<uint64_t>(v);
}

uint64_t rows_pr(const int64_t* s, uint32_t n) { return static_cast<uint64_t>(s[n == 11 ? 7 : 6]); }

}  // namespace

void register_graph(std::vector<KernelDef>& r) {
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS;
  // y = A x over rows [lo,hi)
  r.push_back({"b200", "pagerank_spmv", {I, I, I, I, I, O, S, S, S, S}, {P, P, P, P, P, X, N, N, N, N},
               launch_pr<false>, nullptr, rows_pr});
  // x' = (1-d)/V + d (A x + dangling/V) over rows [lo,hi)
  r.push_back({"b200", "pagerank_step", {I, I, I, I, I, I, O, S, S, S, S}, {P, P, P, P, P, P, X, N, N, N, N},
               launch_pr<true>, nullptr, rows_pr});
  r.push_back({"b200", "pagerank_dangling", {I, I, O, S}, {P, P, P, N}, launch_pr_dangling, nullptr, nullptr});
}

}  // namespace hcl
