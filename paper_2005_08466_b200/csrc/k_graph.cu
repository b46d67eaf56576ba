// PageRank SpMV on the pull CSR of an R-MAT graph (config C3; SURVEY.md §8(a)
// a13 spmv_compute iterated, proj/src/kernels.cpp:132-152), int32 indices and
// fp32 values, HBM-bound.
//
// Warp-granular schedule, no block-wide barriers: the unit array
// (hcl_pagerank_units) holds, sorted by row,
//   * multi-row units: consecutive rows with <= warp_nnz products in total. The
//     warp streams the products val[p]*x[col[p]] (coalesced, 4 loads in flight
//     per lane) into its own shared-memory slice; then a row of <= 32 products
//     is summed by one lane in ascending order (the reference's order,
//     reference.cpp:22-25) and a longer row by the whole warp (lane-strided
//     partial sums + xor butterfly);
//   * chunk units: one 4096-product chunk of a longer row, summed by a warp in
//     the same lane-strided + butterfly order into a per-unit scratch slot; a
//     fixup pass folds each long row's chunk totals in chunk order.
// The per-row order depends only on the row's length — restated exactly in the
// oracle (ho_spmv_f32_b200) — so results are bit-identical to that oracle and
// identical for every partition P of the NDRange (units are global, a part
// clips multi-row units to its rows [lo,hi); rows are never split). The
// PageRank update x' = base + d*(y + dangling/V) is fused into the stores,
// every operation separately rounded (oracle ho_pagerank).
#include <cuda_runtime.h>

#include <cstdint>
#include <tuple>
#include <mutex>
#include <map>
#include <cstdlib>
#include <string>

#include "common.hpp"
#include "../../include/hcl_cabi.h"

namespace hcl {
namespace {

constexpr int PR_T = 256;
constexpr int PR_WARPS = PR_T / 32;
constexpr int PR_CHUNK = 4096;  // long-row chunk (part of the summation-order definition)

// sum over j with outdeg[j]==0 of trunc(x_j * 2^56): integer, so order free
__global__ void __launch_bounds__(256) pr_dangling_kernel(const float* __restrict__ x, const int* __restrict__ outdeg,
                                                          int64_t v, unsigned long long* __restrict__ out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0;
  const int64_t v4 = v / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const int4* d4 = reinterpret_cast<const int4*>(outdeg);
  for (int64_t i = tid; i < v4; i += 2 * stride) {
    int4 da = __ldcs(d4 + i);
    int4 db = i + stride < v4 ? __ldcs(d4 + i + stride) : make_int4(1, 1, 1, 1);
    float4 xa = __ldcs(x4 + i);
    float4 xb = i + stride < v4 ? __ldcs(x4 + i + stride) : make_float4(0, 0, 0, 0);
#define HCL_DANG(dv, xv) \
  if ((dv) == 0) s += static_cast<unsigned long long>(__float2ll_rz(__fmul_rn((xv), 0x1p56f)))
    HCL_DANG(da.x, xa.x); HCL_DANG(da.y, xa.y); HCL_DANG(da.z, xa.z); HCL_DANG(da.w, xa.w);
    HCL_DANG(db.x, xb.x); HCL_DANG(db.y, xb.y); HCL_DANG(db.z, xb.z); HCL_DANG(db.w, xb.w);
  }
  for (int64_t i = v4 * 4 + tid; i < v; i += stride) HCL_DANG(outdeg[i], x[i]);
#undef HCL_DANG
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// The CSR arrays stream through once (2 GiB per iteration): keep them out of L1
// and first in line for L2 eviction, so the gathered x lines stay cached.
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_x(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ float butterfly(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct Update {
  float base, damp, t;
};

template <bool UPDATE>
__device__ __forceinline__ float pr_store(float* __restrict__ y, int r, int lo, float s, const Update& u) {
  float v = s;
  if constexpr (UPDATE) v = __fadd_rn(u.base, __fmul_rn(u.damp, __fadd_rn(s, u.t)));
  y[r - lo] = v;
  return v;
}

// Fused step (pagerank_step_exchange): besides x'[r], each row also yields the
// next iteration's gather input xs'[r] = fl(1/outdeg(r)) * x'[r] (what
// pagerank_prep computes, bit for bit; the reciprocals come precomputed), stored into this device's xs' and
// into every peer's xs' (NVLink stores into peer / IPC-mapped memory), and
// dangling rows add x'[r] to dsum' (2^-56 fixed point, order-free). The
// separate prep pass and the rank-vector allgather disappear; an allreduce
// of dsum' is the only collective, and it doubles as the step barrier.
constexpr int PR_MAX_PEERS = 7;
struct Fanout {
  float* p[PR_MAX_PEERS];
  int n;
  float* xs;            // this device's xs'
  const float* inv;     // fl(1/outdeg), 0 for dangling vertices
};

__device__ __forceinline__ Fanout load_fanout(const unsigned long long* peers, int n, float* xs, const float* inv) {
  Fanout f;
  f.n = n;
  f.xs = xs;
  f.inv = inv;
#pragma unroll
  for (int k = 0; k < PR_MAX_PEERS; ++k) f.p[k] = k < n ? reinterpret_cast<float*>(__ldg(peers + k)) : nullptr;
  return f;
}

template <bool UPDATE, bool XCH>
__device__ __forceinline__ void pr_store_x(float* __restrict__ y, int r, int lo, float s, const Update& u,
                                           const Fanout& f, unsigned long long& dang) {
  const float v = pr_store<UPDATE>(y, r, lo, s, u);
  if constexpr (XCH) {
    const float inv = __ldg(f.inv + r);  // the division is done once per graph, not per step
    const float xs = __fmul_rn(inv, v);
    f.xs[r] = xs;
#pragma unroll
    for (int k = 0; k < PR_MAX_PEERS; ++k)
      if (k < f.n) f.p[k][r] = xs;
    if (inv == 0.f) dang += static_cast<unsigned long long>(__float2ll_rz(__fmul_rn(v, 0x1p56f)));
  }
}

// end of an exchange kernel: the block's dangling partial into dsum', and the
// peer stores made visible system-wide before the allreduce that follows
__device__ __forceinline__ void pr_exchange_flush(unsigned long long dang, unsigned long long* dsum_next) {
  for (int o = 16; o > 0; o >>= 1) dang += __shfl_xor_sync(0xffffffffu, dang, o);
  if ((threadIdx.x & 31) == 0 && dang) atomicAdd(dsum_next, dang);
  __threadfence_system();
}

template <bool UPDATE>
__device__ __forceinline__ Update pr_update(const unsigned long long* dsum, float base, float damp, float inv_v) {
  Update u{base, damp, 0.f};
  if constexpr (UPDATE) {
    float dangling = static_cast<float>(static_cast<double>(*dsum) * 0x1p-56);
    u.t = __fmul_rn(dangling, inv_v);
  }
  return u;
}

// lane-strided partial sums over [p, e) then the butterfly (all lanes hold the total)
// IMP: the values are implicit -- x holds xs = val(src) * x(src) (pagerank_prep),
// so a product is one gather; the same rounded product as val[p] * x[col[p]].
template <bool IMP>
__device__ __forceinline__ float product(const float* __restrict__ valp, const float* __restrict__ x, int q, int c) {
  if constexpr (IMP)
    return ld_x(x + c);
  else
    return __fmul_rn(ld_stream(valp + q), ld_x(x + c));
}

template <bool IMP>
__device__ __forceinline__ float warp_row_sum(const int* __restrict__ colp, const float* __restrict__ valp,
                                              const float* __restrict__ x, int p, int e, int lane) {
  float v = 0.f;
  int q = p + lane;
  for (; q + 96 < e; q += 128) {
    int i0 = ld_stream(colp + q), i1 = ld_stream(colp + q + 32), i2 = ld_stream(colp + q + 64), i3 = ld_stream(colp + q + 96);
    const float p0 = product<IMP>(valp, x, q, i0), p1 = product<IMP>(valp, x, q + 32, i1);
    const float p2 = product<IMP>(valp, x, q + 64, i2), p3 = product<IMP>(valp, x, q + 96, i3);
    v = __fadd_rn(v, p0);
    v = __fadd_rn(v, p1);
    v = __fadd_rn(v, p2);
    v = __fadd_rn(v, p3);
  }
  for (; q < e; q += 32) v = __fadd_rn(v, product<IMP>(valp, x, q, ld_stream(colp + q)));
  return butterfly(v);
}

template <bool UPDATE, bool IMP, bool XCH = false>
__global__ void __launch_bounds__(PR_T) pr_units_kernel(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                        const float* __restrict__ val, int64_t nnz_off,
                                                        const int4* __restrict__ units, int n_units,
                                                        const float* __restrict__ x,
                                                        const unsigned long long* __restrict__ dsum,
                                                        float* __restrict__ y, int lo, int hi, float base, float damp,
                                                        float inv_v, int warp_nnz, float* __restrict__ chunk_tot,
                                                        const unsigned long long* __restrict__ peers, int n_peers,
                                                        const float* __restrict__ inv_outdeg, float* __restrict__ xs_next,
                                                        unsigned long long* __restrict__ dsum_next) {
  extern __shared__ float prod_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* prod = prod_all + warp * warp_nnz;
  const Update upd = pr_update<UPDATE>(dsum, base, damp, inv_v);
  Fanout fo{};
  unsigned long long dang = 0;
  if constexpr (XCH) fo = load_fanout(peers, n_peers, xs_next, inv_outdeg);
  // units overlapping [lo, hi): row1 > lo and row0 < hi (both monotone in u)
  int a = 0, b = n_units;
  while (a < b) {
    int m = (a + b) >> 1;
    if (__ldg(&units[m].y) > lo) b = m; else a = m + 1;
  }
  const int u_first = a;
  b = n_units;
  while (a < b) {
    int m = (a + b) >> 1;
    if (__ldg(&units[m].x) >= hi) b = m; else a = m + 1;
  }
  const int u_last = a;
  const int* colp = col - nnz_off;
  const float* valp = val - nnz_off;
  const int nw = gridDim.x * PR_WARPS;
  for (int u = u_first + blockIdx.x * PR_WARPS + warp; u < u_last; u += nw) {
    const int4 U = units[u];
    if (U.y - U.x == 1 && __ldg(row_ptr + U.x + 1) - __ldg(row_ptr + U.x) > warp_nnz) {
      // one chunk of a long row
      const float v = warp_row_sum<IMP>(colp, valp, x, U.z, U.w, lane);
      if (lane == 0) chunk_tot[u] = v;
      continue;
    }
    const int r0 = max(U.x, lo), r1 = min(U.y, hi);
    const int p0 = __ldg(row_ptr + r0), n = __ldg(row_ptr + r1) - p0;
    int i = lane;
    for (; i + 96 < n; i += 128) {
      int c0 = ld_stream(colp + p0 + i), c1 = ld_stream(colp + p0 + i + 32), c2 = ld_stream(colp + p0 + i + 64),
          c3 = ld_stream(colp + p0 + i + 96);
      const float q0 = product<IMP>(valp, x, p0 + i, c0), q1 = product<IMP>(valp, x, p0 + i + 32, c1);
      const float q2 = product<IMP>(valp, x, p0 + i + 64, c2), q3 = product<IMP>(valp, x, p0 + i + 96, c3);
      prod[i] = q0;
      prod[i + 32] = q1;
      prod[i + 64] = q2;
      prod[i + 96] = q3;
    }
    for (; i < n; i += 32) prod[i] = product<IMP>(valp, x, p0 + i, ld_stream(colp + p0 + i));
    __syncwarp();
    for (int rb = r0; rb < r1; rb += 32) {
      const int r = rb + lane;
      const bool in = r < r1;
      const int q0 = in ? __ldg(row_ptr + r) - p0 : 0;
      const int len = in ? __ldg(row_ptr + r + 1) - p0 - q0 : 0;
      if (in && len <= 32) {
        float s = 0.f;
        for (int q = q0; q < q0 + len; ++q) s = __fadd_rn(s, prod[q]);
        pr_store_x<UPDATE, XCH>(y, r, lo, s, upd, fo, dang);
      }
      unsigned mask = __ballot_sync(0xffffffffu, in && len > 32);
      while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        const int rq0 = __shfl_sync(0xffffffffu, q0, j), rlen = __shfl_sync(0xffffffffu, len, j);
        float v = 0.f;
        for (int q = lane; q < rlen; q += 32) v = __fadd_rn(v, prod[rq0 + q]);
        v = butterfly(v);
        if (lane == 0) pr_store_x<UPDATE, XCH>(y, rb + j, lo, v, upd, fo, dang);
      }
    }
    __syncwarp();
  }
  if constexpr (XCH) pr_exchange_flush(dang, dsum_next);
}

// long rows: fold the chunk totals in chunk order
template <bool UPDATE, bool XCH = false>
__global__ void pr_fixup_kernel(const int* __restrict__ long_rows, int n_long, const float* __restrict__ chunk_tot,
                                const unsigned long long* __restrict__ dsum, float* __restrict__ y, int lo, int hi,
                                float base, float damp, float inv_v, const unsigned long long* __restrict__ peers,
                                int n_peers, const float* __restrict__ inv_outdeg, float* __restrict__ xs_next,
                                unsigned long long* __restrict__ dsum_next) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long dang = 0;
  if (i < n_long) {
    const int row = long_rows[3 * i];
    if (row >= lo && row < hi) {
      const int u0 = long_rows[3 * i + 1], nc = long_rows[3 * i + 2];
      float total = chunk_tot[u0];
      for (int c = 1; c < nc; ++c) total = __fadd_rn(total, chunk_tot[u0 + c]);
      Fanout fo{};
      if constexpr (XCH) fo = load_fanout(peers, n_peers, xs_next, inv_outdeg);
      pr_store_x<UPDATE, XCH>(y, row, lo, total, pr_update<UPDATE>(dsum, base, damp, inv_v), fo, dang);
    }
  }
  if constexpr (XCH) pr_exchange_flush(dang, dsum_next);
}

// validated (row_ptr version, slice) -> row_ptr[lo], row_ptr[hi]
struct PrCheckKey {
  int dev;
  const void* ptr;
  uint64_t version, lo, rows, col_bytes;
  int64_t nnz_off;
  bool operator<(const PrCheckKey& o) const {
    return std::tie(dev, ptr, version, lo, rows, col_bytes, nnz_off) <
           std::tie(o.dev, o.ptr, o.version, o.lo, o.rows, o.col_bytes, o.nnz_off);
  }
};
std::mutex g_pr_check_mu;
std::map<PrCheckKey, std::pair<int, int>> g_pr_check;

bool pr_check_cached(int dev, const BufView& R, uint64_t lo, uint64_t rows, uint64_t col_bytes, int64_t nnz_off,
                     int (&rp)[2]) {
  if (R.version == 0) return false;
  std::lock_guard<std::mutex> lock(g_pr_check_mu);
  auto it = g_pr_check.find({dev, R.ptr, R.version, lo, rows, col_bytes, nnz_off});
  if (it == g_pr_check.end()) return false;
  rp[0] = it->second.first;
  rp[1] = it->second.second;
  return true;
}

void pr_check_store(int dev, const BufView& R, uint64_t lo, uint64_t rows, uint64_t col_bytes, int64_t nnz_off,
                    const int (&rp)[2]) {
  if (R.version == 0) return;
  std::lock_guard<std::mutex> lock(g_pr_check_mu);
  if (g_pr_check.size() > 4096) g_pr_check.clear();
  g_pr_check[{dev, R.ptr, R.version, lo, rows, col_bytes, nnz_off}] = {rp[0], rp[1]};
}

// args: row_ptr col val units long_rows x [dsum] y | V nnz_off n_units n_long warp_nnz
// (IMP: no val argument; x is xs from pagerank_prep)
template <bool UPDATE, bool IMP = false, bool XCH = false>
uint64_t launch_pr(LaunchCtx& c) {
  const char* what = XCH ? "pagerank_step_exchange"
                         : IMP ? "pagerank_step_implicit" : UPDATE ? "pagerank_step" : "pagerank_spmv";
  constexpr uint32_t o = IMP ? 1 : 0;  // argument shift when there is no val buffer
  const uint32_t iy = (UPDATE ? 7 : 6) - o, s0 = iy + 1;
  const int64_t v = scalar_arg(c, s0, what), nnz_off = scalar_arg(c, s0 + 1, what);
  const int64_t n_units = scalar_arg(c, s0 + 2, what), n_long = scalar_arg(c, s0 + 3, what);
  const int64_t warp_nnz = scalar_arg(c, s0 + 4, what);
  if (v < 1 || v > INT32_MAX - 1) fail(ErrorCode::argument, std::string(what) + ": V out of range");
  if (warp_nnz < 1 || warp_nnz > PR_CHUNK)
    fail(ErrorCode::argument, std::string(what) + ": warp_nnz must be in [1, 4096]");
  const BufView& R = buffer_arg(c, 0, what);
  const BufView& Cb = buffer_arg(c, 1, what);
  const BufView& Vb = IMP ? Cb : buffer_arg(c, 2, what);
  const BufView& U = buffer_arg(c, 3 - o, what);
  const BufView& L = buffer_arg(c, 4 - o, what);
  const BufView& X = buffer_arg(c, 5 - o, what);
  if (R.first_byte != 0 || R.bytes != static_cast<uint64_t>(v + 1) * 4)
    fail(ErrorCode::argument, std::string(what) + ": row_ptr must hold V+1 int32");
  if (U.bytes != static_cast<uint64_t>(n_units) * 16 || L.bytes < static_cast<uint64_t>(n_long) * 12)
    fail(ErrorCode::argument, std::string(what) + ": units / long_rows sizes do not match their counts");
  if (Cb.bytes != Vb.bytes || Cb.first_byte != 0 || Vb.first_byte != 0)
    fail(ErrorCode::argument, std::string(what) + ": col_idx/values must be equal whole buffers (nnz_off for slices)");
  if (X.first_byte != 0 || X.bytes != static_cast<uint64_t>(v) * 4)
    fail(ErrorCode::argument, std::string(what) + ": x must hold V floats");
  const unsigned long long* dsum = nullptr;
  if (UPDATE) {
    const BufView& D = buffer_arg(c, 6 - o, what);
    if (D.bytes != 8) fail(ErrorCode::argument, std::string(what) + ": dangling sum is one uint64");
    dsum = reinterpret_cast<const unsigned long long*>(D.ptr);
  }
  const unsigned long long* peers = nullptr;
  int n_peers = 0;
  const float* inv_outdeg = nullptr;
  float* xs_next = nullptr;
  unsigned long long* dsum_next = nullptr;
  if (XCH) {  // peers (device addresses of the peers' xs'), their count, inv_outdeg, xs', dsum'
    n_peers = static_cast<int>(scalar_arg(c, s0 + 6, what));
    const BufView& PB = buffer_arg(c, s0 + 5, what);
    if (n_peers < 0 || n_peers > PR_MAX_PEERS || PB.first_byte != 0 || PB.bytes < static_cast<uint64_t>(n_peers) * 8)
      fail(ErrorCode::argument, std::string(what) + ": peers must list 0..7 device addresses");
    peers = reinterpret_cast<const unsigned long long*>(PB.ptr);
    const BufView& OD = buffer_arg(c, s0 + 7, what);
    const BufView& XN = buffer_arg(c, s0 + 8, what);
    const BufView& DN = buffer_arg(c, s0 + 9, what);
    if (OD.first_byte != 0 || OD.bytes != static_cast<uint64_t>(v) * 4 || XN.first_byte != 0 ||
        XN.bytes != static_cast<uint64_t>(v) * 4 || DN.bytes != 8)
      fail(ErrorCode::argument, std::string(what) + ": inv_outdeg and xs' must hold V elements, dsum' one uint64");
    inv_outdeg = reinterpret_cast<const float*>(OD.ptr);
    xs_next = reinterpret_cast<float*>(XN.ptr);
    dsum_next = reinterpret_cast<unsigned long long*>(DN.ptr);
    HCL_CUDA(cudaMemsetAsync(dsum_next, 0, 8, c.stream));
  }
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(v), lo, rows, what);
  float* y = at_byte<float>(buffer_arg(c, iy, what), lo * 4, rows * 4, what);
  if (!rows || !n_units) return 0;
  const int* row_ptr = reinterpret_cast<const int*>(R.ptr);
  // the non-zeros of [lo, hi) must be resident: two int32 reads of row_ptr with a
  // host round trip -- done once per (row_ptr contents, slice) and cached by
  // the buffer's write version, so iterations do not stall the stream
  int rp[2];
  if (!pr_check_cached(c.dev, R, lo, rows, Cb.bytes, nnz_off, rp)) {
    HCL_CUDA(cudaMemcpyAsync(&rp[0], row_ptr + lo, 4, cudaMemcpyDeviceToHost, c.stream));
    HCL_CUDA(cudaMemcpyAsync(&rp[1], row_ptr + lo + rows, 4, cudaMemcpyDeviceToHost, c.stream));
    HCL_CUDA(cudaStreamSynchronize(c.stream));
    if (rp[0] < nnz_off || static_cast<uint64_t>(rp[1] - nnz_off) * 4 > Cb.bytes)
      fail(ErrorCode::argument, std::string(what) + ": col_idx/values do not cover the rows' non-zeros");
    pr_check_store(c.dev, R, lo, rows, Cb.bytes, nnz_off, rp);
  }
  float* chunk_tot = static_cast<float*>(c.scratch(c.dev, static_cast<size_t>(n_units) * 4));
  const float base = static_cast<float>((1.0 - 0.85) / v), damp = 0.85f, inv_v = static_cast<float>(1.0 / v);
  const size_t smem = static_cast<size_t>(warp_nnz) * 4 * PR_WARPS;
  auto kern = pr_units_kernel<UPDATE, IMP, XCH>;
  HCL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  HCL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PR_T, smem));
  const int grid = std::max(1, per_sm) * c.sm_count;
  kern<<<grid, PR_T, smem, c.stream>>>(row_ptr, reinterpret_cast<const int*>(Cb.ptr),
                                       IMP ? nullptr : reinterpret_cast<const float*>(Vb.ptr), nnz_off,
                                       reinterpret_cast<const int4*>(U.ptr), static_cast<int>(n_units),
                                       reinterpret_cast<const float*>(X.ptr), dsum, y, static_cast<int>(lo),
                                       static_cast<int>(lo + rows), base, damp, inv_v, static_cast<int>(warp_nnz),
                                       chunk_tot, peers, n_peers, inv_outdeg, xs_next, dsum_next);
  HCL_LAUNCHED();
  if (n_long) {
    pr_fixup_kernel<UPDATE, XCH><<<static_cast<unsigned>(ceil_div(n_long, 128)), 128, 0, c.stream>>>(
        reinterpret_cast<const int*>(L.ptr), static_cast<int>(n_long), chunk_tot, dsum, y, static_cast<int>(lo),
        static_cast<int>(lo + rows), base, damp, inv_v, peers, n_peers, inv_outdeg, xs_next, dsum_next);
    HCL_LAUNCHED();
  }
  return 2ull * static_cast<uint64_t>(rp[1] - rp[0]);
}

// xs[i] = val(i) * x[i], val(i) = 1/outdeg(i) rounded to fp32 exactly as the CSR
// builder stores it (hcl_pagerank_csr), 0 for dangling vertices; fused with the
// dangling sum. With xs the SpMV's products are single gathers, bit-identical
// to val[p] * x[col[p]], and the 4-byte-per-edge value stream disappears.
__global__ void __launch_bounds__(256) pr_prep_kernel(const float* __restrict__ x, const int* __restrict__ outdeg,
                                                      int64_t v, float* __restrict__ xs,
                                                      unsigned long long* __restrict__ out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0;
  for (int64_t i = tid; i < v; i += stride) {
    const int d = __ldcs(outdeg + i);
    const float xi = __ldcs(x + i);
    if (d == 0) s += static_cast<unsigned long long>(__float2ll_rz(__fmul_rn(xi, 0x1p56f)));
    xs[i] = d ? __fmul_rn(__fdiv_rn(1.0f, static_cast<float>(d)), xi) : 0.f;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// pagerank_prep(x, outdeg, dsum, xs, V)
uint64_t launch_pr_prep(LaunchCtx& c) {
  int64_t v = scalar_arg(c, 4, "pagerank_prep V");
  const BufView& X = buffer_arg(c, 0, "pagerank_prep x");
  const BufView& O = buffer_arg(c, 1, "pagerank_prep outdeg");
  const BufView& D = buffer_arg(c, 2, "pagerank_prep dsum");
  const BufView& XS = buffer_arg(c, 3, "pagerank_prep xs");
  if (X.first_byte != 0 || X.bytes != static_cast<uint64_t>(v) * 4 || O.first_byte != 0 ||
      O.bytes != static_cast<uint64_t>(v) * 4 || D.bytes != 8 || XS.first_byte != 0 ||
      XS.bytes != static_cast<uint64_t>(v) * 4)
    fail(ErrorCode::argument, "pagerank_prep: x, outdeg, xs must hold V elements, dsum one uint64");
  HCL_CUDA(cudaMemsetAsync(D.ptr, 0, 8, c.stream));
  int grid = static_cast<int>(std::min<uint64_t>(c.sm_count * 8, ceil_div(v, 256)));
  pr_prep_kernel<<<grid, 256, 0, c.stream>>>(reinterpret_cast<const float*>(X.ptr),
                                             reinterpret_cast<const int*>(O.ptr), v,
                                             reinterpret_cast<float*>(XS.ptr),
                                             reinterpret_cast<unsigned long long*>(D.ptr));
  HCL_LAUNCHED();
  return static_cast<uint64_t>(v);
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
  int grid = static_cast<int>(std::min<uint64_t>(c.sm_count * 8, ceil_div(v / 8 + 1, 256)));
  pr_dangling_kernel<<<grid, 256, 0, c.stream>>>(reinterpret_cast<const float*>(X.ptr),
                                                 reinterpret_cast<const int*>(O.ptr), v,
                                                 reinterpret_cast<unsigned long long*>(D.ptr));
  HCL_LAUNCHED();
  return static_cast<uint64_t>(v);
}

uint64_t rows_pr(const int64_t* s, uint32_t n) { return static_cast<uint64_t>(s[n == 13 ? 8 : 7]); }
uint64_t rows_pr_imp(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[7]); }

}  // namespace

void register_graph(std::vector<KernelDef>& r) {
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS;
  // y = A x over rows [lo,hi): row_ptr col val units long_rows x y | V nnz_off n_units n_long warp_nnz
  r.push_back({"b200", "pagerank_spmv", {I, I, I, I, I, I, O, S, S, S, S, S}, {P, P, P, P, P, P, X, N, N, N, N, N},
               launch_pr<false>, nullptr, rows_pr});
  // x' = (1-d)/V + d (A x + dangling/V): row_ptr col val units long_rows x dsum x' | V nnz_off n_units n_long warp_nnz
  r.push_back({"b200", "pagerank_step", {I, I, I, I, I, I, I, O, S, S, S, S, S},
               {P, P, P, P, P, P, P, X, N, N, N, N, N}, launch_pr<true>, nullptr, rows_pr});
  r.push_back({"b200", "pagerank_dangling", {I, I, O, S}, {P, P, P, N}, launch_pr_dangling, nullptr, nullptr});
  // implicit values (val = 1/outdeg(src)): pagerank_prep(x, outdeg, dsum, xs, V), then
  // pagerank_step_implicit(row_ptr col units long_rows xs dsum x' | V nnz_off n_units n_long warp_nnz)
  r.push_back({"b200", "pagerank_prep", {I, I, O, O, S}, {P, P, P, P, N}, launch_pr_prep, nullptr, nullptr});
  r.push_back({"b200", "pagerank_step_implicit", {I, I, I, I, I, I, O, S, S, S, S, S},
               {P, P, P, P, P, P, X, N, N, N, N, N}, launch_pr<true, true>, nullptr, rows_pr_imp});
  // the implicit step fused with the next prep and the exchange: x' rows, xs' rows here and on
  // every peer (peers = device addresses of their xs', uint64[n_peers]), dangling partial dsum':
  // row_ptr col units long_rows xs dsum x' | V nnz_off n_units n_long warp_nnz | peers n_peers inv_outdeg xs' dsum'
  // (inv_outdeg = fl(1/outdeg) as fp32, 0 for dangling vertices: datagen.pagerank_inv_outdeg)
  constexpr uint8_t XG = HCL_PART_EXCHANGE, PR = HCL_PART_PEERS, RS = HCL_PART_REDUCE_SUM;
  r.push_back({"b200", "pagerank_step_exchange", {I, I, I, I, I, I, O, S, S, S, S, S, I, S, I, O, O},
               {P, P, P, P, P, P, X, N, N, N, N, N, PR, N, P, XG, RS}, launch_pr<true, true, true>, nullptr,
               rows_pr_imp});
}

}  // namespace hcl
