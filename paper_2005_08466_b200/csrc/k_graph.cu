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
#include "ptx.cuh"
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
  float* mc;            // NVSwitch multicast address of xs' on every rank (n_peers == PR_MULTICAST), else null
  float scale;          // xs' = fl(inv * x') * scale: 1, or 2^56 for the binned step (exact: a power of two)
};

// n_peers == PR_MULTICAST: peers[0] is the multicast mapping of the ranks' xs'
// buffers (one store reaches every GPU through the switch: the egress per row
// is 4 bytes whatever the rank count, not 4 * (N - 1))
constexpr int PR_MULTICAST = -1;

__device__ __forceinline__ Fanout load_fanout(const unsigned long long* peers, int n, float* xs, const float* inv,
                                              float scale = 1.f) {
  Fanout f;
  f.scale = scale;
  f.mc = n == PR_MULTICAST ? reinterpret_cast<float*>(__ldg(peers)) : nullptr;
  f.n = n < 0 ? 0 : n;
  f.xs = xs;
  f.inv = inv;
#pragma unroll
  for (int k = 0; k < PR_MAX_PEERS; ++k) f.p[k] = k < f.n ? reinterpret_cast<float*>(__ldg(peers + k)) : nullptr;
  return f;
}

__device__ __forceinline__ void multimem_st(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}

template <bool UPDATE, bool XCH>
__device__ __forceinline__ void pr_store_x(float* __restrict__ y, int r, int lo, float s, const Update& u,
                                           const Fanout& f, unsigned long long& dang) {
  const float v = pr_store<UPDATE>(y, r, lo, s, u);
  if constexpr (XCH) {
    const float inv = __ldg(f.inv + r);  // the division is done once per graph, not per step
    const float xs = __fmul_rn(__fmul_rn(inv, v), f.scale);
    f.xs[r] = xs;  // (the multicast store lands here too, the same value)
    if (f.mc) multimem_st(f.mc + r, xs);
#pragma unroll
    for (int k = 0; k < PR_MAX_PEERS; ++k)
      if (k < f.n) f.p[k][r] = xs;
    if (inv == 0.f) dang += static_cast<unsigned long long>(__float2ll_rz(__fmul_rn(v, 0x1p56f)));
  }
}

// end of an exchange kernel: the block's dangling partial into dsum', and the
// peer stores made visible system-wide before the allreduce that follows
__device__ __forceinline__ void pr_exchange_flush(unsigned long long dang, unsigned long long* dsum_next,
                                                  int n_peers = 1) {
  for (int o = 16; o > 0; o >>= 1) dang += __shfl_xor_sync(0xffffffffu, dang, o);
  if ((threadIdx.x & 31) == 0 && dang) atomicAdd(dsum_next, dang);
  if (n_peers) __threadfence_system();  // same-device readers are ordered by the kernel boundary
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
                                                      unsigned long long* __restrict__ out, float scale) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0;
  for (int64_t i = tid; i < v; i += stride) {
    const int d = __ldcs(outdeg + i);
    const float xi = __ldcs(x + i);
    if (d == 0) s += static_cast<unsigned long long>(__float2ll_rz(__fmul_rn(xi, 0x1p56f)));
    xs[i] = d ? __fmul_rn(__fmul_rn(__fdiv_rn(1.0f, static_cast<float>(d)), xi), scale) : 0.f;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// pagerank_prep(x, outdeg, dsum, xs, V); pagerank_prep_fixed: the same with xs scaled by
// 2^56 (the binned step's gather input: its fixed-point terms are then one conversion)
template <bool FIXED>
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
                                             reinterpret_cast<unsigned long long*>(D.ptr), FIXED ? 0x1p56f : 1.f);
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

// ---------------------------------------------------------------------------
// Binned PageRank step (propagation blocking; layout: csrc/host/pagerank_bins.cpp).
//
// The pull formulation gathers x at 2^28 random column indices per iteration:
// one 32-byte sector per 4-byte value, bounded by the L1TEX wavefront rate
// (~0.95 ms at C3), a quarter of HBM speed. The binned step replaces the
// random gathers by two streaming passes:
//   scatter: per chunk of the edges in source order, stage the chunk's gather
//            inputs c[u0 .. u0+span) in shared memory and write each edge's
//            value c[src] into its destination bin's segment (bin-major
//            stream; consecutive lanes write consecutive addresses);
//   gather:  per bin (heavy bins split into units), stream the bin's values
//            and uint16 destination offsets into a shared-memory accumulator
//            of the bin's rows, then finish the rows (the PageRank update, the
//            next gather input xs' = fl(1/outdeg) x' into every device's copy,
//            the dangling partial) -- the same epilogue as
//            pagerank_step_exchange.
// Row sums are order free: each value is rounded to the 2^-56 fixed-point grid
// (RN; values are < 1, sums <= 1 < 2^8) and summed exactly in uint64, so the
// result does not depend on the layout, the unit split or the atomics' order;
// the oracle restates it (ho_spmv_f32_fixed). Bytes per edge and iteration:
// 2 (src_local) + 4 (value write) + 4 (value read) + 2 (dst16) = 12, against
// 8 for the pull CSR's col_idx + gathered x sector-free ideal -- but streamed.

constexpr int PB_T = 512;
constexpr int PB_WARPS = PB_T / 32;

// parts table row (int64): one per partition of the rows, built by
// paper_2005_08466_b200/pagerank.py from hcl_pagerank_bins_build
enum PbPart {
  PB_LO = 0, PB_HI, PB_CHUNK0, PB_NCHUNKS, PB_NBINS, PB_GSTRIDE, PB_DESC0, PB_SRC0, PB_ENT0, PB_UNIT0,
  PB_NUNITS, PB_SLOT0, PB_NSLOTS, PB_BINROWS, PB_SPAN, PB_NEDGES, PB_CHUNK_EDGES, PB_FIELDS = 20
};

__device__ __forceinline__ int ld_stream_u16(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

// block-wide exclusive scan of n <= PB_T * 8 ints in shared memory (in place);
// returns the total. tmp: PB_WARPS ints.
__device__ int block_exclusive_scan(int* a, int n, int* tmp) {
  constexpr int PER = 8;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  int v[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = t * PER + k;
    v[k] = i < n ? a[i] : 0;
    sum += v[k];
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) tmp[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < PB_WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane < PB_WARPS) tmp[lane] = x;
  }
  __syncthreads();
  int run = incl - sum + (w ? tmp[w - 1] : 0);
  const int total = tmp[PB_WARPS - 1];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = t * PER + k;
    if (i < n) a[i] = run;
    run += v[k];
  }
  __syncthreads();
  return total;
}

// Phase 1, persistent CTAs (2 per SM) walking the chunks; each CTA keeps two
// stages, so chunk i+1's bulk copies (TMA) fly while chunk i is written out.
// A stage holds the chunk's descriptor (per 32-entry window {bitmap of the
// entries that start a non-empty segment, segments started before the
// window}, then per segment delta = bin-major start - chunk-local start), its
// src_local and the gather inputs c[u0 .. u0+span) (from the 16-byte aligned
// address below u0). Entry f of window w belongs to segment k = k_base[w] +
// popcount(bitmap[w] & lanes <= f) - 1 and goes to vals[delta[k] + f]: each
// warp writes a contiguous run of windows, consecutive lanes to consecutive
// addresses inside a segment. No search and no block-wide step per chunk.
__global__ void __launch_bounds__(PB_T, 2) pr_bin_scatter_kernel(const int64_t* __restrict__ part,
                                                                 const int4* __restrict__ chunks,
                                                                 const uint16_t* __restrict__ src_local,
                                                                 const uint32_t* __restrict__ cdesc,
                                                                 const float* __restrict__ xs, int64_t v,
                                                                 float* __restrict__ vals, int nst) {
  extern __shared__ __align__(128) uint8_t pb_smem[];
  const int64_t n_chunks = part[PB_NCHUNKS], nb = part[PB_NBINS];
  const int64_t span_max = part[PB_SPAN], ce = part[PB_CHUNK_EDGES];
  const int64_t nwin_max = (ce + 31) >> 5;
  const int64_t wcap = (2 * nwin_max + 3) & ~int64_t(3), dcap = (nb + 3) & ~int64_t(3);  // words
  const int64_t scap = ((ce + 7) & ~int64_t(7)) / 2, ccap = (span_max + 6) & ~int64_t(3);
  const int64_t stage_words = wcap + dcap + scap + ccap;
  uint64_t* bar = reinterpret_cast<uint64_t*>(pb_smem + nst * stage_words * 4);  // nst stages + the records
  int4* rec = reinterpret_cast<int4*>(bar + 4);  // this CTA's chunk records (2 int4 each)
  chunks += 2 * part[PB_CHUNK0];
  src_local += part[PB_SRC0];
  cdesc += part[PB_DESC0];
  vals += part[PB_ENT0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lanemask_le = 0xffffffffu >> (31 - lane);
  auto stage = [&](int b) { return pb_smem + static_cast<int64_t>(b) * stage_words * 4; };
  // one elected thread: the chunk's bulk copies into stage b
  auto issue = [&](const int4& C, const int4& D, int b) {
    uint8_t* st = stage(b);
    const int nwin = (C.w + 31) >> 5;
    const int64_t ua = C.x & ~3, cnt = ((C.x - ua) + C.y + 3) & ~3;
    const int wwords = (2 * nwin + 3) & ~3, dwords = (D.y + 3) & ~3;
    const uint32_t sbytes = C.y > 1 ? ((C.w + 7) & ~7) * 2 : 0;
    const uint32_t cbytes = ua + cnt <= v ? static_cast<uint32_t>(cnt * 4) : 0;
    ptx::mbar_arrive_expect_tx(&bar[b], static_cast<uint32_t>(wwords + dwords) * 4 + sbytes + cbytes);
    ptx::bulk_load(st, cdesc + D.x, static_cast<uint32_t>(wwords) * 4, &bar[b]);
    if (dwords) ptx::bulk_load(st + wcap * 4, cdesc + D.x + wwords, static_cast<uint32_t>(dwords) * 4, &bar[b]);
    if (sbytes) ptx::bulk_load(st + (wcap + dcap) * 4, src_local + C.z, sbytes, &bar[b]);
    if (cbytes) ptx::bulk_load(st + (wcap + dcap + scap) * 4, xs + ua, cbytes, &bar[b]);
  };
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::mbar_init(&bar[2], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // this CTA's chunks: blockIdx.x, + gridDim.x, ... (neighbouring CTAs write
  // neighbouring segments of each bin at about the same time); their records
  // are copied into shared memory once (no global load on the per-chunk path)
  const int nrec = static_cast<int>((n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x);
  if (nrec <= 0) return;
  for (int i = threadIdx.x; i < 2 * nrec; i += PB_T)
    rec[i] = __ldg(chunks + 2 * (blockIdx.x + static_cast<int64_t>(i >> 1) * gridDim.x) + (i & 1));
  __syncthreads();
  if (threadIdx.x == 0) issue(rec[0], rec[1], 0);
  for (int it = 0; it < nrec; ++it) {
    const int b = nst == 2 ? (it & 1) : 0;
    if (nst == 2 && it + 1 < nrec && threadIdx.x == 0) issue(rec[2 * it + 2], rec[2 * it + 3], b ^ 1);
    const int4 C = rec[2 * it];  // u0, span, src_off, n
    uint8_t* st = stage(b);
    const uint2* win = reinterpret_cast<const uint2*>(st);
    const int* delta = reinterpret_cast<const int*>(st + wcap * 4);
    const uint16_t* sl = reinterpret_cast<const uint16_t*>(st + (wcap + dcap) * 4);
    float* cs = reinterpret_cast<float*>(st + (wcap + dcap + scap) * 4);
    const int64_t ua = C.x & ~3, cnt = ((C.x - ua) + C.y + 3) & ~3;
    if (ua + cnt > v) {  // c's tail is not 16-byte complete: plain loads
      for (int i = threadIdx.x; i < C.y; i += PB_T) cs[C.x - ua + i] = __ldg(xs + C.x + i);
      __syncthreads();
    }
    ptx::mbar_wait(&bar[b], static_cast<uint32_t>((nst == 2 ? it >> 1 : it) & 1));
    const float* csu = cs + (C.x - ua);
    const int nwin = (C.w + 31) >> 5;
    const int per = (nwin + PB_WARPS - 1) / PB_WARPS;
    const int w0 = warp * per, w1 = min(nwin, w0 + per);
    const int wfull = min(w1, C.w >> 5);  // windows without a ragged tail
    auto dest = [&](int w, int f) -> unsigned {
      const uint2 d = win[w];
      return static_cast<unsigned>(delta[static_cast<int>(d.y + __popc(d.x & lanemask_le)) - 1] + f);
    };
    if (C.y == 1) {  // single-source piece: every entry is c[u0]
      const float val = csu[0];
      int w = w0;
      for (; w < wfull; ++w) vals[dest(w, 32 * w + lane)] = val;
      if (w < w1 && 32 * w + lane < C.w) vals[dest(w, 32 * w + lane)] = val;
    } else {
      int w = w0;
#pragma unroll 4
      for (; w < wfull; ++w) {
        const int f = 32 * w + lane;
        vals[dest(w, f)] = csu[sl[f]];
      }
      if (w < w1 && 32 * w + lane < C.w) vals[dest(w, 32 * w + lane)] = csu[sl[32 * w + lane]];
    }
    __syncthreads();  // every warp is done with stage b before it is refilled
    if (nst == 1 && it + 1 < nrec && threadIdx.x == 0) issue(rec[2 * it + 2], rec[2 * it + 3], 0);
  }
}

// shared-memory 32-bit add under a predicate, without a branch (atom returns
// the old value; 0 when the predicate is off)
__device__ __forceinline__ unsigned atoms_add_if(unsigned* p, unsigned v, bool pred) {
  unsigned old;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tmov.u32 %0, 0;\n\t"
      "@q atom.shared.add.u32 %0, [%1], %2;\n\t}"
      : "=r"(old)
      : "r"(ptx::smem_u32(p)), "r"(v), "r"(static_cast<unsigned>(pred))
      : "memory");
  return old;
}
__device__ __forceinline__ void reds_add_if(unsigned* p, unsigned v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}" ::"r"(
          ptx::smem_u32(p)),
      "r"(v), "r"(static_cast<unsigned>(pred))
      : "memory");
}

// Phase 2, one unit per CTA. The unit's entries stream through shared memory
// by bulk copies (TMA): one elected thread keeps PBG_STAGES stages of
// PBG_STAGE entries (values + uint16 destinations) in flight, so the HBM
// stream does not wait for the atomics; each thread takes 8 consecutive
// entries of a stage. The bin's row sums live in shared memory as two uint32
// words per row (64-bit shared atomics compile to CAS loops; the low word's
// carry goes into the high word, so (hi, lo) is the exact 64-bit sum in any
// order).
// T threads per CTA, a stage of 8 T entries: T = 1024 with 16384-row bins (one
// CTA per SM), T = 512 with <= 8192-row bins (two CTAs per SM)
constexpr int PBG_STAGES = 2;
// Row r of a bin accumulates at shared word pb_swz(r): the low 5 bits (the bank)
// XOR-folded with bits 5-9 and 10-14, a bijection inside each 32-row block. R-MAT
// ids are skewed toward 0 in every bit, so dst mod 32 alone puts ~25% of the
// entries on bank 0: the busiest bank of an atomic instruction averages 4.1
// lanes, folded 2.7 (scratch evaluation of the C3 layout). ncu at C3: 66.5M ->
// 39.4M atomic wavefronts, gather 545 -> 481 us alone (issue-bound after); inside
// the step the gather is memory-bound and gains ~2%.
__device__ __forceinline__ int pb_swz(int r) { return r ^ ((r >> 5) & 31) ^ ((r >> 10) & 31); }
template <int PBG_T>
__global__ void __launch_bounds__(PBG_T) pr_bin_gather_kernel(const int64_t* __restrict__ part,
                                                             const int4* __restrict__ units,
                                                             const int* __restrict__ slot_units,
                                                             const float* __restrict__ vals,
                                                             const uint16_t* __restrict__ dst16,
                                                             unsigned long long* __restrict__ slot_acc,
                                                             unsigned int* __restrict__ slot_cnt,
                                                             const unsigned long long* __restrict__ dsum,
                                                             float* __restrict__ y, int lo, float base, float damp,
                                                             float inv_v, const unsigned long long* __restrict__ peers,
                                                             int n_peers, const float* __restrict__ inv_outdeg,
                                                             float* __restrict__ xs_next,
                                                             unsigned long long* __restrict__ dsum_next) {
  constexpr int PBG_STAGE = 8 * PBG_T, PBG_STAGE_BYTES = PBG_STAGE * 6;
  extern __shared__ __align__(128) uint8_t pg_smem[];
  __shared__ int last_flag;
  const int64_t W = part[PB_BINROWS], hi = part[PB_HI];
  uint8_t* stage0 = pg_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + PBG_STAGES * PBG_STAGE_BYTES);
  uint64_t* empty = full + PBG_STAGES;
  unsigned* acc_lo = reinterpret_cast<unsigned*>(empty + PBG_STAGES);
  // whole 32-row blocks (pb_swz); with <= 8192-row bins the high words sit at a
  // constant offset, so each atomic pair shares one address register
  unsigned* acc_hi = acc_lo + (PBG_T == 512 ? 8192 : ((W + 31) & ~int64_t(31)));
  const int4 U = __ldg(units + part[PB_UNIT0] + blockIdx.x);  // bin, e0, e1, slot
  const int64_t row0 = lo + static_cast<int64_t>(U.x) * W;
  const int64_t rem = hi - row0;
  const int nrows = static_cast<int>(W < rem ? W : rem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  vals += part[PB_ENT0];
  dst16 += part[PB_ENT0];
  const int64_t n_ent = U.z - U.y, n_st = (n_ent + PBG_STAGE - 1) / PBG_STAGE;
  auto issue = [&](int64_t st) {  // stage st of the unit into buffer st % PBG_STAGES
    const int b = static_cast<int>(st % PBG_STAGES);
    uint8_t* sp = stage0 + b * PBG_STAGE_BYTES;
    const int64_t e = U.y + st * PBG_STAGE;
    const uint32_t cnt = static_cast<uint32_t>(min(static_cast<int64_t>(PBG_STAGE), U.z - e));  // multiple of 8
    ptx::mbar_arrive_expect_tx(&full[b], cnt * 6);
    ptx::bulk_load(sp, vals + e, cnt * 4, &full[b]);
    ptx::bulk_load(sp + PBG_STAGE * 4, dst16 + e, cnt * 2, &full[b]);
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < PBG_STAGES; ++b) {
      ptx::mbar_init(&full[b], 1);
      ptx::mbar_init(&empty[b], PBG_T / 32);
    }
    ptx::fence_mbar_init();
    for (int64_t st = 0; st < min(n_st, static_cast<int64_t>(PBG_STAGES)); ++st) issue(st);
  }
  for (int r = threadIdx.x; r < nrows; r += PBG_T) acc_lo[pb_swz(r)] = acc_hi[pb_swz(r)] = 0u;
  __syncthreads();
  for (int64_t st = 0; st < n_st; ++st) {
    const int b = static_cast<int>(st % PBG_STAGES);
    ptx::mbar_wait(&full[b], static_cast<uint32_t>((st / PBG_STAGES) & 1));
    const uint8_t* sp = stage0 + b * PBG_STAGE_BYTES;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(PBG_STAGE), n_ent - st * PBG_STAGE));
    // this thread's group of 8 consecutive entries: the lanes of a warp take
    // groups 32 apart (skewed by the warp so the stage reads spread over the
    // banks), so the lanes of one atomic rarely share a hub row's run
    const int grp = lane * (PBG_T / 32) + ((warp + lane) & (PBG_T / 32 - 1));
    {
      // segments are sorted by destination, so a hub row's entries come in
      // runs -- each run is added up in registers and lands with one
      // (predicated, branch-free) atomic at its last entry. Lanes past a
      // ragged last stage carry value 0 (no atomics) but stay converged.
      const bool valid = 8 * grp < cnt;
      const float4 zf = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 va = valid ? reinterpret_cast<const float4*>(sp)[2 * grp] : zf;
      const float4 vb = valid ? reinterpret_cast<const float4*>(sp)[2 * grp + 1] : zf;
      const uint4 d = valid ? reinterpret_cast<const uint4*>(sp + PBG_STAGE * 4)[grp] : make_uint4(0, 0, 0, 0);
      const float vv[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
      const unsigned dd[8] = {d.x & 0xffffu, d.x >> 16, d.y & 0xffffu, d.y >> 16,
                              d.z & 0xffffu, d.z >> 16, d.w & 0xffffu, d.w >> 16};
      unsigned long long run = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // the gather input is scaled by 2^56 (pagerank_prep_fixed / the epilogue below):
        // the fixed-point term is one conversion, the same value as fl(v * 2^56)
        const unsigned long long q = __float2ull_rn(vv[k]);
        run = (k > 0 && dd[k] == dd[k - 1]) ? run + q : q;
        const bool last = k == 7 || dd[k] != dd[k + 1];
        const unsigned ql = static_cast<unsigned>(run);
        const int sw = static_cast<int>(dd[k]);  // dst16 is stored bank-folded (pb_swz)
        const unsigned old = atoms_add_if(acc_lo + sw, ql, last);  // (a zero ql adds nothing)
        // carry out of the low word: add with carry-out, then the high half plus the carry
        unsigned qh;
        asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}"
            : "=r"(qh)
            : "r"(old), "r"(ql), "r"(static_cast<unsigned>(run >> 32)));
        // predicated, not branched on a vote: the vote's convergence barriers cost more
        // issue slots than the mostly-off red (gather 469 -> 449 us at C3)
        reds_add_if(acc_hi + sw, qh, last && qh != 0u);
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[b]);
    if (threadIdx.x == 0 && st + PBG_STAGES < n_st) {  // refill once every warp is done with the stage
      ptx::mbar_wait(&empty[b], static_cast<uint32_t>((st / PBG_STAGES) & 1));
      issue(st + PBG_STAGES);
    }
  }
  __syncthreads();
  auto acc = [&](int r) -> unsigned long long {  // row r's sum
    const int sw = pb_swz(r);
    return (static_cast<unsigned long long>(acc_hi[sw]) << 32) | acc_lo[sw];
  };
  if (U.w >= 0) {  // a heavy bin split into units: combine in the slot, the last unit finishes the rows
    const int slot = static_cast<int>(part[PB_SLOT0]) + U.w;
    unsigned long long* sa = slot_acc + static_cast<int64_t>(slot) * W;
    for (int r = threadIdx.x; r < nrows; r += PBG_T)
      if (const unsigned long long a = acc(r)) atomicAdd(sa + r, a);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
      last_flag = atomicAdd(slot_cnt + slot, 1u) == static_cast<unsigned>(__ldg(slot_units + slot) - 1);
    __syncthreads();
    if (!last_flag) return;
    __threadfence();
    for (int r = threadIdx.x; r < nrows; r += PBG_T) {
      const unsigned long long a = __ldcg(sa + r);
      acc_lo[pb_swz(r)] = static_cast<unsigned>(a);
      acc_hi[pb_swz(r)] = static_cast<unsigned>(a >> 32);
      sa[r] = 0ull;  // the slot is zero again for the next step
    }
    if (threadIdx.x == 0) slot_cnt[slot] = 0u;
    __syncthreads();
  }
  const Update upd = pr_update<true>(dsum, base, damp, inv_v);
  const Fanout fo = load_fanout(peers, n_peers, xs_next, inv_outdeg, 0x1p56f);
  unsigned long long dang = 0;
  for (int r = threadIdx.x; r < nrows; r += PBG_T) {
    const float s = static_cast<float>(__ll2double_rn(static_cast<long long>(acc(r))) * 0x1p-56);
    pr_store_x<true, true>(y, static_cast<int>(row0 + r), lo, s, upd, fo, dang);
  }
  pr_exchange_flush(dang, dsum_next, n_peers);
}

struct PbPartRow {
  int64_t f[PB_FIELDS];
};
struct PbKey {
  int dev;
  const void* ptr;
  uint64_t version;
  bool operator<(const PbKey& o) const { return std::tie(dev, ptr, version) < std::tie(o.dev, o.ptr, o.version); }
};
std::mutex g_pb_mu;
std::map<PbKey, std::vector<PbPartRow>> g_pb_parts;

// pagerank_step_binned(parts chunks src_local gtab dst16 units slot_units xs dsum x' | V n_parts |
// (xs and xs' are the gather inputs scaled by 2^56: pagerank_prep_fixed, this epilogue)
//                      peers n_peers inv_outdeg xs' dsum' | vals(LOCAL) slot_acc(LOCAL))
uint64_t launch_pr_binned(LaunchCtx& c) {
  const char* what = "pagerank_step_binned";
  const int64_t v = scalar_arg(c, 10, what), n_parts = scalar_arg(c, 11, what);
  const int n_peers = static_cast<int>(scalar_arg(c, 13, what));
  if (v < 1 || v > INT32_MAX - 1 || n_parts < 1) fail(ErrorCode::argument, std::string(what) + ": bad V or parts");
  const BufView& PT = buffer_arg(c, 0, what);
  if (PT.first_byte != 0 || PT.bytes != static_cast<uint64_t>(n_parts) * PB_FIELDS * 8)
    fail(ErrorCode::argument, std::string(what) + ": the parts table holds " + std::to_string(PB_FIELDS) +
                                  " int64 per part");
  const BufView& CH = buffer_arg(c, 1, what);
  const BufView& SL = buffer_arg(c, 2, what);
  const BufView& GT = buffer_arg(c, 3, what);
  const BufView& DS = buffer_arg(c, 4, what);
  const BufView& UN = buffer_arg(c, 5, what);
  const BufView& SU = buffer_arg(c, 6, what);
  const BufView& XS = buffer_arg(c, 7, what);
  const BufView& D = buffer_arg(c, 8, what);
  const BufView& PB = buffer_arg(c, 12, what);
  const BufView& OD = buffer_arg(c, 14, what);
  const BufView& XN = buffer_arg(c, 15, what);
  const BufView& DN = buffer_arg(c, 16, what);
  const BufView& VA = buffer_arg(c, 17, what);
  const BufView& SA = buffer_arg(c, 18, what);
  if (XS.bytes != static_cast<uint64_t>(v) * 4 || OD.bytes != static_cast<uint64_t>(v) * 4 ||
      XN.bytes != static_cast<uint64_t>(v) * 4 || D.bytes != 8 || DN.bytes != 8)
    fail(ErrorCode::argument, std::string(what) + ": xs, inv_outdeg, xs' must hold V floats, dsum/dsum' one uint64");
  if (n_peers < PR_MULTICAST || n_peers > PR_MAX_PEERS || PB.bytes < static_cast<uint64_t>(n_peers < 0 ? 1 : n_peers) * 8)
    fail(ErrorCode::argument, std::string(what) + ": peers must list 0..7 device addresses (or -1: one multicast address)");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(v), lo, rows, what);
  float* y = at_byte<float>(buffer_arg(c, 9, what), lo * 4, rows * 4, what);
  HCL_CUDA(cudaMemsetAsync(DN.ptr, 0, 8, c.stream));
  if (!rows) return 0;
  // the host copy of the parts table (read once per table contents)
  std::vector<PbPartRow> parts;
  {
    std::lock_guard<std::mutex> lock(g_pb_mu);
    auto it = PT.version ? g_pb_parts.find({c.dev, PT.ptr, PT.version}) : g_pb_parts.end();
    if (it != g_pb_parts.end()) parts = it->second;
  }
  if (parts.empty()) {
    parts.resize(static_cast<size_t>(n_parts));
    HCL_CUDA(cudaMemcpyAsync(parts.data(), PT.ptr, PT.bytes, cudaMemcpyDeviceToHost, c.stream));
    HCL_CUDA(cudaStreamSynchronize(c.stream));
    if (PT.version) {
      std::lock_guard<std::mutex> lock(g_pb_mu);
      if (g_pb_parts.size() > 256) g_pb_parts.clear();
      g_pb_parts[{c.dev, PT.ptr, PT.version}] = parts;
    }
  }
  int pi = -1;
  for (int i = 0; i < static_cast<int>(parts.size()); ++i)
    if (parts[i].f[PB_LO] == static_cast<int64_t>(lo) && parts[i].f[PB_HI] == static_cast<int64_t>(lo + rows)) pi = i;
  if (pi < 0) fail(ErrorCode::argument, std::string(what) + ": no part of the layout covers rows [" +
                                            std::to_string(lo) + ", " + std::to_string(lo + rows) + ")");
  const int64_t* P = parts[pi].f;
  const int64_t nb = P[PB_NBINS], gs = P[PB_GSTRIDE], W = P[PB_BINROWS], span = P[PB_SPAN];
  if (nb > PB_T * 8 || nb < 1 || gs < nb + 1 || (gs & 3) || W < 8 || W > 65536 || span < 1 || (P[PB_ENT0] & 7) ||
      (P[PB_SRC0] & 7) || (P[PB_DESC0] & 3) || P[PB_CHUNK_EDGES] < 8 || P[PB_CHUNK_EDGES] > 65536)
    fail(ErrorCode::argument, std::string(what) + ": bad layout geometry");
  // bounds of every array this part touches
  auto need = [&](const BufView& b, uint64_t bytes, const char* name) {
    if (b.first_byte != 0 || b.bytes < bytes) fail(ErrorCode::argument, std::string(what) + ": " + name + " too short");
  };
  need(CH, static_cast<uint64_t>(P[PB_CHUNK0] + P[PB_NCHUNKS]) * 32, "chunks");
  need(GT, static_cast<uint64_t>(P[PB_DESC0]) * 4, "chunk descriptors");
  need(UN, static_cast<uint64_t>(P[PB_UNIT0] + P[PB_NUNITS]) * 16, "units");
  need(SU, static_cast<uint64_t>(P[PB_SLOT0] + P[PB_NSLOTS]) * 4, "slot_units");
  need(SL, static_cast<uint64_t>(P[PB_SRC0]) * 2, "src_local");
  need(SA, static_cast<uint64_t>(P[PB_SLOT0] + P[PB_NSLOTS]) * (W * 8 + 4), "slot accumulators");
  if (VA.bytes / 4 < DS.bytes / 2 || VA.first_byte != 0 || DS.first_byte != 0 || (DS.bytes / 2) < 8)
    fail(ErrorCode::argument, std::string(what) + ": vals must hold one float per dst16 entry");
  const int64_t* dpart = reinterpret_cast<const int64_t*>(PT.ptr) + static_cast<int64_t>(pi) * PB_FIELDS;
  // phase 1
  const int64_t ce = P[PB_CHUNK_EDGES];
  const int64_t nwin_max = (ce + 31) >> 5;
  const int64_t stage_words = ((2 * nwin_max + 3) & ~int64_t(3)) + ((nb + 3) & ~int64_t(3)) +
                              ((ce + 7) & ~int64_t(7)) / 2 + ((span + 6) & ~int64_t(3));
  const int64_t recs_max = (P[PB_NCHUNKS] + c.sm_count - 1) / c.sm_count + 1;  // any grid >= sm_count
  // two CTAs per SM; two stages per CTA when they fit (copies of chunk i+1 in
  // flight while chunk i is written), else one (the other CTA overlaps)
  auto smem_for = [&](int nst) {
    return static_cast<size_t>(nst * stage_words) * 4 + 32 + static_cast<size_t>(recs_max) * 32 + 64;
  };
  int nst = 2 * (smem_for(2) + 1024) <= 228 * 1024 ? 2 : 1;
  if (const char* e = std::getenv("HCL_PB_NST")) nst = std::atoi(e) == 2 && smem_for(2) <= 227 * 1024 ? 2 : 1;
  const size_t smem1 = smem_for(nst);
  HCL_CUDA(cudaFuncSetAttribute(pr_bin_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem1)));
  int per_sm = 1;
  HCL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pr_bin_scatter_kernel, PB_T, smem1));
  const int grid1 = static_cast<int>(std::min<int64_t>(P[PB_NCHUNKS],
                                                       static_cast<int64_t>(std::min(2, std::max(1, per_sm))) * c.sm_count));
  if (grid1 > 0) {
    pr_bin_scatter_kernel<<<grid1, PB_T, smem1, c.stream>>>(
        dpart, reinterpret_cast<const int4*>(CH.ptr), reinterpret_cast<const uint16_t*>(SL.ptr),
        reinterpret_cast<const uint32_t*>(GT.ptr), reinterpret_cast<const float*>(XS.ptr), v,
        reinterpret_cast<float*>(VA.ptr), nst);
    HCL_LAUNCHED();
  }
  // phase 2
  const bool small_bins = W <= 8192;
  const int gt = small_bins ? 512 : 1024;
  const size_t smem2 = static_cast<size_t>(PBG_STAGES) * 8 * gt * 6 + 2 * PBG_STAGES * 8 +
                       (small_bins ? 8192 * 8 : static_cast<size_t>((W + 31) & ~int64_t(31)) * 8);
  auto gkern = small_bins ? pr_bin_gather_kernel<512> : pr_bin_gather_kernel<1024>;
  HCL_CUDA(cudaFuncSetAttribute(gkern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2)));
  const int64_t n_slots_total = static_cast<int64_t>(SA.bytes / (W * 8 + 4));
  unsigned long long* slot_acc = reinterpret_cast<unsigned long long*>(SA.ptr);
  unsigned int* slot_cnt = reinterpret_cast<unsigned int*>(slot_acc + n_slots_total * W);
  const float base = static_cast<float>((1.0 - 0.85) / v), damp = 0.85f, inv_v = static_cast<float>(1.0 / v);
  if (P[PB_NUNITS] > 0) {
    gkern<<<static_cast<unsigned>(P[PB_NUNITS]), gt, smem2, c.stream>>>(
        dpart, reinterpret_cast<const int4*>(UN.ptr), reinterpret_cast<const int*>(SU.ptr),
        reinterpret_cast<const float*>(VA.ptr), reinterpret_cast<const uint16_t*>(DS.ptr), slot_acc, slot_cnt,
        reinterpret_cast<const unsigned long long*>(D.ptr), y, static_cast<int>(lo), base, damp, inv_v,
        reinterpret_cast<const unsigned long long*>(PB.ptr), n_peers, reinterpret_cast<const float*>(OD.ptr),
        reinterpret_cast<float*>(XN.ptr), reinterpret_cast<unsigned long long*>(DN.ptr));
    HCL_LAUNCHED();
  }
  return 2ull * static_cast<uint64_t>(P[PB_NEDGES]);  // the reference's spmv_compute units (kernels.cpp:292)
}

uint64_t rows_pr(const int64_t* s, uint32_t n) { return static_cast<uint64_t>(s[n == 13 ? 8 : 7]); }
uint64_t rows_pr_imp(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[7]); }
uint64_t rows_pr_binned(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[10]); }

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
  r.push_back({"b200", "pagerank_prep", {I, I, O, O, S}, {P, P, P, P, N}, launch_pr_prep<false>, nullptr, nullptr});
  r.push_back({"b200", "pagerank_prep_fixed", {I, I, O, O, S}, {P, P, P, P, N}, launch_pr_prep<true>, nullptr,
               nullptr});
  r.push_back({"b200", "pagerank_step_implicit", {I, I, I, I, I, I, O, S, S, S, S, S},
               {P, P, P, P, P, P, X, N, N, N, N, N}, launch_pr<true, true>, nullptr, rows_pr_imp});
  // the implicit step fused with the next prep and the exchange: x' rows, xs' rows here and on
  // every peer (peers = device addresses of their xs', uint64[n_peers]), dangling partial dsum':
  // row_ptr col units long_rows xs dsum x' | V nnz_off n_units n_long warp_nnz | peers n_peers inv_outdeg xs' dsum'
  // (inv_outdeg = fl(1/outdeg) as fp32, 0 for dangling vertices: datagen.pagerank_inv_outdeg)
  constexpr uint8_t XG = HCL_PART_EXCHANGE, PR = HCL_PART_PEERS, RS = HCL_PART_REDUCE_SUM;
  // binned step (propagation blocking): the layout of hcl_pagerank_bins_build per part + the exchange epilogue
  constexpr uint8_t IO = HCL_ARG_INOUT, LC = HCL_PART_LOCAL;
  r.push_back({"b200", "pagerank_step_binned",
               {I, I, I, I, I, I, I, I, I, O, S, S, I, S, I, O, O, IO, IO},
               {P, P, P, P, P, P, P, P, P, X, N, N, PR, N, P, XG, RS, LC, LC}, launch_pr_binned, nullptr,
               rows_pr_binned});
  r.push_back({"b200", "pagerank_step_exchange", {I, I, I, I, I, I, O, S, S, S, S, S, I, S, I, O, O},
               {P, P, P, P, P, P, X, N, N, N, N, N, PR, N, P, XG, RS}, launch_pr<true, true, true>, nullptr,
               rows_pr_imp});
}

}  // namespace hcl
