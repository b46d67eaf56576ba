// k-means assignment and update (config C4; assignment =
// the reference's knn with k=1, proj/src/kernels.cpp:195-233).
//
// kmeans_assign: dist(x, c_k) = sum_j (c_kj - x_j)^2 in fp32 with every
//   subtract, multiply and add separately rounded and j ascending, argmin with
//   strict < so ties keep the smaller k — bit-identical to the oracle
//   (ho_kmeans_assign). Blackwell's packed FP32x2 instructions (FADD2/FMUL2,
//   IEEE round-to-nearest per lane) evaluate two centroids per instruction:
//   each thread owns one point (coordinates duplicated into register pairs) and
//   streams centroid pairs from shared memory (interleaved [k/2][j][2]).
// kmeans_accumulate: exact per-cluster sums in 2^-12 fixed point (points are
//   multiples of 2^-12), int32 shared-memory tables per block flushed with
//   int64 atomics — integer sums, so the result is independent of order,
//   blocks and partitions; partial sums of a partitioned launch are combined
//   by the runtime (REDUCE_SUM class) or by an NCCL allreduce across ranks.
// kmeans_finalize: c_k = (sum_k * 2^-12) / count_k in fp64, rounded to fp32;
//   empty clusters keep their centroid.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.hpp"
#include "ptx.cuh"
#include "../../include/hcl_cabi.h"

namespace hcl {
namespace {

constexpr int KM_D = 32;         // fast-path dimension
constexpr int KM_KCHUNK = 1024;  // centroids staged per pass (128 KB of smem)
constexpr int KM_T = 512;

__global__ void __launch_bounds__(KM_T, 1) kmeans_assign32_kernel(const float* __restrict__ pts, int64_t n,
                                                                 const float* __restrict__ cent, int k,
                                                                 int32_t* __restrict__ assign) {
  extern __shared__ float4 cs4[];  // [KM_KCHUNK/2][KM_D/2] of (c_k[j], c_k+1[j], c_k[j+1], c_k+1[j+1])
  float* cs = reinterpret_cast<float*>(cs4);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t first = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // all threads of the block walk the same number of points (block-uniform loop)
  const int64_t iters = (n + stride - 1) / stride;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = first + it * stride;
    const bool active = i < n;
    float2 xn[KM_D];  // (-x_j, -x_j)
#pragma unroll
    for (int j = 0; j < KM_D; j += 4) {
      float4 v = active ? __ldcs(reinterpret_cast<const float4*>(pts + i * KM_D + j)) : make_float4(0, 0, 0, 0);
      xn[j] = make_float2(-v.x, -v.x);
      xn[j + 1] = make_float2(-v.y, -v.y);
      xn[j + 2] = make_float2(-v.z, -v.z);
      xn[j + 3] = make_float2(-v.w, -v.w);
    }
    float best = 0.f;
    int bi = 0;
    for (int k0 = 0; k0 < k; k0 += KM_KCHUNK) {
      const int kc = min(KM_KCHUNK, k - k0);
      const int kpairs = (kc + 1) / 2;
      __syncthreads();
      for (int e = threadIdx.x; e < kpairs * KM_D; e += blockDim.x) {
        const int p = e / KM_D, j = e % KM_D;
        const int ka = k0 + 2 * p, kb = ka + 1;
        cs[(p * KM_D + j) * 2] = cent[(int64_t)ka * KM_D + j];
        cs[(p * KM_D + j) * 2 + 1] = kb < k ? cent[(int64_t)kb * KM_D + j] : __int_as_float(0x7f800000);
      }
      __syncthreads();
      for (int p = 0; p < kpairs; ++p) {
        const float4* row = cs4 + p * (KM_D / 2);
        float2 s = make_float2(0.f, 0.f);
        // squares stay scalar FMUL: ptxas contracts mul.rn.f32x2 + add.rn.f32x2
        // into FFMA2 (single rounding) even under -fmad=false, which would
        // break bit-exactness with the oracle's rounded multiply-then-add
#pragma unroll
        for (int j = 0; j < KM_D; j += 2) {
          const float4 c = row[j / 2];
          float2 d0 = __fadd2_rn(make_float2(c.x, c.y), xn[j]);
          s = __fadd2_rn(s, make_float2(__fmul_rn(d0.x, d0.x), __fmul_rn(d0.y, d0.y)));
          float2 d1 = __fadd2_rn(make_float2(c.z, c.w), xn[j + 1]);
          s = __fadd2_rn(s, make_float2(__fmul_rn(d1.x, d1.x), __fmul_rn(d1.y, d1.y)));
        }
        const int ka = k0 + 2 * p;
        if (ka == 0 || s.x < best) { best = s.x; bi = ka; }
        if (ka + 1 < k && s.y < best) { best = s.y; bi = ka + 1; }
      }
    }
    if (active) assign[i] = bi;
  }
}

// Generic D (any <= 256): scalar, same arithmetic order.
__global__ void __launch_bounds__(256) kmeans_assign_generic_kernel(const float* __restrict__ pts, int64_t n, int d,
                                                                   const float* __restrict__ cent, int k,
                                                                   int32_t* __restrict__ assign) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* x = pts + i * d;
  float best = 0.f;
  int bi = 0;
  for (int c = 0; c < k; ++c) {
    const float* m = cent + (int64_t)c * d;
    float s = 0.f;
    for (int j = 0; j < d; ++j) {
      float diff = __fsub_rn(__ldg(m + j), x[j]);
      s = __fadd_rn(s, __fmul_rn(diff, diff));
    }
    if (c == 0 || s < best) { best = s; bi = c; }
  }
  assign[i] = bi;
}

// sums[k*d + j] += x_ij * 4096 (exact integer), counts[k] += 1
__global__ void __launch_bounds__(1024) kmeans_accumulate_kernel(const float* __restrict__ pts,
                                                                const int32_t* __restrict__ assign, int64_t n, int d,
                                                                int k, unsigned long long* __restrict__ sums,
                                                                unsigned long long* __restrict__ counts,
                                                                int use_smem) {
  extern __shared__ int tbl[];  // [k*d] sums + [k] counts, int32 (a block's points cannot overflow)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
  if (use_smem) {
    for (int e = threadIdx.x; e < k * d + k; e += blockDim.x) tbl[e] = 0;
    __syncthreads();
  }
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  if (use_smem && d == 32) {
    // D = 32: lane = dimension; 8 points per warp iteration so the loads of
    // the next points are in flight together (the loop is latency-bound
    // otherwise). A cluster row is flushed to the int64 totals whenever its
    // block-local count reaches 2^15, so |int32 sum| <= (2^15 + 32) * 2^15 < 2^31
    // for any data (points on the 2^-12 grid in [-8, 8)).
    constexpr int U = 8;
    for (int64_t base = lo + static_cast<int64_t>(warp) * U; base < hi; base += static_cast<int64_t>(nwarps) * U) {
      int cs[U], qs[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = base + u;
        cs[u] = i < hi ? __ldg(assign + i) : -1;
        qs[u] = i < hi ? __float2int_rz(__fmul_rn(__ldg(pts + i * 32 + lane), 4096.0f)) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = cs[u];
        if (c < 0) continue;
        atomicAdd(&tbl[c * 32 + lane], qs[u]);
        int old = 0;
        if (lane == 0) old = atomicAdd(&tbl[k * 32 + c], 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old + 1 == (1 << 15)) {
          __syncwarp();
          const int v = atomicExch(&tbl[c * 32 + lane], 0);
          atomicAdd(&sums[static_cast<int64_t>(c) * 32 + lane],
                    static_cast<unsigned long long>(static_cast<long long>(v)));
          if (lane == 0) atomicAdd(&counts[c], static_cast<unsigned long long>(atomicExch(&tbl[k * 32 + c], 0)));
        }
      }
    }
  } else
  for (int64_t i = lo + warp; i < hi; i += nwarps) {
    const int c = assign[i];
    for (int j = lane; j < d; j += 32) {
      int q = __float2int_rz(__fmul_rn(pts[i * d + j], 4096.0f));
      if (use_smem)
        atomicAdd(&tbl[c * d + j], q);
      else
        atomicAdd(&sums[(int64_t)c * d + j], static_cast<unsigned long long>(static_cast<long long>(q)));
    }
    if (lane == 0) {
      if (use_smem)
        atomicAdd(&tbl[k * d + c], 1);
      else
        atomicAdd(&counts[c], 1ull);
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int e = threadIdx.x; e < k * d; e += blockDim.x)
      if (tbl[e]) atomicAdd(&sums[e], static_cast<unsigned long long>(static_cast<long long>(tbl[e])));
    for (int e = threadIdx.x; e < k; e += blockDim.x)
      if (tbl[k * d + e]) atomicAdd(&counts[e], static_cast<unsigned long long>(tbl[k * d + e]));
  }
}

// D = 32, points streamed through shared memory by 1D bulk copies (TMA): one
// elected thread keeps AC_STAGES chunks of AC_CHUNK points (and their
// assignments) in flight per SM, so the HBM stream does not depend on how
// many loads the warps keep outstanding; the warps add each staged point into
// the block's int32 table (lane = dimension, conflict-free, one shared atomic
// per point) and count the chunk's assignments 32 at a time.
// PT = float: the caller's fp32 points (scaled by 2^12 here); PT = int16_t: the
// points' 2^-12 fixed-point copy (kmeans_quantize_points), half the bytes per
// point and twice the points per chunk -- the accumulation streams HBM, so the
// half-size copy halves its time.
constexpr int AC_FLUSH = 64;
// int16 stream: two stages of 672 points (fewer, larger chunks: each refill waits
// for every warp, so the per-chunk hand-off dominates small chunks). 2^27 points,
// K=1024: 384 x 3 2.94 ms, 512 x 2 2.49, 640 x 2 2.33, 672 x 2 2.30 (the largest
// pair that fits beside the K=1024 table)
#ifndef HCL_AC_Q_CHUNK
#define HCL_AC_Q_CHUNK 672
#endif
#ifndef HCL_AC_Q_STAGES
#define HCL_AC_Q_STAGES 2
#endif
template <typename PT>
struct AcCfg {
  static constexpr int kChunk = sizeof(PT) == 4 ? 192 : HCL_AC_Q_CHUNK;
  static constexpr int kStages = sizeof(PT) == 4 ? 3 : HCL_AC_Q_STAGES;
  static constexpr int kStageBytes = kChunk * 32 * static_cast<int>(sizeof(PT)) + kChunk * 4;
  static constexpr int kFlush = ((1 << 15) - 1) / kChunk < AC_FLUSH ? ((1 << 15) - 1) / kChunk : AC_FLUSH;
  static_assert(kFlush * kChunk < (1 << 15), "rows must stay below 2^16 points between flushes");
};
constexpr int AC_CHUNK = AcCfg<float>::kChunk;  // the fp32 path's chunk (host tail split)
__device__ __forceinline__ int ac_fixed(float x) { return __float2int_rz(__fmul_rn(x, 4096.0f)); }
__device__ __forceinline__ int ac_fixed(int16_t x) { return x; }

template <typename PT>
__global__ void __launch_bounds__(1024) kmeans_accumulate32_bulk_kernel(const PT* __restrict__ pts,
                                                                       const int32_t* __restrict__ assign,
                                                                       int64_t n, int k,
                                                                       unsigned long long* __restrict__ sums,
                                                                       unsigned long long* __restrict__ counts) {
  constexpr int AC_CHUNK = AcCfg<PT>::kChunk, AC_STAGE_BYTES = AcCfg<PT>::kStageBytes, AC_STAGES = AcCfg<PT>::kStages;
  constexpr int PB = 32 * static_cast<int>(sizeof(PT));  // bytes per point
  extern __shared__ __align__(128) uint8_t ac_smem[];
  int* tbl = reinterpret_cast<int*>(ac_smem);  // [k*32] sums + [k] counts
  const size_t tbl_bytes = (static_cast<size_t>(k) * 33 * 4 + 127) & ~size_t(127);
  uint8_t* stage0 = ac_smem + tbl_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + AC_STAGES * AC_STAGE_BYTES);
  uint64_t* empty = full + AC_STAGES;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
  for (int e = threadIdx.x; e < k * 33; e += blockDim.x) tbl[e] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < AC_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], nwarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // this block's range, in whole chunks (the host hands the tail to the other kernel)
  const int64_t nchunks = n / AC_CHUNK;
  const int64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
  if (threadIdx.x == 0) {  // producer: prime the ring
    for (int64_t ch = c0; ch < min(c1, c0 + AC_STAGES); ++ch) {
      const int s = static_cast<int>((ch - c0) % AC_STAGES);
      uint8_t* st = stage0 + s * AC_STAGE_BYTES;
      ptx::mbar_arrive_expect_tx(&full[s], AC_STAGE_BYTES);
      ptx::bulk_load(st, pts + ch * AC_CHUNK * 32, AC_CHUNK * PB, &full[s]);
      ptx::bulk_load(st + AC_CHUNK * PB, assign + ch * AC_CHUNK, AC_CHUNK * 4, &full[s]);
    }
  }
  for (int64_t ch = c0; ch < c1; ++ch) {
    const int64_t it = ch - c0;
    const int s = static_cast<int>(it % AC_STAGES);
    const uint32_t ph = static_cast<uint32_t>((it / AC_STAGES) & 1);
    ptx::mbar_wait(&full[s], ph);
    const PT* sp = reinterpret_cast<const PT*>(stage0 + s * AC_STAGE_BYTES);
    const int* sa = reinterpret_cast<const int*>(stage0 + s * AC_STAGE_BYTES + AC_CHUNK * PB);
    for (int w = warp; w < AC_CHUNK / 32; w += nwarps)  // counts: 32 points per atomic
      atomicAdd(&tbl[k * 32 + sa[w * 32 + lane]], 1);
    for (int p = warp; p < AC_CHUNK; p += nwarps) atomicAdd(&tbl[sa[p] * 32 + lane], ac_fixed(sp[p * 32 + lane]));
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && ch + AC_STAGES < c1) {  // refill this stage once every warp is done with it
      ptx::mbar_wait(&empty[s], ph);
      uint8_t* st = stage0 + s * AC_STAGE_BYTES;
      const int64_t nx = ch + AC_STAGES;
      ptx::mbar_arrive_expect_tx(&full[s], AC_STAGE_BYTES);
      ptx::bulk_load(st, pts + nx * AC_CHUNK * 32, AC_CHUNK * PB, &full[s]);
      ptx::bulk_load(st + AC_CHUNK * PB, assign + nx * AC_CHUNK, AC_CHUNK * 4, &full[s]);
    }
    // int32 overflow guard: |q| <= 2^15, so a row is exact while its block-local
    // count stays below 2^16. Rows past 2^15 are flushed every kFlush chunks
    // (at most kFlush * AC_CHUNK < 2^15 more points in between).
    if ((it + 1) % AcCfg<PT>::kFlush == 0) {
      __syncthreads();
      for (int r = threadIdx.x; r < k; r += blockDim.x)
        if (tbl[k * 32 + r] >= (1 << 15)) {
          for (int j = 0; j < 32; ++j) {
            atomicAdd(&sums[static_cast<int64_t>(r) * 32 + j],
                      static_cast<unsigned long long>(static_cast<long long>(tbl[r * 32 + j])));
            tbl[r * 32 + j] = 0;
          }
          atomicAdd(&counts[r], static_cast<unsigned long long>(tbl[k * 32 + r]));
          tbl[k * 32 + r] = 0;
        }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * 32; e += blockDim.x)
    if (tbl[e]) atomicAdd(&sums[e], static_cast<unsigned long long>(static_cast<long long>(tbl[e])));
  for (int e = threadIdx.x; e < k; e += blockDim.x)
    if (tbl[k * 32 + e]) atomicAdd(&counts[e], static_cast<unsigned long long>(tbl[k * 32 + e]));
}

__global__ void kmeans_finalize_kernel(const long long* __restrict__ sums, const long long* __restrict__ counts, int k,
                                       int d, float* __restrict__ cent) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * d) return;
  long long cnt = counts[e / d];
  if (cnt == 0) return;
  cent[e] = static_cast<float>(__ddiv_rn(__dmul_rn(static_cast<double>(sums[e]), 0x1p-12), static_cast<double>(cnt)));
}

__global__ void add_i64_kernel(long long* __restrict__ dst, const long long* __restrict__ src, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] += src[i];
}

// kmeans_assign(points, centroids, assign, N, D, K)
uint64_t launch_assign(LaunchCtx& c) {
  int64_t n = scalar_arg(c, 3, "kmeans_assign N");
  int64_t d = scalar_arg(c, 4, "kmeans_assign D");
  int64_t k = scalar_arg(c, 5, "kmeans_assign K");
  if (n < 0 || d < 1 || d > 256 || k < 1 || k > (1 << 24))
    fail(ErrorCode::argument, "kmeans_assign: need N >= 0, 1 <= D <= 256, 1 <= K");
  const BufView& P = buffer_arg(c, 0, "kmeans_assign points");
  const BufView& C = buffer_arg(c, 1, "kmeans_assign centroids");
  const BufView& A = buffer_arg(c, 2, "kmeans_assign assign");
  if (C.first_byte != 0 || C.bytes != static_cast<uint64_t>(k * d) * 4)
    fail(ErrorCode::argument, "kmeans_assign: centroids size != K*D");
  if (c.whole && P.bytes != static_cast<uint64_t>(n * d) * 4)
    fail(ErrorCode::argument, "kmeans_assign: points size != N*D");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "kmeans_assign");
  const float* pts = at_byte<const float>(P, lo * d * 4, rows * d * 4, "kmeans_assign points");
  int32_t* as = at_byte<int32_t>(A, lo * 4, rows * 4, "kmeans_assign assign");
  if (!rows) return 0;
  const float* cent = reinterpret_cast<const float*>(C.ptr);
  if (d == KM_D && (reinterpret_cast<uintptr_t>(pts) & 15) == 0) {
    const size_t smem = static_cast<size_t>(KM_KCHUNK) * KM_D * 4;
    HCL_CUDA(cudaFuncSetAttribute(kmeans_assign32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    int grid = static_cast<int>(std::min<uint64_t>(c.sm_count, ceil_div(rows, KM_T)));
    kmeans_assign32_kernel<<<grid, KM_T, smem, c.stream>>>(pts, static_cast<int64_t>(rows), cent,
                                                           static_cast<int>(k), as);
  } else {
    kmeans_assign_generic_kernel<<<static_cast<unsigned>(ceil_div(rows, 256)), 256, 0, c.stream>>>(
        pts, static_cast<int64_t>(rows), static_cast<int>(d), cent, static_cast<int>(k), as);
  }
  HCL_LAUNCHED();
  return 3ull * rows * static_cast<uint64_t>(k) * static_cast<uint64_t>(d);  // 3 flop per term
}

// kmeans_accumulate(points, assign, sums(int64 K*D), counts(int64 K), N, D, K)
uint64_t launch_accumulate(LaunchCtx& c) {
  int64_t n = scalar_arg(c, 4, "kmeans_accumulate N");
  int64_t d = scalar_arg(c, 5, "kmeans_accumulate D");
  int64_t k = scalar_arg(c, 6, "kmeans_accumulate K");
  if (n < 0 || d < 1 || d > 256 || k < 1) fail(ErrorCode::argument, "kmeans_accumulate: bad N/D/K");
  const BufView& P = buffer_arg(c, 0, "kmeans_accumulate points");
  const BufView& A = buffer_arg(c, 1, "kmeans_accumulate assign");
  const BufView& S = buffer_arg(c, 2, "kmeans_accumulate sums");
  const BufView& Cn = buffer_arg(c, 3, "kmeans_accumulate counts");
  if (S.first_byte != 0 || S.bytes != static_cast<uint64_t>(k * d) * 8 || Cn.first_byte != 0 ||
      Cn.bytes != static_cast<uint64_t>(k) * 8)
    fail(ErrorCode::argument, "kmeans_accumulate: sums must be K*D int64 and counts K int64");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "kmeans_accumulate");
  const float* pts = at_byte<const float>(P, lo * d * 4, rows * d * 4, "kmeans_accumulate points");
  const int32_t* as = at_byte<const int32_t>(A, lo * 4, rows * 4, "kmeans_accumulate assign");
  HCL_CUDA(cudaMemsetAsync(S.ptr, 0, S.bytes, c.stream));
  HCL_CUDA(cudaMemsetAsync(Cn.ptr, 0, Cn.bytes, c.stream));
  if (!rows) return 0;
  const uint64_t work = rows * static_cast<uint64_t>(d);
  const size_t bulk_smem = ((static_cast<size_t>(k) * 33 * 4 + 127) & ~size_t(127)) +
                           AcCfg<float>::kStages * AcCfg<float>::kStageBytes + 2 * AcCfg<float>::kStages * 8;
  const char* bulk_env = std::getenv("HCL_KM_ACC_BULK");  // 0: the register-pipelined kernel only
  const bool bulk = (bulk_env ? std::atoi(bulk_env) != 0 : true) && d == 32 && bulk_smem <= 227 * 1024 &&
                    rows >= static_cast<uint64_t>(AC_CHUNK) && (reinterpret_cast<uintptr_t>(pts) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(as) & 15) == 0;
  if (bulk) {  // whole chunks streamed by TMA; the < AC_CHUNK-point tail by the kernel below
    HCL_CUDA(cudaFuncSetAttribute(kmeans_accumulate32_bulk_kernel<float>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bulk_smem)));
    const int bgrid = static_cast<int>(std::min<uint64_t>(c.sm_count, rows / AC_CHUNK));
    kmeans_accumulate32_bulk_kernel<float><<<bgrid, 1024, bulk_smem, c.stream>>>(
        pts, as, static_cast<int64_t>(rows), static_cast<int>(k), reinterpret_cast<unsigned long long*>(S.ptr),
        reinterpret_cast<unsigned long long*>(Cn.ptr));
    HCL_LAUNCHED();
    const uint64_t done = rows / AC_CHUNK * AC_CHUNK;
    pts += done * 32;
    as += done;
    rows -= done;
    if (!rows) return work;
  }
  const size_t smem = static_cast<size_t>(k * d + k) * 4;
  const bool use_smem = smem <= 200 * 1024 && rows > static_cast<uint64_t>(k) * 4;
  if (use_smem)
    HCL_CUDA(cudaFuncSetAttribute(kmeans_accumulate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  int grid = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(c.sm_count) * 2, ceil_div(rows, 1024)));
  if (use_smem) grid = static_cast<int>(std::min<uint64_t>(c.sm_count, ceil_div(rows, 4096)));
  grid = std::max(grid, 1);
  kmeans_accumulate_kernel<<<grid, 1024, use_smem ? smem : 0, c.stream>>>(
      pts, as, static_cast<int64_t>(rows), static_cast<int>(d), static_cast<int>(k),
      reinterpret_cast<unsigned long long*>(S.ptr), reinterpret_cast<unsigned long long*>(Cn.ptr), use_smem);
  HCL_LAUNCHED();
  return work;
}

// the < one-chunk tail of the fixed-point accumulation: a warp per point, lane = dimension
__global__ void kmeans_accumulate_q16_tail_kernel(const int16_t* __restrict__ pts, const int32_t* __restrict__ assign,
                                                  int64_t n, unsigned long long* __restrict__ sums,
                                                  unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; p < n; p += gridDim.x * (blockDim.x / 32)) {
    const int a = assign[p];
    atomicAdd(&sums[static_cast<int64_t>(a) * 32 + lane],
              static_cast<unsigned long long>(static_cast<long long>(pts[p * 32 + lane])));
    if (lane == 0) atomicAdd(&counts[a], 1ull);
  }
}

// kmeans_quantize_points(points f32, q16 out, N, D): q = x * 2^12 as int16 -- exact for
// points on kmeans_check_points' grid (multiples of 2^-12 in [-8, 8))
__global__ void quantize_points_kernel(const float4* __restrict__ pts, uint2* __restrict__ q, int64_t n4) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = pts[i];
    const int a = __float2int_rz(__fmul_rn(v.x, 4096.0f)), b = __float2int_rz(__fmul_rn(v.y, 4096.0f));
    const int c = __float2int_rz(__fmul_rn(v.z, 4096.0f)), d = __float2int_rz(__fmul_rn(v.w, 4096.0f));
    q[i] = make_uint2((static_cast<uint32_t>(a) & 0xffffu) | (static_cast<uint32_t>(b) << 16),
                      (static_cast<uint32_t>(c) & 0xffffu) | (static_cast<uint32_t>(d) << 16));
  }
}

uint64_t launch_quantize_points(LaunchCtx& c) {
  const int64_t n = scalar_arg(c, 2, "kmeans_quantize_points N"), d = scalar_arg(c, 3, "kmeans_quantize_points D");
  if (n < 0 || d < 1 || d % 4) fail(ErrorCode::argument, "kmeans_quantize_points: need D a multiple of 4");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "kmeans_quantize_points");
  const float* p = at_byte<const float>(buffer_arg(c, 0, "kmeans_quantize_points points"), lo * d * 4, rows * d * 4,
                                        "kmeans_quantize_points points");
  int16_t* q = at_byte<int16_t>(buffer_arg(c, 1, "kmeans_quantize_points q16"), lo * d * 2, rows * d * 2,
                                "kmeans_quantize_points q16");
  if (!rows) return 0;
  const int64_t n4 = static_cast<int64_t>(rows) * d / 4;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n4, 256), 8LL * c.sm_count));
  quantize_points_kernel<<<grid, 256, 0, c.stream>>>(reinterpret_cast<const float4*>(p), reinterpret_cast<uint2*>(q),
                                                     n4);
  HCL_LAUNCHED();
  return rows * static_cast<uint64_t>(d);
}

// kmeans_accumulate_q16(q16 points, assign, sums, counts, N, D, K): kmeans_accumulate over the
// 2^-12 fixed-point copy (D = 32), the same integer sums
uint64_t launch_accumulate_q16(LaunchCtx& c) {
  const char* what = "kmeans_accumulate_q16";
  int64_t n = scalar_arg(c, 4, what), d = scalar_arg(c, 5, what), k = scalar_arg(c, 6, what);
  if (n < 0 || d != 32 || k < 1) fail(ErrorCode::argument, std::string(what) + ": needs D = 32, N >= 0, K >= 1");
  const BufView& P = buffer_arg(c, 0, what);
  const BufView& A = buffer_arg(c, 1, what);
  const BufView& S = buffer_arg(c, 2, what);
  const BufView& Cn = buffer_arg(c, 3, what);
  if (S.first_byte != 0 || S.bytes != static_cast<uint64_t>(k * d) * 8 || Cn.first_byte != 0 ||
      Cn.bytes != static_cast<uint64_t>(k) * 8)
    fail(ErrorCode::argument, std::string(what) + ": sums must be K*D int64 and counts K int64");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, what);
  const int16_t* pts = at_byte<const int16_t>(P, lo * d * 2, rows * d * 2, what);
  const int32_t* as = at_byte<const int32_t>(A, lo * 4, rows * 4, what);
  HCL_CUDA(cudaMemsetAsync(S.ptr, 0, S.bytes, c.stream));
  HCL_CUDA(cudaMemsetAsync(Cn.ptr, 0, Cn.bytes, c.stream));
  if (!rows) return 0;
  const uint64_t work = rows * static_cast<uint64_t>(d);
  using Q = AcCfg<int16_t>;
  const size_t smem = ((static_cast<size_t>(k) * 33 * 4 + 127) & ~size_t(127)) + Q::kStages * Q::kStageBytes +
                      2 * Q::kStages * 8;
  if (smem > 227 * 1024) fail(ErrorCode::argument, std::string(what) + ": K too large for the shared-memory table");
  if (rows >= static_cast<uint64_t>(Q::kChunk) && (reinterpret_cast<uintptr_t>(pts) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(as) & 15) == 0) {
    HCL_CUDA(cudaFuncSetAttribute(kmeans_accumulate32_bulk_kernel<int16_t>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int bgrid = static_cast<int>(std::min<uint64_t>(c.sm_count, rows / Q::kChunk));
    kmeans_accumulate32_bulk_kernel<int16_t><<<bgrid, 1024, smem, c.stream>>>(
        pts, as, static_cast<int64_t>(rows), static_cast<int>(k), reinterpret_cast<unsigned long long*>(S.ptr),
        reinterpret_cast<unsigned long long*>(Cn.ptr));
    HCL_LAUNCHED();
    const uint64_t done = rows / Q::kChunk * Q::kChunk;
    pts += done * 32;
    as += done;
    rows -= done;
  }
  if (rows) {
    kmeans_accumulate_q16_tail_kernel<<<static_cast<unsigned>(ceil_div(rows, 8)), 256, 0, c.stream>>>(
        pts, as, static_cast<int64_t>(rows), reinterpret_cast<unsigned long long*>(S.ptr),
        reinterpret_cast<unsigned long long*>(Cn.ptr));
    HCL_LAUNCHED();
  }
  return work;
}

// kmeans_finalize(sums, counts, centroids(inout), K, D)
uint64_t launch_finalize(LaunchCtx& c) {
  int64_t k = scalar_arg(c, 3, "kmeans_finalize K");
  int64_t d = scalar_arg(c, 4, "kmeans_finalize D");
  const BufView& S = buffer_arg(c, 0, "kmeans_finalize sums");
  const BufView& Cn = buffer_arg(c, 1, "kmeans_finalize counts");
  const BufView& Ce = buffer_arg(c, 2, "kmeans_finalize centroids");
  if (S.bytes != static_cast<uint64_t>(k * d) * 8 || Cn.bytes != static_cast<uint64_t>(k) * 8 ||
      Ce.bytes != static_cast<uint64_t>(k * d) * 4)
    fail(ErrorCode::argument, "kmeans_finalize: sizes do not match K and D");
  kmeans_finalize_kernel<<<static_cast<unsigned>(ceil_div(k * d, 256)), 256, 0, c.stream>>>(
      reinterpret_cast<const long long*>(S.ptr), reinterpret_cast<const long long*>(Cn.ptr), static_cast<int>(k),
      static_cast<int>(d), reinterpret_cast<float*>(Ce.ptr));
  HCL_LAUNCHED();
  return static_cast<uint64_t>(k * d);
}

// reduce_add_i64(dst(inout), src, n): dst += src — the runtime's REDUCE_SUM combine step
uint64_t launch_add_i64(LaunchCtx& c) {
  int64_t n = scalar_arg(c, 2, "reduce_add_i64 n");
  const BufView& D = buffer_arg(c, 0, "reduce_add_i64 dst");
  const BufView& S = buffer_arg(c, 1, "reduce_add_i64 src");
  if (D.bytes < static_cast<uint64_t>(n) * 8 || S.bytes < static_cast<uint64_t>(n) * 8)
    fail(ErrorCode::argument, "reduce_add_i64: buffers shorter than n");
  if (!n) return 0;
  int grid = static_cast<int>(std::min<uint64_t>(ceil_div(n, 256), c.sm_count * 4));
  add_i64_kernel<<<grid, 256, 0, c.stream>>>(reinterpret_cast<long long*>(D.ptr),
                                             reinterpret_cast<const long long*>(S.ptr), n);
  HCL_LAUNCHED();
  return static_cast<uint64_t>(n);
}

// Device-side synthetic points, bit-identical to hcl_gen_kmeans_points (host)
// and oracle ho_kmeans_points: counter-based SplitMix64, so a partitioned
// launch generates each rank's rows in place.
__device__ __forceinline__ uint64_t sm_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void gen_points_kernel(float* __restrict__ out, uint64_t first, uint64_t count, int d, uint64_t blobs,
                                  uint64_t seed) {
  const uint64_t total = count * d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = first + e / d, j = e % d;
    const uint64_t b = sm_at(seed ^ 0xB10BULL, i) % blobs;
    const int64_t c = static_cast<int64_t>(sm_at(seed ^ 0xCE47E2ULL, b * d + j) >> 49) - 16384;
    const uint64_t r = sm_at(seed, i * d + j);
    const int64_t nsum = static_cast<int64_t>(r & 0xffff) + static_cast<int64_t>((r >> 16) & 0xffff) +
                         static_cast<int64_t>((r >> 32) & 0xffff) + static_cast<int64_t>(r >> 48) - 131070;
    int64_t q = c + (nsum >> 5);
    q = q < -32768 ? -32768 : (q > 32767 ? 32767 : q);
    out[e] = static_cast<float>(q) * 0x1p-12f;
  }
}

// gen_kmeans_points(points(out), N, D, blobs, seed)
uint64_t launch_gen_points(LaunchCtx& c) {
  int64_t n = scalar_arg(c, 1, "gen_kmeans_points N"), d = scalar_arg(c, 2, "gen_kmeans_points D");
  int64_t blobs = scalar_arg(c, 3, "gen_kmeans_points blobs"), seed = scalar_arg(c, 4, "gen_kmeans_points seed");
  if (n < 0 || d < 1 || blobs < 1) fail(ErrorCode::argument, "gen_kmeans_points: bad N/D/blobs");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "gen_kmeans_points");
  float* out = at_byte<float>(buffer_arg(c, 0, "gen_kmeans_points out"), lo * d * 4, rows * d * 4, "gen points");
  if (!rows) return 0;
  gen_points_kernel<<<c.sm_count * 16, 256, 0, c.stream>>>(out, lo, rows, static_cast<int>(d),
                                                           static_cast<uint64_t>(blobs), static_cast<uint64_t>(seed));
  HCL_LAUNCHED();
  return rows * static_cast<uint64_t>(d);
}

__global__ void check_perm_kernel(const int32_t* __restrict__ perm, int64_t lo, int64_t rows, int* __restrict__ bad) {
  int mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    mine |= perm[i] < lo || perm[i] >= lo + rows;
  if (__syncthreads_or(mine) && threadIdx.x == 0) atomicOr(bad, 1);
}

// kmeans_accumulate's exact int32/int64 tables assume every coordinate is a
// multiple of 2^-12 inside [-8, 8) (|x * 4096| <= 2^15). This check flags
// any other value (NaN and inf included) before the data is used.
__global__ void check_points_kernel(const float* __restrict__ pts, uint64_t count, int* __restrict__ bad) {
  int mine = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count; e += (uint64_t)gridDim.x * blockDim.x) {
    const float x = pts[e];
    const float q = __fmul_rn(x, 4096.0f);
    mine |= !(x >= -8.0f && x < 8.0f) || q != truncf(q);
  }
  if (__syncthreads_or(mine) && threadIdx.x == 0) atomicOr(bad, 1);
}

// kmeans_check_points(points, N, D): argument error unless every coordinate of
// the launch's rows is on the 2^-12 grid inside [-8, 8) (KMeans.load_points)
uint64_t launch_check_points(LaunchCtx& c) {
  int64_t n = scalar_arg(c, 1, "kmeans_check_points N"), d = scalar_arg(c, 2, "kmeans_check_points D");
  if (n < 0 || d < 1) fail(ErrorCode::argument, "kmeans_check_points: bad N/D");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "kmeans_check_points");
  const float* pts = at_byte<const float>(buffer_arg(c, 0, "kmeans_check_points points"), lo * d * 4, rows * d * 4,
                                          "kmeans_check_points");
  if (!rows) return 0;
  int* bad = static_cast<int*>(c.scratch(c.dev, sizeof(int)));
  HCL_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
  check_points_kernel<<<c.sm_count * 8, 256, 0, c.stream>>>(pts, rows * static_cast<uint64_t>(d), bad);
  HCL_LAUNCHED();
  int h = 0;
  HCL_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  if (h)
    fail(ErrorCode::argument,
         "k-means points must be multiples of 2^-12 inside [-8, 8): the exact fixed-point centroid sums need it");
  return rows * static_cast<uint64_t>(d);
}

// dst row i = src row perm[i] (perm: absolute rows inside the launch's range)
__global__ void gather_rows_kernel(const float4* __restrict__ src, const int32_t* __restrict__ perm,
                                   float4* __restrict__ dst, int64_t lo, int64_t rows, int v4) {
  const int64_t total = rows * v4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / v4;
    const int64_t from = static_cast<int64_t>(__ldg(perm + i)) - lo;
    dst[e] = __ldg(src + from * v4 + (e - i * v4));
  }
}

// kmeans_gather_points(points, perm, out, N, D): out[i] = points[perm[i]] for the
// launch's rows; perm must stay inside them (argument error otherwise)
uint64_t launch_gather_points(LaunchCtx& c) {
  int64_t n = scalar_arg(c, 3, "kmeans_gather_points N"), d = scalar_arg(c, 4, "kmeans_gather_points D");
  if (n < 0 || d < 1 || d % 4) fail(ErrorCode::argument, "kmeans_gather_points: bad N or D (a multiple of 4)");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "kmeans_gather_points");
  const float* src = at_byte<const float>(buffer_arg(c, 0, "gather src"), lo * d * 4, rows * d * 4, "gather src");
  const int32_t* perm = at_byte<const int32_t>(buffer_arg(c, 1, "gather perm"), lo * 4, rows * 4, "gather perm");
  float* dst = at_byte<float>(buffer_arg(c, 2, "gather dst"), lo * d * 4, rows * d * 4, "gather dst");
  if (!rows) return 0;
  // the permutation must stay inside [lo, lo + rows): check on the device
  int* bad = static_cast<int*>(c.scratch(c.dev, 8));
  HCL_CUDA(cudaMemsetAsync(bad, 0, 8, c.stream));
  check_perm_kernel<<<c.sm_count * 4, 256, 0, c.stream>>>(perm, static_cast<int64_t>(lo), static_cast<int64_t>(rows), bad);
  HCL_LAUNCHED();
  int h = 0;
  HCL_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, c.stream));
  HCL_CUDA(cudaStreamSynchronize(c.stream));
  if (h) fail(ErrorCode::argument, "kmeans_gather_points: perm leaves the launch's rows");
  gather_rows_kernel<<<c.sm_count * 8, 256, 0, c.stream>>>(reinterpret_cast<const float4*>(src), perm,
                                                          reinterpret_cast<float4*>(dst), static_cast<int64_t>(lo),
                                                          static_cast<int64_t>(rows), static_cast<int>(d / 4));
  HCL_LAUNCHED();
  return rows * static_cast<uint64_t>(d);
}

uint64_t rows_km(const int64_t* s, uint32_t n) { return static_cast<uint64_t>(s[n == 6 ? 3 : 4]); }
uint64_t rows_gen(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[1]); }
uint64_t rows_gather(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[3]); }
uint64_t rows_quant(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[2]); }

}  // namespace

void register_kmeans(std::vector<KernelDef>& r) {
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT, IO = HCL_ARG_INOUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS, R = HCL_PART_REDUCE_SUM;
  r.push_back({"b200", "kmeans_assign", {I, I, O, S, S, S}, {X, P, X, N, N, N}, launch_assign, nullptr, rows_km});
  r.push_back({"b200", "kmeans_accumulate", {I, I, O, O, S, S, S}, {X, X, R, R, N, N, N}, launch_accumulate, nullptr,
               rows_km});
  r.push_back({"b200", "kmeans_accumulate_q16", {I, I, O, O, S, S, S}, {X, X, R, R, N, N, N}, launch_accumulate_q16,
               nullptr, rows_km});
  r.push_back({"b200", "kmeans_quantize_points", {I, O, S, S}, {X, X, N, N}, launch_quantize_points, nullptr,
               rows_quant});
  r.push_back({"b200", "kmeans_finalize", {I, I, IO, S, S}, {P, P, P, N, N}, launch_finalize, nullptr, nullptr});
  r.push_back({"b200", "reduce_add_i64", {IO, I, S}, {P, P, N}, launch_add_i64, nullptr, nullptr});
  r.push_back({"b200", "kmeans_check_points", {I, S, S}, {X, N, N}, launch_check_points, nullptr, rows_gen});
  r.push_back({"b200", "kmeans_gather_points", {I, I, O, S, S}, {X, X, X, N, N}, launch_gather_points, nullptr,
               rows_gather});
  r.push_back({"b200", "gen_kmeans_points", {O, S, S, S, S}, {X, N, N, N, N}, launch_gen_points, nullptr, rows_gen});
}

}  // namespace hcl
