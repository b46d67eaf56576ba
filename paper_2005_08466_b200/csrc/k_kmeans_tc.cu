// Tensor-core filtered k-means assignment (config C4; SURVEY.md §8(d) C4 "with
// tensor filtering"). Same result as kmeans_assign -- the exact fp32 argmin of
// sum_j (c_kj - x_j)^2 (every operation separately rounded, j ascending, ties
// to the smaller k; the reference's knn k=1, proj/src/kernels.cpp:195-233) --
// but the 2*N*K*D distance work runs on the 5th-generation tensor cores:
//
//   1. score: s~_k = x . c_k by tcgen05 bf16 MMAs with fp32 accumulation, on
//      split operands x = xh + xl (exact for points on a 2^-12 grid, else
//      |x - xh - xl| <= 2^-16 |x|) and c = ch + cl (+ |residual| <= 2^-16 |c|):
//      xh.ch + xl.ch + xh.cl + xl.cl as 8 MMAs of K=16 over the A row [xh|xl]
//      and the B rows [ch|ch], [cl|cl]. t_k = |c_k|^2 - 2 s~_k ranks the
//      centroids like |x - c_k|^2 (|x|^2 is common to the row).
//   2. filter (epilogue, per point): every k with t_k <= min_j t_j + 2 eps is a
//      candidate, eps = 2^-10 (|x| max|c| + |x|^2 + max|c|^2) -- at least 8x
//      the bound on |t_k + |x|^2 - d_k| from the split, the tensor-core
//      accumulation (<= 2^-13 |x||c|) and the fp32 evaluation of the exact
//      distance d_k (<= 2^-19 (|x|^2 + |c|^2 + 2|x||c|)). The exact argmin is
//      always a candidate, and so is every k tied with it.
//   3. verify: the candidates' exact fp32 distances (the oracle's operation
//      order) pick the result; a point whose candidate list overflows is
//      scanned exactly over all K.
// On the C4 data (2^28 points, K=1024, 1024 Gaussian blobs) the filter keeps
// 1.26 candidates per point on average (max 5; scripts in profiles/).
//
// Layout: points are stored twice -- fp32 (the exact pass and the update) and
// split bf16 [xh(32) | xl(32)] (128 B per point = one SWIZZLE_128B row) with
// |x|^2 per point, made once by kmeans_split_points. Per launch the centroids
// are split into B1 = [ch|ch], B2 = [cl|cl] (bf16, K x 64) with |c|^2. One
// persistent CTA pair (cta_group::2) per 2 SMs: the pair's B halves for all K
// are resident (K/2 x 256 B per CTA, <= 128 KB), A tiles of 2 x 128 points
// stream through 2 stages, and each tile runs K/256 chunks of N=256 MMAs into
// two TMEM accumulators. Scan warps 0-3 take columns 0-127 of every chunk,
// warps 4-7 columns 128-255, and hand each tile's candidate lists
// (double-buffered in shared memory, mbarrier handshakes) to verify warps 8-11,
// which filter, check exactly and store while the scan runs on.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.hpp"
#include "ptx.cuh"
#include "../../include/hcl_cabi.h"

namespace hcl {

CUtensorMap make_tmap_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                              uint32_t box_outer);

namespace {

constexpr int KT_D = 32;
constexpr int KT_SCAN = 8;                   // scan warps 0-7 (TMEM scores -> candidate lists)
constexpr int KT_VER = 4;                    // verify warps 8-11 (exact fp32 check, store)
constexpr int KT_PROD = KT_SCAN + KT_VER;    // TMA producer warp 12, MMA warp 13
constexpr int KT_MMA = KT_PROD + 1;
constexpr int KT_THREADS = (KT_MMA + 1) * 32;
constexpr int KT_ROWS = 128;                 // points per CTA per tile
constexpr int KT_A = KT_ROWS * 128;          // 16 KB A tile per CTA
constexpr int KT_STAGES = 2;
constexpr int KT_BH = 128 * 128;             // per CTA, chunk and split part: 128 centroids x 128 B
constexpr int KT_LIST = 8;                   // candidate slots per point and scan group
constexpr int KT_KMAX = 1024;
constexpr int KT_LBUF = 2 * KT_ROWS * KT_LIST;  // float2 slots of one tile's lists (both groups)

struct KtLayout {
  size_t b, a, q, lists, xch, vq, bars, total;
  __host__ __device__ KtLayout(int K) {
    const int nch = K / 256;
    b = 0;
    a = b + static_cast<size_t>(nch) * 2 * KT_BH;
    q = a + static_cast<size_t>(KT_STAGES) * KT_A;
    lists = q + static_cast<size_t>(K) * 4;
    xch = lists + 2ull * KT_LBUF * 8;             // 2 buffers x (bmin, k) float2 slots
    vq = xch + 2ull * 2 * KT_ROWS * 16;           // 2 buffers x 2 groups x (min, count, overflow)
    bars = vq + static_cast<size_t>(KT_VER) * 32 * 2 * KT_LIST * 8;  // verify queues
    total = bars + 16 * 8 + 16 + 1024;            // barriers, TMEM slot, alignment slack
  }
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// exact fp32 distance in the oracle's order (ho_kmeans_assign)
__device__ __forceinline__ float exact_dist(const float (&x)[KT_D], const float* __restrict__ c) {
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < KT_D; j += 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(c + j));
    float d0 = __fsub_rn(v.x, x[j]), d1 = __fsub_rn(v.y, x[j + 1]);
    float d2 = __fsub_rn(v.z, x[j + 2]), d3 = __fsub_rn(v.w, x[j + 3]);
    s = __fadd_rn(s, __fmul_rn(d0, d0));
    s = __fadd_rn(s, __fmul_rn(d1, d1));
    s = __fadd_rn(s, __fmul_rn(d2, d2));
    s = __fadd_rn(s, __fmul_rn(d3, d3));
  }
  return s;
}

__global__ void __launch_bounds__(KT_THREADS, 1)
    kmeans_assign_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB1,
                            const __grid_constant__ CUtensorMap tmB2, const float* __restrict__ qg,
                            const float* __restrict__ stats, const float* __restrict__ cent,
                            const float* __restrict__ pts, const float* __restrict__ xxg,
                            int32_t* __restrict__ assign, int rows, int K, int* __restrict__ n_overflow,
                            int dbg) {
  // dbg (HCL_KM_DBG, diagnostics only; wrong results): bit 0 skips the exact
  // verification, bit 1 the candidate masks, bit 2 the whole verify stage
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const KtLayout L(K);
  uint8_t* sb = smem + L.b;
  uint8_t* sa = smem + L.a;
  float* sq = reinterpret_cast<float*>(smem + L.q);
  float2* lists = reinterpret_cast<float2*>(smem + L.lists);
  float4* xch = reinterpret_cast<float4*>(smem + L.xch);
  int2* vq = reinterpret_cast<int2*>(smem + L.vq);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + KT_STAGES;
  uint64_t* tfull = empty + KT_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* lfull = tempty + 2;   // [2] scan -> verify: a tile's candidate lists are complete
  uint64_t* lempty = lfull + 2;   // [2] verify -> scan: list buffer free again
  uint64_t* bfull = lempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const int nch = K / 256;

  if (warp == KT_PROD && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB1);
    ptx::prefetch_tmap(&tmB2);
    for (int s = 0; s < KT_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * KT_SCAN);  // every scan warp, both CTAs
      ptx::mbar_init(&lfull[a], KT_SCAN);
      ptx::mbar_init(&lempty[a], KT_VER);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == KT_MMA) ptx::tmem_alloc<2>(tmem_slot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int tiles = (rows + 2 * KT_ROWS - 1) / (2 * KT_ROWS);

  if (warp == KT_PROD) {
    if (lane == 0) {
      // resident B: this CTA's 128-centroid half of every 256-centroid chunk
      if (rank == 0) ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(nch) * 2 * KT_BH * 2);
      const uint32_t bb = ptx::mapa(ptx::smem_u32(bfull), 0);
      for (int c = 0; c < nch; ++c) {
        const int row = c * 256 + static_cast<int>(rank) * 128;
        ptx::tma_load_2d_pair(sb + (2 * c) * KT_BH, &tmB1, bb, 0, row);
        ptx::tma_load_2d_pair(sb + (2 * c + 1) * KT_BH, &tmB2, bb, 0, row);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < tiles; t += nclusters) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], KT_A * 2);
        const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
        ptx::tma_load_2d_pair(sa + stage * KT_A, &tmA, bar, 0, t * 2 * KT_ROWS + static_cast<int>(rank) * KT_ROWS);
        if (++stage == KT_STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == KT_MMA) {
    if (rank == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc(1, 0, 0, 2 * KT_ROWS, 256);
      ptx::mbar_wait(bfull, 0);
      const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(sa), 16, 1024);
      const uint64_t bdesc0 = ptx::umma_desc_sw128(ptx::smem_u32(sb), 16, 1024);
      int stage = 0;
      uint32_t phase = 0, ph0 = 0, ph1 = 0;
      for (int t = cluster; t < tiles; t += nclusters) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t adesc = adesc0 + static_cast<uint64_t>((stage * KT_A) >> 4);
        for (int c = 0; c < nch; ++c) {
          const int acc = c & 1;
          if (acc == 0) {
            ptx::mbar_wait(&tempty[0], ph0 ^ 1);
            ph0 ^= 1;
          } else {
            ptx::mbar_wait(&tempty[1], ph1 ^ 1);
            ph1 ^= 1;
          }
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
          const uint64_t b1 = bdesc0 + static_cast<uint64_t>(((2 * c) * KT_BH) >> 4);
          const uint64_t b2 = bdesc0 + static_cast<uint64_t>(((2 * c + 1) * KT_BH) >> 4);
#pragma unroll
          for (int i = 0; i < 4; ++i) ptx::mma_elect<2, false>(d_tmem, adesc + 2 * i, b1 + 2 * i, idesc, i != 0);
#pragma unroll
          for (int i = 0; i < 4; ++i) ptx::mma_elect<2, false>(d_tmem, adesc + 2 * i, b2 + 2 * i, idesc, 1);
          ptx::mma_commit_elect<2>(&tfull[acc]);
        }
        ptx::mma_commit_elect<2>(&empty[stage]);
        if (++stage == KT_STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp < KT_SCAN) {
    // ---------------- scan: group g = column half g of every chunk ----------------
    const int g = warp / 4, quad = warp % 4;
    const int pl = quad * 32 + lane;  // point within the CTA tile = TMEM lane
    for (int i = threadIdx.x; i < K; i += KT_SCAN * 32) sq[i] = qg[i];
    const float qmax = stats[0];
    const float cmax = sqrtf(qmax);
    epi_bar();
    uint32_t ph0 = 0, ph1 = 0;
    int it = 0;
    for (int t = cluster; t < tiles; t += nclusters, ++it) {
      const int buf = it & 1;
      const int row = t * 2 * KT_ROWS + static_cast<int>(rank) * KT_ROWS + pl;
      const bool valid = row < rows;
      const float xx = valid ? __ldg(xxg + row) : 0.f;
      const float two_eps = 0x1p-9f * (sqrtf(xx) * cmax + xx + qmax);
      float m = __int_as_float(0x7f800000);
      int cnt = 0, ovf = 0;
      ptx::mbar_wait(&lempty[buf], ((it >> 1) & 1) ^ 1);  // the verify warps are done with this buffer
      float2* my = lists + buf * KT_LBUF + (g * KT_ROWS + pl) * KT_LIST;
      for (int c = 0; c < nch; ++c) {
        const int acc = c & 1;
        if (acc == 0) {
          ptx::mbar_wait(&tfull[0], ph0);
          ph0 ^= 1;
        } else {
          ptx::mbar_wait(&tfull[1], ph1);
          ph1 ^= 1;
        }
        ptx::tc_fence_after();
        const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                               static_cast<uint32_t>(acc * 256 + g * 128);
        uint32_t r[2][32];
        ptx::tmem_ld_32x32b_x32(tbase, r[0]);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          uint32_t (&cur)[32] = r[b & 1];
          if (b < 3) {
            ptx::tmem_ld_32x32b_x32(tbase + (b + 1) * 32, r[(b + 1) & 1]);  // next batch in flight
          } else {  // our half of the accumulator drained: hand it back to the MMA warp
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
          }
          const int k0 = c * 256 + g * 128 + b * 32;
          const float4* q4 = reinterpret_cast<const float4*>(sq + k0);
          float g4[8];  // independent group minima: a shallow dependency tree, not a 32-long chain
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 qv = q4[j / 4];
            const float t0 = fmaf(-2.f, __uint_as_float(cur[j]), qv.x);
            const float t1 = fmaf(-2.f, __uint_as_float(cur[j + 1]), qv.y);
            const float t2 = fmaf(-2.f, __uint_as_float(cur[j + 2]), qv.z);
            const float t3 = fmaf(-2.f, __uint_as_float(cur[j + 3]), qv.w);
            cur[j] = __float_as_uint(t0);
            cur[j + 1] = __float_as_uint(t1);
            cur[j + 2] = __float_as_uint(t2);
            cur[j + 3] = __float_as_uint(t3);
            g4[j / 4] = fminf(fminf(t0, t1), fminf(t2, t3));
          }
          const float bmin = fminf(fminf(fminf(g4[0], g4[1]), fminf(g4[2], g4[3])),
                                   fminf(fminf(g4[4], g4[5]), fminf(g4[6], g4[7])));
          m = fminf(m, bmin);
          const float thr = m + two_eps;
          // branch-free candidate mask (four independent partial masks); the
          // (rare) appends loop over its bits. Entries carry their batch
          // minimum, a lower bound of their t (no dynamic register indexing):
          // an entry whose batch minimum exceeds the final threshold is
          // certainly stale; the rest are verified exactly.
          uint32_t mask = 0;
          if (!(dbg & 2)) {
            uint32_t pm[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 32; ++j) pm[j & 3] |= (__uint_as_float(cur[j]) <= thr ? 1u : 0u) << j;
            mask = (pm[0] | pm[1]) | (pm[2] | pm[3]);
            if (dbg & 8) {  // diagnostics: build the mask but skip the appends
              ovf |= mask == 0x5a5a5a5au;
              mask = 0;
            }
          }
          while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            if (cnt == KT_LIST) {  // drop entries the running minimum has excluded
              int w = 0;
              for (int e = 0; e < KT_LIST; ++e)
                if (my[e].x <= thr) my[w++] = my[e];
              cnt = w;
            }
            if (cnt < KT_LIST)
              my[cnt++] = make_float2(bmin, __int_as_float(k0 + j));
            else
              ovf = 1;
          }
          if (b < 3) ptx::tmem_ld_wait();
        }
      }
      xch[(buf * 2 + g) * KT_ROWS + pl] = make_float4(m, __int_as_float(cnt), __int_as_float(ovf), two_eps);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&lfull[buf]);
    }
  } else if (warp < KT_SCAN + KT_VER) {
    // ---------------- verify: final filter, exact check of multi-candidate points, store ----------------
    const int vw = warp - KT_SCAN;
    const int pl = vw * 32 + lane;
    int2* wq = vq + vw * (32 * 2 * KT_LIST);
    int it = 0;
    for (int t = cluster; t < tiles; t += nclusters, ++it) {
      const int buf = it & 1;
      const int row = t * 2 * KT_ROWS + static_cast<int>(rank) * KT_ROWS + pl;
      const bool valid = row < rows;
      ptx::mbar_wait(&lfull[buf], (it >> 1) & 1);
      if (dbg & 4) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&lempty[buf]);
        continue;
      }
      const float4 o0 = xch[(buf * 2 + 0) * KT_ROWS + pl];
      const float4 o1 = xch[(buf * 2 + 1) * KT_ROWS + pl];
      const float thr = fminf(o0.x, o1.x) + o0.w;
      const int cnt0 = __float_as_int(o0.y), cnt1 = __float_as_int(o1.y);
      const int ovf = __float_as_int(o0.z) | __float_as_int(o1.z);
      const float2* l0 = lists + buf * KT_LBUF + pl * KT_LIST;
      const float2* l1 = lists + buf * KT_LBUF + (KT_ROWS + pl) * KT_LIST;
      // a single survivor is the exact argmin as it stands; points with several
      // survivors queue their (point, centroid) pairs for the whole warp
      int nc = 0, k1 = 0;
      if (valid && !ovf)
        for (int e = 0; e < cnt0 + cnt1; ++e) {
          const float2 en = e < cnt0 ? l0[e] : l1[e - cnt0];
          if (en.x <= thr) {
            ++nc;
            k1 = __float_as_int(en.y);
          }
        }
      const int nq = (nc >= 2 && !(dbg & 1)) ? nc : 0;
      int off = nq;  // inclusive warp scan of the queue counts
#pragma unroll
      for (int sft = 1; sft < 32; sft <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, off, sft);
        if (lane >= sft) off += v;
      }
      const int total = __shfl_sync(0xffffffffu, off, 31);
      off -= nq;
      if (nq) {
        int w = off;
        for (int e = 0; e < cnt0 + cnt1; ++e) {
          const float2 en = e < cnt0 ? l0[e] : l1[e - cnt0];
          if (en.x <= thr) wq[w++] = make_int2(__float_as_int(en.y) | (lane << 16), 0);
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&lempty[buf]);  // lists consumed (the queue is private)
      const int row0 = row - lane;
      for (int i = lane; i < total; i += 32) {
        const int2 e = wq[i];
        const int p = e.x >> 16, k = e.x & 0xffff;
        float x[KT_D];
#pragma unroll
        for (int j = 0; j < KT_D; j += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(pts + static_cast<int64_t>(row0 + p) * KT_D + j));
          x[j] = v.x;
          x[j + 1] = v.y;
          x[j + 2] = v.z;
          x[j + 3] = v.w;
        }
        wq[i].y = __float_as_int(exact_dist(x, cent + static_cast<int64_t>(k) * KT_D));
      }
      __syncwarp();
      if (valid) {
        int bk = k1;
        if (ovf) {  // candidate list overflowed: exact scan over all K (rare)
          atomicAdd(n_overflow, 1);
          float x[KT_D];
#pragma unroll
          for (int j = 0; j < KT_D; j += 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(pts + static_cast<int64_t>(row) * KT_D + j));
            x[j] = v.x;
            x[j + 1] = v.y;
            x[j + 2] = v.z;
            x[j + 3] = v.w;
          }
          float best = __int_as_float(0x7f800000);
          for (int k = 0; k < K; ++k) {
            const float e = exact_dist(x, cent + static_cast<int64_t>(k) * KT_D);
            if (e < best) { best = e; bk = k; }
          }
        } else if (nq) {
          float best = __int_as_float(0x7f800000);
          bk = 0x7fffffff;
          for (int i = off; i < off + nq; ++i) {
            const int2 e = wq[i];
            const float d = __int_as_float(e.y);
            const int k = e.x & 0xffff;
            if (d < best || (d == best && k < bk)) { best = d; bk = k; }
          }
        }
        assign[row] = bk;
      }
      __syncwarp();
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == KT_MMA) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2>(tmem_base, 512);
  }
}

// points (N x 32 fp32) -> split rows [xh | xl] (N x 64 bf16) and |x|^2
__global__ void kmeans_split_points_kernel(const float4* __restrict__ pts, uint4* __restrict__ split,
                                           float* __restrict__ xx, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t hi[16], lo[16];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 v = pts[i * 8 + j];
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; u += 2) {
      const __nv_bfloat16 h0 = __float2bfloat16_rn(e[u]), h1 = __float2bfloat16_rn(e[u + 1]);
      const __nv_bfloat16 l0 = __float2bfloat16_rn(e[u] - __bfloat162float(h0));
      const __nv_bfloat16 l1 = __float2bfloat16_rn(e[u + 1] - __bfloat162float(h1));
      hi[(j * 4 + u) / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(h0)) |
                            (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16);
      lo[(j * 4 + u) / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(l0)) |
                            (static_cast<uint32_t>(__bfloat16_as_ushort(l1)) << 16);
    }
    s = fmaf(v.x, v.x, s);
    s = fmaf(v.y, v.y, s);
    s = fmaf(v.z, v.z, s);
    s = fmaf(v.w, v.w, s);
  }
  uint4* o = split + i * 8;
#pragma unroll
  for (int j = 0; j < 4; ++j) o[j] = make_uint4(hi[4 * j], hi[4 * j + 1], hi[4 * j + 2], hi[4 * j + 3]);
#pragma unroll
  for (int j = 0; j < 4; ++j) o[4 + j] = make_uint4(lo[4 * j], lo[4 * j + 1], lo[4 * j + 2], lo[4 * j + 3]);
  xx[i] = s;
}

// centroids (K x 32) -> B1 = [ch|ch], B2 = [cl|cl] (K x 64 bf16), q = |c|^2, stats[0] = max q
__global__ void kmeans_split_centroids_kernel(const float* __restrict__ cent, uint16_t* __restrict__ b1,
                                              uint16_t* __restrict__ b2, float* __restrict__ q,
                                              unsigned* __restrict__ stats, int K) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float s = 0.f;
  for (int j = 0; j < KT_D; ++j) {
    const float v = cent[static_cast<int64_t>(k) * KT_D + j];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
    b1[k * 64 + j] = b1[k * 64 + 32 + j] = __bfloat16_as_ushort(h);
    b2[k * 64 + j] = b2[k * 64 + 32 + j] = __bfloat16_as_ushort(l);
    s = fmaf(v, v, s);
  }
  q[k] = s;
  atomicMax(stats, __float_as_uint(s * (1.f + 0x1p-20f)));  // non-negative: bit order = value order
}

// kmeans_assign_tc(points, split, xx, centroids, assign, N, D, K)
uint64_t launch_assign_tc(LaunchCtx& c) {
  const int64_t n = scalar_arg(c, 5, "kmeans_assign_tc N");
  const int64_t d = scalar_arg(c, 6, "kmeans_assign_tc D");
  const int64_t k = scalar_arg(c, 7, "kmeans_assign_tc K");
  if (d != KT_D) fail(ErrorCode::argument, "kmeans_assign_tc: D must be 32");
  if (k < 256 || k > KT_KMAX || k % 256) fail(ErrorCode::argument, "kmeans_assign_tc: K must be 256, 512, 768 or 1024");
  if (n < 1 || n > INT32_MAX) fail(ErrorCode::argument, "kmeans_assign_tc: N out of range");
  const BufView& P = buffer_arg(c, 0, "kmeans_assign_tc points");
  const BufView& S = buffer_arg(c, 1, "kmeans_assign_tc split");
  const BufView& X = buffer_arg(c, 2, "kmeans_assign_tc xx");
  const BufView& Cb = buffer_arg(c, 3, "kmeans_assign_tc centroids");
  if (Cb.first_byte != 0 || Cb.bytes != static_cast<uint64_t>(k * d) * 4)
    fail(ErrorCode::argument, "kmeans_assign_tc: centroids size != K*D");
  if (c.whole && (P.bytes != static_cast<uint64_t>(n * d) * 4 || S.bytes != static_cast<uint64_t>(n) * 128 ||
                  X.bytes != static_cast<uint64_t>(n) * 4))
    fail(ErrorCode::argument, "kmeans_assign_tc: points N*D fp32, split N*128 bytes, xx N fp32");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "kmeans_assign_tc");
  const float* pts = at_byte<const float>(P, lo * d * 4, rows * d * 4, "kmeans_assign_tc points");
  const uint8_t* split = at_byte<const uint8_t>(S, lo * 128, rows * 128, "kmeans_assign_tc split");
  const float* xx = at_byte<const float>(X, lo * 4, rows * 4, "kmeans_assign_tc xx");
  int32_t* asg = at_byte<int32_t>(buffer_arg(c, 4, "kmeans_assign_tc assign"), lo * 4, rows * 4, "kmeans_assign_tc assign");
  if (!rows) return 0;
  // per-launch centroid split + norms in scratch
  const size_t bsz = static_cast<size_t>(k) * 128;
  uint8_t* scr = static_cast<uint8_t*>(c.scratch(c.dev, 2 * bsz + static_cast<size_t>(k) * 4 + 64));
  uint16_t* b1 = reinterpret_cast<uint16_t*>(scr);
  uint16_t* b2 = reinterpret_cast<uint16_t*>(scr + bsz);
  float* q = reinterpret_cast<float*>(scr + 2 * bsz);
  unsigned* stats = reinterpret_cast<unsigned*>(scr + 2 * bsz + static_cast<size_t>(k) * 4);
  int* n_ovf = reinterpret_cast<int*>(stats + 4);
  HCL_CUDA(cudaMemsetAsync(stats, 0, 32, c.stream));
  kmeans_split_centroids_kernel<<<static_cast<unsigned>(ceil_div(k, 128)), 128, 0, c.stream>>>(
      reinterpret_cast<const float*>(Cb.ptr), b1, b2, q, stats, static_cast<int>(k));
  HCL_LAUNCHED();
  CUtensorMap ta = make_tmap_2d_bf16(split, 64, rows, 128, 64, KT_ROWS);
  CUtensorMap tb1 = make_tmap_2d_bf16(b1, 64, static_cast<uint64_t>(k), 128, 64, 128);
  CUtensorMap tb2 = make_tmap_2d_bf16(b2, 64, static_cast<uint64_t>(k), 128, 64, 128);
  const KtLayout Lh(static_cast<int>(k));
  const size_t smem = Lh.total;
  HCL_CUDA(cudaFuncSetAttribute(kmeans_assign_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  const int64_t tiles = ceil_div(static_cast<int64_t>(rows), 2 * KT_ROWS);
  const int64_t clusters = std::min<int64_t>(tiles, c.sm_count / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * 2));
  cfg.blockDim = dim3(KT_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const char* dbg_env = std::getenv("HCL_KM_DBG");
  const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
  HCL_CUDA(cudaLaunchKernelEx(&cfg, kmeans_assign_tc_kernel, ta, tb1, tb2, static_cast<const float*>(q),
                              reinterpret_cast<const float*>(stats), reinterpret_cast<const float*>(Cb.ptr), pts, xx,
                              asg, static_cast<int>(rows), static_cast<int>(k), n_ovf, dbg));
  HCL_LAUNCHED();
  return 3ull * rows * static_cast<uint64_t>(k) * static_cast<uint64_t>(d);
}

// kmeans_split_points(points, split, xx, N, D)
uint64_t launch_split_points(LaunchCtx& c) {
  const int64_t n = scalar_arg(c, 3, "kmeans_split_points N");
  const int64_t d = scalar_arg(c, 4, "kmeans_split_points D");
  if (d != KT_D) fail(ErrorCode::argument, "kmeans_split_points: D must be 32");
  const BufView& P = buffer_arg(c, 0, "kmeans_split_points points");
  if (c.whole && P.bytes != static_cast<uint64_t>(n * d) * 4)
    fail(ErrorCode::argument, "kmeans_split_points: points size != N*D");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(n), lo, rows, "kmeans_split_points");
  const float* pts = at_byte<const float>(P, lo * d * 4, rows * d * 4, "kmeans_split_points points");
  uint8_t* split = at_byte<uint8_t>(buffer_arg(c, 1, "split"), lo * 128, rows * 128, "kmeans_split_points split");
  float* xx = at_byte<float>(buffer_arg(c, 2, "xx"), lo * 4, rows * 4, "kmeans_split_points xx");
  if (!rows) return 0;
  kmeans_split_points_kernel<<<static_cast<unsigned>(ceil_div(rows, 256)), 256, 0, c.stream>>>(
      reinterpret_cast<const float4*>(pts), reinterpret_cast<uint4*>(split), xx, static_cast<int64_t>(rows));
  HCL_LAUNCHED();
  return rows;
}

uint64_t rows_tc(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[5]); }
uint64_t rows_split(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[3]); }

}  // namespace

void register_kmeans_tc(std::vector<KernelDef>& r) {
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS;
  r.push_back({"b200", "kmeans_assign_tc", {I, I, I, I, O, S, S, S}, {X, X, X, P, X, N, N, N}, launch_assign_tc,
               nullptr, rows_tc});
  r.push_back({"b200", "kmeans_split_points", {I, O, O, S, S}, {X, X, X, N, N}, launch_split_points, nullptr,
               rows_split});
}

}  // namespace hcl
