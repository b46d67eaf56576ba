// Tensor-core filtered k-means assignment (config C4; SURVEY.md §8(d) C4 "with
// tensor filtering"). Same result as kmeans_assign -- the exact fp32 argmin of
// sum_j (c_kj - x_j)^2 (every operation separately rounded, j ascending, ties
// to the smaller k; the reference's knn k=1, proj/src/kernels.cpp:195-233) --
// but the 2*N*K*D distance work runs on the 5th-generation tensor cores:
//
//   1. score: t~_k = |c_k|^2 - 2 x . c_k straight out of the tensor core:
//      tcgen05 bf16 MMAs with fp32 accumulation on split operands x = xh + xl
//      (exact for points on a 2^-12 grid, else |x - xh - xl| <= 2^-16 |x|)
//      and c = ch + cl (+ |residual| <= 2^-16 |c|): -2(xh.ch + xl.ch + xh.cl)
//      as 6 MMAs of K=16 over the A row [xh|xl] and the B rows [-2ch|-2ch]
//      (4) and [-2cl|..] (2; xl.cl, <= 2^-18 |x||c|, is dropped), plus one
//      K=16 MMA of a constant "ones" A tile against B2's second half
//      [qh, ql, 0...] (|c|^2 as bf16 hi + lo, |error| <= 2^-17 |c|^2). t_k
//      ranks the centroids like |x - c_k|^2 (|x|^2 is common to the row); the
//      scan reads it from TMEM with no per-score arithmetic.
//   2. filter (epilogue, per point): every k with t_k <= min_j t_j + 2 eps is a
//      candidate, eps = 2^-10 (|x| max|c| + |x|^2 + max|c|^2) -- at least 4x
//      the bound on |t_k + |x|^2 - d_k| from the splits and the dropped term,
//      the tensor-core accumulation (<= 2^-13 (|x||c| + |c|^2)) and the fp32
//      evaluation of the exact distance d_k (<= 2^-19 (|x|^2 + |c|^2 +
//      2|x||c|)). The exact argmin is always a candidate, and so is every k
//      tied with it.
//   3. verify: the candidates' exact fp32 distances (the oracle's operation
//      order) pick the result; a point whose candidate list overflows (or
//      with more than KT_QCAP survivors) is scanned exactly over all K by
//      the whole verify warp.
// On the C4 data (2^28 points, K=1024, 1024 Gaussian blobs) the filter keeps
// 1.26 candidates per point on average (max 5; profiles/r01_kmeans_tc.txt); at 2^26
// points 22% of the points keep several (0.48 exact checks per point) and
// ~900 overflow (HCL_KM_DBG=16 prints these counts).
//
// Layout: points are stored twice -- fp32 (the exact pass and the update) and
// split bf16 [xh(32) | xl(32)] (128 B per point = one SWIZZLE_128B row) with
// |x|^2 per point, made once by kmeans_split_points. Per launch the centroids
// are split into B1 = [-2ch|-2ch], B2 = [-2cl|qh,ql,0..] (bf16, K x 64). One
// persistent CTA pair (cta_group::2) per 2 SMs: the pair's B halves for all K
// are resident (K/2 x 256 B per CTA, <= 128 KB), A tiles of 2 x 128 points
// stream through 2 stages, and each tile runs K/KT_CW chunks of N=KT_CW MMAs
// into 512/KT_CW TMEM accumulators. KT_GROUPS groups of 4 scan warps each take
// a KT_CW/KT_GROUPS column slice of every chunk (score, running minimum,
// candidate mask; one list entry per batch of 32 columns with candidates)
// and hand each tile's lists (double-buffered in shared memory, mbarrier
// handshakes) to the verify warps -- two sets of 4, one per list buffer --
// which filter, check exactly and store while the scan runs on. Measured on
// 2^26 points, K=1024 (round 1 sweeps, profiles/r01_kmeans_tc.txt): 4 groups x 4 slots,
// N=256: 20.2 ms, 17.2 ms with |c|^2 folded into the MMA; 2 groups x 8 slots:
// 24.5 ms; N=128 chunks: 22.0 ms.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
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
#ifndef HCL_KT_GROUPS
#define HCL_KT_GROUPS 4
#endif
#ifndef HCL_KT_CW
#define HCL_KT_CW 256
#endif
constexpr int KT_CW = HCL_KT_CW;             // centroids per chunk (MMA N); TMEM holds 512 / KT_CW accumulators
constexpr int KT_NACC = 512 / KT_CW;
constexpr int KT_GROUPS = HCL_KT_GROUPS;     // scan groups: column slices of every chunk
constexpr int KT_SCAN = 4 * KT_GROUPS;       // scan warps (TMEM scores -> candidate lists)
constexpr int KT_VER = 8;                    // verify warps: two sets of 4, one per list buffer
constexpr int KT_QCAP = 8;                   // queued exact checks per point (more: full scan)
constexpr int KT_PROD = KT_SCAN + KT_VER;    // TMA producer warp, then the MMA warp
constexpr int KT_GCOLS = KT_CW / KT_GROUPS;  // columns per group per chunk
static_assert(KT_GCOLS >= 32 && KT_GCOLS % 32 == 0, "scan groups take whole 32-column batches");
constexpr int KT_MMA = KT_PROD + 1;
constexpr int KT_THREADS = (KT_MMA + 1) * 32;
constexpr int KT_ROWS = 128;                 // points per CTA per tile
constexpr int KT_A = KT_ROWS * 128;          // 16 KB A tile per CTA
constexpr int KT_STAGES = 2;
constexpr int KT_BH = (KT_CW / 2) * 128;     // per CTA, chunk and split part: KT_CW / 2 centroids x 128 B
#ifndef HCL_KT_LIST
#define HCL_KT_LIST (16 / HCL_KT_GROUPS)
#endif
constexpr int KT_LIST = HCL_KT_LIST;         // list entries (32-column batches with candidates) per point and scan group
constexpr int KT_KMAX = 1024;
static_assert((KT_KMAX / KT_CW) * (KT_GCOLS / 32) <= 16, "list keys carry a 4-bit batch index");
constexpr int KT_LBUF = KT_GROUPS * KT_ROWS * KT_LIST;  // float2 slots of one tile's lists (all groups)

struct KtLayout {
  size_t b, a, q, lists, xch, vq, bars, seed, total;
  __host__ __device__ KtLayout(int K) {
    const int nch = K / KT_CW;
    b = 0;
    a = b + static_cast<size_t>(nch) * 2 * KT_BH;
    q = a + static_cast<size_t>(KT_STAGES) * KT_A;
    lists = q + 4096;  // q: the constant "ones" A tile of the |c|^2 MMA (128 rows x 16 bf16, no swizzle)
    xch = lists + 2ull * KT_LBUF * 8;             // 2 buffers x (key | batch index, mask) float2 entries
    vq = xch + 2ull * KT_GROUPS * KT_ROWS * 8 + 2ull * KT_ROWS * 4;  // 2 bufs x groups x (min, count|ovf) + 2 eps
    bars = vq + static_cast<size_t>(KT_VER) * 32 * KT_QCAP * 8;  // verify queues
    seed = bars + 16 * 8 + 16;                    // barriers, TMEM slot
    total = seed + 2 * KT_ROWS * 4 + 1024;        // per-point threshold seeds (2 tiles), alignment slack
  }
};

// first centroid of a list entry's batch: batch index (low 4 key bits) within scan group g
__device__ __forceinline__ int entry_k0(uint32_t key, int g) {
  const int bi = static_cast<int>(key & 0xfu);
  return (bi / (KT_GCOLS / 32)) * KT_CW + g * KT_GCOLS + (bi % (KT_GCOLS / 32)) * 32;
}

// scan -> verify hand-off through named barriers: a waiting warp is parked by
// bar.sync and takes no issue slot (polled mbarriers cost the ALU-bound scan
// warps up to a quarter of their issue slots). Per list buffer b: LF(b) "lists
// of b complete" (scan warps arrive, the verify set of b syncs), LE(b) "b free
// again" (the verify set arrives, the scan warps sync before reusing b).
constexpr int KT_HANDOFF = (KT_SCAN + KT_VER / 2) * 32;
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ int bar_lf(int b) { return 2 + b; }
__device__ __forceinline__ int bar_le(int b) { return 4 + b; }

// three-input minimum (sm_100: one FMNMX3)
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(KT_SCAN * 32) : "memory"); }

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
                            const __grid_constant__ CUtensorMap tmB2, const float* __restrict__ qnorm,
                            const float* __restrict__ stats, const float* __restrict__ cent,
                            const float* __restrict__ pts, const float* __restrict__ xxg,
                            int32_t* __restrict__ assign, int rows, int K, int* __restrict__ n_overflow,
                            int dbg) {
  // dbg (HCL_KM_DBG, diagnostics only; wrong results): bit 0 skips the exact
  // verification, bit 2 the whole verify stage, bit 4 counts exact checks
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // aligned by pointer arithmetic on the shared array (not through an integer
  // cast), so the compiler keeps the shared address space: LDS/STS for the
  // candidate lists instead of generic loads and stores
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const KtLayout L(K);
  uint8_t* sb = smem + L.b;
  uint8_t* sa = smem + L.a;
  uint32_t* ones = reinterpret_cast<uint32_t*>(smem + L.q);
  float2* lists = reinterpret_cast<float2*>(smem + L.lists);
  float2* xch = reinterpret_cast<float2*>(smem + L.xch);              // [buf][group][point] (min, count|ovf<<16)
  float* xeps = reinterpret_cast<float*>(xch + 2 * KT_GROUPS * KT_ROWS);  // [buf][point] 2 eps
  int2* vq = reinterpret_cast<int2*>(smem + L.vq);
  float* seeds = reinterpret_cast<float*>(smem + L.seed);  // per point of the tile: the threshold seed
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + KT_STAGES;
  uint64_t* tfull = empty + KT_STAGES;
  uint64_t* tempty = tfull + KT_NACC;
  uint64_t* lfull = tempty + KT_NACC;   // [2] scan -> verify: a tile's candidate lists are complete
  uint64_t* lempty = lfull + 2;   // [2] verify -> scan: list buffer free again
  uint64_t* bfull = lempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const int nch = K / KT_CW;

  if (warp == KT_PROD && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB1);
    ptx::prefetch_tmap(&tmB2);
    for (int s = 0; s < KT_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 2);  // the MMAs' commit + the scan warps' seed reads of the A rows
    }
    for (int a = 0; a < KT_NACC; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * KT_SCAN);  // every scan warp, both CTAs
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&lfull[a], KT_SCAN);
      ptx::mbar_init(&lempty[a], KT_VER / 2);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == KT_MMA) ptx::tmem_alloc<2>(tmem_slot, 512);
  // every 16-byte core-matrix row = bf16 [1, 1, 0 x 6]: A(m, k) = 1 for k % 8 in {0, 1},
  // against B2 columns 32.. = [qh, ql, 0 ...] (identical core matrices: layout-proof)
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) ones[i] = (i & 3) == 0 ? 0x3F803F80u : 0u;
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int tiles = (rows + 2 * KT_ROWS - 1) / (2 * KT_ROWS);

  if (warp == KT_PROD) {
    if (lane == 0) {
      // resident B: this CTA's half of every chunk's centroids
      if (rank == 0) ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(nch) * 2 * KT_BH * 2);
      const uint32_t bb = ptx::mapa(ptx::smem_u32(bfull), 0);
      for (int c = 0; c < nch; ++c) {
        const int row = c * KT_CW + static_cast<int>(rank) * (KT_CW / 2);
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
      constexpr uint32_t idesc = ptx::umma_idesc(1, 0, 0, 2 * KT_ROWS, KT_CW);
      ptx::mbar_wait(bfull, 0);
      const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(sa), 16, 1024);
      const uint64_t bdesc0 = ptx::umma_desc_sw128(ptx::smem_u32(sb), 16, 1024);
      const uint64_t ones_desc = ptx::umma_desc_noswz(ptx::smem_u32(ones), 128, 256);
      int stage = 0;
      uint32_t phase = 0, tph = 0;  // tph: phase bit per accumulator
      int acc = 0;
      for (int t = cluster; t < tiles; t += nclusters) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t adesc = adesc0 + static_cast<uint64_t>((stage * KT_A) >> 4);
        for (int c = 0; c < nch; ++c) {
          ptx::mbar_wait(&tempty[acc], ((tph >> acc) & 1) ^ 1);
          tph ^= 1u << acc;
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * KT_CW);
          const uint64_t b1 = bdesc0 + static_cast<uint64_t>(((2 * c) * KT_BH) >> 4);
          const uint64_t b2 = bdesc0 + static_cast<uint64_t>(((2 * c + 1) * KT_BH) >> 4);
#pragma unroll
          for (int i = 0; i < 4; ++i) ptx::mma_elect<2, false>(d_tmem, adesc + 2 * i, b1 + 2 * i, idesc, i != 0);
#pragma unroll
          for (int i = 0; i < 2; ++i) ptx::mma_elect<2, false>(d_tmem, adesc + 2 * i, b2 + 2 * i, idesc, 1);
          ptx::mma_elect<2, false>(d_tmem, ones_desc, b2 + 4, idesc, 1);  // + |c|^2 (B2 k-step 2)
          ptx::mma_commit_elect<2>(&tfull[acc]);
          if (++acc == KT_NACC) acc = 0;
        }
        ptx::mma_commit_elect<2>(&empty[stage]);
        if (++stage == KT_STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp < KT_SCAN) {
    // ---------------- scan: group g = column slice g of every chunk ----------------
    const int g = warp / 4, quad = warp % 4;
    const int pl = quad * 32 + lane;  // point within the CTA tile = TMEM lane
    const float qmax = stats[0];
    const float cmax = sqrtf(qmax);
    epi_bar();
    uint32_t tph = 0;  // phase bit per accumulator
    int acc = 0, it = 0;
    for (int t = cluster; t < tiles; t += nclusters, ++it) {
      const int buf = it & 1;
      const int row = t * 2 * KT_ROWS + static_cast<int>(rank) * KT_ROWS + pl;
      const bool valid = row < rows;
      const float xx = valid ? __ldg(xxg + row) : 0.f;
      const float two_eps = 0x1p-9f * (sqrtf(xx) * cmax + xx + qmax);
      float m = __int_as_float(0x7f800000);
      int cnt = 0, ovf = 0;
      if (it >= 2) named_sync(bar_le(buf), KT_HANDOFF);  // the verify warps are done with this buffer
      float2* my = lists + buf * KT_LBUF + (g * KT_ROWS + pl) * KT_LIST;
      for (int c = 0; c < nch; ++c) {
        ptx::mbar_wait(&tfull[acc], (tph >> acc) & 1);
        tph ^= 1u << acc;
        ptx::tc_fence_after();
        if (c == 0) {
          // start the running minimum at an upper bound of min_k t~_k: the score of
          // the point's previous centroid (any centroid bounds the minimum, so stale
          // or zero assignments are safe), t_p = |c_p|^2 - 2 x.c_p in fp32 with x =
          // xh + xl read from this tile's A rows (landed: chunk 0's scores exist, so
          // the MMAs have read them -- the stage's full barrier lives in the pair's
          // leader CTA; resident: the stage is released only after this read,
          // below), plus 2 eps (>= |t~_p - t_p| + fp32 error).
          // With the threshold tight from the first batch, a batch needs the mask
          // pass only where a candidate lies -- the warp skips it otherwise.
          // (computed once per point by scan group 0, shared through shared memory)
          if (g == 0) {
            float m0 = __int_as_float(0x7f800000);
            if (valid) {
              const int kp = min(max(assign[row], 0), K - 1);
              const uint8_t* arow = sa + (it % KT_STAGES) * KT_A + pl * 128;
              const float4* cp = reinterpret_cast<const float4*>(cent + static_cast<int64_t>(kp) * KT_D);
              float dot = 0.f;
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {  // 16-byte chunks q4 (xh) and q4 + 4 (xl), SWIZZLE_128B
                const uint4 hv = *reinterpret_cast<const uint4*>(arow + ((q4 ^ (pl & 7)) << 4));
                const uint4 lv = *reinterpret_cast<const uint4*>(arow + (((q4 + 4) ^ (pl & 7)) << 4));
                const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
                const float4 c0 = __ldg(cp + 2 * q4), c1 = __ldg(cp + 2 * q4 + 1);
                const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float x0 = __uint_as_float(hw[e] << 16) + __uint_as_float(lw[e] << 16);
                  const float x1 = __uint_as_float(hw[e] & 0xffff0000u) + __uint_as_float(lw[e] & 0xffff0000u);
                  dot = fmaf(x0, cc[2 * e], dot);
                  dot = fmaf(x1, cc[2 * e + 1], dot);
                }
              }
              m0 = fmaf(-2.f, dot, __ldg(qnorm + kp)) + two_eps;
            }
            seeds[buf * KT_ROWS + pl] = m0;  // double-buffered by tile parity
          }
          epi_bar();  // every scan warp: the seeds of this tile are written
          // the A rows are read: the stage may be refilled (with K <= 512 the MMAs
          // release it before the scan starts, so the producer also waits for this)
          if (warp == 0 && lane == 0) ptx::mbar_arrive(&empty[it % KT_STAGES]);
          m = seeds[buf * KT_ROWS + pl];
        }
        const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                               static_cast<uint32_t>(acc * KT_CW + g * KT_GCOLS);
#pragma unroll
        for (int b = 0; b < KT_GCOLS / 32; ++b) {
          uint32_t cur[32];
          ptx::tmem_ld_32x32b_x32(tbase + b * 32, cur);
          ptx::tmem_ld_wait();
          if (b == KT_GCOLS / 32 - 1) {  // our slice of the accumulator drained: hand it back
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
          }
          // batch minimum with 3-input mins (FMNMX3: 16 ALU ops for 32 scores instead of 31;
          // the scan is ALU-bound), independent partial minima for a shallow tree
          float g3[11];
#pragma unroll
          for (int j = 0; j < 10; ++j)
            g3[j] = min3f(__uint_as_float(cur[3 * j]), __uint_as_float(cur[3 * j + 1]), __uint_as_float(cur[3 * j + 2]));
          g3[10] = fminf(__uint_as_float(cur[30]), __uint_as_float(cur[31]));
          const float h0 = min3f(g3[0], g3[1], g3[2]), h1 = min3f(g3[3], g3[4], g3[5]);
          const float h2 = min3f(g3[6], g3[7], g3[8]), h3 = fminf(g3[9], g3[10]);
          const float bmin = min3f(h0, h1, fminf(h2, h3));
          m = fminf(m, bmin);
          const float thr = m + two_eps;
          if (__any_sync(0xffffffffu, bmin <= thr))
          // candidate mask: set.le gives exact 1.0/0.0 flags (one ALU op per
          // score) that FFMAs (the FMA pipe) weigh by 2^j into exact integers
          // below 2^24, read back from the float bits. A batch with candidates
          // appends ONE entry (key, mask): the key is a lower bound of the
          // batch minimum (so of every candidate's t) carrying the batch
          // index in its low 4 bits -- an entry whose key exceeds the final
          // threshold is certainly stale; the rest are verified exactly.
          {
            float acc[4] = {0x1p23f, 0.f, 0x1p23f, 0.f};  // 2^23 + bits 0-15 / 2^23 + bits 16-31
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float f;
              asm("set.le.f32.f32 %0, %1, %2;" : "=f"(f) : "f"(__uint_as_float(cur[j])), "f"(thr));
              acc[(j >> 4) * 2 + (j & 1)] = fmaf(f, static_cast<float>(1u << (j & 15)), acc[(j >> 4) * 2 + (j & 1)]);
            }
            const uint32_t lo = __float_as_uint(acc[0] + acc[1]), hi = __float_as_uint(acc[2] + acc[3]);
            const uint32_t mask = __byte_perm(lo, hi, 0x5410);
            if (mask) {
              if (cnt == KT_LIST) {  // drop entries the running minimum has excluded
                int w = 0;
#pragma unroll
                for (int e = 0; e < KT_LIST; ++e) {
                  const float2 en = my[e];
                  if (en.x <= thr) my[w++] = en;
                }
                cnt = w;
              }
              if (cnt < KT_LIST) {
                const float lb = bmin - (fabsf(bmin) * 0x1p-16f + 0x1p-100f);  // < bmin by >= 8 ulps
                const uint32_t key = (__float_as_uint(lb) & ~0xfu) | static_cast<uint32_t>(c * (KT_GCOLS / 32) + b);
                my[cnt++] = make_float2(__uint_as_float(key), __uint_as_float(mask));
              } else {
                ovf = 1;
              }
            }
          }
        }
        if (++acc == KT_NACC) acc = 0;
      }
      xch[(buf * KT_GROUPS + g) * KT_ROWS + pl] = make_float2(m, __int_as_float(cnt | (ovf << 16)));
      if (g == 0) xeps[buf * KT_ROWS + pl] = two_eps;
      __syncwarp();
      named_arrive(bar_lf(buf), KT_HANDOFF);
    }
  } else if (warp < KT_SCAN + KT_VER) {
    // ---------------- verify: final filter, exact check of multi-candidate points, store ----------------
    // set vset = vw / 4 takes the tiles of list buffer vset (every other tile)
    const int vw = warp - KT_SCAN, vset = vw / 4;
    const int pl = (vw % 4) * 32 + lane;
    int2* wq = vq + vw * (32 * KT_QCAP);
    int it = vset;
    for (int t = cluster + vset * nclusters; t < tiles; t += 2 * nclusters, it += 2) {
      const int buf = vset;
      const int row = t * 2 * KT_ROWS + static_cast<int>(rank) * KT_ROWS + pl;
      const bool valid = row < rows;
      named_sync(bar_lf(buf), KT_HANDOFF);  // parked until the scan warps hand this tile over
      if (dbg & 4) {
        __syncwarp();
        named_arrive(bar_le(buf), KT_HANDOFF);
        continue;
      }
      float mall = __int_as_float(0x7f800000);
      int ovf = 0, cnts[KT_GROUPS];
#pragma unroll
      for (int gg = 0; gg < KT_GROUPS; ++gg) {
        const float2 o = xch[(buf * KT_GROUPS + gg) * KT_ROWS + pl];
        mall = fminf(mall, o.x);
        cnts[gg] = __float_as_int(o.y) & 0xffff;
        ovf |= __float_as_int(o.y) >> 16;
      }
      const float thr = mall + xeps[buf * KT_ROWS + pl];
      const float2* lbase = lists + buf * KT_LBUF + pl * KT_LIST;
      // all list entries at once (independent shared loads), stale ones masked off
      float2 ent[KT_GROUPS * KT_LIST];
#pragma unroll
      for (int gg = 0; gg < KT_GROUPS; ++gg)
#pragma unroll
        for (int e = 0; e < KT_LIST; ++e) {
          float2 en = make_float2(0.f, 0.f);
          if (e < cnts[gg]) en = lbase[gg * KT_ROWS * KT_LIST + e];
          if (!(en.x <= thr)) en.y = 0.f;  // mask 0: no candidates
          ent[gg * KT_LIST + e] = en;
        }
      // a single survivor is the exact argmin as it stands; points with several
      // survivors queue their (point, centroid) pairs for the whole warp
      int nc = 0, k1 = 0;
      if (valid && !ovf)
#pragma unroll
        for (int gg = 0; gg < KT_GROUPS; ++gg)
#pragma unroll
          for (int e = 0; e < KT_LIST; ++e) {
            const uint32_t mk = __float_as_uint(ent[gg * KT_LIST + e].y);
            if (mk) {
              nc += __popc(mk);
              k1 = entry_k0(__float_as_uint(ent[gg * KT_LIST + e].x), gg) + __ffs(mk) - 1;
            }
          }
      if (nc > KT_QCAP) {  // more survivors than its queue share: full scan
        ovf = 1;
        nc = 0;
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
      if (dbg & 16) {  // diagnostics: queued exact checks, multi-candidate points
        const uint32_t multi = __ballot_sync(0xffffffffu, nq > 0);
        if (lane == 0) {
          atomicAdd(n_overflow + 1, total);
          atomicAdd(n_overflow + 2, __popc(multi));
        }
      }
      if (nq) {
        int w = off;
#pragma unroll
        for (int gg = 0; gg < KT_GROUPS; ++gg)
#pragma unroll
          for (int e = 0; e < KT_LIST; ++e) {
            const int k0 = entry_k0(__float_as_uint(ent[gg * KT_LIST + e].x), gg);
            for (uint32_t mk = __float_as_uint(ent[gg * KT_LIST + e].y); mk; mk &= mk - 1)
              wq[w++] = make_int2((k0 + __ffs(mk) - 1) | (lane << 16), 0);
          }
      }
      __syncwarp();
      named_arrive(bar_le(buf), KT_HANDOFF);  // lists consumed (the queue is private)
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
      // points whose candidate list overflowed: exact scan over all K, the
      // whole warp sharing one point (lane-strided centroids, then a warp
      // argmin with the lowest index on ties)
      int okb = -1;
      for (uint32_t om = __ballot_sync(0xffffffffu, valid && ovf); om; om &= om - 1) {
        const int p = __ffs(om) - 1;
        float x[KT_D];
#pragma unroll
        for (int j = 0; j < KT_D; j += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(pts + static_cast<int64_t>(row0 + p) * KT_D + j));
          x[j] = v.x;
          x[j + 1] = v.y;
          x[j + 2] = v.z;
          x[j + 3] = v.w;
        }
        float best = __int_as_float(0x7f800000);
        int bkk = 0x7fffffff;
        for (int k = lane; k < K; k += 32) {
          const float e = exact_dist(x, cent + static_cast<int64_t>(k) * KT_D);
          if (e < best) { best = e; bkk = k; }
        }
#pragma unroll
        for (int sft = 16; sft; sft >>= 1) {
          const float ob = __shfl_xor_sync(0xffffffffu, best, sft);
          const int ok = __shfl_xor_sync(0xffffffffu, bkk, sft);
          if (ob < best || (ob == best && ok < bkk)) { best = ob; bkk = ok; }
        }
        if (lane == p) okb = bkk;
      }
      if (valid) {
        int bk = k1;
        if (ovf) {  // candidate list overflowed (rare): the warp scan above
          atomicAdd(n_overflow, 1);
          bk = okb;
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
    // -2c: exact in bf16 (a power-of-two scale), so the MMA accumulates -2 x.c directly
    b1[k * 64 + j] = b1[k * 64 + 32 + j] = __bfloat16_as_ushort(__hmul(h, __float2bfloat16_rn(-2.f)));
    b2[k * 64 + j] = __bfloat16_as_ushort(__hmul(l, __float2bfloat16_rn(-2.f)));
    s = fmaf(v, v, s);
  }
  // B2's second half carries |c|^2 as bf16 hi + lo (|error| <= 2^-17 |c|^2) for the
  // ones-column MMA: the accumulator then holds t = |c|^2 - 2 x.c itself
  const __nv_bfloat16 qh = __float2bfloat16_rn(s);
  const __nv_bfloat16 ql = __float2bfloat16_rn(s - __bfloat162float(qh));
  b2[k * 64 + 32] = __bfloat16_as_ushort(qh);
  b2[k * 64 + 33] = __bfloat16_as_ushort(ql);
  for (int j = 34; j < 64; ++j) b2[k * 64 + j] = 0;
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
  CUtensorMap tb1 = make_tmap_2d_bf16(b1, 64, static_cast<uint64_t>(k), 128, 64, KT_CW / 2);
  CUtensorMap tb2 = make_tmap_2d_bf16(b2, 64, static_cast<uint64_t>(k), 128, 64, KT_CW / 2);
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
  if (dbg & 16) {  // diagnostics: report list overflows of this launch
    int h[3] = {0, 0, 0};
    HCL_CUDA(cudaMemcpyAsync(h, n_ovf, 12, cudaMemcpyDeviceToHost, c.stream));
    HCL_CUDA(cudaStreamSynchronize(c.stream));
    std::fprintf(stderr, "kmeans_assign_tc: %d list overflows, %d queued exact checks, %d multi-candidate points in %lld points\n",
                 h[0], h[1], h[2], static_cast<long long>(rows));
  }
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
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT, IO = HCL_ARG_INOUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS;
  // assign is INOUT: the previous assignment seeds each point's threshold
  r.push_back({"b200", "kmeans_assign_tc", {I, I, I, I, IO, S, S, S}, {X, X, X, P, X, N, N, N}, launch_assign_tc,
               nullptr, rows_tc});
  r.push_back({"b200", "kmeans_split_points", {I, O, O, S, S}, {X, X, X, N, N}, launch_split_points, nullptr,
               rows_split});
}

}  // namespace hcl
