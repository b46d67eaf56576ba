// 3x3 convolution, stride 1, pad 1 (config C5) as an implicit GEMM on the
// 5th-generation tensor cores. Layouts in HBM:
//   input   : zero-padded NHWC bf16, [N][H+2][W+2][C]   (conv_pad_nhwc makes it)
//   weights : KRSC bf16, [K][3][3][C] = a K x 9C matrix
//   output  : NHWK, bf16 or fp32, [N][H][W][K]
// Implicit-GEMM trick: compute outputs on the "virtual" pixel grid of the padded
// image, p = h*(W+2) + w with w in [0, W+2): the input pixel read by tap (r,s) is
// then p + r*(W+2) + s — a uniform row shift of the flattened padded input — so
// an A tile is one plain 2D TMA box of consecutive rows x 64 channels
// (SWIZZLE_128B, exactly the GEMM's K-major operand). The two junk columns per
// image row (w >= W) are computed and not stored (0.9% extra MMA work).
//
// Kernel structure = csrc/k_gemm.cu: persistent CTA pairs (cta_group::2, UMMA
// 256 x 128 x 16), a TMA producer warp, an MMA issuer warp, epilogue warps, an
// smem ring, two TMEM accumulators (2 x 128 columns). A pair tile is 256
// consecutive virtual pixels of one image.
//   v2 (C == 64, default): the weights stay resident in shared memory (each CTA
//     holds its 64 output channels x 9 taps = 72 KB, loaded once), and one A
//     load per filter row r (136 consecutive padded pixels) feeds the three taps
//     s = 0,1,2 through descriptors that start s rows (s*128 bytes) further into
//     the swizzled tile. Measured on B200: the UMMA's 128B swizzle is address
//     based like TMA's, so the descriptor base-offset field stays 0 (setting it
//     to the row phase gives wrong results). 8 epilogue warps (two per TMEM lane
//     quadrant) keep the short K = 576 main loop fed.
//   v1 (any C multiple of 64): one A and one B TMA load per tap and 64-channel
//     chunk, 4 epilogue warps.
// The NDRange is the batch: a partitioned launch splits images (SPLIT_ROWS input
// and output), weights are REPLICATE.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.hpp"
#include "ptx.cuh"
#include "../../include/hcl_cabi.h"

namespace hcl {

// from k_gemm.cu
CUtensorMap make_tmap_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                              uint32_t box_outer);
CUtensorMap make_tmap_4d_bf16(const void* base, const uint64_t dims[4], const uint64_t strides[3],
                              const uint32_t box[4]);

namespace {

constexpr int CV_BM = 128;          // pixels per CTA tile (TMEM lanes)
constexpr int CV_BN = 128;          // output channels (UMMA N)
constexpr int CV_BNL = CV_BN / 2;   // B rows per CTA
constexpr int CV_TMEM = 256;        // 2 accumulators x 128 columns

// v1
constexpr int CV1_A = CV_BM * 128;  // 16 KB
constexpr int CV1_B = CV_BNL * 128; // 8 KB
constexpr int CV1_STAGE = CV1_A + CV1_B;
constexpr int CV1_STAGES = 8;
constexpr int CV1_EPI = 4;          // epilogue warps 0-3, producer 4, MMA 5
constexpr size_t CV1_SMEM = static_cast<size_t>(CV1_STAGES) * CV1_STAGE + 1024 + 256;

// v2
constexpr int CV2_AROWS = 136;              // 128 pixels + 2 shifted rows, padded to 8
constexpr int CV2_A = CV2_AROWS * 128;      // 17 KB
constexpr int CV2_BTAP = CV_BNL * 128;      // 8 KB per tap per CTA
constexpr int CV2_B = 9 * CV2_BTAP;         // 72 KB
constexpr int CV2_EPI = 8;                  // epilogue warps 0-7, producer 8, MMA 9
constexpr int CV2_OSTAGE = 32 * 128;        // per epilogue warp: 32 pixels x 64 bf16 channels (TMA-store staging)
// bf16 output stages its tiles in shared memory for TMA stores (6 A stages);
// fp32 output stores directly from registers (8 A stages)
template <bool OUTF32>
struct CV2Cfg {
  static constexpr int kStages = OUTF32 ? 8 : 6;
  static constexpr size_t kObytes = OUTF32 ? 0 : static_cast<size_t>(CV2_EPI) * CV2_OSTAGE;
  static constexpr size_t kSmem = static_cast<size_t>(CV2_B) + static_cast<size_t>(kStages) * CV2_A + kObytes + 1024 + 256;
};

// One epilogue warp's share of a finished 128-pixel x 128-channel accumulator:
// TMEM lane quadrant warp%4 (32 pixels), channel chunks [c0, c1) of 32.
template <bool OUTF32>
__device__ __forceinline__ void conv_epilogue(uint32_t tmem_base, int acc, int warp, int c0, int c1, bool ok,
                                              int64_t opix, void* __restrict__ out) {
#pragma unroll 1
  for (int chunk = c0; chunk < c1; ++chunk) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>((warp % 4) * 32) << 16) +
                                static_cast<uint32_t>(acc * CV_BN + chunk * 32),
                            r);
    ptx::tmem_ld_wait();
    if (!ok) continue;
    if constexpr (OUTF32) {
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<float*>(out) + opix * CV_BN + chunk * 32);
#pragma unroll
      for (int j = 0; j < 8; ++j) dst[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
    } else {
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        pk[j] = *reinterpret_cast<uint32_t*>(&b2);
      }
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + opix * CV_BN + chunk * 32);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    }
  }
}

struct ConvGeom {
  int Wp, m_img, tiles_img, tiles;
  int64_t img_rows;
  __device__ ConvGeom(int n_img, int H, int W) {
    Wp = W + 2;
    img_rows = static_cast<int64_t>(H + 2) * Wp;
    m_img = H * Wp;
    tiles_img = (m_img + 2 * CV_BM - 1) / (2 * CV_BM);
    tiles = n_img * tiles_img;
  }
};

// Epilogue warps' loop over this cluster's tiles (shared by v1 and v2).
// epi_mode (HCL_CONV_EPI, diagnostics only): 0 normal, 1 skip TMEM loads and
// stores, 2 TMEM loads without stores -- separates MMA, TMEM-read and store costs
template <bool OUTF32, int EPI>
__device__ __forceinline__ void conv_epilogue_loop(const ConvGeom& g, int H, int W, uint32_t rank, int warp, int lane,
                                                   uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty,
                                                   void* __restrict__ out, int epi_mode) {
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int c0 = EPI == 8 ? (warp / 4) * 2 : 0, c1 = EPI == 8 ? c0 + 2 : 4;
  int acc = 0;
  uint32_t acc_phase = 0;
  for (int t = cluster; t < g.tiles; t += nclusters) {
    const int n = t / g.tiles_img;
    const int p = (t % g.tiles_img) * 2 * CV_BM + static_cast<int>(rank) * CV_BM + (warp % 4) * 32 + lane;
    const int h = p / g.Wp, w = p - h * g.Wp;
    const bool ok = p < g.m_img && w < W && epi_mode == 0;
    const int64_t opix = (static_cast<int64_t>(n) * H + h) * W + w;
    ptx::mbar_wait(&tfull[acc], acc_phase);
    ptx::tc_fence_after();
    if (epi_mode != 1) conv_epilogue<OUTF32>(tmem_base, acc, warp, c0, c1, ok, opix, out);
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
  }
}

// bf16 epilogue through shared memory and TMA stores (v2): each epilogue warp
// owns 32 consecutive virtual pixels (TMEM lane quadrant warp%4) x 64 output
// channels (warp/4). It releases the accumulator right after its TMEM loads,
// writes its 32 x 128-byte rows SWIZZLE_128B-swizzled into a private 4 KB
// buffer, and one lane stores them with a 4D TMA box [1,1,32,64]
// of the N x H x W x K output; a group that wraps into the next image row
// stores its wrapped lanes directly from registers; the padding columns
// (w >= W) and rows past the image (h >= H) are out of bounds, so TMA skips them.
__device__ __forceinline__ void conv_epilogue_loop_tma(const ConvGeom& g, int H, int W, uint32_t rank, int warp,
                                                       int lane, uint32_t tmem_base, uint64_t* tfull,
                                                       uint64_t* tempty, const CUtensorMap* tmO, uint8_t* obuf,
                                                       void* __restrict__ out, int epi_mode) {
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int half = warp / 4;
  int acc = 0;
  uint32_t acc_phase = 0;
  for (int t = cluster; t < g.tiles; t += nclusters) {
    const int n = t / g.tiles_img;
    const int p = (t % g.tiles_img) * 2 * CV_BM + static_cast<int>(rank) * CV_BM + (warp % 4) * 32;
    ptx::mbar_wait(&tfull[acc], acc_phase);
    ptx::tc_fence_after();
    uint32_t r0[32], r1[32];
    if (epi_mode != 1) {
      const uint32_t ta = tmem_base + (static_cast<uint32_t>((warp % 4) * 32) << 16) +
                          static_cast<uint32_t>(acc * CV_BN + half * 64);
      ptx::tmem_ld_32x32b_x32(ta, r0);
      ptx::tmem_ld_32x32b_x32(ta + 32, r1);
      ptx::tmem_ld_wait();
    }
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    if (epi_mode != 0) continue;
    if (lane == 0) ptx::bulk_wait_read0();  // the previous store has read this buffer
    __syncwarp();
    uint32_t pk[32];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      __nv_bfloat162 a = __floats2bfloat162_rn(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
      __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]));
      pk[j] = *reinterpret_cast<uint32_t*>(&a);
      pk[16 + j] = *reinterpret_cast<uint32_t*>(&b);
    }
    uint8_t* row = obuf + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) << 4)) =
          make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    ptx::fence_proxy_async_smem();
    __syncwarp();
    const int h = p / g.Wp, w = p - h * g.Wp;
    if (lane == 0) {
      if (h < H) ptx::tma_store_4d(tmO, obuf, half * 64, w, h, n);
      ptx::bulk_commit();
    }
    // a group that wraps into the next image row: those lanes store their
    // 128 bytes directly (TMA box starts cannot be negative)
    const int j0 = g.Wp - w;
    if (lane >= j0 && h + 1 < H) {
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) +
                                            ((static_cast<int64_t>(n) * H + h + 1) * W + (lane - j0)) * CV_BN +
                                            half * 64);
#pragma unroll
      for (int j = 0; j < 8; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    }
  }
  if (lane == 0) ptx::bulk_wait0();
}

template <bool OUTF32>
__global__ void __launch_bounds__((CV1_EPI + 2) * 32, 1)
    conv3x3_v1_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      void* __restrict__ out, int n_img, int H, int W, int C, int epi_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CV1_STAGES * CV1_STAGE);
  uint64_t* empty = full + CV1_STAGES;
  uint64_t* tfull = empty + CV1_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  constexpr int PROD = CV1_EPI, MMA = CV1_EPI + 1;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const ConvGeom g(n_img, H, W);
  const int cb = C / 64, nk = 9 * cb;

  if (warp == PROD && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < CV1_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * CV1_EPI);
    }
    ptx::fence_mbar_init();
  }
  if (warp == MMA) ptx::tmem_alloc<2>(tmem_slot, CV_TMEM);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;

  if (warp == PROD) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < g.tiles; t += nclusters) {
        const int n = t / g.tiles_img;
        const int p0 = (t % g.tiles_img) * 2 * CV_BM + static_cast<int>(rank) * CV_BM;
        const int64_t arow = static_cast<int64_t>(n) * g.img_rows + p0;
        for (int kb = 0; kb < nk; ++kb) {
          const int tap = kb / cb, c0 = (kb % cb) * 64;
          const int r = tap / 3, s = tap % 3;
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * CV1_STAGE;
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CV1_STAGE * 2);
          const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
          ptx::tma_load_2d_pair(sa, &tmA, bar, c0, static_cast<int>(arow + r * g.Wp + s));
          ptx::tma_load_2d_pair(sa + CV1_A, &tmB, bar, tap * C + c0, static_cast<int>(rank) * CV_BNL);
          if (++stage == CV1_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == MMA) {
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc(1, 0, 0, 2 * CV_BM, CV_BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < g.tiles; t += nclusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * CV_BN);
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smem + stage * CV1_STAGE);
          const uint32_t b_addr = a_addr + CV1_A;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            ptx::mma<2, false>(d_tmem, ptx::umma_desc_sw128(a_addr + k * 32, 16, 1024),
                               ptx::umma_desc_sw128(b_addr + k * 32, 16, 1024), idesc, (kb | k) != 0);
          ptx::mma_commit<2>(&empty[stage]);
          if (++stage == CV1_STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit<2>(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    conv_epilogue_loop<OUTF32, CV1_EPI>(g, H, W, rank, warp, lane, tmem_base, tfull, tempty, out, epi_mode);
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == MMA) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2>(tmem_base, CV_TMEM);
  }
}

template <bool OUTF32>
__global__ void __launch_bounds__((CV2_EPI + 2) * 32, 1)
    conv3x3_v2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, void* __restrict__ out, int n_img, int H, int W,
                      int epi_mode) {
  constexpr int CV2_STAGES = CV2Cfg<OUTF32>::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_b = smem;
  uint8_t* smem_a = smem + CV2_B;
  uint8_t* smem_o = smem_a + CV2_STAGES * CV2_A;  // 1024-aligned (72 KB + 6 x 17 KB)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_o + CV2Cfg<OUTF32>::kObytes);
  uint64_t* empty = full + CV2_STAGES;
  uint64_t* tfull = empty + CV2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  constexpr int PROD = CV2_EPI, MMA = CV2_EPI + 1;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const ConvGeom g(n_img, H, W);

  if (warp == PROD && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if constexpr (!OUTF32) ptx::prefetch_tmap(&tmO);
    for (int s = 0; s < CV2_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * CV2_EPI);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == MMA) ptx::tmem_alloc<2>(tmem_slot, CV_TMEM);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;

  if (warp == PROD) {
    if (lane == 0) {
      // resident weights: 9 taps x this CTA's 64 output channels
      if (rank == 0) ptx::mbar_arrive_expect_tx(bfull, CV2_B * 2);
      const uint32_t bb = ptx::mapa(ptx::smem_u32(bfull), 0);
      for (int tap = 0; tap < 9; ++tap)
        ptx::tma_load_2d_pair(smem_b + tap * CV2_BTAP, &tmB, bb, tap * 64, static_cast<int>(rank) * CV_BNL);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < g.tiles; t += nclusters) {
        const int n = t / g.tiles_img;
        const int p0 = (t % g.tiles_img) * 2 * CV_BM + static_cast<int>(rank) * CV_BM;
        const int64_t arow = static_cast<int64_t>(n) * g.img_rows + p0;
        for (int r = 0; r < 3; ++r) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CV2_A * 2);
          const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
          ptx::tma_load_2d_pair(smem_a + stage * CV2_A, &tmA, bar, 0, static_cast<int>(arow + r * g.Wp));
          if (++stage == CV2_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == MMA) {
    if (rank == 0) {
      // the whole warp runs the issue loop (uniform operands, elect.sync inside
      // the MMA asm); descriptors are the base descriptors plus compile-time
      // offsets in 16-byte units (the start-address field, bits 0-13)
      constexpr uint32_t idesc = ptx::umma_idesc(1, 0, 0, 2 * CV_BM, CV_BN);
      ptx::mbar_wait(bfull, 0);
      const uint64_t bdesc0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_b), 16, 1024);
      const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_a), 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < g.tiles; t += nclusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * CV_BN);
        for (int r = 0; r < 3; ++r) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t adesc = adesc0 + static_cast<uint64_t>((stage * CV2_A) >> 4);
#pragma unroll
          for (int s = 0; s < 3; ++s) {
            const int tap = r * 3 + s;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              ptx::mma_elect<2, false>(d_tmem, adesc + static_cast<uint64_t>((s * 128 + k * 32) >> 4),
                                       bdesc0 + static_cast<uint64_t>((tap * CV2_BTAP + k * 32) >> 4), idesc,
                                       (r | s | k) != 0);
          }
          ptx::mma_commit_elect<2>(&empty[stage]);
          if (++stage == CV2_STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit_elect<2>(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    if constexpr (OUTF32)
      conv_epilogue_loop<OUTF32, CV2_EPI>(g, H, W, rank, warp, lane, tmem_base, tfull, tempty, out, epi_mode);
    else
      conv_epilogue_loop_tma(g, H, W, rank, warp, lane, tmem_base, tfull, tempty, &tmO, smem_o + warp * CV2_OSTAGE,
                             out, epi_mode);
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == MMA) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2>(tmem_base, CV_TMEM);
  }
}

// ---------------------------------------------------------------------------
// v3: straight from unpadded NHWC (conv3x3_nhwc, C == 64). A CTA's tile is a
// 16 (h) x 8 (w) block of output pixels (a CTA pair: 16 x 16); TMEM lane
// m = 8 g + j is pixel (h0 + g, w0 + j). The producer loads the tile's input
// halo as ONE 4D TMA box {64 ch, 16 w, 18 h, 1 image} at signed coordinates
// (w0 - 1, h0 - 1): TMA zero-fills everything outside the image, which IS the
// padding -- no padded copy of the input exists. In shared memory halo pixel
// (a, b) is row 16 a + b (128 B, SWIZZLE_128B), so for tap (r, s) the MMA's A
// operand starts at row 16 r + s: 8-row groups (one h each) 16 rows = 2048 B
// apart (the descriptor's stride), 1024-byte aligned plus the row shift s
// (address-based swizzle, as in v2). One 36 KB load feeds all 9 taps; the
// halo re-read is 288 / 128 = 2.25 rows per pixel (v2: 3 x 136 / 128 = 3.2).
constexpr int CV3_TW = 8, CV3_TH = 16;               // CTA tile: 8 w x 16 h = 128 pixels
constexpr int CV3_BW = 16, CV3_BH = CV3_TH + 2;      // halo box: 16 w (>= 8 + 2, 8-row groups) x 18 h
constexpr int CV3_A = CV3_BW * CV3_BH * 128;         // 36 KB
template <bool OUTF32>
struct CV3Cfg {
  static constexpr int kStages = OUTF32 ? 4 : 3;
  static constexpr size_t kObytes = OUTF32 ? 0 : static_cast<size_t>(CV2_EPI) * CV2_OSTAGE;
  static constexpr size_t kSmem = static_cast<size_t>(CV2_B) + static_cast<size_t>(kStages) * CV3_A + kObytes + 1024 + 256;
};

struct Conv3Geom {
  int th, tw, tiles_img, tiles;
  __device__ Conv3Geom(int n_img, int H, int W) {
    th = (H + CV3_TH - 1) / CV3_TH;
    tw = (W + 2 * CV3_TW - 1) / (2 * CV3_TW);
    tiles_img = th * tw;
    tiles = n_img * tiles_img;
  }
  // pair tile t -> image, this CTA's h0, w0
  __device__ void at(int t, uint32_t rank, int& n, int& h0, int& w0) const {
    n = t / tiles_img;
    const int q = t - n * tiles_img;
    h0 = (q / tw) * CV3_TH;
    w0 = (q % tw) * 2 * CV3_TW + static_cast<int>(rank) * CV3_TW;
  }
};

// epilogue, fp32 output: each lane stores its pixel's channel chunks directly
__device__ __forceinline__ void conv3_epilogue_loop_f32(const Conv3Geom& g, int H, int W, uint32_t rank, int warp,
                                                        int lane, uint32_t tmem_base, uint64_t* tfull,
                                                        uint64_t* tempty, void* __restrict__ out, int epi_mode) {
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int c0 = (warp / 4) * 2, c1 = c0 + 2;
  const int m = (warp % 4) * 32 + lane;
  int acc = 0;
  uint32_t acc_phase = 0;
  for (int t = cluster; t < g.tiles; t += nclusters) {
    int n, h0, w0;
    g.at(t, rank, n, h0, w0);
    const int h = h0 + m / CV3_TW, w = w0 + m % CV3_TW;
    const bool ok = h < H && w < W && epi_mode == 0;
    const int64_t opix = (static_cast<int64_t>(n) * H + h) * W + w;
    ptx::mbar_wait(&tfull[acc], acc_phase);
    ptx::tc_fence_after();
    if (epi_mode != 1) conv_epilogue<true>(tmem_base, acc, warp, c0, c1, ok, opix, out);
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
  }
}

// epilogue, bf16 output: a warp's 32 pixels are 4 h x 8 w of the tile; their
// 64-channel half goes through a swizzled 4 KB buffer and one 4D TMA store
// {64 ch, 8 w, 4 h, 1} (pixels outside the image are clipped by TMA)
__device__ __forceinline__ void conv3_epilogue_loop_tma(const Conv3Geom& g, uint32_t rank, int warp, int lane,
                                                        uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty,
                                                        const CUtensorMap* tmO, uint8_t* obuf, int epi_mode) {
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int half = warp / 4, quad = warp % 4;
  int acc = 0;
  uint32_t acc_phase = 0;
  for (int t = cluster; t < g.tiles; t += nclusters) {
    int n, h0, w0;
    g.at(t, rank, n, h0, w0);
    ptx::mbar_wait(&tfull[acc], acc_phase);
    ptx::tc_fence_after();
    uint32_t r0[32], r1[32];
    if (epi_mode != 1) {
      const uint32_t ta = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * CV_BN + half * 64);
      ptx::tmem_ld_32x32b_x32(ta, r0);
      ptx::tmem_ld_32x32b_x32(ta + 32, r1);
      ptx::tmem_ld_wait();
    }
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    if (epi_mode != 0) continue;
    if (lane == 0) ptx::bulk_wait_read0();  // the previous store has read this buffer
    __syncwarp();
    uint32_t pk[32];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      __nv_bfloat162 a = __floats2bfloat162_rn(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
      __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]));
      pk[j] = *reinterpret_cast<uint32_t*>(&a);
      pk[16 + j] = *reinterpret_cast<uint32_t*>(&b);
    }
    uint8_t* row = obuf + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) << 4)) =
          make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_4d(tmO, obuf, half * 64, w0, h0 + quad * 4, n);
      ptx::bulk_commit();
    }
  }
  if (lane == 0) ptx::bulk_wait0();
}

template <bool OUTF32>
__global__ void __launch_bounds__((CV2_EPI + 2) * 32, 1)
    conv3x3_v3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, void* __restrict__ out, int n_img, int H, int W,
                      int epi_mode) {
  constexpr int STAGES = CV3Cfg<OUTF32>::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_b = smem;
  uint8_t* smem_a = smem + CV2_B;                  // 72 KB: 1024-aligned
  uint8_t* smem_o = smem_a + STAGES * CV3_A;       // 36 KB stages: 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_o + CV3Cfg<OUTF32>::kObytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  constexpr int PROD = CV2_EPI, MMA = CV2_EPI + 1;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const Conv3Geom g(n_img, H, W);

  if (warp == PROD && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if constexpr (!OUTF32) ptx::prefetch_tmap(&tmO);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * CV2_EPI);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == MMA) ptx::tmem_alloc<2>(tmem_slot, CV_TMEM);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;

  if (warp == PROD) {
    if (lane == 0) {
      // resident weights: 9 taps x this CTA's 64 output channels
      if (rank == 0) ptx::mbar_arrive_expect_tx(bfull, CV2_B * 2);
      const uint32_t bb = ptx::mapa(ptx::smem_u32(bfull), 0);
      for (int tap = 0; tap < 9; ++tap)
        ptx::tma_load_2d_pair(smem_b + tap * CV2_BTAP, &tmB, bb, tap * 64, static_cast<int>(rank) * CV_BNL);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < g.tiles; t += nclusters) {
        int n, h0, w0;
        g.at(t, rank, n, h0, w0);
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CV3_A * 2);
        const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
        ptx::tma_load_4d_pair(smem_a + stage * CV3_A, &tmA, bar, 0, w0 - 1, h0 - 1, n);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == MMA) {
    if (rank == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc(1, 0, 0, 2 * CV_BM, CV_BN);
      ptx::mbar_wait(bfull, 0);
      const uint64_t bdesc0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_b), 16, 1024);
      const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_a), 16, CV3_BW * 128);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < g.tiles; t += nclusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * CV_BN);
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t adesc = adesc0 + static_cast<uint64_t>((stage * CV3_A) >> 4);
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int r = tap / 3, s = tap % 3;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            ptx::mma_elect<2, false>(d_tmem, adesc + static_cast<uint64_t>(((r * CV3_BW + s) * 128 + k * 32) >> 4),
                                     bdesc0 + static_cast<uint64_t>((tap * CV2_BTAP + k * 32) >> 4), idesc,
                                     (tap | k) != 0);
        }
        ptx::mma_commit_elect<2>(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        ptx::mma_commit_elect<2>(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    if constexpr (OUTF32)
      conv3_epilogue_loop_f32(g, H, W, rank, warp, lane, tmem_base, tfull, tempty, out, epi_mode);
    else
      conv3_epilogue_loop_tma(g, rank, warp, lane, tmem_base, tfull, tempty, &tmO, smem_o + warp * CV2_OSTAGE,
                              epi_mode);
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == MMA) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2>(tmem_base, CV_TMEM);
  }
}

// NHWC -> zero-padded NHWC (one 16-byte vector of 8 channels per thread)
__global__ void pad_nhwc_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n, int H, int W,
                                int c8) {
  const int64_t total = n * (H + 2) * (W + 2) * c8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t pix = e / c8;
    int c = static_cast<int>(e - pix * c8);
    int wp = static_cast<int>(pix % (W + 2));
    int64_t t = pix / (W + 2);
    int hp = static_cast<int>(t % (H + 2));
    int64_t img = t / (H + 2);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (hp >= 1 && hp <= H && wp >= 1 && wp <= W) v = in[((img * H + (hp - 1)) * W + (wp - 1)) * c8 + c];
    out[e] = v;
  }
}

// conv3x3(input_padded, weights, output, N, H, W, C, K, out_f32)
uint64_t launch_conv(LaunchCtx& c) {
  const int64_t n = scalar_arg(c, 3, "conv3x3 N"), H = scalar_arg(c, 4, "conv3x3 H"), W = scalar_arg(c, 5, "conv3x3 W");
  const int64_t C = scalar_arg(c, 6, "conv3x3 C"), K = scalar_arg(c, 7, "conv3x3 K");
  const bool out_f32 = scalar_arg(c, 8, "conv3x3 out_f32") != 0;
  if (n < 1 || H < 1 || W < 1 || C < 64 || C % 64 || K != CV_BN)
    fail(ErrorCode::argument, "conv3x3: need N,H,W >= 1, C a multiple of 64, K == 128 (this kernel's tile)");
  const int64_t img_in = (H + 2) * (W + 2) * C * 2, img_out = H * W * K * (out_f32 ? 4 : 2);
  const BufView& I = buffer_arg(c, 0, "conv3x3 input");
  const BufView& Wt = buffer_arg(c, 1, "conv3x3 weights");
  const BufView& O = buffer_arg(c, 2, "conv3x3 output");
  if (Wt.first_byte != 0 || Wt.bytes != static_cast<uint64_t>(K * 9 * C * 2))
    fail(ErrorCode::argument, "conv3x3: weights must be K x 3 x 3 x C bf16");
  if (c.whole && (I.bytes != static_cast<uint64_t>(n * img_in) || O.bytes != static_cast<uint64_t>(n * img_out)))
    fail(ErrorCode::argument, "conv3x3: input must be padded N x (H+2) x (W+2) x C bf16, output N x H x W x K");
  uint64_t lo, cnt;
  sub_range(c, static_cast<uint64_t>(n), lo, cnt, "conv3x3");
  const uint8_t* in = at_byte<const uint8_t>(I, lo * img_in, cnt * img_in, "conv3x3 input");
  uint8_t* outp = at_byte<uint8_t>(O, lo * img_out, cnt * img_out, "conv3x3 output");
  if (!cnt) return 0;
  const int64_t rows = static_cast<int64_t>(cnt) * (H + 2) * (W + 2);
  const char* mode_env = std::getenv("HCL_CONV_MODE");
  const bool v2 = C == 64 && !(mode_env && std::atoi(mode_env) == 1);
  CUtensorMap ta = make_tmap_2d_bf16(in, C, rows, C * 2, 64, v2 ? CV2_AROWS : CV_BM);
  CUtensorMap tb = make_tmap_2d_bf16(Wt.ptr, 9 * C, K, 9 * C * 2, 64, CV_BNL);
  void* kern = v2 ? (out_f32 ? reinterpret_cast<void*>(conv3x3_v2_kernel<true>)
                             : reinterpret_cast<void*>(conv3x3_v2_kernel<false>))
                  : (out_f32 ? reinterpret_cast<void*>(conv3x3_v1_kernel<true>)
                             : reinterpret_cast<void*>(conv3x3_v1_kernel<false>));
  const size_t smem = v2 ? (out_f32 ? CV2Cfg<true>::kSmem : CV2Cfg<false>::kSmem) : CV1_SMEM;
  // bf16 output tensor N x H x W x K for the v2 TMA-store epilogue
  CUtensorMap to{};
  if (v2 && !out_f32) {
    const uint64_t od[4] = {static_cast<uint64_t>(K), static_cast<uint64_t>(W), static_cast<uint64_t>(H), cnt};
    const uint64_t os[3] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(W) * K * 2,
                            static_cast<uint64_t>(H) * W * K * 2};
    const uint32_t ob[4] = {64, 32, 1, 1};
    to = make_tmap_4d_bf16(outp, od, os, ob);
  }
  HCL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t tiles_img = ceil_div(H * (W + 2), 2 * CV_BM);
  const int64_t clusters = std::min<int64_t>(static_cast<int64_t>(cnt) * tiles_img, c.sm_count / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * 2));
  cfg.blockDim = dim3(((v2 ? CV2_EPI : CV1_EPI) + 2) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* outv = static_cast<void*>(outp);
  int cn = static_cast<int>(cnt), hh = static_cast<int>(H), ww = static_cast<int>(W), cc = static_cast<int>(C);
  const char* epi_env = std::getenv("HCL_CONV_EPI");
  int epi_mode = epi_env ? std::atoi(epi_env) : 0;
  void* params_v1[] = {&ta, &tb, &outv, &cn, &hh, &ww, &cc, &epi_mode};
  void* params_v2[] = {&ta, &tb, &to, &outv, &cn, &hh, &ww, &epi_mode};
  HCL_CUDA(cudaLaunchKernelExC(&cfg, kern, v2 ? params_v2 : params_v1));
  HCL_LAUNCHED();
  return 2ull * cnt * H * W * K * 9 * C;
}

// conv3x3_nhwc(input NHWC bf16 (unpadded), weights KRSC, output NHWK, N, H, W, C, K, out_f32):
// the whole layer from plain NHWC (v3 kernel; C == 64, K == 128)
uint64_t launch_conv_nhwc(LaunchCtx& c) {
  const int64_t n = scalar_arg(c, 3, "conv3x3_nhwc N"), H = scalar_arg(c, 4, "conv3x3_nhwc H");
  const int64_t W = scalar_arg(c, 5, "conv3x3_nhwc W");
  const int64_t C = scalar_arg(c, 6, "conv3x3_nhwc C"), K = scalar_arg(c, 7, "conv3x3_nhwc K");
  const bool out_f32 = scalar_arg(c, 8, "conv3x3_nhwc out_f32") != 0;
  if (n < 1 || H < 1 || W < 1 || C != 64 || K != CV_BN)
    fail(ErrorCode::argument, "conv3x3_nhwc: need N,H,W >= 1, C == 64, K == 128 (this kernel's tile)");
  const int64_t img_in = H * W * C * 2, img_out = H * W * K * (out_f32 ? 4 : 2);
  const BufView& I = buffer_arg(c, 0, "conv3x3_nhwc input");
  const BufView& Wt = buffer_arg(c, 1, "conv3x3_nhwc weights");
  const BufView& O = buffer_arg(c, 2, "conv3x3_nhwc output");
  if (Wt.first_byte != 0 || Wt.bytes != static_cast<uint64_t>(K * 9 * C * 2))
    fail(ErrorCode::argument, "conv3x3_nhwc: weights must be K x 3 x 3 x C bf16");
  if (c.whole && (I.bytes != static_cast<uint64_t>(n * img_in) || O.bytes != static_cast<uint64_t>(n * img_out)))
    fail(ErrorCode::argument, "conv3x3_nhwc: input must be N x H x W x C bf16, output N x H x W x K");
  uint64_t lo, cnt;
  sub_range(c, static_cast<uint64_t>(n), lo, cnt, "conv3x3_nhwc");
  const uint8_t* in = at_byte<const uint8_t>(I, lo * img_in, cnt * img_in, "conv3x3_nhwc input");
  uint8_t* outp = at_byte<uint8_t>(O, lo * img_out, cnt * img_out, "conv3x3_nhwc output");
  if (!cnt) return 0;
  const uint64_t id[4] = {static_cast<uint64_t>(C), static_cast<uint64_t>(W), static_cast<uint64_t>(H), cnt};
  const uint64_t is[3] = {static_cast<uint64_t>(C) * 2, static_cast<uint64_t>(W) * C * 2,
                          static_cast<uint64_t>(H) * W * C * 2};
  const uint32_t ib[4] = {64, CV3_BW, CV3_BH, 1};
  CUtensorMap ta = make_tmap_4d_bf16(in, id, is, ib);
  CUtensorMap tb = make_tmap_2d_bf16(Wt.ptr, 9 * C, K, 9 * C * 2, 64, CV_BNL);
  CUtensorMap to{};
  if (!out_f32) {
    const uint64_t od[4] = {static_cast<uint64_t>(K), static_cast<uint64_t>(W), static_cast<uint64_t>(H), cnt};
    const uint64_t os[3] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(W) * K * 2,
                            static_cast<uint64_t>(H) * W * K * 2};
    const uint32_t ob[4] = {64, CV3_TW, 4, 1};
    to = make_tmap_4d_bf16(outp, od, os, ob);
  }
  void* kern = out_f32 ? reinterpret_cast<void*>(conv3x3_v3_kernel<true>) : reinterpret_cast<void*>(conv3x3_v3_kernel<false>);
  const size_t smem = out_f32 ? CV3Cfg<true>::kSmem : CV3Cfg<false>::kSmem;
  HCL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t tiles = static_cast<int64_t>(cnt) * ceil_div(H, CV3_TH) * ceil_div(W, 2 * CV3_TW);
  const int64_t clusters = std::min<int64_t>(tiles, c.sm_count / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * 2));
  cfg.blockDim = dim3((CV2_EPI + 2) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* outv = static_cast<void*>(outp);
  int cn = static_cast<int>(cnt), hh = static_cast<int>(H), ww = static_cast<int>(W);
  const char* epi_env = std::getenv("HCL_CONV_EPI");
  int epi_mode = epi_env ? std::atoi(epi_env) : 0;
  void* params[] = {&ta, &tb, &to, &outv, &cn, &hh, &ww, &epi_mode};
  HCL_CUDA(cudaLaunchKernelExC(&cfg, kern, params));
  HCL_LAUNCHED();
  return 2ull * cnt * H * W * K * 9 * C;
}

// conv_pad_nhwc(input NHWC bf16, output padded, N, H, W, C)
uint64_t launch_pad(LaunchCtx& c) {
  const int64_t n = scalar_arg(c, 2, "conv_pad_nhwc N"), H = scalar_arg(c, 3, "conv_pad_nhwc H");
  const int64_t W = scalar_arg(c, 4, "conv_pad_nhwc W"), C = scalar_arg(c, 5, "conv_pad_nhwc C");
  if (n < 1 || H < 1 || W < 1 || C < 8 || C % 8) fail(ErrorCode::argument, "conv_pad_nhwc: C must be a multiple of 8");
  const int64_t in_img = H * W * C * 2, out_img = (H + 2) * (W + 2) * C * 2;
  uint64_t lo, cnt;
  sub_range(c, static_cast<uint64_t>(n), lo, cnt, "conv_pad_nhwc");
  const uint8_t* in = at_byte<const uint8_t>(buffer_arg(c, 0, "pad in"), lo * in_img, cnt * in_img, "conv_pad_nhwc in");
  uint8_t* out = at_byte<uint8_t>(buffer_arg(c, 1, "pad out"), lo * out_img, cnt * out_img, "conv_pad_nhwc out");
  if (!cnt) return 0;
  pad_nhwc_kernel<<<c.sm_count * 8, 256, 0, c.stream>>>(reinterpret_cast<const uint4*>(in), reinterpret_cast<uint4*>(out),
                                                       static_cast<int64_t>(cnt), static_cast<int>(H),
                                                       static_cast<int>(W), static_cast<int>(C / 8));
  HCL_LAUNCHED();
  return cnt * (out_img + in_img);
}

uint64_t rows_conv(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[3]); }
uint64_t rows_pad(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[2]); }

}  // namespace

void register_conv(std::vector<KernelDef>& r) {
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS;
  r.push_back({"b200", "conv3x3", {I, I, O, S, S, S, S, S, S}, {X, P, X, N, N, N, N, N, N}, launch_conv, nullptr,
               rows_conv});
  r.push_back({"b200", "conv_pad_nhwc", {I, O, S, S, S, S}, {X, X, N, N, N, N}, launch_pad, nullptr, rows_pad});
  r.push_back({"b200", "conv3x3_nhwc", {I, I, O, S, S, S, S, S, S}, {X, P, X, N, N, N, N, N, N}, launch_conv_nhwc,
               nullptr, rows_conv});
}

}  // namespace hcl
