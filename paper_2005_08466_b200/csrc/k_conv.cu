// 3x3 convolution, stride 1, pad 1 (config C5) as an implicit GEMM on the
// 5th-generation tensor cores. Layouts in HBM:
//   input   : zero-padded NHWC bf16, [N][H+2][W+2][C]   (conv_pad_nhwc makes it)
//   weights : KRSC bf16, [K][3][3][C] = a K x 9C matrix
//   output  : NHWK, bf16 or fp32, [N][H][W][K]
// Implicit-GEMM trick: compute outputs on the "virtual" pixel grid of the padded
// image, p = h*(W+2) + w with w in [0, W+2): then the input pixel read by tap
// (r,s) is p + r*(W+2) + s — a uniform row shift of the flattened padded input —
// so every A tile is one plain 2D TMA box of 128 consecutive rows x 64 channels
// (SWIZZLE_128B, exactly the GEMM's K-major operand). The two junk columns per
// image row (w >= W) are computed and not stored (0.9% extra MMA work).
// Kernel structure = csrc/k_gemm.cu: persistent CTA pairs (cta_group::2, UMMA
// 256 x K x 16), warp 4 TMA producer, warp 5 MMA issuer, warps 0-3 epilogue,
// 8-stage smem ring, two TMEM accumulators. A pair tile is 256 consecutive
// virtual pixels of one image; K loop = 9 taps x C/64.
// The NDRange is the batch: a partitioned launch splits images (SPLIT_ROWS on
// input and output), weights are REPLICATE.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "common.hpp"
#include "ptx.cuh"
#include "../../include/hcl_cabi.h"

namespace hcl {

// from k_gemm.cu
CUtensorMap make_tmap_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                              uint32_t box_outer);

namespace {

constexpr int CV_BM = 128;               // pixels per CTA tile
constexpr int CV_BN = 128;               // output channels (UMMA N)
constexpr int CV_BNL = CV_BN / 2;        // B rows per CTA
constexpr int CV_A = CV_BM * 128;        // 16 KB
constexpr int CV_B = CV_BNL * 128;       // 8 KB
constexpr int CV_STAGE = CV_A + CV_B;
constexpr int CV_STAGES = 8;
constexpr int CV_THREADS = 192;
constexpr int CV_TMEM = 256;             // 2 accumulators x 128 columns
constexpr size_t CV_SMEM = static_cast<size_t>(CV_STAGES) * CV_STAGE + 1024 + 256;

template <bool OUTF32>
__global__ void __launch_bounds__(CV_THREADS, 1)
    conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      void* __restrict__ out, int n_img, int H, int W, int C) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CV_STAGES * CV_STAGE);
  uint64_t* empty = full + CV_STAGES;
  uint64_t* tfull = empty + CV_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const int Wp = W + 2;
  const int64_t img_rows = static_cast<int64_t>(H + 2) * Wp;  // padded pixels per image
  const int m_img = H * Wp;                                    // virtual output pixels per image
  const int tiles_img = (m_img + 2 * CV_BM - 1) / (2 * CV_BM);
  const int tiles = n_img * tiles_img;
  const int cb = C / 64;
  const int nk = 9 * cb;

  if (warp == 4 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < CV_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 8);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 5) ptx::tmem_alloc<2>(tmem_slot, CV_TMEM);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;

  if (warp == 4) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < tiles; t += nclusters) {
        const int n = t / tiles_img;
        const int p0 = (t % tiles_img) * 2 * CV_BM + static_cast<int>(rank) * CV_BM;
        const int64_t arow = static_cast<int64_t>(n) * img_rows + p0;
        for (int kb = 0; kb < nk; ++kb) {
          const int tap = kb / cb, c0 = (kb % cb) * 64;
          const int r = tap / 3, s = tap % 3;
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * CV_STAGE;
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CV_STAGE * 2);
          const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
          ptx::tma_load_2d_pair(sa, &tmA, bar, c0, static_cast<int>(arow + r * Wp + s));
          ptx::tma_load_2d_pair(sa + CV_A, &tmB, bar, tap * C + c0, static_cast<int>(rank) * CV_BNL);
          if (++stage == CV_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc(1, 0, 0, 2 * CV_BM, CV_BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < tiles; t += nclusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * CV_BN);
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smem + stage * CV_STAGE);
          const uint32_t b_addr = a_addr + CV_A;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            ptx::mma<2, false>(d_tmem, ptx::umma_desc_sw128(a_addr + k * 32, 16, 1024),
                               ptx::umma_desc_sw128(b_addr + k * 32, 16, 1024), idesc, (kb | k) != 0);
          ptx::mma_commit<2>(&empty[stage]);
          if (++stage == CV_STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit<2>(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cluster; t < tiles; t += nclusters) {
      const int n = t / tiles_img;
      const int p = (t % tiles_img) * 2 * CV_BM + static_cast<int>(rank) * CV_BM + warp * 32 + lane;
      const int h = p / Wp, w = p - h * Wp;
      const bool ok = p < m_img && w < W;
      const int64_t opix = (static_cast<int64_t>(n) * H + h) * W + w;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int chunk = 0; chunk < CV_BN / 32; ++chunk) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) +
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
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 5) {
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
  CUtensorMap ta = make_tmap_2d_bf16(in, C, rows, C * 2, 64, CV_BM);
  CUtensorMap tb = make_tmap_2d_bf16(Wt.ptr, 9 * C, K, 9 * C * 2, 64, CV_BNL);
  auto kern = out_f32 ? conv3x3_tc_kernel<true> : conv3x3_tc_kernel<false>;
  HCL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(CV_SMEM)));
  const int64_t tiles_img = ceil_div(H * (W + 2), 2 * CV_BM);
  const int64_t clusters = std::min<int64_t>(static_cast<int64_t>(cnt) * tiles_img, c.sm_count / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * 2));
  cfg.blockDim = dim3(CV_THREADS);
  cfg.dynamicSmemBytes = CV_SMEM;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HCL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, static_cast<void*>(outp), static_cast<int>(cnt), static_cast<int>(H),
                              static_cast<int>(W), static_cast<int>(C)));
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
}

}  // namespace hcl
