// Dense GEMM C = A * B for the partitioned NDRange (SURVEY.md §8(a) a9, configs
// C1/C2): the reference's matmul contraction (proj/src/kernels.cpp:96-119) on
// the 5th-generation tensor cores.
//
//   A  M x K row-major (K-major)          -- SPLIT_ROWS in a partitioned launch
//   B  K x N row-major (MN-major operand) -- REPLICATE
//   C  M x N row-major, bf16 or fp32      -- SPLIT_ROWS
//
// Kernel structure (a CTA pair per output tile, cta_group::2; a persistent
// schedule with strided tile lists is kept behind HCL_GEMM_PERSIST=1):
//   warp 4      TMA producer: A tile 128 x 128B and B tile (256/CG) x 128B per
//               stage into a 6-deep SWIZZLE_128B smem ring (mbarrier full/empty)
//   warp 5      MMA issuer (leader CTA; the whole warp runs the loop and
//               elect.sync picks the issuing lane): tcgen05.mma 256x256xK into
//               one of two TMEM accumulators (2 x 256 columns = all 512)
//   warps 0-3   epilogue: tcgen05.ld 32x32b -> registers -> bf16/fp32 -> HBM,
//               overlapped with the next tile's main loop (TMEM double buffer)
// Tiles are visited in an L2-friendly grouped order (8 M-tiles per group).
// K tails and M/N edges are handled by TMA zero fill plus masked stores.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "common.hpp"
#include "ptx.cuh"
#include "../../include/hcl_cabi.h"

namespace hcl {
namespace {

constexpr int kBM = 128;            // A rows per CTA
constexpr int kThreads = 192;       // 4 epilogue warps + producer + MMA
constexpr int kGroupM = 8;          // default tile raster group (HCL_GEMM_GROUP overrides)

// Tile shapes: (CG, BN) = (2, 256) for large problems (256x256 UMMA per CTA
// pair); (2, 128) and (1, 64) when the 256-wide grid would leave SMs idle
// (C1: a 1024^2 output is only 16 pair tiles at 256x256, 128 CTA tiles at 128x64).
// ONE: one tile per CTA pair -- a single TMEM accumulator and ~100 KB of
// stages, so two pairs share each SM pair and one's epilogue overlaps the
// other's main loop (the persistent schedule double-buffers TMEM instead).
template <int CG, bool TF32, int BN, bool ONE = false>
struct Cfg {
  static constexpr int kBN = BN;                 // tile N (UMMA_N)
  static constexpr int kTmemCols = ONE ? BN : 2 * BN;  // accumulators x BN fp32 columns
  static constexpr int kElem = TF32 ? 4 : 2;
  static constexpr int kBK = 128 / kElem;        // one 128-byte swizzle row of K
  static constexpr int kUK = 32 / kElem;         // K per tcgen05.mma
  static constexpr int kBNLocal = kBN / CG;      // B rows (N) loaded by each CTA
  static constexpr int kABytes = kBM * 128;
  static constexpr int kBBytes = kBNLocal * 128;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kBudget = ONE ? 100 * 1024 : 200 * 1024;
  static constexpr int kStages = kBudget / kStage < 8 ? kBudget / kStage : 8;
  static constexpr int kMNAtom = 128 / kElem;    // MN elements per swizzle atom row
  // bf16 C through shared memory + TMA stores (ONE): 4 warps x 32 rows x 64 B
  static constexpr bool kTmaC = ONE && !TF32;
  static constexpr int kCStage = 32 * 64;
  static constexpr size_t kCBytes = kTmaC ? 4 * kCStage : 0;
  static constexpr size_t kSmem = static_cast<size_t>(kStages) * kStage + kCBytes + 1024 + 256;
};

template <int CG, bool TF32, int BN, bool ONE>
struct C_MC_OK {  // MC needs two 64-column B atoms per CTA (one per pair)
  static constexpr bool value = Cfg<CG, TF32, BN, ONE>::kBNLocal / Cfg<CG, TF32, BN, ONE>::kMNAtom == 2;
};

struct TileMap {
  int num_m, num_n, group_m;
  __device__ __forceinline__ void get(int t, int& mt, int& nt) const {
    int group = group_m * num_n;
    int g = t / group;
    int first_m = g * group_m;
    int gm = min(group_m, num_m - first_m);
    int local = t - g * group;
    mt = first_m + local % gm;
    nt = local / gm;
  }
};

// MC: clusters of two CTA pairs computing vertically adjacent tiles (same B
// columns); each CTA loads half of its B half and multicasts it to the
// same-rank CTA of the other pair, so every B byte leaves L2 once per cluster
// instead of twice. The stage's empty barrier then counts both pairs' MMA
// commits (the other pair writes into this CTA's stage).
template <int CG, bool TF32, bool BMN, bool OUTF32, int BN, bool ONE, bool MC = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, void* __restrict__ Cout, int M, int N, int K,
                   int64_t ldc, int group_m, int tma_c, int ksplit, int kseg) {
  // ksplit > 1 (fp32 output only): work unit t = (tile, K slice t / tiles); slice s
  // accumulates k-blocks [nk*s/ksplit, nk*(s+1)/ksplit) into C + s*M*ldc (a workspace
  // the launcher reduces in slice order)
  // kseg > 0 (K-major A and B, kseg % kBK == 0): the K' = 3 kseg operands are stored
  // as [hi | lo] (2 kseg per row) and read as A' = [hi | hi | lo], B' = [hi | lo | hi]
  using C = Cfg<CG, TF32, BN, ONE>;
  constexpr int kBN = C::kBN;
  static_assert(!BMN || C::kBNLocal % C::kMNAtom == 0, "MN-major B needs whole 128-byte atoms per CTA");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* cstage = smem + C::kStages * C::kStage;  // 1024-aligned (stages are 16/32 KB)
  uint64_t* full = reinterpret_cast<uint64_t*>(cstage + C::kCBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = CG == 2 ? ptx::cluster_ctarank() : 0;
  const uint32_t rank = MC ? (crank & 1u) : crank;  // CTA within its pair
  const uint32_t lead = MC ? (crank & ~1u) : 0u;    // the pair's leader (cluster rank)
  const uint32_t pr = MC ? (crank >> 1) : 0u;       // pair within the cluster
  static_assert(!MC || (CG == 2 && BMN && C_MC_OK<CG, TF32, BN, ONE>::value), "MC: 2-CTA pairs, MN-major B");

  if (warp == 4 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], MC ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4 * CG);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 5) ptx::tmem_alloc<CG>(tmem_slot, C::kTmemCols);
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::grid_dep_wait();  // the prologue above overlaps the producing launch's tail (PDL)
  ptx::grid_dep_launch();

  const TileMap map{static_cast<int>((M + kBM * CG - 1) / (kBM * CG)), (N + kBN - 1) / kBN, group_m};
  const int tiles = map.num_m * map.num_n;
  const int units = tiles * ksplit;
  const int cluster = blockIdx.x / CG, nclusters = gridDim.x / CG;
  const int nk = (K + C::kBK - 1) / C::kBK;

  if (warp == 4) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < units; t += nclusters) {
        int mt, nt;
        map.get(t % tiles, mt, nt);
        const int sp = t / tiles;
        const int kb0 = static_cast<int>(static_cast<int64_t>(nk) * sp / ksplit);
        const int kb1 = static_cast<int>(static_cast<int64_t>(nk) * (sp + 1) / ksplit);
        const int m0 = mt * kBM * CG + static_cast<int>(rank) * kBM;
        const int n0 = nt * kBN + static_cast<int>(rank) * C::kBNLocal;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          int ca = kb * C::kBK, cb = ca;  // A / B column of this k-block
          if (kseg) {
            const int sg = ca / kseg, off = ca - sg * kseg;
            ca = (sg == 2 ? kseg : 0) + off;
            cb = (sg == 1 ? kseg : 0) + off;
          }
          uint8_t* sa = smem + stage * C::kStage;
          uint8_t* sb = sa + C::kABytes;
          if constexpr (CG == 1) {
            ptx::mbar_arrive_expect_tx(&full[stage], C::kStage);
            ptx::tma_load_2d(sa, &tmA, &full[stage], ca, m0);
            if constexpr (BMN) {
#pragma unroll
              for (int j = 0; j < C::kBNLocal / C::kMNAtom; ++j)
                ptx::tma_load_2d(sb + j * C::kBK * 128, &tmB, &full[stage], n0 + j * C::kMNAtom, kb * C::kBK);
            } else {
              ptx::tma_load_2d(sb, &tmB, &full[stage], cb, n0);
            }
          } else {
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], C::kStage * 2);
            const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), lead);
            ptx::tma_load_2d_pair(sa, &tmA, bar, ca, m0);
            if constexpr (BMN && MC) {  // atom pr of this CTA's B half, to the same-rank CTA of both pairs
              ptx::tma_load_2d_pair_mc(sb + pr * C::kBK * 128, &tmB, ptx::smem_u32(&full[stage]) & 0xFEFFFFFFu,
                                       static_cast<uint16_t>(0x5u << rank), n0 + static_cast<int>(pr) * C::kMNAtom,
                                       kb * C::kBK);
            } else if constexpr (BMN) {
#pragma unroll
              for (int j = 0; j < C::kBNLocal / C::kMNAtom; ++j)
                ptx::tma_load_2d_pair(sb + j * C::kBK * 128, &tmB, bar, n0 + j * C::kMNAtom, kb * C::kBK);
            } else {
              ptx::tma_load_2d_pair(sb, &tmB, bar, cb, n0);
            }
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      // whole warp issues (uniform operands; elect.sync inside the asm);
      // descriptors = stage-0 descriptors + offsets in 16-byte units
      constexpr uint32_t idesc = ptx::umma_idesc(TF32 ? 2 : 1, 0, BMN ? 1 : 0, kBM * CG, kBN);
      const uint32_t a0 = ptx::smem_u32(smem);
      const uint64_t adesc0 = ptx::umma_desc_sw128(a0, 16, 1024);
      const uint64_t bdesc0 = BMN ? ptx::umma_desc_sw128(a0 + C::kABytes, C::kBK * 128, 1024)
                                  : ptx::umma_desc_sw128(a0 + C::kABytes, 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < units; t += nclusters) {
        const int sp = t / tiles;
        const int kb0 = static_cast<int>(static_cast<int64_t>(nk) * sp / ksplit);
        const int kb1 = static_cast<int>(static_cast<int64_t>(nk) * (sp + 1) / ksplit);
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t so = static_cast<uint64_t>((stage * C::kStage) >> 4);
#pragma unroll
          for (int k = 0; k < C::kBK / C::kUK; ++k) {
            const uint64_t adesc = adesc0 + so + static_cast<uint64_t>((k * 32) >> 4);
            const uint64_t bdesc = bdesc0 + so + static_cast<uint64_t>((BMN ? k * (C::kUK / 8) * 1024 : k * 32) >> 4);
            ptx::mma_elect<CG, TF32>(d_tmem, adesc, bdesc, idesc, (kb != kb0) | (k != 0));
          }
          if constexpr (MC)  // both pairs write into every CTA's stage: release it in all four
            ptx::mma_commit_elect_mask(&empty[stage], 0xF);
          else
            ptx::mma_commit_elect<CG>(&empty[stage]);  // frees the smem slot when these MMAs finish
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        if constexpr (MC)
          ptx::mma_commit_elect_mask(&tfull[acc], static_cast<uint16_t>(0x3u << (2 * pr)));
        else
          ptx::mma_commit_elect<CG>(&tfull[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 0-3 ----------------
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cluster; t < units; t += nclusters) {
      int mt, nt;
      map.get(t % tiles, mt, nt);
      const int64_t slice = static_cast<int64_t>(t / tiles) * M * ldc;  // 0 unless ksplit > 1
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int64_t row = static_cast<int64_t>(mt) * kBM * CG + rank * kBM + warp * 32 + lane;
      const bool row_ok = row < M;
#pragma unroll 1
      for (int chunk = 0; chunk < kBN / 32; ++chunk) {
        uint32_t r[32];
        const uint32_t taddr =
            tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(acc * kBN + chunk * 32);
        ptx::tmem_ld_32x32b_x32(taddr, r);
        ptx::tmem_ld_wait();
        const int col0 = nt * kBN + chunk * 32;
        if (C::kTmaC && !OUTF32 && tma_c) {
          if (col0 >= N) continue;  // warp-uniform; TMA clips rows >= M
        } else {
          if (!row_ok || col0 >= N) continue;
        }
        if constexpr (OUTF32) {
          float* dst = reinterpret_cast<float*>(Cout) + slice + row * ldc + col0;
          if (col0 + 32 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<uint4*>(dst)[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < N) dst[j] = __uint_as_float(r[j]);
          }
        } else if (Cfg<CG, TF32, BN, ONE>::kTmaC && tma_c) {
          // SWIZZLE_64B staging: row = lane, 16-byte chunk j at j ^ ((row >> 1) & 3);
          // TMA clips rows >= M and columns >= N
          uint32_t p[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
            p[j] = *reinterpret_cast<uint32_t*>(&h);
          }
          uint8_t* buf = cstage + warp * C::kCStage;
          if (lane == 0) ptx::bulk_wait_read0();  // the previous chunk's store has read the buffer
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
                make_uint4(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(&tmC, buf, col0, static_cast<int>(row - lane));
            ptx::bulk_commit();
          }
        } else {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(Cout) + row * ldc + col0;
          uint32_t p[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
            p[j] = *reinterpret_cast<uint32_t*>(&h);
          }
          if (col0 + 32 <= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              reinterpret_cast<uint4*>(dst)[j] = make_uint4(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < N) dst[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        // relaxed: this barrier only returns the TMEM accumulator (no global-store ordering needed)
        ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&tempty[acc]), lead));
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  if constexpr (C::kTmaC)
    if (tma_c && warp < 4 && lane == 0) ptx::bulk_wait0();
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 5) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) fail(ErrorCode::internal, "cuTensorMapEncodeTiled unavailable from the driver");
  return fn;
}

// A (rows x cols) -> At (cols x pitch), pitch >= rows
__global__ void transpose_pitched_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t rows,
                                         int64_t cols, int64_t pitch) {
  __shared__ float tile[32][33];
  const int64_t c = blockIdx.x * 32 + threadIdx.x, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (r0 + i < rows && c < cols) tile[i][threadIdx.x] = in[(r0 + i) * cols + c];
  __syncthreads();
  const int64_t oc = r0 + threadIdx.x, or0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (or0 + i < cols && oc < rows) out[(or0 + i) * pitch + oc] = tile[threadIdx.x][i];
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// TMA L2 sector promotion (HCL_GEMM_PROMO 0..3 = none/64B/128B/256B). Default
// none: measured at 16384^3 bf16, 17.2 GB DRAM reads per launch vs 19.6 GB with
// 256B promotion, same or better time (profiles/r01_gemm_sweep.txt).
CUtensorMapL2promotion l2_promotion() {
  switch (env_int("HCL_GEMM_PROMO", 0)) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// 2D row-major tensor [outer][inner] with a SWIZZLE_128B box [box_outer][box_inner].
CUtensorMap make_tmap(const void* base, bool f32, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                      uint32_t box_inner, uint32_t box_outer,
                      CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, promo,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(ErrorCode::argument, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) +
                                  "): base/row pitch must be 16-byte aligned");
  return m;
}

template <int CG, bool TF32, bool BMN, bool OUTF32, int BN = 256, bool ONE = false, bool MC = false>
void run_gemm(const void* A, const void* B, void* Cp, int64_t M, int64_t N, int64_t K, int64_t ldc,
              int sm_count, cudaStream_t stream, int group_m, bool persistent, int ksplit = 1, bool pdl = false,
              int kseg = 0) {
  using C = Cfg<CG, TF32, BN, ONE>;
  const uint64_t es = C::kElem;
  const CUtensorMapL2promotion promo = l2_promotion();
  const int64_t kst = kseg ? 2 * kseg : K;  // stored K extent of A and K-major B
  CUtensorMap ta = make_tmap(A, TF32, kst, M, kst * es, C::kBK, kBM, promo);
  CUtensorMap tb = BMN ? make_tmap(B, TF32, N, K, N * es, C::kMNAtom, C::kBK, promo)
                       : make_tmap(B, TF32, kst, N, kst * es, C::kBK, C::kBNLocal, promo);
  CUtensorMap tc{};
  const int tma_c = C::kTmaC && !OUTF32 && env_int("HCL_GEMM_TMAC", 1) ? 1 : 0;
  if (tma_c) {  // C (M x N bf16), box 32 x 32, SWIZZLE_64B
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldc) * 2};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&tc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Cp, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(ErrorCode::argument, "cuTensorMapEncodeTiled (C) failed");
  }
  auto kern = gemm_tc_kernel<CG, TF32, BMN, OUTF32, BN, ONE, MC>;
  // per launch: the attribute is per device context and launches may target several GPUs
  HCL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::kSmem)));
  const int64_t tiles = ceil_div(M, kBM * CG) * ceil_div(N, BN) * ksplit;
  // One cluster per tile (default): the hardware launches clusters in raster
  // order as SMs free up, so the running tiles stay a compact window of the
  // grouped raster and L2 serves the panel re-reads. Measured at 16384^3:
  // 9.8 GB DRAM reads per launch and 1.40 GHz under the power cap, vs 18.4 GB
  // and 1.23 GHz for persistent CTA pairs walking strided tile lists, whose
  // drift spreads the live panels over several waves (profiles/r01_gemm_sweep.txt).
  // The persistent schedule (HCL_GEMM_PERSIST=1) is also what an SM budget
  // needs: its grid is sized to the budget (emulated heterogeneous devices).
  const int64_t clusters = !ONE && persistent ? std::min<int64_t>(tiles, sm_count / CG) : tiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * CG));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MC ? 2 * CG : CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  HCL_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, Cp, static_cast<int>(M), static_cast<int>(N),
                              static_cast<int>(K), ldc, group_m, tma_c, ksplit, kseg));
  HCL_LAUNCHED();
}

// B (K x N) -> Bt (N x K): used only by the K-major debug variant.
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t rows, int64_t cols) {
  __shared__ T tile[32][33];
  int64_t c = blockIdx.x * 32 + threadIdx.x, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (r0 + i < rows && c < cols) tile[i][threadIdx.x] = in[(r0 + i) * cols + c];
  __syncthreads();
  int64_t oc = r0 + threadIdx.x, or0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (or0 + i < cols && oc < rows) out[(or0 + i) * rows + oc] = tile[threadIdx.x][i];
}

// Tile shape with the smallest estimated time: waves x (BN + 32), i.e. the
// per-SM work of a tile (128 x BN) plus a fixed per-tile cost (prologue,
// pipeline fill, epilogue tail) in column units.
int pick_shape(int64_t M, int64_t N, int sm_count, int ksplit = 1) {
  static constexpr int kCG[4] = {2, 1, 2, 1}, kBNs[4] = {256, 256, 128, 64};
  int best = 0;
  int64_t best_t = INT64_MAX;
  for (int i : {0, 2, 3}) {
    const int64_t units = ceil_div(M, kBM * kCG[i]) * ceil_div(N, kBNs[i]) * ksplit;
    const int64_t clusters = std::max<int64_t>(1, std::min<int64_t>(units, sm_count / kCG[i]));
    const int64_t t = ceil_div(units, clusters) * (kBNs[i] + 32);
    if (t < best_t) { best_t = t; best = i; }
  }
  return best;
}

// B multicast across two CTA pairs (HCL_GEMM_MC=1): the clusters' two tiles must be
// vertically adjacent with the same B columns -- whole raster groups of an even
// number of M tiles, an even tile count, no K split
bool mc_ok(int64_t M, int64_t N, int group_m, int ksplit) {
  if (env_int("HCL_GEMM_MC", 0) == 0 || ksplit != 1 || group_m % 2) return false;
  const int64_t num_m = ceil_div(M, kBM * 2), num_n = ceil_div(N, 256);
  return num_m % group_m == 0 && (num_m * num_n) % 2 == 0;
}

template <bool TF32, bool BMN, bool OUTF32>
void dispatch_shape(int shape, const void* a, const void* b, void* cp, int64_t M, int64_t n, int64_t k,
                    const LaunchCtx& c, int group_m, int ksplit = 1, bool pdl = false, int kseg = 0) {
  const bool persist = c.sm_budgeted || env_int("HCL_GEMM_PERSIST", 0) != 0;
  switch (shape) {
    case 1:
      run_gemm<1, TF32, BMN, OUTF32, 256>(a, b, cp, M, n, k, n, c.sm_count, c.stream, group_m, persist, ksplit, pdl, kseg);
      break;
    case 2:
      run_gemm<2, TF32, BMN, OUTF32, 128>(a, b, cp, M, n, k, n, c.sm_count, c.stream, group_m, persist, ksplit, pdl, kseg);
      break;
    case 3:
      run_gemm<1, TF32, BMN, OUTF32, 64>(a, b, cp, M, n, k, n, c.sm_count, c.stream, group_m, persist, ksplit, pdl, kseg);
      break;
    default:
      if (!persist && env_int("HCL_GEMM_ONE", 1) == 0 && mc_ok(M, n, group_m, ksplit) && BMN && !TF32)
        run_gemm<2, TF32, BMN, OUTF32, 256, false, BMN && !TF32>(a, b, cp, M, n, k, n, c.sm_count, c.stream, group_m,
                                                                false, ksplit, pdl, kseg);
      else if (persist || env_int("HCL_GEMM_ONE", 1) == 0)
        run_gemm<2, TF32, BMN, OUTF32, 256>(a, b, cp, M, n, k, n, c.sm_count, c.stream, group_m, persist, ksplit, pdl, kseg);
      else if (mc_ok(M, n, group_m, ksplit) && BMN && !TF32)
        run_gemm<2, TF32, BMN, OUTF32, 256, true, BMN && !TF32>(a, b, cp, M, n, k, n, c.sm_count, c.stream, group_m,
                                                               false, ksplit, pdl, kseg);
      else
        run_gemm<2, TF32, BMN, OUTF32, 256, true>(a, b, cp, M, n, k, n, c.sm_count, c.stream, group_m, false,
                                                  ksplit, pdl, kseg);
      break;
  }
}

// C = sum over the ksplit workspace slices, in slice order (deterministic)
__global__ void __launch_bounds__(256) ksplit_reduce_kernel(const float4* __restrict__ ws, float4* __restrict__ out,
                                                            int64_t n4, int ksplit) {
  ptx::grid_dep_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = ws[i];
    for (int s = 1; s < ksplit; ++s) {
      const float4 b = ws[s * n4 + i];
      a.x = __fadd_rn(a.x, b.x);
      a.y = __fadd_rn(a.y, b.y);
      a.z = __fadd_rn(a.z, b.z);
      a.w = __fadd_rn(a.w, b.w);
    }
    out[i] = a;
  }
}

// gemm_bf16(A, B, C, M, K, N, out_f32) and gemm_tf32(A, B, C, M, K, N)
template <bool TF32>
uint64_t launch_gemm_tc(LaunchCtx& c) {
  const char* what = TF32 ? "gemm_tf32" : "gemm_bf16";
  int64_t m = scalar_arg(c, 3, "gemm M");
  int64_t k = scalar_arg(c, 4, "gemm K");
  int64_t n = scalar_arg(c, 5, "gemm N");
  bool out_f32 = TF32 ? true : scalar_arg(c, 6, "gemm out_f32") != 0;
  if (m < 1 || k < 1 || n < 1) fail(ErrorCode::argument, std::string(what) + ": dimensions must be >= 1");
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) fail(ErrorCode::argument, std::string(what) + ": dimension too large");
  const uint64_t es = TF32 ? 4 : 2, os = out_f32 ? 4 : 2;
  if ((k * es) % 16 || (n * es) % 16)
    fail(ErrorCode::argument, std::string(what) + ": K and N must be multiples of " + std::to_string(16 / es) +
                                  " (16-byte TMA row pitch)");
  const BufView& A = buffer_arg(c, 0, "gemm A");
  const BufView& B = buffer_arg(c, 1, "gemm B");
  const BufView& Cb = buffer_arg(c, 2, "gemm C");
  if (c.whole && A.bytes != static_cast<uint64_t>(m * k) * es)
    fail(ErrorCode::argument, std::string(what) + ": A size != M*K");
  if (B.first_byte != 0 || B.bytes != static_cast<uint64_t>(k * n) * es)
    fail(ErrorCode::argument, std::string(what) + ": B size != K*N");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(m), lo, rows, what);
  const void* a = at_byte<const uint8_t>(A, lo * k * es, rows * k * es, "gemm A");
  void* cp = at_byte<uint8_t>(Cb, lo * n * os, rows * n * os, "gemm C");
  if (rows == 0) return 0;
  const int cg = env_int("HCL_GEMM_CG", 0);  // 1/2 force the 256-wide shapes; 0 = auto
  // tf32 B goes K-major: an MN-major 32-bit operand needs the 128B_BASE32B
  // swizzle atom, which this kernel does not stage (measured: zeros)
  const bool kmajor = TF32 || env_int("HCL_GEMM_B_KMAJOR", 0) != 0;
  const void* b = B.ptr;
  if (kmajor) {  // debug/validation variant: transpose B to N x K first
    void* bt = c.scratch(c.dev, static_cast<size_t>(k * n * es));
    dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(k, 32)));
    if (TF32)
      transpose_kernel<float><<<grid, dim3(32, 8), 0, c.stream>>>(static_cast<const float*>(b), static_cast<float*>(bt), k, n);
    else
      transpose_kernel<uint16_t><<<grid, dim3(32, 8), 0, c.stream>>>(static_cast<const uint16_t*>(b), static_cast<uint16_t*>(bt), k, n);
    HCL_LAUNCHED();
    b = bt;
  }
  const int64_t M = static_cast<int64_t>(rows);
  const int group_m = std::max(1, env_int("HCL_GEMM_GROUP", kGroupM));
  int shape = env_int("HCL_GEMM_SHAPE", -1);  // debug override: 0..3 = (2,256) (1,256) (2,128) (1,64)
  if (shape < 0 || shape > 3) shape = cg == 1 ? 1 : cg == 2 ? 0 : pick_shape(M, n, c.sm_count);
  if (kmajor && !TF32) shape &= 1;  // the K-major bf16 debug variant exists for the 256-wide shapes only
  if (kmajor) {
    if (out_f32) dispatch_shape<TF32, false, true>(shape, a, b, cp, M, n, k, c, group_m);
    else dispatch_shape<TF32, false, false>(shape, a, b, cp, M, n, k, c, group_m);
  } else if constexpr (!TF32) {
    if (out_f32) dispatch_shape<TF32, true, true>(shape, a, b, cp, M, n, k, c, group_m);
    else dispatch_shape<TF32, true, false>(shape, a, b, cp, M, n, k, c, group_m);
  }
  return 2ull * rows * static_cast<uint64_t>(n) * static_cast<uint64_t>(k);
}

// ---------------------------------------------------------------------------
// fp32 GEMM as 3xTF32 on the tensor cores (gemm_f32x3). Each fp32 operand is
// split x = hi + lo with hi = tf32_rna(x) and lo = x - hi (exact in fp32);
// C = hi_a*hi_b + hi_a*lo_b + lo_a*hi_b (lo_a*lo_b ~ 2^-22 |a||b| dropped).
// The three products become ONE K-major TF32 GEMM over K' = 3K:
//   A'[r] = [hi(a_r) | hi(a_r) | lo(a_r)],  B'^T[n] = [hi(b_n) | lo(b_n) | hi(b_n)]
// built by one memory-bound split launch (A rows and B columns), then the same tcgen05 kernel as
// gemm_tf32 (and the K-slice reduction), chained as programmatic dependent launches. The split products are exact, but the tensor core's fp32
// accumulation truncates per MMA, so the measured normwise error is ~2^-19 at
// K=1024 and ~2^-17 at K=16384 (SIMT gemm_f32: ~2^-22) -- at 1/3 of the TF32
// tensor rate instead of the FFMA rate (16384^3: 192 vs 37 TFLOP/s).

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Both splits in one launch (small GEMMs are launch-bound): blocks [0, a_blocks)
// split A's rows, the rest transpose-split B in 32x32 tiles (256 threads = 32 x 8)
__global__ void __launch_bounds__(256) split3_both_kernel(const float4* __restrict__ a, float4* __restrict__ a3,
                                                          int64_t rows, int64_t k4, int a_blocks,
                                                          const float* __restrict__ b, float* __restrict__ b3,
                                                          int64_t K, int64_t N, int gx, bool seg) {
  if (static_cast<int>(blockIdx.x) < a_blocks) {
    const int64_t total = rows * k4;
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += static_cast<int64_t>(a_blocks) * 256) {
      const int64_t r = i / k4, c = i - r * k4;
      float4 v = a[i], h, l;
      h.x = tf32_hi(v.x); h.y = tf32_hi(v.y); h.z = tf32_hi(v.z); h.w = tf32_hi(v.w);
      l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
      if (seg) {  // [hi | lo]
        float4* o = a3 + r * 2 * k4 + c;
        o[0] = h;
        o[k4] = l;
      } else {
        float4* o = a3 + r * 3 * k4 + c;
        o[0] = h;
        o[k4] = h;
        o[2 * k4] = l;
      }
    }
    return;
  }
  __shared__ float tile[32][33];
  const int bid = static_cast<int>(blockIdx.x) - a_blocks;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t n0 = static_cast<int64_t>(bid % gx) * 32, k0 = static_cast<int64_t>(bid / gx) * 32;
  for (int i = ty; i < 32; i += 8) {
    const int64_t k = k0 + i, n = n0 + tx;
    tile[i][tx] = (k < K && n < N) ? b[k * N + n] : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t n = n0 + i, k = k0 + tx;
    if (n < N && k < K) {
      const float v = tile[tx][i], h = tf32_hi(v);
      float* o = b3 + n * (seg ? 2 : 3) * K + k;
      o[0] = h;
      o[K] = v - h;
      if (!seg) o[2 * K] = h;
    }
  }
}

// gemm_f32x3(A, B, C, M, K, N): same arguments and classes as gemm_f32
uint64_t launch_gemm_f32x3(LaunchCtx& c) {
  int64_t m = scalar_arg(c, 3, "gemm_f32x3 M");
  int64_t k = scalar_arg(c, 4, "gemm_f32x3 K");
  int64_t n = scalar_arg(c, 5, "gemm_f32x3 N");
  if (m < 1 || k < 1 || n < 1) fail(ErrorCode::argument, "gemm_f32x3: dimensions must be >= 1");
  if (m > INT32_MAX || n > INT32_MAX || 3 * k > INT32_MAX) fail(ErrorCode::argument, "gemm_f32x3: dimension too large");
  if (k % 4 || n % 4) fail(ErrorCode::argument, "gemm_f32x3: K and N must be multiples of 4 (16-byte TMA row pitch)");
  const BufView& A = buffer_arg(c, 0, "gemm_f32x3 A");
  const BufView& B = buffer_arg(c, 1, "gemm_f32x3 B");
  const BufView& Cb = buffer_arg(c, 2, "gemm_f32x3 C");
  if (c.whole && A.bytes != static_cast<uint64_t>(m * k) * 4) fail(ErrorCode::argument, "gemm_f32x3: A size != M*K");
  if (B.first_byte != 0 || B.bytes != static_cast<uint64_t>(k * n) * 4)
    fail(ErrorCode::argument, "gemm_f32x3: B size != K*N");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(m), lo, rows, "gemm_f32x3");
  const float* a = at_byte<const float>(A, lo * k * 4, rows * k * 4, "gemm_f32x3 A");
  float* cp = at_byte<float>(Cb, lo * n * 4, rows * n * 4, "gemm_f32x3 C");
  if (rows == 0) return 0;
  const int64_t r = static_cast<int64_t>(rows);
  // K split (slices of K' = 3K reduced in slice order, fp32 round-to-nearest). The
  // tensor core's fp32 accumulation truncates per MMA, so its error grows with the
  // accumulation length: each halving of K' per slice halves it (C1, 1024^3, measured
  // normwise: 2^-18.8 unsplit, 2^-19.9 with 2 slices, 2^-20.8 with 4, 2^-22.0 with 8).
  // Default: slices of ~768 K' (at most 4) when the fp32 slice workspace stays small
  // (M N <= 2^24); HCL_GEMM_KSPLIT overrides. A function of M, N and K only, so every
  // row partition of one GEMM sums in the same order (P-invariance).
  const int64_t nkb = ceil_div(3 * k, 32);
  const int64_t ks_default = m * n <= (int64_t(1) << 24) ? std::max<int64_t>(1, std::min<int64_t>(4, 3 * k / 768)) : 1;
  const int ksplit = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(env_int("HCL_GEMM_KSPLIT", static_cast<int>(ks_default)), nkb)));
  // K-block aligned K: the operands are stored once as [hi | lo] and the GEMM's
  // producer reads the three segments from them (HCL_GEMM_SEG=0: materialised 3K rows)
  const bool seg = k % 32 == 0 && env_int("HCL_GEMM_SEG", 1) != 0;
  const size_t a3_bytes = static_cast<size_t>(r * (seg ? 2 : 3) * k * 4);
  const size_t b3_bytes = static_cast<size_t>(n * (seg ? 2 : 3) * k * 4);
  const size_t ws_bytes = ksplit > 1 ? static_cast<size_t>(ksplit) * r * n * 4 : 0;
  uint8_t* s = static_cast<uint8_t*>(c.scratch(c.dev, a3_bytes + b3_bytes + ws_bytes));
  float* a3 = reinterpret_cast<float*>(s);
  float* b3 = reinterpret_cast<float*>(s + a3_bytes);
  float* ws = reinterpret_cast<float*>(s + a3_bytes + b3_bytes);
  {
    const int64_t total = r * (k / 4);
    const int a_blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 64LL * c.sm_count));
    const int gx = static_cast<int>(ceil_div(n, 32));
    const int64_t b_blocks = static_cast<int64_t>(gx) * ceil_div(k, 32);
    split3_both_kernel<<<static_cast<unsigned>(a_blocks + b_blocks), 256, 0, c.stream>>>(
        reinterpret_cast<const float4*>(a), reinterpret_cast<float4*>(a3), r, k / 4, a_blocks,
        reinterpret_cast<const float*>(B.ptr), b3, k, n, gx, seg);
    HCL_LAUNCHED();
  }
  const int group_m = std::max(1, env_int("HCL_GEMM_GROUP", kGroupM));
  int shape = env_int("HCL_GEMM_SHAPE", -1);
  if (shape < 0 || shape > 3) shape = pick_shape(r, n, c.sm_count, ksplit);
  // programmatic dependent launches: split -> GEMM -> reduce overlap each launch's
  // prologue with the previous one's tail (HCL_GEMM_PDL=0: plain stream order)
  const bool pdl = env_int("HCL_GEMM_PDL", 1) != 0;
  dispatch_shape<true, false, true>(shape, a3, b3, ksplit > 1 ? ws : cp, r, n, 3 * k, c, group_m, ksplit, pdl,
                                    seg ? static_cast<int>(k) : 0);
  if (ksplit > 1) {
    const int64_t n4 = r * n / 4;  // N % 4 == 0
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(n4, 256), 8LL * c.sm_count));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    HCL_CUDA(cudaLaunchKernelEx(&cfg, ksplit_reduce_kernel, reinterpret_cast<const float4*>(ws),
                                reinterpret_cast<float4*>(cp), n4, ksplit));
    HCL_LAUNCHED();
  }
  return 2ull * rows * static_cast<uint64_t>(n) * static_cast<uint64_t>(k);
}

// ---------------------------------------------------------------------------
// fp32 SIMT GEMM (exact fp32 products, FFMA accumulate in ascending k; the
// multistage kernel below may run K slices, each such a chain, summed in order): BMxBN
// tile per 256-thread block, TMxTN outputs per thread, K panels of 16
// double-buffered in shared memory with register-staged prefetch (the next
// panel's global loads are in flight while the current one is multiplied).
// A is stored k-major in smem with a 4-float pad so the transposing stores are
// conflict-free. 128x128 tiles (8x8 per thread) for large problems, 64x64
// (4x4) when the 128 grid would leave SMs idle (C1: 1024^3 = 64 vs 256 tiles).

constexpr int SG_K = 16;  // k per smem panel: 16 keeps a panel of FFMA work ahead of the global-load latency

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(256) gemm_f32_simt_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                            float* __restrict__ Cc, int64_t M, int64_t N, int64_t K) {
  static_assert((BM / TM) * (BN / TN) == 256, "256 threads");
  constexpr int AP = BM + 4;                      // padded k-row of the A panel
  constexpr int A_PER = BM * SG_K / 256, B_PER = BN * SG_K / 256;
  constexpr int RSTEP = BM * 4 / TM, CSTEP = BN * 4 / TN;  // distance between a thread's 4-groups
  __shared__ __align__(16) float sa[2][SG_K][AP];
  __shared__ __align__(16) float sb[2][SG_K][BN];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int64_t row0 = blockIdx.y * (int64_t)BM, col0 = blockIdx.x * (int64_t)BN;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  float ra[A_PER], rb[B_PER];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      int idx = tid + e * 256;
      int64_t gr = row0 + idx / SG_K, gk = k0 + idx % SG_K;
      ra[e] = (gr < M && gk < K) ? A[gr * K + gk] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      int idx = tid + e * 256;
      int64_t gk = k0 + idx / BN, gc = col0 + idx % BN;
      rb[e] = (gk < K && gc < N) ? B[gk * N + gc] : 0.f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      int idx = tid + e * 256;
      sa[buf][idx % SG_K][idx / SG_K] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      int idx = tid + e * 256;
      sb[buf][idx / BN][idx % BN] = rb[e];
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < K; k0 += SG_K) {
    const bool more = k0 + SG_K < K;
    if (more) fetch(k0 + SG_K);
#pragma unroll
    for (int kk = 0; kk < SG_K; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int g = 0; g < TM / 4; ++g) {
        float4 v = *reinterpret_cast<const float4*>(&sa[buf][kk][g * RSTEP + ty * 4]);
        av[g * 4] = v.x; av[g * 4 + 1] = v.y; av[g * 4 + 2] = v.z; av[g * 4 + 3] = v.w;
      }
#pragma unroll
      for (int g = 0; g < TN / 4; ++g) {
        float4 v = *reinterpret_cast<const float4*>(&sb[buf][kk][g * CSTEP + tx * 4]);
        bv[g * 4] = v.x; bv[g * 4 + 1] = v.y; bv[g * 4 + 2] = v.z; bv[g * 4 + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t r = row0 + (i / 4) * RSTEP + ty * 4 + i % 4;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int64_t cc = col0 + (j / 4) * CSTEP + tx * 4 + j % 4;
      if (cc < N) Cc[r * N + cc] = acc[i][j];
    }
  }
}

// Multistage variant (N % 4 == 0): A is first transposed to At (K x rows,
// pitch padded to 4 floats) so both operand tiles are contiguous k-rows, copied
// with 16-byte cp.async (zero-filled past the edges) into a 3-stage ring; the
// register tile and the FFMA chain per output are those of gemm_f32_simt_kernel
// (k ascending), so results are bit-identical to it with one K slice.
constexpr int MS_K = 16, MS_STAGES = 3;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ptx::smem_u32(smem)), "l"(gmem),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(256) gemm_f32_ms_kernel(const float* __restrict__ At, int64_t lda,
                                                          const float* __restrict__ B, float* __restrict__ Cc,
                                                          int64_t M, int64_t N, int64_t K) {
  // gridDim.z > 1: K slice blockIdx.z (k-tiles [nkt z / Z, nkt (z+1) / Z)) into C + z M N
  static_assert((BM / TM) * (BN / TN) == 256, "256 threads");
  constexpr int RSTEP = BM * 4 / TM, CSTEP = BN * 4 / TN;
  constexpr int A_CH = MS_K * BM / 4, B_CH = MS_K * BN / 4;  // 16-byte chunks per stage
  extern __shared__ __align__(16) float ms_smem[];
  float* sa = ms_smem;                          // [stage][MS_K][BM]
  float* sb = ms_smem + MS_STAGES * MS_K * BM;  // [stage][MS_K][BN]
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int64_t row0 = blockIdx.y * (int64_t)BM, col0 = blockIdx.x * (int64_t)BN;
  const int nkt = static_cast<int>((K + MS_K - 1) / MS_K);
  const int kt0 = static_cast<int>(static_cast<int64_t>(nkt) * blockIdx.z / gridDim.z);
  const int nk = static_cast<int>(static_cast<int64_t>(nkt) * (blockIdx.z + 1) / gridDim.z) - kt0;
  Cc += static_cast<int64_t>(blockIdx.z) * M * N;
  auto issue = [&](int stage, int kt) {
    kt += kt0;
    const int64_t k0 = static_cast<int64_t>(kt) * MS_K;
    for (int ch = tid; ch < A_CH; ch += 256) {
      const int kk = ch / (BM / 4), m4 = (ch % (BM / 4)) * 4;
      const int64_t gk = k0 + kk, gm = row0 + m4;
      const int64_t rem = M - gm;
      const int bytes = gk < K ? static_cast<int>(rem >= 4 ? 4 : (rem > 0 ? rem : 0)) * 4 : 0;
      cp_async16(sa + (stage * MS_K + kk) * BM + m4, bytes ? At + gk * lda + gm : At, bytes);
    }
    for (int ch = tid; ch < B_CH; ch += 256) {
      const int kk = ch / (BN / 4), n4 = (ch % (BN / 4)) * 4;
      const int64_t gk = k0 + kk, gn = col0 + n4;
      const int64_t rem = N - gn;
      const int bytes = gk < K ? static_cast<int>(rem >= 4 ? 4 : (rem > 0 ? rem : 0)) * 4 : 0;
      cp_async16(sb + (stage * MS_K + kk) * BN + n4, bytes ? B + gk * N + gn : B, bytes);
    }
  };
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  ptx::grid_dep_wait();  // At is the previous launch's output (PDL)
  ptx::grid_dep_launch();
#pragma unroll
  for (int st = 0; st < MS_STAGES - 1; ++st) {
    if (st < nk) issue(st, st);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<MS_STAGES - 2>();
    __syncthreads();
    const int nxt = kt + MS_STAGES - 1;
    if (nxt < nk) issue(nxt % MS_STAGES, nxt);
    cp_async_commit();
    const float* a = sa + (kt % MS_STAGES) * MS_K * BM;
    const float* b = sb + (kt % MS_STAGES) * MS_K * BN;
#pragma unroll
    for (int kk = 0; kk < MS_K; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int g = 0; g < TM / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(a + kk * BM + g * RSTEP + ty * 4);
        av[g * 4] = v.x; av[g * 4 + 1] = v.y; av[g * 4 + 2] = v.z; av[g * 4 + 3] = v.w;
      }
#pragma unroll
      for (int g = 0; g < TN / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(b + kk * BN + g * CSTEP + tx * 4);
        bv[g * 4] = v.x; bv[g * 4 + 1] = v.y; bv[g * 4 + 2] = v.z; bv[g * 4 + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t r = row0 + (i / 4) * RSTEP + ty * 4 + i % 4;
    if (r >= M) continue;
#pragma unroll
    for (int g = 0; g < TN / 4; ++g) {
      const int64_t cc = col0 + g * CSTEP + tx * 4;
      if (cc + 3 < N) {
        *reinterpret_cast<float4*>(Cc + r * N + cc) =
            make_float4(acc[i][g * 4], acc[i][g * 4 + 1], acc[i][g * 4 + 2], acc[i][g * 4 + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (cc + j < N) Cc[r * N + cc + j] = acc[i][g * 4 + j];
      }
    }
  }
}

template <int BM, int BN, int TM, int TN>
void run_gemm_f32_ms(const float* At, int64_t lda, const float* b, float* cp, int64_t r, int64_t n, int64_t k,
                     cudaStream_t stream, int ksplit = 1, bool pdl = false) {
  const size_t smem = static_cast<size_t>(MS_STAGES) * MS_K * (BM + BN) * 4;
  auto kern = gemm_f32_ms_kernel<BM, BN, TM, TN>;
  HCL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  dim3 grid(static_cast<unsigned>(ceil_div(n, BN)), static_cast<unsigned>(ceil_div(r, BM)),
            static_cast<unsigned>(ksplit));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  HCL_CUDA(cudaLaunchKernelEx(&cfg, kern, At, lda, b, cp, r, n, k));
  HCL_LAUNCHED();
}

uint64_t launch_gemm_f32(LaunchCtx& c) {
  int64_t m = scalar_arg(c, 3, "gemm_f32 M");
  int64_t k = scalar_arg(c, 4, "gemm_f32 K");
  int64_t n = scalar_arg(c, 5, "gemm_f32 N");
  if (m < 1 || k < 1 || n < 1) fail(ErrorCode::argument, "gemm_f32: dimensions must be >= 1");
  const BufView& A = buffer_arg(c, 0, "gemm_f32 A");
  const BufView& B = buffer_arg(c, 1, "gemm_f32 B");
  const BufView& Cb = buffer_arg(c, 2, "gemm_f32 C");
  if (c.whole && A.bytes != static_cast<uint64_t>(m * k) * 4)
    fail(ErrorCode::argument, "gemm_f32: A size != M*K");
  if (B.first_byte != 0 || B.bytes != static_cast<uint64_t>(k * n) * 4)
    fail(ErrorCode::argument, "gemm_f32: B size != K*N");
  uint64_t lo, rows;
  sub_range(c, static_cast<uint64_t>(m), lo, rows, "gemm_f32");
  const float* a = at_byte<const float>(A, lo * k * 4, rows * k * 4, "gemm_f32 A");
  float* cp = at_byte<float>(Cb, lo * n * 4, rows * n * 4, "gemm_f32 C");
  if (rows == 0) return 0;
  const float* bp = reinterpret_cast<const float*>(B.ptr);
  const int64_t r = static_cast<int64_t>(rows);
  // tile: 128x128 (8x8 per thread) when the grid fills the GPU twice, else
  // 64x64 (4x4); 128x64 (8x4) is available; HCL_SIMT_TILE=0|1|2 forces one
  // (every shape computes each output with the same FMA chains, so results
  // are identical for a given K split)
  const int64_t sms = c.sm_count;
  int tile = env_int("HCL_SIMT_TILE", -1);
  if (tile < 0 || tile > 2)
    tile = ceil_div(r, 128) * ceil_div(n, 128) >= 2 * sms ? 0 : 2;  // without a K split: 64x64 at 1024^3 (24.5 TF)
  if (n % 4 == 0 && env_int("HCL_SIMT_MS", 1)) {
    // multistage path: At = A^T (K x rows, pitch rounded up to 4 floats).
    // K split when the 128x128 grid is small: slices of the k-tiles, each one FMA
    // chain in ascending k, summed in slice order by ksplit_reduce_kernel; a
    // function of M, N and K only, so row partitions agree. 128x128 tiles then
    // fill the GPU. HCL_SIMT_KSPLIT overrides (1 = one chain per output).
    const int64_t t128 = ceil_div(m, 128) * ceil_div(n, 128), nkt = ceil_div(k, MS_K);
    const int64_t ks_default = std::max<int64_t>(1, std::min<int64_t>({8, 2 * sms / t128, nkt / 4}));
    const int ksplit = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(env_int("HCL_SIMT_KSPLIT", static_cast<int>(ks_default)), nkt)));
    if (ksplit > 1 && env_int("HCL_SIMT_TILE", -1) < 0) tile = 0;
    const int64_t lda = (r + 3) / 4 * 4;
    const size_t at_floats = static_cast<size_t>(k * lda + 3) & ~size_t(3);  // the workspace stays 16-byte aligned
    float* at = static_cast<float*>(
        c.scratch(c.dev, (at_floats + (ksplit > 1 ? static_cast<size_t>(ksplit) * r * n : 0)) * 4));
    float* out = ksplit > 1 ? at + at_floats : cp;
    dim3 tg(static_cast<unsigned>(ceil_div(k, 32)), static_cast<unsigned>(ceil_div(r, 32)));
    transpose_pitched_kernel<<<tg, dim3(32, 8), 0, c.stream>>>(a, at, r, k, lda);
    HCL_LAUNCHED();
    // transpose -> GEMM -> reduction as programmatic dependent launches (HCL_GEMM_PDL)
    const bool pdl = env_int("HCL_GEMM_PDL", 1) != 0;
    if (tile == 0) run_gemm_f32_ms<128, 128, 8, 8>(at, lda, bp, out, r, n, k, c.stream, ksplit, pdl);
    else if (tile == 1) run_gemm_f32_ms<128, 64, 8, 4>(at, lda, bp, out, r, n, k, c.stream, ksplit, pdl);
    else run_gemm_f32_ms<64, 64, 4, 4>(at, lda, bp, out, r, n, k, c.stream, ksplit, pdl);
    if (ksplit > 1) {
      const int64_t n4 = r * n / 4;
      const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(n4, 256), 8LL * c.sm_count));
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(256);
      cfg.stream = c.stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl ? 1 : 0;
      HCL_CUDA(cudaLaunchKernelEx(&cfg, ksplit_reduce_kernel, reinterpret_cast<const float4*>(out),
                                  reinterpret_cast<float4*>(cp), n4, ksplit));
      HCL_LAUNCHED();
    }
    return 2ull * rows * static_cast<uint64_t>(n) * static_cast<uint64_t>(k);
  }
  if (tile == 0) {
    dim3 grid(static_cast<unsigned>(ceil_div(n, 128)), static_cast<unsigned>(ceil_div(r, 128)));
    gemm_f32_simt_kernel<128, 128, 8, 8><<<grid, 256, 0, c.stream>>>(a, bp, cp, r, n, k);
  } else if (tile == 1) {
    dim3 grid(static_cast<unsigned>(ceil_div(n, 64)), static_cast<unsigned>(ceil_div(r, 128)));
    gemm_f32_simt_kernel<128, 64, 8, 4><<<grid, 256, 0, c.stream>>>(a, bp, cp, r, n, k);
  } else {
    dim3 grid(static_cast<unsigned>(ceil_div(n, 64)), static_cast<unsigned>(ceil_div(r, 64)));
    gemm_f32_simt_kernel<64, 64, 4, 4><<<grid, 256, 0, c.stream>>>(a, bp, cp, r, n, k);
  }
  HCL_LAUNCHED();
  return 2ull * rows * static_cast<uint64_t>(n) * static_cast<uint64_t>(k);
}

uint64_t rows_gemm(const int64_t* s, uint32_t) { return static_cast<uint64_t>(s[3]); }
uint64_t rowbytes_gemm_bf16(const int64_t* s, uint32_t, uint32_t i) {
  return i == 0 ? static_cast<uint64_t>(s[4]) * 2 : static_cast<uint64_t>(s[5]) * (s[6] ? 4 : 2);
}
uint64_t rowbytes_gemm_f32(const int64_t* s, uint32_t, uint32_t i) {
  return static_cast<uint64_t>(i == 0 ? s[4] : s[5]) * 4;
}

}  // namespace

// shared with the implicit-GEMM conv (k_conv.cu)
CUtensorMap make_tmap_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                              uint32_t box_outer) {
  return make_tmap(base, false, inner, outer, row_bytes, box_inner, box_outer);
}

// 4D bf16 tensor (dims[0] innermost), SWIZZLE_128B box; strides[i] = byte
// pitch of dimension i+1. Out-of-bounds box elements are skipped by stores.
CUtensorMap make_tmap_4d_bf16(const void* base, const uint64_t dims[4], const uint64_t strides[3],
                              const uint32_t box[4]) {
  CUtensorMap m;
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t s[3] = {strides[0], strides[1], strides[2]};
  cuuint32_t b[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t e[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, s, b, e,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(ErrorCode::argument, "cuTensorMapEncodeTiled (4D) failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

void register_gemm(std::vector<KernelDef>& r) {
  constexpr uint8_t S = HCL_ARG_SCALAR, I = HCL_ARG_IN, O = HCL_ARG_OUT;
  constexpr uint8_t N = HCL_PART_NONE, P = HCL_PART_REPLICATE, X = HCL_PART_SPLIT_ROWS;
  r.push_back({"b200", "gemm_bf16", {I, I, O, S, S, S, S}, {X, P, X, N, N, N, N}, launch_gemm_tc<false>,
               rowbytes_gemm_bf16, rows_gemm, true});
  r.push_back({"b200", "gemm_tf32", {I, I, O, S, S, S}, {X, P, X, N, N, N}, launch_gemm_tc<true>,
               rowbytes_gemm_f32, rows_gemm, true});
  r.push_back({"b200", "gemm_f32", {I, I, O, S, S, S}, {X, P, X, N, N, N}, launch_gemm_f32, rowbytes_gemm_f32,
               rows_gemm, true});
  r.push_back({"b200", "gemm_f32x3", {I, I, O, S, S, S}, {X, P, X, N, N, N}, launch_gemm_f32x3, rowbytes_gemm_f32,
               rows_gemm, true});
}

}  // namespace hcl
