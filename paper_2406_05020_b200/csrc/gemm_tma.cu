// FP64 tensor-core GEMM for the Kronecker mode products:
// TMA-fed, mbarrier-pipelined, warp-specialised DMMA kernel for sm_100a.
//
//   C[b] = alpha * sum_seg A_seg[b] B_seg[b] + beta * C[b]     (two batch levels
//   b = (b1, b2), each operand with its own strides or broadcast per level)
//
// FP64 on sm_100a has no tcgen05 kind: the tensor-core instruction is
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, 256 FMA, one per 16 cycles per SM
// sub-partition at the measured 37 TF/s).  What this kernel adds over an
// sm80-style cp.async GEMM is the Blackwell data movement:
//   * one producer warp issues cp.async.bulk.tensor (TMA, SASS UTMALDG) for
//     every stage of a STAGES-deep ring; consumers wait on a per-stage "full"
//     mbarrier (transaction-count completion) and release the slot through a
//     per-stage "empty" mbarrier — no CTA-wide __syncthreads in the main loop;
//   * tiles land 128-byte swizzled (CU_TENSOR_MAP_SWIZZLE_128B): a K-contiguous
//     operand tile is [rows][16 doubles], a 16-byte chunk c of row r stored at
//     chunk c ^ (r & 7), so each DMMA fragment load (8 rows x 4 k) is exactly
//     2 shared-memory wavefronts (the minimum for 256 bytes);
//   * an N-contiguous (row-major) B operand is loaded as [N/16][16 k][16 n]
//     swizzled boxes and each k4 step of the DMMA contracts k = {s, s+4, s+8,
//     s+12} instead of {4s..4s+3} (a K permutation inside the 16-block, exact:
//     the same permutation is applied to A), which puts the four k rows of a B
//     fragment in two different 64-byte bank halves: again 2 wavefronts.
//   * out-of-range rows/columns/k are zero-filled by the TMA unit (no
//     predication in the main loop).
// Requirements (else the caller uses the generic kernels in gemm.cu): 16-byte
// aligned base pointers, even element strides, a_cs == c_cs == 1, b_cs == 1 or
// b_rs == 1, at most two batch levels (the extra term: one).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace gpfvm {

namespace {

struct TmaArgs {
  int M, N, batch;
  int batch1;  // size of batch level 1 (b = b1 + batch1 * b2)
  int kt_seg;  // 16-wide k tiles per segment
  int kt_extra;  // k tiles of the extra term (tmA2 / tmB2), after the segments
  int nseg;
  int a_bc1, a_bc2, b_bc1, b_bc2;  // operand shared along batch level 1 / 2
  int dbg;               // debugging switches (GPFVM_TMA_DBG bits)
  double alpha, beta;
  double* C;
  int64_t c_rs, c_b1, c_b2;
};

// ---- PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int STAGES>
struct TmaSmem {
  static constexpr int A_BYTES = BM * 128;  // [BM][16] doubles
  static constexpr int B_BYTES = BN * 128;  // [BN][16] or [BN/16][16][16]
  static constexpr size_t raw_bytes = 1024 + (size_t)STAGES * (A_BYTES + B_BYTES) + 2 * STAGES * sizeof(uint64_t);
  // Shared memory asked for at launch: the ring, or at least `floor_kb` KB.  A
  // floor above half of the SM's 227 KB keeps ONE CTA of this kernel per SM;
  // that was the first mitigation of the wrong-tile failure of DESIGN.md 4.4,
  // whose root cause (a missing fence.proxy.async, fixed in the consumer loop)
  // does not need it.  GPFVM_TMA_SMEM_FLOOR_KB sets it (default 0: the small
  // tile variants run 2 CTAs per SM).
  static size_t bytes_at_launch() {
    static const size_t floor_kb = getenv("GPFVM_TMA_SMEM_FLOOR_KB") ? (size_t)atoi(getenv("GPFVM_TMA_SMEM_FLOOR_KB")) : 0;
    return std::max(raw_bytes, floor_kb * 1024);
  }
};

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool BROW, int MINB>
__global__ void __launch_bounds__((WARPS_M * WARPS_N + 1) * 32, MINB)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2, TmaArgs g) {
  constexpr int NCW = WARPS_M * WARPS_N;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int TM = WM / 8, TN = WN / 8;
  static_assert(!BROW || WN % 16 == 0, "row-major B: warp tile must cover whole 16-column blocks");
  using L = TmaSmem<BM, BN, STAGES>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sA = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* sB = sA + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * L::B_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int KTm = g.kt_seg * g.nseg, KT = KTm + g.kt_extra;
  const int tiles_n = (g.N + BN - 1) / BN, tiles_m = (g.M + BM - 1) / BM;
  const int64_t ntiles = (int64_t)tiles_n * tiles_m * g.batch;

  if (warp == NCW) {
    // ---- TMA producer: runs ahead across tile boundaries (persistent CTA) ----
    if (lane == 0) {
      if (g.dbg & 4) {
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      }
      if (!(g.dbg & 1)) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      }
      if (g.dbg & 2) asm volatile("fence.proxy.async.global;\n" ::: "memory");
      int it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tn = (int)(t % tiles_n);
        const int64_t r = t / tiles_n;
        const int tm = (int)(r % tiles_m), b = (int)(r / tiles_m);
        const int m0 = tm * BM, n0 = tn * BN;
        const int b1 = b % g.batch1, b2 = b / g.batch1;
        const int a1 = g.a_bc1 ? 0 : b1, a2 = g.a_bc2 ? 0 : b2, bq1 = g.b_bc1 ? 0 : b1, bq2 = g.b_bc2 ? 0 : b2;
        for (int kt = 0; kt < KT; kt++, it++) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
          if (kt >= KTm) {  // extra low-rank term (same layout class, own maps)
            const int k0 = (kt - KTm) * 16;
            tma_load_5d(sA + s * L::A_BYTES, &tmA2, k0, m0, 0, b, 0, &full[s]);
            tma_load_5d(sB + s * L::B_BYTES, &tmB2, k0, n0, 0, b, 0, &full[s]);
            continue;
          }
          const int seg = kt / g.kt_seg, k0 = (kt - seg * g.kt_seg) * 16;
          tma_load_5d(sA + s * L::A_BYTES, &tmA, k0, m0, seg, a1, a2, &full[s]);
          if (BROW) {
#pragma unroll
            for (int j = 0; j < BN / 16; j++)
              tma_load_5d(sB + s * L::B_BYTES + j * 2048, &tmB, n0 + 16 * j, k0, seg, bq1, bq2, &full[s]);
          } else {
            tma_load_5d(sB + s * L::B_BYTES, &tmB, k0, n0, seg, bq1, bq2, &full[s]);
          }
        }
      }
    }
    return;
  }

  // ---- DMMA consumers ----
  const int wm0 = (warp / WARPS_N) * WM, wn0 = (warp % WARPS_N) * WN;
  const int g8 = lane >> 2, q = lane & 3;
  // per-lane byte offsets inside a stage (swizzle: chunk ^ (row & 7); every
  // fragment row is wm0 + 8i + g8, so row & 7 == g8)
  uint32_t a_off[4], b_off[4];
#pragma unroll
  for (int st = 0; st < 4; st++) {
    if (BROW) {
      const int k = st + 4 * q;  // permuted k set {st, st+4, st+8, st+12}
      a_off[st] = (uint32_t)((wm0 + g8) * 128 + (((k >> 1) ^ g8) << 4) + ((k & 1) << 3));
      // B: [n/16][k][16 n], n = wn0 + 8j + g8 (wn0 % 16 == 0): block wn0/16 + j/2,
      // in-block column 8(j&1) + g8, chunk ((n & 15) >> 1) ^ (k & 7)
      b_off[st] = (uint32_t)((wn0 >> 4) * 2048 + k * 128 + (((g8 >> 1) ^ (k & 7)) << 4) + ((g8 & 1) << 3));
    } else {
      const int k = 4 * st + q;
      a_off[st] = (uint32_t)((wm0 + g8) * 128 + (((k >> 1) ^ g8) << 4) + ((k & 1) << 3));
      b_off[st] = (uint32_t)((wn0 + g8) * 128 + (((k >> 1) ^ g8) << 4) + ((k & 1) << 3));
    }
  }

  // odd j: column + 8 flips bit 2 of the swizzled chunk; that bit is (k & 4) >> 2
  // = q & 1 for every step, so the byte offset moves by -64 or +64
  const int b_odd = (q & 1) ? -64 : 64;
  const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tn = (int)(t % tiles_n);
    const int64_t r = t / tiles_n;
    const int tm = (int)(r % tiles_m), b = (int)(r / tiles_m);
    const int m0 = tm * BM, n0 = tn * BN;
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; kt++, it++) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const uint32_t as = sA0 + s * L::A_BYTES, bs = sB0 + s * L::B_BYTES;
#pragma unroll
      for (int st = 0; st < 4; st++) {
        double af[TM], bf[TN];
#pragma unroll
        for (int i = 0; i < TM; i++) af[i] = lds64(as + a_off[st] + i * 8 * 128);
#pragma unroll
        for (int j = 0; j < TN; j++) {
          if (BROW)
            bf[j] = lds64(bs + b_off[st] + ((j & 1) ? b_odd : 0) + (j >> 1) * 2048);
          else
            bf[j] = lds64(bs + b_off[st] + j * 8 * 128);
        }
#pragma unroll
        for (int i = 0; i < TM; i++)
#pragma unroll
          for (int j = 0; j < TN; j++) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      // The fragment loads above are generic-proxy reads of the stage; the TMA
      // refill is an async-proxy write.  The mbarrier release alone does not
      // order accesses across the two proxies: without this fence the refill
      // could land before a queued fragment load had read the old tile (whole
      // warp tiles wrong, only under shared-memory pressure from co-resident
      // CTAs, tools/gemm_race.cu).
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---- epilogue: C = alpha acc + beta C (two consecutive doubles per lane);
    // the producer is already filling the ring with the next tile ----
    double* C = g.C + (int64_t)(b % g.batch1) * g.c_b1 + (int64_t)(b / g.batch1) * g.c_b2;
#pragma unroll
    for (int i = 0; i < TM; i++) {
      const int row = m0 + wm0 + i * 8 + g8;
      if (row >= g.M) continue;
      double* crow = C + (int64_t)row * g.c_rs + n0 + wn0 + 2 * q;
      const int col0 = n0 + wn0 + 2 * q;
      // beta != 0: all the row's old values first (TN independent 16-byte loads
      // in flight per lane instead of a load -> fma -> store chain per pair)
      double2 old[TN];
      if (g.beta != 0.0) {
#pragma unroll
        for (int j = 0; j < TN; j++)
          old[j] = (col0 + j * 8 + 1 < g.N) ? *reinterpret_cast<const double2*>(crow + j * 8) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < TN; j++) {
        const int col = col0 + j * 8;
        double* cp = crow + j * 8;
        double v0 = g.alpha * acc[i][j][0], v1 = g.alpha * acc[i][j][1];
        if (col + 1 < g.N) {
          if (g.beta != 0.0) {
            v0 += g.beta * old[j].x;
            v1 += g.beta * old[j].y;
          }
          *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
        } else if (col < g.N) {
          if (g.beta != 0.0) v0 += g.beta * cp[0];
          cp[0] = v0;
        }
      }
    }
  }
}

// ---- host side -------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 5D tiled map over doubles: dims (d0 contiguous, d1, d2, d3, d4) with element strides s1..s4
bool make_map(CUtensorMap* m, const double* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint64_t d4,
              int64_t s1, int64_t s2, int64_t s3, int64_t s4, uint32_t b0, uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return false;
  // size-1 dims: any legal stride
  if (d2 == 1) s2 = std::max<int64_t>(s1, 2);
  if (d3 == 1) s3 = std::max<int64_t>(s2, 2);
  if (d4 == 1) s4 = std::max<int64_t>(s3, 2);
  if (s2 <= 0 || s3 <= 0 || s4 <= 0) return false;
  cuuint64_t dims[5] = {d0, d1, d2, d3, d4};
  cuuint64_t strides[4] = {(cuuint64_t)s1 * 8, (cuuint64_t)s2 * 8, (cuuint64_t)s3 * 8, (cuuint64_t)s4 * 8};
  cuuint32_t box[5] = {b0, b1, 1, 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool BROW, int MINB>
void launch_tma(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& ma2, const CUtensorMap& mb2,
                const TmaArgs& a, int batch, cudaStream_t s) {
  using L = TmaSmem<BM, BN, STAGES>;
  auto kern = dgemm_tma_kernel<BM, BN, WARPS_M, WARPS_N, STAGES, BROW, MINB>;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    GPFVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes_at_launch()));
    if (getenv("GPFVM_CARVEOUT_TMA"))
      GPFVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(getenv("GPFVM_CARVEOUT_TMA"))));
    configured_dev = dev;
  }
  static int sms = 0, per_sm = 0;
  if (sms == 0) {
    GPFVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GPFVM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (WARPS_M * WARPS_N + 1) * 32, L::bytes_at_launch()));
    per_sm = std::max(per_sm, 1);
  }
  const int64_t tiles = (int64_t)((a.N + BN - 1) / BN) * ((a.M + BM - 1) / BM) * batch;
  // persistent (one CTA per resident slot, the producer runs ahead across
  // tiles) unless GPFVM_TMA_NONPERSIST: one CTA per tile, which lets the light
  // IC/BC branches of the matvec graph interleave at CTA granularity
  static const bool nonpersist = getenv("GPFVM_TMA_NONPERSIST") != nullptr;
  const int grid = nonpersist ? (int)std::min<int64_t>(tiles, 1 << 30) : (int)std::min<int64_t>(tiles, (int64_t)sms * per_sm);
  kern<<<grid, (WARPS_M * WARPS_N + 1) * 32, L::bytes_at_launch(), s>>>(ma, mb, ma2, mb2, a);
  count_launch();
  check_launch("dgemm_tma_kernel");
}

// CTA tile BM x BN, WMr x WNr consumer warps, ST stages, MINB CTAs per SM
template <int BM_, int BN_, int WM_, int WN_, int ST_, int MINB_>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, WMr = WM_, WNr = WN_, ST = ST_, MINB = MINB_;
};
// every variant: 8 consumer warps, one CTA per SM (see TmaSmem::bytes)
using V0 = TileCfg<128, 64, 4, 2, 6, 1>;   // 32x32 warp tiles
using V1 = TileCfg<64, 64, 4, 2, 6, 1>;    // 16x32 warp tiles (small grids)
using V2 = TileCfg<128, 64, 2, 2, 4, 2>;   // 64x32 warp tiles, 4 consumer warps, 2 CTAs per SM
using V3 = TileCfg<128, 128, 2, 4, 4, 1>;  // 64x32 warp tiles
using V4 = TileCfg<128, 128, 4, 2, 4, 1>;  // 32x64 warp tiles
using V5 = TileCfg<256, 64, 4, 2, 3, 1>;   // 64x32 warp tiles
// 96-wide tiles for the half sizes of 192-cell dimensions (config 4 after the
// parity split: M or N = 96 wastes a quarter of a 128-wide tile)
using W0 = TileCfg<96, 192, 3, 4, 4, 1>;   // 32x48 warp tiles, 12 consumer warps: one M = 96, N = 192 batch entry per tile
using W1 = TileCfg<128, 96, 4, 2, 4, 1>;   // 32x48 warp tiles
using W2 = TileCfg<96, 128, 3, 4, 4, 1>;   // 32x32 warp tiles, 12 consumer warps

#ifdef GPFVM_TMA_SHARED_SMS  // extra shapes for tools/gemm_race.cu
using V6 = TileCfg<64, 64, 2, 2, 4, 2>;    // round-2 start: 32x32 warp tiles, 4 stages
using V7 = TileCfg<64, 64, 4, 2, 4, 1>;    // V1 with 4 stages
using V8 = TileCfg<64, 64, 2, 2, 6, 2>;    // 32x32 warp tiles, 6 stages
using V9 = TileCfg<128, 64, 2, 2, 4, 2>;   // V2 with launch bounds for 2 CTAs per SM
#endif

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool ev(int64_t v) { return (v & 1) == 0; }

}  // namespace

static bool try_tma_gemm_impl(const Gemm& g, cudaStream_t s) {
  static const bool off = getenv("GPFVM_NO_TMA") != nullptr;
  if (off) return false;
  if (g.batch3 != 1 || (g.K2 > 0 && g.batch2 != 1)) return false;
  if (g.a_cs != 1 || g.c_cs != 1) return false;
  const bool brow = (g.b_cs == 1);
  if (!brow && g.b_rs != 1) return false;
  if (g.M < 32 || g.N < 32 || g.K * g.nseg < 16) return false;
  if (!al16(g.A) || !al16(g.B) || !al16(g.C)) return false;
  const int64_t b_ld = brow ? g.b_rs : g.b_cs;
  if (!ev(g.a_rs) || !ev(b_ld) || !ev(g.c_rs) || !ev(g.a_sg) || !ev(g.b_sg) || !ev(g.a_b1) || !ev(g.b_b1) ||
      !ev(g.c_b1) || !ev(g.a_b2) || !ev(g.b_b2) || !ev(g.c_b2))
    return false;
  const int batch = g.batch1 * g.batch2;
  if ((int64_t)g.batch1 * g.batch2 > (1 << 30)) return false;
  if (g.K2 > 0 && (brow || !al16(g.A2) || !al16(g.B2) || !ev(g.a2_rs) || !ev(g.b2_rs) || !ev(g.a2_b1) ||
                   !ev(g.b2_b1)))
    return false;
  const bool a_bc1 = (g.a_b1 == 0) || g.batch1 == 1, b_bc1 = (g.b_b1 == 0) || g.batch1 == 1;
  const bool a_bc2 = (g.a_b2 == 0) || g.batch2 == 1, b_bc2 = (g.b_b2 == 0) || g.batch2 == 1;
  CUtensorMap ma, mb, ma2, mb2;
  memset(&ma2, 0, sizeof(ma2));
  memset(&mb2, 0, sizeof(mb2));
  TmaArgs a;
  a.kt_extra = g.K2 > 0 ? (g.K2 + 15) / 16 : 0;
  a.M = g.M; a.N = g.N; a.batch = batch; a.batch1 = g.batch1;
  a.kt_seg = (g.K + 15) / 16;
  a.nseg = g.nseg;
  a.a_bc1 = a_bc1; a.a_bc2 = a_bc2; a.b_bc1 = b_bc1; a.b_bc2 = b_bc2;
  a.alpha = g.alpha; a.beta = g.beta;
  static const int dbgbits = getenv("GPFVM_TMA_DBG") ? atoi(getenv("GPFVM_TMA_DBG")) : 0;
  a.dbg = dbgbits;
  a.C = g.C; a.c_rs = g.c_rs; a.c_b1 = g.c_b1; a.c_b2 = g.c_b2;
  static const int variant = getenv("GPFVM_TMA_VARIANT") ? atoi(getenv("GPFVM_TMA_VARIANT")) : -1;
  auto run = [&](auto cfg) -> bool {
    using Cfg = decltype(cfg);
    if (!make_map(&ma, g.A, g.K, g.M, g.nseg, a_bc1 ? 1 : g.batch1, a_bc2 ? 1 : g.batch2, g.a_rs, g.a_sg, g.a_b1,
                  g.a_b2, 16, Cfg::BM))
      return false;
    if (brow) {
      if (!make_map(&mb, g.B, g.N, g.K, g.nseg, b_bc1 ? 1 : g.batch1, b_bc2 ? 1 : g.batch2, g.b_rs, g.b_sg, g.b_b1,
                    g.b_b2, 16, 16))
        return false;
      launch_tma<Cfg::BM, Cfg::BN, Cfg::WMr, Cfg::WNr, Cfg::ST, true, Cfg::MINB>(ma, mb, ma2, mb2, a, batch, s);
    } else {
      if (!make_map(&mb, g.B, g.K, g.N, g.nseg, b_bc1 ? 1 : g.batch1, b_bc2 ? 1 : g.batch2, g.b_cs, g.b_sg, g.b_b1,
                    g.b_b2, 16, Cfg::BN))
        return false;
      if (g.K2 > 0) {
        if (!make_map(&ma2, g.A2, g.K2, g.M, 1, batch, 1, g.a2_rs, 0, g.a2_b1, 0, 16, Cfg::BM)) return false;
        if (!make_map(&mb2, g.B2, g.K2, g.N, 1, batch, 1, g.b2_rs, 0, g.b2_b1, 0, 16, Cfg::BN)) return false;
      }
      launch_tma<Cfg::BM, Cfg::BN, Cfg::WMr, Cfg::WNr, Cfg::ST, false, Cfg::MINB>(ma, mb, ma2, mb2, a, batch, s);
    }
    return true;
  };
  switch (variant) {
    case 0: return run(V0{});
    case 1: return run(V1{});
    case 2: return run(V2{});
    case 3: return run(V3{});
    case 4: return run(V4{});
    case 5: return run(V5{});
    case 10: return run(W0{});
    case 11: return run(W1{});
    case 12: return run(W2{});
#ifdef GPFVM_TMA_SHARED_SMS
    case 6: return run(V6{});
    case 7: return run(V7{});
    case 8: return run(V8{});
    case 9: return run(V9{});
#endif
    default: break;
  }
  // Tile choice: estimated time = waves x tile work / relative DMMA efficiency
  // of the tile shape (128x128 with 32x64 warp tiles 1.0, 128x64 with 32x32
  // warp tiles 0.92, 64x64 with 16x32 warp tiles 0.8), waves = ceil(tiles / 148).
  auto cost = [&](int bm, int bn, double eff) {
    const int64_t tiles = ((g.M + bm - 1) / bm) * (int64_t)((g.N + bn - 1) / bn) * batch;
    return (double)((tiles + 147) / 148) * bm * bn / eff;
  };
  // grids that cannot fill the machine even with 64x64 tiles go to the
  // cp.async kernel's 32x32 tiles (more CTAs; these are the short IC/BC
  // coupling GEMMs that run concurrently with the PDE branch; config 2:
  // 0.68 -> 0.62 ms).  While the consumer loop lacked its proxy fence this
  // mix was what exposed the wrong tiles; GPFVM_TMA_MIN_TILES=0
  // sends every eligible GEMM here.
  static const int min_tiles = getenv("GPFVM_TMA_MIN_TILES") ? atoi(getenv("GPFVM_TMA_MIN_TILES")) : 148;
  if (((g.M + 63) / 64) * (int64_t)((g.N + 63) / 64) * batch < min_tiles) return false;
  // 128x64: 8 warps of 32x32 on one CTA per SM (V0), or 4 warps of 64x32 on two (V2, GPFVM_TMA_MID=2)
  static const int mid = getenv("GPFVM_TMA_MID") ? atoi(getenv("GPFVM_TMA_MID")) : 0;
  auto cost2 = [&](int bm, int bn, double eff) {  // two CTAs per SM
    const int64_t tiles = ((g.M + bm - 1) / bm) * (int64_t)((g.N + bn - 1) / bn) * batch;
    return (double)((tiles + 295) / 296) * bm * bn * 2 / eff;
  };
  const double c4 = cost(128, 128, 1.0), c0 = mid == 2 ? cost2(128, 64, 0.98) : cost(128, 64, 0.92),
               c1 = cost2(64, 64, 0.8);
  // 96-wide tiles only where a dimension is a multiple of 96 but not of 128
  // (they exist for the half sizes of 192-cell dimensions)
  static const bool no96 = getenv("GPFVM_TMA_NO96") != nullptr;
  const bool m96 = !no96 && g.M % 96 == 0 && g.M % 128 != 0, n96 = !no96 && g.N % 96 == 0 && g.N % 128 != 0;
  const double big = 1e300;
  const double w0 = (m96 && g.N % 192 == 0) ? cost(96, 192, 0.95) : big, w1 = n96 ? cost(128, 96, 0.97) : big,
               w2 = m96 ? cost(96, 128, 0.93) : big;
  const double best = std::min(std::min(std::min(c4, c0), std::min(c1, w0)), std::min(w1, w2));
  if (best == w0) return run(W0{});
  if (best == w1) return run(W1{});
  if (best == w2) return run(W2{});
  if (best == c4) return run(V4{});
  if (best == c0) return mid == 2 ? run(V2{}) : run(V0{});
  return run(V1{});
}

// GPFVM_TMA_VERIFY=1 (debugging): every TMA GEMM is recomputed by a naive
// kernel and compared entry by entry (synchronous; prints mismatches).
__global__ void verify_gather_kernel(const double* C, int64_t c_rs, int64_t c_b1, double* out, int M, int N) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y, b = blockIdx.z;
  if (n < N) out[((int64_t)b * M + m) * N + n] = C[b * c_b1 + (int64_t)m * c_rs + n];
}
__global__ void verify_ref_kernel(Gemm g, double* out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y, b = blockIdx.z;
  if (n >= g.N) return;
  const double* A = g.A + b * g.a_b1;
  const double* B = g.B + b * g.b_b1;
  double acc = 0.0;
  for (int sg = 0; sg < g.nseg; sg++)
    for (int k = 0; k < g.K; k++)
      acc = fma(A[sg * g.a_sg + (int64_t)m * g.a_rs + k], B[sg * g.b_sg + (int64_t)k * g.b_rs + (int64_t)n * g.b_cs], acc);
  double* o = out + ((int64_t)b * g.M + m) * g.N + n;
  *o = g.alpha * acc + (g.beta != 0.0 ? g.beta * *o : 0.0);
}

bool try_tma_gemm(const Gemm& g, cudaStream_t s) {
  static const bool verify = getenv("GPFVM_TMA_VERIFY") != nullptr;
  if (verify) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusNone && g.K2 == 0 && g.batch2 == 1 && g.batch3 == 1 && g.a_cs == 1 && g.c_cs == 1) {
      const size_t n = (size_t)g.M * g.N * g.batch1;
      double *ref = nullptr, *got = nullptr;
      GPFVM_CUDA(cudaMalloc(&ref, n * 8));
      GPFVM_CUDA(cudaMalloc(&got, n * 8));
      const dim3 gr((g.N + 127) / 128, g.M, g.batch1);
      verify_gather_kernel<<<gr, 128, 0, s>>>(g.C, g.c_rs, g.c_b1, ref, g.M, g.N);
      verify_ref_kernel<<<gr, 128, 0, s>>>(g, ref);
      const bool ok = try_tma_gemm_impl(g, s);
      verify_gather_kernel<<<gr, 128, 0, s>>>(g.C, g.c_rs, g.c_b1, got, g.M, g.N);
      std::vector<double> hr(n), hg(n);
      GPFVM_CUDA(cudaMemcpyAsync(hr.data(), ref, n * 8, cudaMemcpyDeviceToHost, s));
      GPFVM_CUDA(cudaMemcpyAsync(hg.data(), got, n * 8, cudaMemcpyDeviceToHost, s));
      GPFVM_CUDA(cudaStreamSynchronize(s));
      cudaFree(ref);
      cudaFree(got);
      if (ok) {
        double mx = 0.0, err = 0.0;
        int64_t nbad = 0, first = -1;
        for (size_t i = 0; i < n; i++) mx = std::max(mx, std::fabs(hr[i]));
        for (size_t i = 0; i < n; i++) {
          const double e = std::fabs(hr[i] - hg[i]);
          err = std::max(err, e);
          if (!(e <= 1e-13 * mx)) { nbad++; if (first < 0) first = (int64_t)i; }
        }
        fprintf(stderr, "[tma-verify] M=%d N=%d K=%d nseg=%d batch=%d a(rs=%lld b1=%lld) b(rs=%lld cs=%lld b1=%lld) c(rs=%lld b1=%lld) beta=%g: %s rel %.2e nbad %lld first %lld\n",
                g.M, g.N, g.K, g.nseg, g.batch1, (long long)g.a_rs, (long long)g.a_b1, (long long)g.b_rs, (long long)g.b_cs,
                (long long)g.b_b1, (long long)g.c_rs, (long long)g.c_b1, g.beta, nbad ? "MISMATCH" : "ok", err / (mx > 0 ? mx : 1.0),
                (long long)nbad, (long long)first);
      }
      return ok;
    }
  }
  const bool ok = try_tma_gemm_impl(g, s);
  static const bool sync_each = getenv("GPFVM_TMA_SYNC") != nullptr;
  if (ok && sync_each) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusNone) GPFVM_CUDA(cudaStreamSynchronize(s));
  }
  static const bool dbg = getenv("GPFVM_DEBUG") != nullptr;
  if (!ok && dbg && g.M >= 32 && g.N >= 32)
    fprintf(stderr, "[gemm] TMA path not taken: M=%d N=%d K=%d nseg=%d batch=%d,%d,%d\n", g.M, g.N, g.K, g.nseg,
            g.batch1, g.batch2, g.batch3);
  return ok;
}

}  // namespace gpfvm
