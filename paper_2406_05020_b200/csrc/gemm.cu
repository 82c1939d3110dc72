// FP64 tensor-core GEMM (DMMA m8n8k4) for the batched mode-n contractions of
// the Kronecker matvec.
//
//   C[b] = alpha * sum_seg A_seg[b] B_seg[b] + beta * C[b]
//   b = (b1, b2, b3) three-level batch, seg = 0..nseg-1 K-segments
//   (A_seg = A + seg*a_sg, B_seg = B + seg*b_sg): a sum of Kronecker terms
//   whose contraction inputs live side by side becomes ONE GEMM with
//   K_total = nseg*K (DESIGN.md §4.2 "K-concatenation").
// Fast path: A row-major (a_cs == 1), C row-major (c_cs == 1), B row-major
// (b_cs == 1) or column-major (b_rs == 1).  Tiles are staged through shared
// memory by a multi-stage cp.async pipeline (16-byte copies when every
// address is 16-byte aligned, else 8-byte), each warp owns a (TM*8)x(TN*8)
// sub-tile and issues TM*TN DMMA per k4 step (SASS DMMA.8x8x4 — the FP64
// tensor-core instruction of sm_100a; tcgen05 has no f64 kind).  Shared rows
// are padded so fragment loads hit each 8-byte bank pair exactly twice per
// warp (2 wavefronts, the minimum for 256 B).
#include <cstdio>
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace gpfvm {

namespace {

constexpr int BK = 16;
constexpr int APAD = 4;   // As row stride BK+4 doubles (160 B, 16-B aligned)
constexpr int BPAD = 4;   // Bs (row layout) row stride BN+4 doubles: (k*stride) mod 16 in {0,4,8,12} per half-warp

__device__ __forceinline__ void cp_async8(void* smem, const double* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const double* gmem, int valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid * 8;  // 0, 8 or 16 bytes, rest zero-filled
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, bool B_ROW>
struct SmemLayout {
  static constexpr int AS = BK + APAD;
  static constexpr int BS_ROW = BN + BPAD;
  static constexpr int A_STAGE = BM * AS;
  static constexpr int B_STAGE = B_ROW ? BK * BS_ROW : BN * AS;
};

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool B_ROW, bool V16>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32)
    dgemm_dmma_kernel(Gemm g) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int TM = WM / 8, TN = WN / 8;
  using L = SmemLayout<BM, BN, B_ROW>;
  constexpr int AS = L::AS, BS_ROW = L::BS_ROW;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * L::A_STAGE;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / WARPS_N) * WM, wn0 = (warp % WARPS_N) * WN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
  const int KT = (g.K + BK - 1) / BK;
  const int KT_all = KT * g.nseg;

  for (int64_t z = blockIdx.z; z < nbatch; z += gridDim.z) {
    const int64_t b1 = z % g.batch1, b23 = z / g.batch1;
    const int64_t b2 = b23 % g.batch2, b3 = b23 / g.batch2;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2 + b3 * g.a_b3;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2 + b3 * g.b_b3;
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2 + b3 * g.c_b3;

    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto load_tile = [&](int stage, int kt_all) {
      const int seg = kt_all / KT;
      const int k0 = (kt_all - seg * KT) * BK;
      const double* Aseg = A + seg * g.a_sg;
      const double* Bseg = B + seg * g.b_sg;
      double* as = As + stage * L::A_STAGE;
      double* bs = Bs + stage * L::B_STAGE;
      if (V16) {
#pragma unroll
        for (int i = tid; i < BM * BK / 2; i += NT) {
          int r = i / (BK / 2), c = (i % (BK / 2)) * 2;
          int gm = m0 + r, gk = k0 + c;
          int valid = (gm < g.M) ? max(0, min(2, g.K - gk)) : 0;
          const double* src = valid ? (Aseg + (int64_t)gm * g.a_rs + gk) : Aseg;
          cp_async16(as + r * AS + c, src, valid);
        }
        if (B_ROW) {
#pragma unroll
          for (int i = tid; i < BK * BN / 2; i += NT) {
            int r = i / (BN / 2), c = (i % (BN / 2)) * 2;
            int gk = k0 + r, gn = n0 + c;
            int valid = (gk < g.K) ? max(0, min(2, g.N - gn)) : 0;
            const double* src = valid ? (Bseg + (int64_t)gk * g.b_rs + gn) : Bseg;
            cp_async16(bs + r * BS_ROW + c, src, valid);
          }
        } else {
#pragma unroll
          for (int i = tid; i < BN * BK / 2; i += NT) {
            int r = i / (BK / 2), c = (i % (BK / 2)) * 2;  // r: n, c: k
            int gn = n0 + r, gk = k0 + c;
            int valid = (gn < g.N) ? max(0, min(2, g.K - gk)) : 0;
            const double* src = valid ? (Bseg + (int64_t)gn * g.b_cs + gk) : Bseg;
            cp_async16(bs + r * AS + c, src, valid);
          }
        }
      } else {
#pragma unroll
        for (int i = tid; i < BM * BK; i += NT) {
          int r = i / BK, c = i % BK;
          int gm = m0 + r, gk = k0 + c;
          bool p = (gm < g.M) && (gk < g.K);
          cp_async8(as + r * AS + c, p ? (Aseg + (int64_t)gm * g.a_rs + gk) : Aseg, p);
        }
        if (B_ROW) {
#pragma unroll
          for (int i = tid; i < BK * BN; i += NT) {
            int r = i / BN, c = i % BN;
            int gk = k0 + r, gn = n0 + c;
            bool p = (gk < g.K) && (gn < g.N);
            cp_async8(bs + r * BS_ROW + c, p ? (Bseg + (int64_t)gk * g.b_rs + gn) : Bseg, p);
          }
        } else {
#pragma unroll
          for (int i = tid; i < BK * BN; i += NT) {
            int r = i / BK, c = i % BK;
            int gn = n0 + r, gk = k0 + c;
            bool p = (gk < g.K) && (gn < g.N);
            cp_async8(bs + r * AS + c, p ? (Bseg + (int64_t)gn * g.b_cs + gk) : Bseg, p);
          }
        }
      }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
      if (s < KT_all) load_tile(s, s);
      cp_async_commit();
    }
    for (int kt = 0; kt < KT_all; kt++) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        int nk = kt + STAGES - 1;
        if (nk < KT_all) load_tile(nk % STAGES, nk);
        cp_async_commit();
      }
      const double* as = As + (kt % STAGES) * L::A_STAGE;
      const double* bs = Bs + (kt % STAGES) * L::B_STAGE;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[TM], bf[TN];
#pragma unroll
        for (int i = 0; i < TM; i++) af[i] = as[(wm0 + i * 8 + (lane >> 2)) * AS + kk + (lane & 3)];
#pragma unroll
        for (int j = 0; j < TN; j++) {
          if (B_ROW)
            bf[j] = bs[(kk + (lane & 3)) * BS_ROW + wn0 + j * 8 + (lane >> 2)];
          else
            bf[j] = bs[(wn0 + j * 8 + (lane >> 2)) * AS + kk + (lane & 3)];
        }
#pragma unroll
        for (int i = 0; i < TM; i++)
#pragma unroll
          for (int j = 0; j < TN; j++) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();

    // epilogue: C = alpha acc + beta C  (2 consecutive doubles per thread)
#pragma unroll
    for (int i = 0; i < TM; i++) {
      int row = m0 + wm0 + i * 8 + (lane >> 2);
      if (row >= g.M) continue;
#pragma unroll
      for (int j = 0; j < TN; j++) {
        int col = n0 + wn0 + j * 8 + 2 * (lane & 3);
        double* cp = C + (int64_t)row * g.c_rs + col;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          if (col + e < g.N) {
            double v = g.alpha * acc[i][j][e];
            if (g.beta != 0.0) v += g.beta * cp[e];
            cp[e] = v;
          }
        }
      }
    }
  }
}

// Generic strided fallback (tiny / irregular shapes): one thread per C entry.
__global__ void dgemm_generic_kernel(Gemm g) {
  // 2D mapping without 64-bit divisions: x covers columns n (coalesced for
  // row-major B/C), y loops rows m; z covers the batch.
  const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.N) return;
  for (int64_t z = blockIdx.z; z < nbatch; z += gridDim.z) {
    const int64_t b1 = z % g.batch1, b23 = z / g.batch1;
    const int64_t b2 = b23 % g.batch2, b3 = b23 / g.batch2;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2 + b3 * g.a_b3;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2 + b3 * g.b_b3;
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2 + b3 * g.c_b3;
    for (int m = blockIdx.y; m < g.M; m += gridDim.y) {
      double acc = 0.0;
      for (int seg = 0; seg < g.nseg; seg++) {
        const double* As = A + seg * g.a_sg + (int64_t)m * g.a_rs;
        const double* Bs = B + seg * g.b_sg + (int64_t)n * g.b_cs;
        for (int k = 0; k < g.K; k++) acc = fma(As[k * g.a_cs], Bs[k * g.b_rs], acc);
      }
      double* cp = C + (int64_t)m * g.c_rs + (int64_t)n * g.c_cs;
      double v = g.alpha * acc;
      if (g.beta != 0.0) v += g.beta * *cp;
      *cp = v;
    }
  }
}

// Skinny fallback (few outputs, long K): one warp per C entry, lanes stride K
// (coalesced when A is row-major or B column-major), shuffle reduction.
__global__ void dgemm_skinny_kernel(Gemm g) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_per_block = blockDim.x >> 5;
  const int64_t total = (int64_t)g.M * g.N;
  const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
  for (int64_t z = blockIdx.y; z < nbatch; z += gridDim.y) {
    const int64_t b1 = z % g.batch1, b23 = z / g.batch1;
    const int64_t b2 = b23 % g.batch2, b3 = b23 / g.batch2;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2 + b3 * g.a_b3;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2 + b3 * g.b_b3;
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2 + b3 * g.c_b3;
    for (int64_t idx = blockIdx.x * warps_per_block + (threadIdx.x >> 5); idx < total;
         idx += (int64_t)gridDim.x * warps_per_block) {
      const int m = (int)(idx / g.N), n = (int)(idx % g.N);
      double acc = 0.0;
      for (int seg = 0; seg < g.nseg; seg++) {
        const double* Ar = A + seg * g.a_sg + (int64_t)m * g.a_rs;
        const double* Bc = B + seg * g.b_sg + (int64_t)n * g.b_cs;
        for (int k = lane; k < g.K; k += 32) acc = fma(Ar[k * g.a_cs], Bc[k * g.b_rs], acc);
      }
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        double* cp = C + (int64_t)m * g.c_rs + (int64_t)n * g.c_cs;
        double v = g.alpha * acc;
        if (g.beta != 0.0) v += g.beta * *cp;
        *cp = v;
      }
    }
  }
}

// Few-row GEMM with a row-major B (b_cs == 1): C[m, n] = alpha sum_k A[m, k] B[k, n]
// (+ beta C), M <= 8.  One thread per output column n: consecutive threads read
// consecutive B elements (coalesced rows), A is broadcast; 8 rows of B in
// flight per thread.  E.g. the time-point functional of an IC block applied to
// a PDE-shaped vector (K = n_t, N = n_x).
template <int MM>
__global__ void __launch_bounds__(256) dgemm_gemvt_kernel(Gemm g) {
  const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
  const int64_t ncol_blocks = (g.N + blockDim.x - 1) / blockDim.x;
  for (int64_t w = blockIdx.x; w < nbatch * ncol_blocks; w += gridDim.x) {
    const int64_t z = w / ncol_blocks;
    const int n = (int)((w - z * ncol_blocks) * blockDim.x + threadIdx.x);
    if (n >= g.N) continue;
    const int64_t b1 = z % g.batch1, b23 = z / g.batch1;
    const int64_t b2 = b23 % g.batch2, b3 = b23 / g.batch2;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2 + b3 * g.a_b3;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2 + b3 * g.b_b3 + n;
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2 + b3 * g.c_b3 + (int64_t)n * g.c_cs;
    double acc[MM];
#pragma unroll
    for (int m = 0; m < MM; m++) acc[m] = 0.0;
    for (int seg = 0; seg < g.nseg; seg++) {
      const double* As = A + seg * g.a_sg;
      const double* Bs = B + seg * g.b_sg;
      int k = 0;
      for (; k + 8 <= g.K; k += 8) {
        double bv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) bv[u] = __ldg(Bs + (int64_t)(k + u) * g.b_rs);
#pragma unroll
        for (int u = 0; u < 8; u++)
#pragma unroll
          for (int m = 0; m < MM; m++)
            if (m < g.M) acc[m] = fma(__ldg(As + (int64_t)m * g.a_rs + (int64_t)(k + u) * g.a_cs), bv[u], acc[m]);
      }
      for (; k < g.K; k++) {
        const double bv = __ldg(Bs + (int64_t)k * g.b_rs);
#pragma unroll
        for (int m = 0; m < MM; m++)
          if (m < g.M) acc[m] = fma(__ldg(As + (int64_t)m * g.a_rs + (int64_t)k * g.a_cs), bv, acc[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < MM; m++)
      if (m < g.M) {
        double* cp = C + (int64_t)m * g.c_rs;
        double v = g.alpha * acc[m];
        if (g.beta != 0.0) v += g.beta * *cp;
        *cp = v;
      }
  }
}

// Few-column GEMM with A contiguous along K (a_cs == 1): C[m, n] for N <= 8.
// One warp per output row m computes all N columns, so each row of A is read
// once (lanes along K, coalesced), 4 rows of A in flight per lane.  E.g. the
// space-point functionals of BC blocks applied to a PDE-shaped vector.
template <int NN>
__global__ void __launch_bounds__(256) dgemm_gemvn_kernel(Gemm g) {
  const int lane = threadIdx.x & 31;
  const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nbatch * g.M; w += warps) {
    const int64_t z = w / g.M;
    const int m = (int)(w - z * g.M);
    const int64_t b1 = z % g.batch1, b23 = z / g.batch1;
    const int64_t b2 = b23 % g.batch2, b3 = b23 / g.batch2;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2 + b3 * g.a_b3 + (int64_t)m * g.a_rs;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2 + b3 * g.b_b3;
    double acc[NN];
#pragma unroll
    for (int n = 0; n < NN; n++) acc[n] = 0.0;
    for (int seg = 0; seg < g.nseg; seg++) {
      const double* As = A + seg * g.a_sg;
      const double* Bs = B + seg * g.b_sg;
      int k = lane;
      if (g.b_rs == 1 && ((reinterpret_cast<uintptr_t>(As) | reinterpret_cast<uintptr_t>(Bs)) & 15) == 0 &&
          (g.b_cs & 1) == 0) {
        // 16-byte loads over full 256-element chunks (lane: elements 2*lane, 2*lane+1
        // of each 64-wide slice), then the tail with scalar loads
        const int nfull = g.K / 256;
        for (int c = 0; c < nfull; c++) {
          const int k2 = 256 * c + 2 * lane;
          double2 av[4];
#pragma unroll
          for (int u = 0; u < 4; u++) av[u] = __ldg(reinterpret_cast<const double2*>(As + k2 + 64 * u));
#pragma unroll
          for (int u = 0; u < 4; u++)
#pragma unroll
            for (int n = 0; n < NN; n++)
              if (n < g.N) {
                const double2 bv = __ldg(reinterpret_cast<const double2*>(Bs + k2 + 64 * u + (int64_t)n * g.b_cs));
                acc[n] = fma(av[u].x, bv.x, fma(av[u].y, bv.y, acc[n]));
              }
        }
        k = 256 * nfull + lane;
      }
      for (; k + 96 < g.K; k += 128) {
        double av[4];
#pragma unroll
        for (int u = 0; u < 4; u++) av[u] = __ldg(As + k + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
          for (int n = 0; n < NN; n++)
            if (n < g.N) acc[n] = fma(av[u], __ldg(Bs + (int64_t)(k + 32 * u) * g.b_rs + (int64_t)n * g.b_cs), acc[n]);
      }
      for (; k < g.K; k += 32) {
        const double av = __ldg(As + k);
#pragma unroll
        for (int n = 0; n < NN; n++)
          if (n < g.N) acc[n] = fma(av, __ldg(Bs + (int64_t)k * g.b_rs + (int64_t)n * g.b_cs), acc[n]);
      }
    }
#pragma unroll
    for (int n = 0; n < NN; n++) {
      double v = acc[n];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[n] = v;
    }
    if (lane == 0) {
      double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2 + b3 * g.c_b3 + (int64_t)m * g.c_rs;
#pragma unroll
      for (int n = 0; n < NN; n++)
        if (n < g.N) {
          double* cp = C + (int64_t)n * g.c_cs;
          double v = g.alpha * acc[n];
          if (g.beta != 0.0) v += g.beta * *cp;
          *cp = v;
        }
    }
  }
}

// gemvt for 16-byte aligned B with even N and row stride: a 256-thread block
// covers 64 columns (double2 per thread) x 8 K-slices (one warp each), 8 rows
// in flight per thread, partial sums reduced through shared memory.
template <int MM>
__global__ void __launch_bounds__(256) dgemm_gemvt2_kernel(Gemm g) {
  __shared__ double2 red[8][MM][32];
  const int lane = threadIdx.x & 31, ks = threadIdx.x >> 5;
  const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
  const int64_t ctiles = (g.N + 63) / 64;
  const int kchunk = (g.K + 7) / 8;
  const int k0 = ks * kchunk, k1 = min(g.K, k0 + kchunk);
  for (int64_t w = blockIdx.x; w < nbatch * ctiles; w += gridDim.x) {
    const int64_t z = w / ctiles;
    const int n = (int)((w - z * ctiles) * 64 + 2 * lane);
    const int64_t b1 = z % g.batch1, b23 = z / g.batch1;
    const int64_t b2 = b23 % g.batch2, b3 = b23 / g.batch2;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2 + b3 * g.a_b3;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2 + b3 * g.b_b3 + n;
    double2 acc[MM];
#pragma unroll
    for (int m = 0; m < MM; m++) acc[m] = make_double2(0.0, 0.0);
    if (n < g.N) {
      for (int seg = 0; seg < g.nseg; seg++) {
        const double* As = A + seg * g.a_sg;
        const double* Bs = B + seg * g.b_sg;
        int k = k0;
        for (; k + 8 <= k1; k += 8) {
          double2 bv[8];
#pragma unroll
          for (int u = 0; u < 8; u++) bv[u] = __ldg(reinterpret_cast<const double2*>(Bs + (int64_t)(k + u) * g.b_rs));
#pragma unroll
          for (int u = 0; u < 8; u++)
#pragma unroll
            for (int m = 0; m < MM; m++)
              if (m < g.M) {
                const double a = __ldg(As + (int64_t)m * g.a_rs + (int64_t)(k + u) * g.a_cs);
                acc[m].x = fma(a, bv[u].x, acc[m].x);
                acc[m].y = fma(a, bv[u].y, acc[m].y);
              }
        }
        for (; k < k1; k++) {
          const double2 bv = __ldg(reinterpret_cast<const double2*>(Bs + (int64_t)k * g.b_rs));
#pragma unroll
          for (int m = 0; m < MM; m++)
            if (m < g.M) {
              const double a = __ldg(As + (int64_t)m * g.a_rs + (int64_t)k * g.a_cs);
              acc[m].x = fma(a, bv.x, acc[m].x);
              acc[m].y = fma(a, bv.y, acc[m].y);
            }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MM; m++) red[ks][m][lane] = acc[m];
    __syncthreads();
    if (ks < MM && ks < g.M && n < g.N) {
      double2 v = red[0][ks][lane];
#pragma unroll
      for (int j = 1; j < 8; j++) {
        v.x += red[j][ks][lane].x;
        v.y += red[j][ks][lane].y;
      }
      double* cp = g.C + b1 * g.c_b1 + b2 * g.c_b2 + b3 * g.c_b3 + (int64_t)ks * g.c_rs + (int64_t)n * g.c_cs;
      double r0 = g.alpha * v.x, r1 = g.alpha * v.y;
      if (g.beta != 0.0) {
        r0 += g.beta * cp[0];
        r1 += g.beta * cp[g.c_cs];
      }
      cp[0] = r0;
      cp[g.c_cs] = r1;
    }
    __syncthreads();
  }
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool B_ROW, bool V16>
void launch_dmma(const Gemm& g, cudaStream_t s) {
  using L = SmemLayout<BM, BN, B_ROW>;
  size_t smem = (size_t)STAGES * (L::A_STAGE + L::B_STAGE) * sizeof(double);
  auto kern = dgemm_dmma_kernel<BM, BN, WARPS_M, WARPS_N, STAGES, B_ROW, V16>;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    GPFVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (getenv("GPFVM_CARVEOUT"))
      GPFVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(getenv("GPFVM_CARVEOUT"))));
    configured_dev = dev;
  }
  int64_t nb = (int64_t)g.batch1 * g.batch2 * g.batch3;
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, (unsigned)std::min<int64_t>(nb, 65535));
  kern<<<grid, WARPS_M * WARPS_N * 32, smem, s>>>(g);
  count_launch();
  check_launch("dgemm_dmma_kernel");
}

template <int BM, int BN, int WM_, int WN_, int ST, bool V16>
void launch_b(const Gemm& g, bool brow, cudaStream_t s) {
  if (brow) launch_dmma<BM, BN, WM_, WN_, ST, true, V16>(g, s);
  else launch_dmma<BM, BN, WM_, WN_, ST, false, V16>(g, s);
}

template <bool V16>
void dispatch(const Gemm& g, bool brow, cudaStream_t s) {
  // Tile choice (measured on B200, tools/gemm_bench.cu): 128x64 CTA tiles
  // with 8 warps of 32x32 (2 CTAs/SM) give the best DMMA throughput for the
  // mode-product shapes (~28-30 TF/s of 37); smaller tiles when the grid would
  // not fill the 148 SMs.
  const int64_t nb = (int64_t)g.batch1 * g.batch2 * g.batch3;
  const int64_t t12864 = ((g.M + 127) / 128) * (int64_t)((g.N + 63) / 64) * nb;
  const int64_t t64 = ((g.M + 63) / 64) * (int64_t)((g.N + 63) / 64) * nb;
  static const int variant = getenv("GPFVM_GEMM_VARIANT") ? atoi(getenv("GPFVM_GEMM_VARIANT")) : -1;
  if (variant == 0) { launch_b<128, 128, 2, 4, 3, V16>(g, brow, s); return; }
  if (variant == 3) { launch_b<64, 32, 2, 2, 4, V16>(g, brow, s); return; }
  if (t12864 >= 148) launch_b<128, 64, 4, 2, 3, V16>(g, brow, s);
  else if (t64 >= 148) launch_b<64, 64, 2, 2, 4, V16>(g, brow, s);
  else launch_b<32, 32, 2, 2, 4, V16>(g, brow, s);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool even(int64_t v) { return (v & 1) == 0; }

}  // namespace

double gemm_flops(const Gemm& g) {
  return 2.0 * g.M * (double)g.N * g.K * g.nseg * g.batch1 * g.batch2 * g.batch3;
}

// B (cols x rows) = A^T for A (rows x cols, leading dimension lda), tiled
__global__ void transpose_any_kernel(const double* __restrict__ A, int64_t lda, double* __restrict__ B, int rows,
                                     int cols) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = by + j, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[j][threadIdx.x] = A[(int64_t)r * lda + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = bx + j, c = by + threadIdx.x;
    if (r < cols && c < rows) B[(int64_t)r * rows + c] = tile[threadIdx.x][j];
  }
}

void run_gemm(const Gemm& g0, cudaStream_t s) {
  if (g0.K2 > 0) {
    // extra low-rank term: fused into the TMA kernel's k loop, else a second GEMM
    if (try_tma_gemm(g0, s)) return;
    Gemm m = g0;
    m.K2 = 0;
    run_gemm(m, s);
    Gemm e;
    e.M = g0.M; e.N = g0.N; e.K = g0.K2; e.batch1 = g0.batch1;
    e.A = g0.A2; e.a_rs = g0.a2_rs; e.a_cs = 1; e.a_b1 = g0.a2_b1;
    e.B = g0.B2; e.b_rs = 1; e.b_cs = g0.b2_rs; e.b_b1 = g0.b2_b1;
    e.C = g0.C; e.c_rs = g0.c_rs; e.c_cs = g0.c_cs; e.c_b1 = g0.c_b1;
    e.alpha = g0.alpha; e.beta = 1.0;
    run_gemm(e, s);
    return;
  }
  Gemm g = g0;
  // A single-row GEMM batched over right-hand sides that share B is one GEMM
  // with the batch as its M dimension (e.g. IC-block contractions).
  if (g.M == 1 && g.batch1 > 1 && g.batch2 == 1 && g.batch3 == 1 && g.b_b1 == 0) {
    g.M = g.batch1;
    g.a_rs = g.a_b1;
    g.c_rs = g.c_b1;
    g.batch1 = 1;
    g.a_b1 = g.c_b1 = 0;
  }
  // Symmetric case: a single-column GEMM batched over right-hand sides that
  // share A (e.g. the time factor of a BC block applied to per-vector
  // contractions) is C^T = B^T A^T with the batch as M — one DMMA GEMM that
  // reads A once instead of once per vector.
  if (g.N == 1 && g.batch1 > 1 && g.batch2 == 1 && g.batch3 == 1 && g.a_b1 == 0) {
    Gemm t = g;
    t.M = g.batch1; t.N = g.M; t.K = g.K;
    t.A = g.B; t.a_rs = g.b_b1; t.a_cs = g.b_rs; t.a_sg = g.b_sg;
    t.B = g.A; t.b_rs = g.a_cs; t.b_cs = g.a_rs; t.b_sg = g.a_sg;
    t.C = g.C; t.c_rs = g.c_b1; t.c_cs = g.c_rs;
    t.batch1 = 1;
    t.a_b1 = t.b_b1 = t.c_b1 = 0;
    g = t;
  }
  if (g.M <= 0 || g.N <= 0 || g.batch1 <= 0 || g.batch2 <= 0 || g.batch3 <= 0) return;
  static const bool trace = getenv("GPFVM_TRACE_GEMM") != nullptr;
  if (trace)
    fprintf(stderr, "[gemm] M=%d N=%d K=%d nseg=%d batch=%d,%d,%d a(rs=%lld cs=%lld b=%lld,%lld,%lld sg=%lld) "
            "b(rs=%lld cs=%lld b=%lld,%lld,%lld sg=%lld) c(rs=%lld cs=%lld b=%lld,%lld,%lld) beta=%g\n",
            g.M, g.N, g.K, g.nseg, g.batch1, g.batch2, g.batch3, (long long)g.a_rs, (long long)g.a_cs, (long long)g.a_b1,
            (long long)g.a_b2, (long long)g.a_b3, (long long)g.a_sg, (long long)g.b_rs, (long long)g.b_cs,
            (long long)g.b_b1, (long long)g.b_b2, (long long)g.b_b3, (long long)g.b_sg, (long long)g.c_rs,
            (long long)g.c_cs, (long long)g.c_b1, (long long)g.c_b2, (long long)g.c_b3, g.beta);
  GPFVM_CHECK(g.K > 0 && g.nseg > 0, GPFVM_ERR_INVALID, "run_gemm: K and nseg must be positive");
  const bool fast = (g.a_cs == 1) && (g.c_cs == 1) && (g.b_cs == 1 || g.b_rs == 1) && g.M >= 8 &&
                    g.N >= 8 && g.K * g.nseg >= 4;
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  if (!fast) GPFVM_CUDA(cudaStreamIsCapturing(s, &cap_status));
  if (!fast && cap_status == cudaStreamCaptureStatusNone && g.a_rs == 1 && g.a_cs >= g.M && g.c_cs == 1 &&
      (g.b_cs == 1 || g.b_rs == 1) && g.M >= 8 && g.N >= 8 && g.K >= 8 && g.nseg == 1 &&
      g.batch1 * g.batch2 * g.batch3 == 1) {
    // (not while a CUDA graph is being captured: the scratch copy is returned
    // to the pool after a stream synchronisation)
    // transposed A (setup GEMMs such as S^T T or L^{-T} L^{-1}): materialise
    // A^T once (K x M -> M x K) so the tensor-core path applies
    DevBuf At;
    At.ensure((size_t)g.M * g.K);
    const dim3 tg((g.M + 31) / 32, (g.K + 31) / 32);
    transpose_any_kernel<<<tg, dim3(32, 8), 0, s>>>(g.A, g.a_cs, At.ptr, g.K, g.M);
    count_launch();
    Gemm t = g;
    t.A = At.ptr;
    t.a_rs = g.K;
    t.a_cs = 1;
    run_gemm(t, s);
    GPFVM_CUDA(cudaStreamSynchronize(s));  // At is returned to the pool on scope exit
    return;
  }
  if (!fast) {
    int64_t total = (int64_t)g.M * g.N;
    const int64_t kk = (int64_t)g.K * g.nseg;
    static const bool no_gemvt = getenv("GPFVM_NO_GEMVT") != nullptr;
    if (!no_gemvt && g.b_cs == 1 && g.M <= 8 && g.N >= 64 && g.K >= 64 && (g.N & 1) == 0 && (g.b_rs & 1) == 0 &&
        (g.b_b1 & 1) == 0 && (g.b_b2 & 1) == 0 && (g.b_b3 & 1) == 0 && (g.b_sg & 1) == 0 &&
        aligned16(g.B)) {
      const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
      const unsigned grid = (unsigned)std::min<int64_t>(nbatch * ((g.N + 63) / 64), 148 * 16);
      if (g.M <= 2) dgemm_gemvt2_kernel<2><<<grid, 256, 0, s>>>(g);
      else if (g.M <= 4) dgemm_gemvt2_kernel<4><<<grid, 256, 0, s>>>(g);
      else dgemm_gemvt2_kernel<8><<<grid, 256, 0, s>>>(g);
      count_launch();
      check_launch("dgemm_gemvt2_kernel");
      return;
    }
    if (!no_gemvt && g.b_cs == 1 && g.M <= 8 && g.N >= 64 && kk >= 8) {
      const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
      const int64_t work = nbatch * ((g.N + 127) / 128);
      const unsigned grid = (unsigned)std::min<int64_t>(work, 148 * 32);
      if (g.M <= 2) dgemm_gemvt_kernel<2><<<grid, 128, 0, s>>>(g);
      else if (g.M <= 4) dgemm_gemvt_kernel<4><<<grid, 128, 0, s>>>(g);
      else dgemm_gemvt_kernel<8><<<grid, 128, 0, s>>>(g);
      count_launch();
      check_launch("dgemm_gemvt_kernel");
      return;
    }
    if (!no_gemvt && g.a_cs == 1 && g.N <= 8 && g.M >= 32 && kk >= 64) {
      const int64_t nbatch = (int64_t)g.batch1 * g.batch2 * g.batch3;
      const unsigned grid = (unsigned)std::min<int64_t>((nbatch * g.M + 7) / 8, 148 * 16);
      if (g.N <= 2) dgemm_gemvn_kernel<2><<<grid, 256, 0, s>>>(g);
      else if (g.N <= 4) dgemm_gemvn_kernel<4><<<grid, 256, 0, s>>>(g);
      else dgemm_gemvn_kernel<8><<<grid, 256, 0, s>>>(g);
      count_launch();
      check_launch("dgemm_gemvn_kernel");
      return;
    }
    if (kk >= 32 && total <= (1 << 20)) {
      const int threads = 256;  // 8 warps, one output each
      unsigned bx = (unsigned)std::min<int64_t>((total + 7) / 8, 4096);
      unsigned by = (unsigned)std::min<int64_t>((int64_t)g.batch1 * g.batch2 * g.batch3, 65535);
      dgemm_skinny_kernel<<<dim3(bx, by), threads, 0, s>>>(g);
      count_launch();
      check_launch("dgemm_skinny_kernel");
      return;
    }
    const int threads = g.N >= 128 ? 128 : 32;
    unsigned bx = (unsigned)((g.N + threads - 1) / threads);
    // enough blocks to fill the machine; each thread loops over M / by rows
    const int64_t nbz = std::min<int64_t>((int64_t)g.batch1 * g.batch2 * g.batch3, 65535);
    unsigned by = (unsigned)std::min<int64_t>(g.M, std::max<int64_t>(16, 4096 / std::max<int64_t>(1, (int64_t)bx * nbz)));
    unsigned bz = (unsigned)std::min<int64_t>((int64_t)g.batch1 * g.batch2 * g.batch3, 65535);
    dgemm_generic_kernel<<<dim3(bx, by, bz), threads, 0, s>>>(g);
    count_launch();
    check_launch("dgemm_generic_kernel");
    return;
  }
  if (try_tma_gemm(g, s)) return;
  const bool brow = (g.b_cs == 1);
  const int64_t b_ld = brow ? g.b_rs : g.b_cs;
  const bool v16 = aligned16(g.A) && aligned16(g.B) && even(g.a_rs) && even(b_ld) && even(g.a_b1) &&
                   even(g.a_b2) && even(g.a_b3) && even(g.b_b1) && even(g.b_b2) && even(g.b_b3) &&
                   even(g.a_sg) && even(g.b_sg);
  if (v16) dispatch<true>(g, brow, s);
  else dispatch<false>(g, brow, s);
}

}  // namespace gpfvm
