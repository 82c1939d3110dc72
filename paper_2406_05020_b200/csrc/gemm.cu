// FP64 tensor-core GEMM (DMMA m8n8k4) for the batched mode-n contractions of
// the Kronecker matvec.
//
// C[b] = alpha * A[b] B[b] + beta * C[b],  b = (b1, b2) two-level batch.
// Fast path: A row-major (a_cs == 1), C row-major (c_cs == 1), B row-major
// (b_cs == 1) or column-major (b_rs == 1).  Tiles are staged through shared
// memory with a 3-stage cp.async pipeline; each warp owns a (TM*8)x(TN*8)
// sub-tile and issues TM*TN DMMA per k4 step (SASS: DMMA.8x8x4, the only
// FP64 tensor-core instruction on sm_100a — tcgen05 has no f64 kind).
// Shared-memory rows are padded so the fragment loads hit each 8-byte bank
// pair exactly twice per warp (2 wavefronts, the minimum for 256 B).
#include "internal.h"

namespace gpfvm {

namespace {

constexpr int BK = 16;
constexpr int STAGES = 3;
constexpr int APAD = 4;   // As row stride BK+4 doubles
constexpr int BPAD = 8;   // Bs (row layout) row stride BN+8 doubles

__device__ __forceinline__ void cp_async8(void* smem, const double* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
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

template <int BM, int BN, int WARPS_M, int WARPS_N, bool B_ROW>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32)
    dgemm_dmma_kernel(Gemm g) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int TM = WM / 8, TN = WN / 8;
  constexpr int AS = BK + APAD;
  constexpr int BS_ROW = BN + BPAD;
  constexpr int B_STAGE = B_ROW ? BK * BS_ROW : BN * AS;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                       // [STAGES][BM][AS]
  double* Bs = smem + STAGES * BM * AS;    // [STAGES][BK][BS_ROW] or [STAGES][BN][AS]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / WARPS_N) * WM, wn0 = (warp % WARPS_N) * WN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

  for (int64_t z = blockIdx.z; z < (int64_t)g.batch1 * g.batch2; z += gridDim.z) {
    const int64_t b1 = z % g.batch1, b2 = z / g.batch1;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2;
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2;

    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int KT = (g.K + BK - 1) / BK;
    auto load_tile = [&](int stage, int kt) {
      const int k0 = kt * BK;
      double* as = As + stage * BM * AS;
#pragma unroll
      for (int i = tid; i < BM * BK; i += NT) {
        int r = i / BK, c = i % BK;
        int gm = m0 + r, gk = k0 + c;
        bool p = (gm < g.M) && (gk < g.K);
        const double* src = p ? (A + (int64_t)gm * g.a_rs + gk) : A;
        cp_async8(as + r * AS + c, src, p);
      }
      double* bs = Bs + stage * B_STAGE;
      if (B_ROW) {
#pragma unroll
        for (int i = tid; i < BK * BN; i += NT) {
          int r = i / BN, c = i % BN;
          int gk = k0 + r, gn = n0 + c;
          bool p = (gk < g.K) && (gn < g.N);
          const double* src = p ? (B + (int64_t)gk * g.b_rs + gn) : B;
          cp_async8(bs + r * BS_ROW + c, src, p);
        }
      } else {
#pragma unroll
        for (int i = tid; i < BK * BN; i += NT) {
          int r = i / BK, c = i % BK;  // r: n, c: k
          int gn = n0 + r, gk = k0 + c;
          bool p = (gk < g.K) && (gn < g.N);
          const double* src = p ? (B + (int64_t)gn * g.b_cs + gk) : B;
          cp_async8(bs + r * AS + c, src, p);
        }
      }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
      if (s < KT) load_tile(s, s);
      cp_async_commit();
    }
    for (int kt = 0; kt < KT; kt++) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        int nk = kt + STAGES - 1;
        if (nk < KT) load_tile(nk % STAGES, nk);
        cp_async_commit();
      }
      const double* as = As + (kt % STAGES) * BM * AS;
      const double* bs = Bs + (kt % STAGES) * B_STAGE;
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

    // epilogue: C = alpha acc + beta C
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

// Generic strided fallback (small / irregular shapes): one thread per C entry.
__global__ void dgemm_generic_kernel(Gemm g) {
  int64_t total = (int64_t)g.M * g.N;
  for (int64_t z = blockIdx.y; z < (int64_t)g.batch1 * g.batch2; z += gridDim.y) {
    const int64_t b1 = z % g.batch1, b2 = z / g.batch1;
    const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2;
    const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2;
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
      int m = (int)(idx / g.N), n = (int)(idx % g.N);
      double acc = 0.0;
      for (int k = 0; k < g.K; k++) acc = fma(A[m * g.a_rs + k * g.a_cs], B[k * g.b_rs + n * g.b_cs], acc);
      double* cp = C + m * g.c_rs + n * g.c_cs;
      double v = g.alpha * acc;
      if (g.beta != 0.0) v += g.beta * *cp;
      *cp = v;
    }
  }
}

template <int BM, int BN, int WARPS_M, int WARPS_N, bool B_ROW>
void launch_dmma(const Gemm& g, cudaStream_t s) {
  constexpr int AS = BK + APAD;
  constexpr int B_STAGE = B_ROW ? BK * (BN + BPAD) : BN * AS;
  size_t smem = (size_t)STAGES * (BM * AS + B_STAGE) * sizeof(double);
  auto kern = dgemm_dmma_kernel<BM, BN, WARPS_M, WARPS_N, B_ROW>;
  static bool configured = false;
  if (!configured) {
    GPFVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM,
            (unsigned)std::min<int64_t>((int64_t)g.batch1 * g.batch2, 65535));
  kern<<<grid, WARPS_M * WARPS_N * 32, smem, s>>>(g);
  count_launch();
  check_launch("dgemm_dmma_kernel");
}

}  // namespace

double gemm_flops(const Gemm& g) { return 2.0 * g.M * (double)g.N * g.K * g.batch1 * g.batch2; }

void run_gemm(const Gemm& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch1 <= 0 || g.batch2 <= 0) return;
  if (g.K <= 0) {
    GPFVM_CHECK(false, GPFVM_ERR_INVALID, "run_gemm: K must be positive");
  }
  const bool fast = (g.a_cs == 1) && (g.c_cs == 1) && (g.b_cs == 1 || g.b_rs == 1) && g.M >= 8 &&
                    g.N >= 8 && g.K >= 4;
  if (!fast) {
    int64_t total = (int64_t)g.M * g.N;
    int threads = 256;
    unsigned bx = (unsigned)std::min<int64_t>((total + threads - 1) / threads, 4096);
    unsigned by = (unsigned)std::min<int64_t>((int64_t)g.batch1 * g.batch2, 65535);
    dgemm_generic_kernel<<<dim3(bx, by), threads, 0, s>>>(g);
    count_launch();
    check_launch("dgemm_generic_kernel");
    return;
  }
  const bool brow = (g.b_cs == 1);
  const int64_t nb = (int64_t)g.batch1 * g.batch2;
  const int64_t tiles64 = ((g.M + 63) / 64) * (int64_t)((g.N + 63) / 64) * nb;
  const int64_t tiles128 = ((g.M + 127) / 128) * (int64_t)((g.N + 63) / 64) * nb;
  if (tiles128 >= 4 * 148) {
    if (brow) launch_dmma<128, 64, 4, 2, true>(g, s);
    else launch_dmma<128, 64, 4, 2, false>(g, s);
  } else if (tiles64 >= 2 * 148) {
    if (brow) launch_dmma<64, 64, 2, 2, true>(g, s);
    else launch_dmma<64, 64, 2, 2, false>(g, s);
  } else {
    if (brow) launch_dmma<32, 32, 2, 2, true>(g, s);
    else launch_dmma<32, 32, 2, 2, false>(g, s);
  }
}

}  // namespace gpfvm
