// C-ABI primitives used by the sharded multi-GPU path:
//   gpfvm_gemm     row-major DMMA GEMM (the time contraction after the all-to-all)
//   gpfvm_permute  <=4D tensor permutation (layout changes around the all-to-all)
//   gpfvm_sygv     generalised symmetric-definite eigensolver (FD factors)
#include <algorithm>

#include "problem.h"

namespace gpfvm {
namespace {
__global__ void permute_kernel(const double* __restrict__ src, double* __restrict__ dst, int4 shape, int4 perm,
                               int64_t total) {
  // dst index order = (shape[perm[0]], shape[perm[1]], ...) row-major
  const int sh[4] = {shape.x, shape.y, shape.z, shape.w};
  const int pm[4] = {perm.x, perm.y, perm.z, perm.w};
  int64_t sstride[4];
  sstride[3] = 1;
  for (int i = 2; i >= 0; i--) sstride[i] = sstride[i + 1] * sh[i + 1];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = o, sidx = 0;
    for (int k = 3; k >= 0; k--) {
      int64_t ext = sh[pm[k]];
      int64_t c = rem % ext;
      rem /= ext;
      sidx += c * sstride[pm[k]];
    }
    dst[o] = src[sidx];
  }
}

// register-only DMMA throughput probe (8 independent accumulator chains per warp)
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, int iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
int guarded2(F&& f) {
  try {
    f();
    return GPFVM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GPFVM_ERR_INVALID;
  }
}
}  // namespace
}  // namespace gpfvm

using namespace gpfvm;

extern "C" int gpfvm_probe_fp64_peak(double* tflops, void* stream) {
  return guarded2([&] {
    GPFVM_CHECK(tflops, GPFVM_ERR_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    GPFVM_CUDA(cudaGetDevice(&dev));
    GPFVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 4, threads = 256, iters = 4096;
    DevBuf out;
    out.ensure((size_t)blocks * threads);
    cudaEvent_t e0, e1;
    GPFVM_CUDA(cudaEventCreate(&e0));
    GPFVM_CUDA(cudaEventCreate(&e1));
    dmma_probe_kernel<<<blocks, threads, 0, s>>>(out.ptr, 16);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 2; rep++) {
      GPFVM_CUDA(cudaEventRecord(e0, s));
      dmma_probe_kernel<<<blocks, threads, 0, s>>>(out.ptr, iters);
      GPFVM_CUDA(cudaEventRecord(e1, s));
      GPFVM_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      GPFVM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    count_launch(3);
    check_launch("dmma_probe_kernel");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    *tflops = flops / (best * 1e-3) / 1e12;
  });
}

extern "C" int gpfvm_gemm(int M, int N, int K, double alpha, const double* A, int64_t lda, const double* B,
                          int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  return guarded2([&] {
    GPFVM_CHECK(M >= 0 && N >= 0 && K >= 1 && A && B && C, GPFVM_ERR_INVALID, "bad gemm arguments");
    GPFVM_CHECK(lda >= K && ldb >= N && ldc >= N, GPFVM_ERR_INVALID, "leading dimension too small");
    Gemm g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.a_rs = lda; g.a_cs = 1;
    g.B = B; g.b_rs = ldb; g.b_cs = 1;
    g.C = C; g.c_rs = ldc; g.c_cs = 1;
    g.alpha = alpha; g.beta = beta;
    run_gemm(g, (cudaStream_t)stream);
  });
}

extern "C" int gpfvm_permute(int ndim, const int* shape, const int* perm, const double* src, double* dst,
                             void* stream) {
  return guarded2([&] {
    GPFVM_CHECK(ndim >= 1 && ndim <= 4 && shape && perm && src && dst && src != dst, GPFVM_ERR_INVALID,
                "bad permute arguments");
    int sh[4] = {1, 1, 1, 1}, pm[4] = {0, 1, 2, 3};
    int off = 4 - ndim;  // right-align into 4D
    int64_t total = 1;
    int seen = 0;
    for (int i = 0; i < ndim; i++) {
      GPFVM_CHECK(shape[i] >= 1 && perm[i] >= 0 && perm[i] < ndim && !(seen & (1 << perm[i])), GPFVM_ERR_INVALID,
                  "bad permutation");
      seen |= 1 << perm[i];
      sh[off + i] = shape[i];
      pm[off + i] = off + perm[i];
      total *= shape[i];
    }
    for (int i = 0; i < off; i++) pm[i] = i;
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 4096));
    permute_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(src, dst, make_int4(sh[0], sh[1], sh[2], sh[3]),
                                                             make_int4(pm[0], pm[1], pm[2], pm[3]), total);
    count_launch();
    check_launch("permute_kernel");
  });
}

extern "C" int gpfvm_sygv(int n, const double* A, const double* B, double* V, double* w, void* stream) {
  return guarded2([&] {
    GPFVM_CHECK(n >= 1 && A && B && V && w, GPFVM_ERR_INVALID, "bad sygv arguments");
    sygv(A, B, n, V, w, (cudaStream_t)stream);
  });
}

// Fused solver vector ops for the sharded solver (same kernels as gpfvm_solve):
//   out[j] = X_j . v  (k vectors, deterministic two-pass reduction), y += sign * sum_j coef[j] X_j
extern "C" int gpfvm_dot_many(const double* X, int64_t ldx, const double* v, int64_t n, int k, double* out,
                              void* stream) {
  return guarded2([&] {
    GPFVM_CHECK(X && v && out && k >= 1 && n >= 0, GPFVM_ERR_INVALID, "bad dot_many arguments");
    dot_many(X, ldx, v, n, k, out, (cudaStream_t)stream);
  });
}

extern "C" int gpfvm_axpy_many(double* y, const double* X, int64_t ldx, const double* coef, double sign, int64_t n,
                               int k, void* stream) {
  return guarded2([&] {
    GPFVM_CHECK(y && X && coef && k >= 1 && n >= 0, GPFVM_ERR_INVALID, "bad axpy_many arguments");
    axpy_many(y, X, ldx, coef, sign, n, k, (cudaStream_t)stream);
  });
}
