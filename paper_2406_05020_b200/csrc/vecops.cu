// Fused solver vector operations: multi-dot products with
// warp-shuffle + deterministic two-pass block reduction (fixed order, so the
// same inputs always give bitwise-identical scalars), multi-axpy for the
// IterGP reorthogonalisation, and element-wise helpers.  All memory-bound,
// vectorised over a grid sized to 2 x 148 SMs.
#include <algorithm>
#include "internal.h"

namespace gpfvm {

namespace {
constexpr int RED_BLOCKS = 296;
constexpr int RED_THREADS = 256;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void dot_partial_kernel(const double* __restrict__ X, int64_t ldx, const double* __restrict__ v,
                                   int64_t n, double* __restrict__ partial) {
  const int j = blockIdx.y;
  const double* x = X + j * ldx;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], v[i], s);
  s = warp_sum(s);
  __shared__ double ws[RED_THREADS / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < RED_THREADS / 32) ? ws[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) partial[(int64_t)j * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void dot_final_kernel(const double* __restrict__ partial, int nparts, double* __restrict__ out) {
  const int j = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[(int64_t)j * nparts + i];
  s = warp_sum(s);
  __shared__ double ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < (int)(blockDim.x >> 5)) ? ws[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[j] = t;
  }
}

__global__ void axpy_many_kernel(double* __restrict__ y, const double* __restrict__ X, int64_t ldx,
                                 const double* __restrict__ coef, double sign, int64_t n, int k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < k; j++) acc = fma(coef[j], X[j * ldx + i], acc);
    y[i] = fma(sign, acc, y[i]);
  }
}

__global__ void noise_kernel(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ noise,
                             int64_t n, int64_t ld) {
  const int r = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[r * ld + i] = noise[i] * x[r * ld + i];
}

__global__ void fill_kernel(double* x, double v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}

__global__ void gather_kernel(double* __restrict__ dst, const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) dst[i] = src[idx[i]];
}
__global__ void scatter_kernel(double* __restrict__ dst, const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) dst[idx[i]] = src[i];
}

unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8));
}
}  // namespace

void dot_many(const double* X, int64_t ldx, const double* v, int64_t n, int k, double* out, cudaStream_t s) {
  if (k <= 0) return;
  // blocks per dot from the length (>= 4 elements per thread), so short dots
  // (e.g. the n_b-long rows of S^{-1}) do not launch 296 near-empty CTAs each;
  // fixed for a given n, hence still deterministic
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(RED_BLOCKS, (n + 4 * RED_THREADS - 1) / (4 * RED_THREADS)));
  DevBuf& partial = scratch(s, 0);
  partial.ensure((size_t)RED_BLOCKS * k);
  dot_partial_kernel<<<dim3(nblk, k), RED_THREADS, 0, s>>>(X, ldx, v, n, partial.ptr);
  dot_final_kernel<<<k, 512, 0, s>>>(partial.ptr, nblk, out);
  count_launch(2);
  check_launch("dot_many");
}

void axpy_many(double* y, const double* X, int64_t ldx, const double* coef, double sign, int64_t n, int k,
               cudaStream_t s) {
  if (k <= 0 || n <= 0) return;
  axpy_many_kernel<<<grid_for(n, 256), 256, 0, s>>>(y, X, ldx, coef, sign, n, k);
  count_launch();
  check_launch("axpy_many");
}

void vec_scale_add(double* y, const double* x, const double* noise, int64_t n, int nrhs, int64_t ld, cudaStream_t s) {
  if (n <= 0 || nrhs <= 0) return;
  noise_kernel<<<dim3(grid_for(n, 256), nrhs), 256, 0, s>>>(y, x, noise, n, ld);
  count_launch();
  check_launch("noise_kernel");
}

void fill(double* x, double v, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, v, n);
  count_launch();
}

void copy(double* dst, const double* src, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  GPFVM_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

void gather(double* dst, const double* src, const int64_t* idx, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  gather_kernel<<<grid_for(n, 256), 256, 0, s>>>(dst, src, idx, n);
  count_launch();
}

void scatter(double* dst, const double* src, const int64_t* idx, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  scatter_kernel<<<grid_for(n, 256), 256, 0, s>>>(dst, src, idx, n);
  count_launch();
}

}  // namespace gpfvm
