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

// ---- IterGP/PCG iteration with device-resident scalars ----
// state[ST_*] lives in device memory; every kernel returns immediately once
// state[ST_DONE] != 0, so the host only has to look at the state every few
// iterations (no per-iteration host synchronisation).
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[32];
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = (threadIdx.x < (blockDim.x >> 5)) ? ws[threadIdx.x] : 0.0;
  if (threadIdx.x < 32) t = warp_sum(t);
  return t;  // valid in thread 0
}

// c_j = (Kd_j . gd) / eta_j   (final pass of the reorthogonalisation dots)
__global__ void reorth_final_kernel(const double* __restrict__ partial, int nparts, const double* __restrict__ eta,
                                    double* __restrict__ c, const double* __restrict__ state) {
  if (state[ST_DONE] != 0.0) return;
  const int j = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[(int64_t)j * nparts + i];
  s = block_sum(s);
  if (threadIdx.x == 0) c[j] = s / eta[j];
}

// d' = d - sum_j c_j Kd_j ; g' = g - sum_j c_j Kg_j (written to the Krylov slot);
// partial sums of d'.g' and d'.r.  HBM-bound on the 2 w N reads of the kept
// actions: two consecutive elements per thread (16-byte loads) and four
// actions per step keep 16 loads in flight per thread (n, ld even, 16-byte
// aligned pointers: checked by the host wrapper; a scalar variant otherwise).
template <bool V2>
__global__ void __launch_bounds__(RED_THREADS) itergp_update_kernel(
    const double* __restrict__ d, const double* __restrict__ g, const double* __restrict__ Kd,
    const double* __restrict__ Kg, int64_t ld, int w, const double* __restrict__ c, const double* __restrict__ r,
    double* __restrict__ dout, double* __restrict__ gout, int64_t n, double* __restrict__ partial,
    const double* __restrict__ state) {
  if (state[ST_DONE] != 0.0) return;
  double s_eta = 0.0, s_del = 0.0;
  if (V2) {
    const int64_t n2 = n >> 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
      // projection first, then one subtraction (the rounding of axpy_many)
      double2 pd = make_double2(0.0, 0.0), pg = make_double2(0.0, 0.0);
      int j = 0;
      for (; j + 4 <= w; j += 4) {
        double2 kd[4], kg[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          kd[u] = __ldcs(reinterpret_cast<const double2*>(Kd + (j + u) * ld) + i);
          kg[u] = __ldcs(reinterpret_cast<const double2*>(Kg + (j + u) * ld) + i);
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const double cj = c[j + u];
          pd.x = fma(cj, kd[u].x, pd.x); pd.y = fma(cj, kd[u].y, pd.y);
          pg.x = fma(cj, kg[u].x, pg.x); pg.y = fma(cj, kg[u].y, pg.y);
        }
      }
      for (; j < w; j++) {
        const double cj = c[j];
        const double2 kd = __ldcs(reinterpret_cast<const double2*>(Kd + j * ld) + i);
        const double2 kg = __ldcs(reinterpret_cast<const double2*>(Kg + j * ld) + i);
        pd.x = fma(cj, kd.x, pd.x); pd.y = fma(cj, kd.y, pd.y);
        pg.x = fma(cj, kg.x, pg.x); pg.y = fma(cj, kg.y, pg.y);
      }
      const double2 dv2 = reinterpret_cast<const double2*>(d)[i], gv2 = reinterpret_cast<const double2*>(g)[i];
      const double2 rv = reinterpret_cast<const double2*>(r)[i];
      const double2 dn = make_double2(dv2.x - pd.x, dv2.y - pd.y), gn = make_double2(gv2.x - pg.x, gv2.y - pg.y);
      reinterpret_cast<double2*>(dout)[i] = dn;
      reinterpret_cast<double2*>(gout)[i] = gn;
      s_eta = fma(dn.x, gn.x, s_eta); s_eta = fma(dn.y, gn.y, s_eta);
      s_del = fma(dn.x, rv.x, s_del); s_del = fma(dn.y, rv.y, s_del);
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      double pd = 0.0, pg = 0.0;
      for (int j = 0; j < w; j++) {
        const double cj = c[j];
        pd = fma(cj, Kd[j * ld + i], pd);
        pg = fma(cj, Kg[j * ld + i], pg);
      }
      const double dv = d[i] - pd, gv = g[i] - pg;
      dout[i] = dv;
      gout[i] = gv;
      s_eta = fma(dv, gv, s_eta);
      s_del = fma(dv, r[i], s_del);
    }
  }
  s_eta = block_sum(s_eta);
  s_del = block_sum(s_del);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = s_eta;
    partial[gridDim.x + blockIdx.x] = s_del;
  }
}

// eta = d'.g', a = d'.r / eta; breakdown (eta <= 0 or not finite) stops the iteration
__global__ void itergp_update_final_kernel(const double* __restrict__ partial, int nparts, double* __restrict__ state,
                                           double* __restrict__ eta_slot) {
  if (state[ST_DONE] != 0.0) return;
  double se = 0.0, sd = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    se += partial[i];
    sd += partial[nparts + i];
  }
  se = block_sum(se);
  sd = block_sum(sd);
  if (threadIdx.x == 0) {
    if (!(se > 0.0) || !isfinite(se) || !isfinite(sd)) {
      state[ST_DONE] = 2.0;  // breakdown: the trace so far is kept
      return;
    }
    *eta_slot = se;
    state[ST_ETA] = se;
    state[ST_A] = sd / se;
  }
}

// x += a d', r -= a g', partial sums of r.r
__global__ void __launch_bounds__(RED_THREADS) itergp_step_kernel(double* __restrict__ x, double* __restrict__ r,
                                                                  const double* __restrict__ dn,
                                                                  const double* __restrict__ gn, int64_t n,
                                                                  double* __restrict__ partial,
                                                                  const double* __restrict__ state) {
  if (state[ST_DONE] != 0.0) return;
  const double a = state[ST_A];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(a, dn[i], x[i]);
    const double rv = fma(-a, gn[i], r[i]);
    r[i] = rv;
    s = fma(rv, rv, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// ||r||, convergence flag, iteration counter
__global__ void itergp_step_final_kernel(const double* __restrict__ partial, int nparts, double* __restrict__ state) {
  if (state[ST_DONE] != 0.0) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    const double nr = sqrt(s);
    state[ST_NR] = nr;
    state[ST_COUNT] += 1.0;
    if (nr <= state[ST_THR]) state[ST_DONE] = 1.0;
  }
}

// ||y|| and the initial state
__global__ void itergp_init_kernel(const double* __restrict__ partial, int nparts, double rtol, double* __restrict__ state) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    const double ny = sqrt(s);
    state[ST_NY] = ny;
    state[ST_NR] = ny;
    state[ST_THR] = rtol * ny;
    state[ST_COUNT] = 0.0;
    state[ST_A] = state[ST_ETA] = 0.0;
    state[ST_DONE] = (ny == 0.0 || ny <= rtol * ny) ? 1.0 : 0.0;
  }
}

__global__ void iter_coefs_kernel(const double* __restrict__ dots, int w, const double* __restrict__ eta,
                                  double* __restrict__ c, const double* __restrict__ state) {
  if (state[ST_DONE] != 0.0) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < w; j += gridDim.x * blockDim.x) c[j] = dots[j] / eta[j];
}

unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8));
}
}  // namespace

int red_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(RED_BLOCKS, (n + 4 * RED_THREADS - 1) / (4 * RED_THREADS)));
}

void dot_many(const double* X, int64_t ldx, const double* v, int64_t n, int k, double* out, cudaStream_t s) {
  if (k <= 0) return;
  // blocks per dot from the length (>= 4 elements per thread), so short dots
  // (e.g. the n_b-long rows of S^{-1}) do not launch 296 near-empty CTAs each;
  // fixed for a given n, hence still deterministic
  const int nblk = red_blocks(n);
  DevBuf& partial = scratch(s, 0);
  partial.ensure((size_t)RED_BLOCKS * k);
  dot_partial_kernel<<<dim3(nblk, k), RED_THREADS, 0, s>>>(X, ldx, v, n, partial.ptr);
  dot_final_kernel<<<k, 512, 0, s>>>(partial.ptr, nblk, out);
  count_launch(2);
  check_launch("dot_many");
}

void itergp_init(const double* y, int64_t n, double rtol, double* state, cudaStream_t s) {
  const int nblk = red_blocks(n);
  DevBuf& partial = scratch(s, 3);
  partial.ensure((size_t)2 * RED_BLOCKS);
  dot_partial_kernel<<<dim3(nblk, 1), RED_THREADS, 0, s>>>(y, n, y, n, partial.ptr);
  itergp_init_kernel<<<1, 256, 0, s>>>(partial.ptr, nblk, rtol, state);
  count_launch(2);
  check_launch("itergp_init");
}

void itergp_reorth_coefs(const double* Kd, int64_t ld, int w, const double* gd, int64_t n, const double* eta,
                         double* c, const double* state, cudaStream_t s) {
  if (w <= 0) return;
  const int nblk = red_blocks(n);
  DevBuf& partial = scratch(s, 4);
  partial.ensure((size_t)RED_BLOCKS * w);
  dot_partial_kernel<<<dim3(nblk, w), RED_THREADS, 0, s>>>(Kd, ld, gd, n, partial.ptr);
  reorth_final_kernel<<<w, 256, 0, s>>>(partial.ptr, nblk, eta, c, state);
  count_launch(2);
  check_launch("itergp_reorth_coefs");
}

// the fused update pass; block partial sums [eta..][delta..] into scratch, returns the block count
static int itergp_update_blocks(const double* d, const double* g, const double* Kd, const double* Kg, int64_t ld,
                                int w, const double* c, const double* r, double* dout, double* gout, int64_t n,
                                const double* state, double** partial_out, cudaStream_t s);

void itergp_update(const double* d, const double* g, const double* Kd, const double* Kg, int64_t ld, int w,
                   const double* c, const double* r, double* dout, double* gout, int64_t n, double* state,
                   double* eta_slot, cudaStream_t s) {
  double* part = nullptr;
  const int nblk = itergp_update_blocks(d, g, Kd, Kg, ld, w, c, r, dout, gout, n, state, &part, s);
  itergp_update_final_kernel<<<1, 256, 0, s>>>(part, nblk, state, eta_slot);
  count_launch();
  check_launch("itergp_update");
}

static int itergp_update_blocks(const double* d, const double* g, const double* Kd, const double* Kg, int64_t ld,
                                int w, const double* c, const double* r, double* dout, double* gout, int64_t n,
                                const double* state, double** partial_out, cudaStream_t s) {
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool v2 = (n % 2 == 0) && (ld % 2 == 0) && a16(d) && a16(g) && a16(Kd) && a16(Kg) && a16(r) && a16(dout) &&
                  a16(gout);
  // enough CTAs to keep 2 w N streaming loads in flight (8 per SM), fixed for
  // a given n so the reduction order (and the scalars) stay deterministic
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n / (v2 ? 2 : 1) + RED_THREADS - 1) / RED_THREADS));
  DevBuf& partial = scratch(s, 5);
  partial.ensure((size_t)2 * 148 * 8);
  if (v2)
    itergp_update_kernel<true><<<nblk, RED_THREADS, 0, s>>>(d, g, Kd, Kg, ld, w, c, r, dout, gout, n, partial.ptr, state);
  else
    itergp_update_kernel<false><<<nblk, RED_THREADS, 0, s>>>(d, g, Kd, Kg, ld, w, c, r, dout, gout, n, partial.ptr, state);
  count_launch();
  *partial_out = partial.ptr;
  return nblk;
}

void itergp_step(double* x, double* r, const double* dn, const double* gn, int64_t n, double* state, cudaStream_t s) {
  const int nblk = red_blocks(n);
  DevBuf& partial = scratch(s, 3);
  partial.ensure((size_t)2 * RED_BLOCKS);
  itergp_step_kernel<<<nblk, RED_THREADS, 0, s>>>(x, r, dn, gn, n, partial.ptr, state);
  itergp_step_final_kernel<<<1, 256, 0, s>>>(partial.ptr, nblk, state);
  count_launch(2);
  check_launch("itergp_step");
}

// ---- C ABI: the iteration steps with explicit partial sums (sharded solve) ----
template <class F>
static int guarded_vec(F&& f) {
  try {
    f();
    return GPFVM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  }
}

}  // namespace gpfvm

extern "C" {
using namespace gpfvm;

int gpfvm_iter_init(const double* yy, double rtol, double* state, void* stream) {
  return guarded_vec([&] {
    GPFVM_CHECK(yy && state, GPFVM_ERR_INVALID, "null argument");
    itergp_init_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(yy, 1, rtol, state);
    count_launch();
    check_launch("gpfvm_iter_init");
  });
}

int gpfvm_iter_coefs(const double* dots, int w, const double* eta, double* c, const double* state, void* stream) {
  return guarded_vec([&] {
    GPFVM_CHECK(w >= 0 && (w == 0 || (dots && eta && c)) && state, GPFVM_ERR_INVALID, "bad arguments");
    if (w == 0) return;
    iter_coefs_kernel<<<(w + 255) / 256, 256, 0, (cudaStream_t)stream>>>(dots, w, eta, c, state);
    count_launch();
    check_launch("gpfvm_iter_coefs");
  });
}

int gpfvm_iter_update_local(const double* d, const double* g, const double* Kd, const double* Kg, int64_t ld, int w,
                            const double* c, const double* r, double* dout, double* gout, int64_t n, double* partial,
                            const double* state, void* stream) {
  return guarded_vec([&] {
    GPFVM_CHECK(d && g && r && dout && gout && partial && state && n >= 0 && w >= 0 && (w == 0 || (Kd && Kg && c)),
                GPFVM_ERR_INVALID, "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    double* part = nullptr;
    const int nblk = itergp_update_blocks(d, g, Kd, Kg, ld, w, c, r, dout, gout, n, state, &part, s);
    dot_final_kernel<<<2, 512, 0, s>>>(part, nblk, partial);  // [eta, delta] local sums
    count_launch();
    check_launch("gpfvm_iter_update_local");
  });
}

int gpfvm_iter_update_final(const double* sums, double* state, double* eta_slot, void* stream) {
  return guarded_vec([&] {
    GPFVM_CHECK(sums && state && eta_slot, GPFVM_ERR_INVALID, "null argument");
    itergp_update_final_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(sums, 1, state, eta_slot);
    count_launch();
    check_launch("gpfvm_iter_update_final");
  });
}

int gpfvm_iter_step_local(double* x, double* r, const double* dn, const double* gn, int64_t n, double* partial,
                          const double* state, void* stream) {
  return guarded_vec([&] {
    GPFVM_CHECK(x && r && dn && gn && partial && state && n >= 0, GPFVM_ERR_INVALID, "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    const int nblk = red_blocks(n);
    DevBuf& part = scratch(s, 3);
    part.ensure((size_t)2 * RED_BLOCKS);
    itergp_step_kernel<<<nblk, RED_THREADS, 0, s>>>(x, r, dn, gn, n, part.ptr, state);
    dot_final_kernel<<<1, 512, 0, s>>>(part.ptr, nblk, partial);
    count_launch(2);
    check_launch("gpfvm_iter_step_local");
  });
}

int gpfvm_iter_step_final(const double* sum, double* state, void* stream) {
  return guarded_vec([&] {
    GPFVM_CHECK(sum && state, GPFVM_ERR_INVALID, "null argument");
    itergp_step_final_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(sum, 1, state);
    count_launch();
    check_launch("gpfvm_iter_step_final");
  });
}

}  // extern "C"

namespace gpfvm {

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
