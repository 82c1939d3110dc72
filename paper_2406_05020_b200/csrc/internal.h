// Internal declarations shared by the libgpfvm translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/gpfvm.h"
#include "dd.cuh"

namespace gpfvm {

// ---- errors -----------------------------------------------------------------
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};

#define GPFVM_CUDA(call)                                                                  \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::gpfvm::Error{GPFVM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + \
                                               " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
  } while (0)

#define GPFVM_CHECK(cond, code, msg)                  \
  do {                                                \
    if (!(cond)) throw ::gpfvm::Error{(code), (msg)}; \
  } while (0)

extern std::atomic<int64_t> g_launches;
inline void count_launch(int64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void check_launch(const char* what);

// ---- device buffer -------------------------------------------------------------
// Device allocations go through a size-bucketed caching pool: releasing a
// buffer returns it to the pool instead of calling cudaFree (which would
// synchronise the whole device and serialise concurrent streams).  A pooled
// block is handed out again only to a later allocation; temporaries are
// released after the stream that used them has been synchronised or when the
// next user is on the same stream (stream order), as everywhere in this library.
void* pool_alloc(size_t bytes);              // on the current device
void pool_free(void* p, size_t bytes, int dev);  // back to the bucket of the device it came from
void pool_trim();  // cudaFree every cached block of the current device
int current_device();

struct DevBuf {
  double* ptr = nullptr;
  size_t n = 0;
  int dev = -1;  // device the block was allocated on
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n), dev(o.dev) { o.ptr = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); ptr = o.ptr; n = o.n; dev = o.dev; o.ptr = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) pool_free(ptr, n * sizeof(double), dev);
    ptr = nullptr;
    n = 0;
  }
  void ensure(size_t count) {
    if (count <= n && (ptr == nullptr || dev == current_device())) return;
    release();
    if (count == 0) return;
    ptr = static_cast<double*>(pool_alloc(count * sizeof(double)));
    n = count;
    dev = current_device();
  }
};
// Scratch buffer private to (calling thread, current device, stream, slot):
// library-internal temporaries of stream-ordered calls (no sharing across
// devices or concurrently used streams).
DevBuf& scratch(cudaStream_t s, int slot);

// ---- Matérn parameters in double-double ----------------------------------------
struct MaternDD {
  int q;
  dd lam;
  dd a[4];  // k(d) = exp(-lam d) * sum_k a[k] d^k  for d >= 0
};
MaternDD matern_dd(int q, double lengthscale, double variance);

// site list resident on the device
struct Sites {
  int kind = GPFVM_SITE_INTERVAL;
  int n = 0;
  std::vector<double> lo, hi;
  DevBuf d_lo, d_hi;
};

void launch_factor(const MaternDD& K, const Sites& L, int mL, const Sites& R, int mR, double* out,
                   int64_t ld, cudaStream_t s);

// ---- GEMM ------------------------------------------------------------------------
// C[b] = alpha * sum_seg A_seg[b] * B_seg[b] + beta * C[b]; b = (b1, b2, b3),
// element strides; A_seg = A + seg * a_sg, B_seg = B + seg * b_sg.
struct Gemm {
  int M = 0, N = 0, K = 0;
  int nseg = 1;
  int batch1 = 1, batch2 = 1, batch3 = 1;
  const double* A = nullptr;
  int64_t a_rs = 0, a_cs = 0, a_b1 = 0, a_b2 = 0, a_b3 = 0, a_sg = 0;
  const double* B = nullptr;
  int64_t b_rs = 0, b_cs = 0, b_b1 = 0, b_b2 = 0, b_b3 = 0, b_sg = 0;
  double* C = nullptr;
  int64_t c_rs = 0, c_cs = 0, c_b1 = 0, c_b2 = 0, c_b3 = 0;
  double alpha = 1.0, beta = 0.0;
  // optional extra term  C[b] += alpha * A2[b] B2[b]^T  (A2: M x K2 rows a2_rs,
  // B2: N x K2 rows b2_rs, both K-contiguous, one batch level): a low-rank
  // update appended to the contraction as extra k-tiles
  int K2 = 0;
  const double* A2 = nullptr;
  int64_t a2_rs = 0, a2_b1 = 0;
  const double* B2 = nullptr;
  int64_t b2_rs = 0, b2_b1 = 0;
};
void run_gemm(const Gemm& g, cudaStream_t s);
bool try_tma_gemm(const Gemm& g, cudaStream_t s);  // gemm_tma.cu (TMA + mbarrier DMMA kernel)
double gemm_flops(const Gemm& g);

// ---- small dense linear algebra (linalg.cu) ---------------------------------------
// In-place lower Cholesky of an n x n row-major SPD matrix (strict upper part zeroed).
// Returns 0 on success, or the (1-based) failing column.
int cholesky_inplace(double* A, int n, cudaStream_t s, int* d_info);
// Solve L L^T X = B in place (B: n x nrhs, row-major, ld = nrhs) with L from cholesky_inplace.
void cholesky_solve(const double* L, int n, double* B, int nrhs, cudaStream_t s);
// X <- L^{-1} X  (forward substitution only)
void trsm_lower(const double* L, int n, double* B, int nrhs, cudaStream_t s);
// X <- U^{-1} X with U upper triangular (row-major, e.g. U = L^T)
void trsm_upper(const double* U, int n, double* B, int nrhs, cudaStream_t s);
// B (cols x rows) = A^T, A rows x cols, both row-major
void transpose(const double* A, double* B, int rows, int cols, cudaStream_t s);
// Generalised symmetric-definite eigenproblem  A V = Bm V diag(w),  V^T Bm V = I.
// A, Bm: n x n row-major device; V: n x n row-major device (columns = eigenvectors); w: n.
void sygv(const double* A, const double* Bm, int n, double* V, double* w, cudaStream_t s);

// ---- vector ops (vecops.cu) --------------------------------------------------------
void vec_scale_add(double* y, const double* x, const double* noise, int64_t n, int nrhs, int64_t ld,
                   cudaStream_t s);  // y = noise .* x (per rhs)
void dot_many(const double* X, int64_t ldx, const double* v, int64_t n, int k, double* out,
              cudaStream_t s);  // out[j] = X_j . v   (j < k)
void axpy_many(double* y, const double* X, int64_t ldx, const double* coef, double sign, int64_t n,
               int k, cudaStream_t s);  // y += sign * sum_j coef[j] X_j
// IterGP/PCG iteration kernels with device-resident scalars: state[ST_*]
enum { ST_NY = 0, ST_NR = 1, ST_THR = 2, ST_A = 3, ST_ETA = 4, ST_DONE = 5, ST_COUNT = 6, ST_SIZE = 8 };
void itergp_init(const double* y, int64_t n, double rtol, double* state, cudaStream_t s);  // ||y||, flags
// c_j = Kd_j . gd / eta_j (j < w)
void itergp_reorth_coefs(const double* Kd, int64_t ld, int w, const double* gd, int64_t n, const double* eta,
                         double* c, const double* state, cudaStream_t s);
// dout = d - sum c_j Kd_j, gout = g - sum c_j Kg_j; eta = dout.gout -> *eta_slot, a = dout.r / eta
void itergp_update(const double* d, const double* g, const double* Kd, const double* Kg, int64_t ld, int w,
                   const double* c, const double* r, double* dout, double* gout, int64_t n, double* state,
                   double* eta_slot, cudaStream_t s);
// x += a dn, r -= a gn, ||r|| -> state, convergence flag, iteration counter
void itergp_step(double* x, double* r, const double* dn, const double* gn, int64_t n, double* state, cudaStream_t s);
void fill(double* x, double v, int64_t n, cudaStream_t s);
void copy(double* dst, const double* src, int64_t n, cudaStream_t s);
void gather(double* dst, const double* src, const int64_t* idx, int64_t n, cudaStream_t s);
void scatter(double* dst, const double* src, const int64_t* idx, int64_t n, cudaStream_t s);

}  // namespace gpfvm
