// Small dense FP64 linear algebra for the preconditioner:
//   * blocked right-looking Cholesky (panel in one CTA, trailing update on DMMA GEMM)
//   * blocked triangular solves (diagonal block per column thread, GEMM updates)
//   * symmetric eigensolver: block one-sided (Hestenes) Jacobi — each CTA
//     orthogonalises a pair of 16-column blocks held in shared memory
//     (Gram -> in-smem parallel cyclic Jacobi -> rotate columns), tournament
//     ordering across CTAs; converged columns X = C V = V diag(lambda).
//   * generalised symmetric-definite eigenproblem via Cholesky reduction.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace gpfvm {

namespace {

constexpr int PB = 32;  // panel width

__global__ void potrf_diag_kernel(double* A, int n, int k, int kb, int* info) {
  __shared__ double s[PB][PB + 1];
  int t = threadIdx.x;
  for (int i = t; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    s[r][c] = A[(int64_t)(k + r) * n + k + c];
  }
  __syncthreads();
  for (int j = 0; j < kb; j++) {
    if (t == 0) {
      double d = s[j][j];
      if (!(d > 0.0)) {
        if (*info == 0) *info = k + j + 1;
        d = NAN;
      }
      s[j][j] = sqrt(d);
    }
    __syncthreads();
    double ljj = s[j][j];
    for (int r = j + 1 + t; r < kb; r += blockDim.x) s[r][j] /= ljj;
    __syncthreads();
    // update trailing columns of the diagonal block
    for (int i = t; i < kb * kb; i += blockDim.x) {
      int r = i / kb, c = i % kb;
      if (c > j && r >= c) s[r][c] -= s[r][j] * s[c][j];
    }
    __syncthreads();
  }
  for (int i = t; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    A[(int64_t)(k + r) * n + k + c] = (c <= r) ? s[r][c] : 0.0;
  }
}

// rows r >= k+kb:  A[r, k:k+kb] <- A[r, k:k+kb] L11^{-T}
__global__ void potrf_panel_kernel(double* A, int n, int k, int kb) {
  __shared__ double L[PB][PB + 1];
  for (int i = threadIdx.x; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    L[r][c] = A[(int64_t)(k + r) * n + k + c];
  }
  __syncthreads();
  int r = k + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[PB];
  double* row = A + (int64_t)r * n + k;
  for (int j = 0; j < kb; j++) {
    double v = row[j];
    for (int i = 0; i < j; i++) v -= x[i] * L[j][i];
    x[j] = v / L[j][j];
  }
  for (int j = 0; j < kb; j++) row[j] = x[j];
}

// Forward substitution on a diagonal block: B[k:k+kb, c] <- L11^{-1} B[k:k+kb, c]
__global__ void trsm_lower_diag_kernel(const double* L, int n, double* B, int nrhs, int k, int kb) {
  __shared__ double s[PB][PB + 1];
  for (int i = threadIdx.x; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    s[r][c] = L[(int64_t)(k + r) * n + k + c];
  }
  __syncthreads();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  double x[PB];
  for (int i = 0; i < kb; i++) {
    double v = B[(int64_t)(k + i) * nrhs + c];
    for (int j = 0; j < i; j++) v -= s[i][j] * x[j];
    x[i] = v / s[i][i];
    B[(int64_t)(k + i) * nrhs + c] = x[i];
  }
}

// Backward substitution with U = L^T (U upper, row-major): B[k:k+kb] <- U11^{-1} B[k:k+kb]
__global__ void trsm_upper_diag_kernel(const double* U, int n, double* B, int nrhs, int k, int kb) {
  __shared__ double s[PB][PB + 1];
  for (int i = threadIdx.x; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    s[r][c] = U[(int64_t)(k + r) * n + k + c];
  }
  __syncthreads();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  double x[PB];
  for (int i = kb - 1; i >= 0; i--) {
    double v = B[(int64_t)(k + i) * nrhs + c];
    for (int j = i + 1; j < kb; j++) v -= s[i][j] * x[j];
    x[i] = v / s[i][i];
    B[(int64_t)(k + i) * nrhs + c] = x[i];
  }
}

__global__ void transpose_kernel(const double* __restrict__ A, double* __restrict__ B, int rows, int cols) {
  __shared__ double t[32][33];
  int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int r = by + j, c = bx + threadIdx.x;
    if (r < rows && c < cols) t[j][threadIdx.x] = A[(int64_t)r * cols + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int r = bx + j, c = by + threadIdx.x;  // B is cols x rows
    if (r < cols && c < rows) B[(int64_t)r * rows + c] = t[threadIdx.x][j];
  }
}

__global__ void symmetrize_kernel(double* A, int n) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int r = (int)(idx / n), c = (int)(idx % n);
  if (c <= r) return;
  double v = 0.5 * (A[(int64_t)r * n + c] + A[(int64_t)c * n + r]);
  A[(int64_t)r * n + c] = v;
  A[(int64_t)c * n + r] = v;
}

__global__ void zero_upper_kernel(double* A, int n) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  if ((idx % n) > (idx / n)) A[idx] = 0.0;
}

__global__ void eye_kernel(double* A, int n) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  A[idx] = ((idx / n) == (idx % n)) ? 1.0 : 0.0;
}

// ---- block one-sided Jacobi ----------------------------------------------------
constexpr int JB = 16;          // columns per block
constexpr int JC = 2 * JB;      // columns per CTA (pair of blocks)
constexpr int JT = 256;         // threads per CTA (<= 255 registers: no spills in the X.Q update)
__constant__ int c_inner_sweeps = 1;

// Xc, Vc: column-major n x n (column j at Xc + j*n).  pairs: (blk_a, blk_b) per CTA.
__global__ void __launch_bounds__(JT) jacobi_round_kernel(double* Xc, double* Vc, int n, int nblk,
                                                          const int* __restrict__ pairs,
                                                          unsigned long long* offmax) {
  extern __shared__ double sm[];
  double* Xs = sm;                  // [JC][n] column-major (column c at Xs + c*n)
  double* H = Xs + (size_t)JC * n;  // [JC][JC+1]
  double* Q = H + JC * (JC + 1);    // [JC][JC+1]
  __shared__ double cs[JC / 2], sn[JC / 2];
  __shared__ int col_of[JC];
  __shared__ int cnt_s;
  const int t = threadIdx.x;
  const int pa = pairs[2 * blockIdx.x], pb = pairs[2 * blockIdx.x + 1];
  if (t == 0) {
    int c = 0;
    for (int b : {pa, pb}) {
      if (b < 0) continue;
      int j0 = b * JB, j1 = min(n, j0 + JB);
      for (int j = j0; j < j1; j++) col_of[c++] = j;
    }
    cnt_s = c;
  }
  __syncthreads();
  const int cnt = cnt_s;
  if (cnt < 2) return;
  // load columns
  for (int i = t; i < cnt * n; i += JT) {
    int c = i / n, r = i % n;
    Xs[(size_t)c * n + r] = Xc[(size_t)col_of[c] * n + r];
  }
  __syncthreads();
  // Gram H = Xs^T Xs: one warp per (a, b) entry, lanes stride the rows
  // (consecutive lanes -> consecutive banks), shuffle reduction.
  {
    const int warp = t >> 5, lane = t & 31, nw = JT / 32;
    const int npair = cnt * (cnt + 1) / 2;
    for (int e = warp; e < npair; e += nw) {
      int a = 0, rem = e;
      while (rem >= cnt - a) { rem -= cnt - a; a++; }
      int b = a + rem;
      const double* xa = Xs + (size_t)a * n;
      const double* xb = Xs + (size_t)b * n;
      double s = 0.0;
      for (int r = lane; r < n; r += 32) s = fma(xa[r], xb[r], s);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        H[a * (JC + 1) + b] = s;
        H[b * (JC + 1) + a] = s;
      }
    }
  }
  for (int i = t; i < JC * (JC + 1); i += JT) Q[i] = 0.0;
  __syncthreads();
  for (int i = t; i < cnt; i += JT) Q[i * (JC + 1) + i] = 1.0;
  // convergence measure (only pairs across the two blocks + within: all)
  if (t < 32) {
    double m = 0.0;
    for (int i = t; i < cnt * cnt; i += 32) {
      int a = i / cnt, b = i % cnt;
      if (b <= a) continue;
      double d = sqrt(fabs(H[a * (JC + 1) + a]) * fabs(H[b * (JC + 1) + b]));
      double v = (d > 0.0) ? fabs(H[a * (JC + 1) + b]) / d : 0.0;
      m = fmax(m, v);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (t == 0) atomicMax(offmax, (unsigned long long)__double_as_longlong(m));
  }
  __syncthreads();
  // parallel cyclic two-sided Jacobi on H (cnt x cnt), round-robin pairing
  const int m = (cnt + 1) & ~1;  // even player count (a dummy if cnt odd)
  const int inner_sweeps = c_inner_sweeps;
  for (int sweep = 0; sweep < inner_sweeps; sweep++) {
    __shared__ int done;
    if (t == 0) done = 1;
    __syncthreads();
    for (int rnd = 0; rnd < m - 1; rnd++) {
      // pairs: player 0 fixed, others rotate
      if (t < m / 2) {
        int a = (t == 0) ? 0 : 1 + ((t - 1 + rnd) % (m - 1));
        int b = 1 + ((m - 2 - t + rnd) % (m - 1));
        int p = min(a, b), q = max(a, b);
        double c = 1.0, s = 0.0;
        if (q < cnt) {
          double hpp = H[p * (JC + 1) + p], hqq = H[q * (JC + 1) + q], hpq = H[p * (JC + 1) + q];
          if (fabs(hpq) > 1e-300 && fabs(hpq) > 1e-16 * sqrt(fabs(hpp * hqq))) {
            double zeta = (hqq - hpp) / (2.0 * hpq);
            double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = 1.0 / sqrt(1.0 + tt * tt);
            s = c * tt;
            done = 0;
          }
        }
        cs[t] = c;
        sn[t] = s;
        col_of[2 * t] = p;  // reuse as pair table (col_of no longer needed... keep copy below)
        col_of[2 * t + 1] = q;
      }
      __syncthreads();
      // columns: H <- H J ; Q <- Q J   (for each pair, each row)
      for (int i = t; i < (m / 2) * cnt; i += JT) {
        int pr = i / cnt, r = i % cnt;
        int p = col_of[2 * pr], q = col_of[2 * pr + 1];
        if (q >= cnt) continue;
        double c = cs[pr], s = sn[pr];
        double hp = H[r * (JC + 1) + p], hq = H[r * (JC + 1) + q];
        H[r * (JC + 1) + p] = c * hp - s * hq;
        H[r * (JC + 1) + q] = s * hp + c * hq;
        double qp = Q[r * (JC + 1) + p], qq = Q[r * (JC + 1) + q];
        Q[r * (JC + 1) + p] = c * qp - s * qq;
        Q[r * (JC + 1) + q] = s * qp + c * qq;
      }
      __syncthreads();
      // rows: H <- J^T H
      for (int i = t; i < (m / 2) * cnt; i += JT) {
        int pr = i / cnt, r = i % cnt;
        int p = col_of[2 * pr], q = col_of[2 * pr + 1];
        if (q >= cnt) continue;
        double c = cs[pr], s = sn[pr];
        double hp = H[p * (JC + 1) + r], hq = H[q * (JC + 1) + r];
        H[p * (JC + 1) + r] = c * hp - s * hq;
        H[q * (JC + 1) + r] = s * hp + c * hq;
      }
      __syncthreads();
    }
    if (done) break;
  }
  // restore column ids
  if (t == 0) {
    int c = 0;
    for (int b : {pa, pb}) {
      if (b < 0) continue;
      int j0 = b * JB, j1 = min(n, j0 + JB);
      for (int j = j0; j < j1; j++) col_of[c++] = j;
    }
  }
  __syncthreads();
  // X <- X Q, then V <- V Q (V staged through the same shared buffer).  Rows
  // in parallel; per row JC independent register accumulators (fully unrolled,
  // no local-memory arrays), operands from shared memory (X column-major:
  // consecutive rows -> consecutive banks; Q broadcast).  Unused columns
  // (cnt < JC) carry zeros in Q.
  for (int pass = 0; pass < 2; pass++) {
    double* dst = pass == 0 ? Xc : Vc;
    if (pass == 1) {
      __syncthreads();
      for (int i = t; i < cnt * n; i += JT) {
        int c = i / n, r = i % n;
        Xs[(size_t)c * n + r] = Vc[(size_t)col_of[c] * n + r];
      }
      __syncthreads();
    }
    for (int r = t; r < n; r += JT) {
      double acc[JC];
#pragma unroll
      for (int j = 0; j < JC; j++) acc[j] = 0.0;
#pragma unroll
      for (int c = 0; c < JC; c++) {
        const double xv = (c < cnt) ? Xs[(size_t)c * n + r] : 0.0;
#pragma unroll
        for (int j = 0; j < JC; j++) acc[j] = fma(xv, Q[c * (JC + 1) + j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < JC; j++)
        if (j < cnt) dst[(size_t)col_of[j] * n + r] = acc[j];
    }
  }
}

__global__ void colnorm_kernel(const double* Xc, int n, double* w, bool squared) {
  int j = blockIdx.x;
  double s = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) s = fma(Xc[(size_t)j * n + r], Xc[(size_t)j * n + r], s);
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) w[j] = squared ? red[0] : sqrt(red[0]);
}

}  // namespace

int cholesky_inplace(double* A, int n, cudaStream_t s, int* d_info) {
  GPFVM_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), s));
  for (int k = 0; k < n; k += PB) {
    int kb = std::min(PB, n - k);
    potrf_diag_kernel<<<1, 256, 0, s>>>(A, n, k, kb, d_info);
    count_launch();
    int rest = n - k - kb;
    if (rest > 0) {
      potrf_panel_kernel<<<(rest + 127) / 128, 128, 0, s>>>(A, n, k, kb);
      count_launch();
      Gemm g;
      g.M = rest; g.N = rest; g.K = kb;
      g.A = A + (int64_t)(k + kb) * n + k; g.a_rs = n; g.a_cs = 1;
      g.B = A + (int64_t)(k + kb) * n + k; g.b_rs = 1; g.b_cs = n;  // L21^T
      g.C = A + (int64_t)(k + kb) * n + k + kb; g.c_rs = n; g.c_cs = 1;
      g.alpha = -1.0; g.beta = 1.0;
      run_gemm(g, s);
    }
  }
  zero_upper_kernel<<<(unsigned)(((int64_t)n * n + 255) / 256), 256, 0, s>>>(A, n);
  count_launch();
  check_launch("cholesky");
  int info = 0;
  GPFVM_CUDA(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, s));
  GPFVM_CUDA(cudaStreamSynchronize(s));
  return info;
}

void trsm_lower(const double* L, int n, double* B, int nrhs, cudaStream_t s) {
  for (int k = 0; k < n; k += PB) {
    int kb = std::min(PB, n - k);
    trsm_lower_diag_kernel<<<(nrhs + 127) / 128, 128, 0, s>>>(L, n, B, nrhs, k, kb);
    count_launch();
    int rest = n - k - kb;
    if (rest > 0) {
      Gemm g;
      g.M = rest; g.N = nrhs; g.K = kb;
      g.A = L + (int64_t)(k + kb) * n + k; g.a_rs = n; g.a_cs = 1;
      g.B = B + (int64_t)k * nrhs; g.b_rs = nrhs; g.b_cs = 1;
      g.C = B + (int64_t)(k + kb) * nrhs; g.c_rs = nrhs; g.c_cs = 1;
      g.alpha = -1.0; g.beta = 1.0;
      run_gemm(g, s);
    }
  }
  check_launch("trsm_lower");
}

void trsm_upper(const double* U, int n, double* B, int nrhs, cudaStream_t s) {
  int last = ((n - 1) / PB) * PB;
  for (int k = last; k >= 0; k -= PB) {
    int kb = std::min(PB, n - k);
    trsm_upper_diag_kernel<<<(nrhs + 127) / 128, 128, 0, s>>>(U, n, B, nrhs, k, kb);
    count_launch();
    if (k > 0) {
      Gemm g;
      g.M = k; g.N = nrhs; g.K = kb;
      g.A = U + k; g.a_rs = n; g.a_cs = 1;  // U[0:k, k:k+kb]
      g.B = B + (int64_t)k * nrhs; g.b_rs = nrhs; g.b_cs = 1;
      g.C = B; g.c_rs = nrhs; g.c_cs = 1;
      g.alpha = -1.0; g.beta = 1.0;
      run_gemm(g, s);
    }
  }
  check_launch("trsm_upper");
}

void transpose(const double* A, double* B, int rows, int cols, cudaStream_t s) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(A, B, rows, cols);
  count_launch();
}

void cholesky_solve(const double* L, int n, double* B, int nrhs, cudaStream_t s) {
  trsm_lower(L, n, B, nrhs, s);
  DevBuf U;
  U.ensure((size_t)n * n);
  transpose(L, U.ptr, n, n, s);
  trsm_upper(U.ptr, n, B, nrhs, s);
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

// One-sided (Hestenes) block Jacobi on the columns of X (column-major n x n):
// X W = U Sigma.  Eigenvectors of X^T X are the columns of W (returned row-major
// in V, eigenvectors in columns); w = Sigma^2 (squared = true) or Sigma.
static void jacobi_cols(const double* X0, int n, double* V, double* w, bool squared, cudaStream_t s) {
  DevBuf Xc, Vc;
  Xc.ensure((size_t)n * n);
  Vc.ensure((size_t)n * n);
  GPFVM_CUDA(cudaMemcpyAsync(Xc.ptr, X0, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  eye_kernel<<<(unsigned)(((int64_t)n * n + 255) / 256), 256, 0, s>>>(Vc.ptr, n);
  count_launch();
  int nblk = (n + JB - 1) / JB;
  int players = nblk + (nblk & 1);
  std::vector<std::vector<int>> rounds;
  for (int r = 0; r < players - 1; r++) {
    std::vector<int> pr;
    for (int i = 0; i < players / 2; i++) {
      int a = (i == 0) ? 0 : 1 + ((i - 1 + r) % (players - 1));
      int b = 1 + ((players - 2 - i + r) % (players - 1));
      pr.push_back(a < nblk ? a : -1);
      pr.push_back(b < nblk ? b : -1);
    }
    rounds.push_back(pr);
  }
  int* d_pairs = nullptr;
  unsigned long long* d_off = nullptr;
  GPFVM_CUDA(cudaMalloc(&d_pairs, sizeof(int) * players * (players - 1) + sizeof(int)));
  GPFVM_CUDA(cudaMalloc(&d_off, sizeof(unsigned long long)));
  for (int r = 0; r < players - 1; r++)
    GPFVM_CUDA(cudaMemcpyAsync(d_pairs + r * players, rounds[r].data(), sizeof(int) * players,
                               cudaMemcpyHostToDevice, s));
  size_t smem = sizeof(double) * ((size_t)JC * n + 2 * JC * (JC + 1));
  GPFVM_CHECK(smem <= 227 * 1024, GPFVM_ERR_UNSUPPORTED, "eigensolver: dimension too large (n > 800)");
  GPFVM_CUDA(cudaFuncSetAttribute(jacobi_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int sweeps = 0;
  double offd = 1.0;
  if (getenv("GPFVM_INNER")) { int v = atoi(getenv("GPFVM_INNER")); GPFVM_CUDA(cudaMemcpyToSymbol(c_inner_sweeps, &v, sizeof(int))); }
  for (int sweep = 0; sweep < 40; sweep++) {
    sweeps++;
    GPFVM_CUDA(cudaMemsetAsync(d_off, 0, sizeof(unsigned long long), s));
    for (int r = 0; r < players - 1; r++) {
      jacobi_round_kernel<<<players / 2, JT, smem, s>>>(Xc.ptr, Vc.ptr, n, nblk, d_pairs + r * players, d_off);
      count_launch();
    }
    check_launch("jacobi_round_kernel");
    unsigned long long off = 0;
    GPFVM_CUDA(cudaMemcpyAsync(&off, d_off, sizeof(off), cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
    memcpy(&offd, &off, sizeof(double));
    if (getenv("GPFVM_DEBUG") && atoi(getenv("GPFVM_DEBUG")) > 1) fprintf(stderr, "[gpfvm]   sweep %d off %.3e\n", sweep, offd);
    // one-sided Jacobi orthogonality floor ~ n eps (rounding of the column dots)
    if (offd < std::max(4e-15, 2e-16 * n)) break;
  }
  if (getenv("GPFVM_DEBUG")) fprintf(stderr, "[gpfvm] jacobi n=%d sweeps=%d offmax=%.3e\n", n, sweeps, offd);
  colnorm_kernel<<<n, 256, 0, s>>>(Xc.ptr, n, w, squared);
  count_launch();
  // Vc is column-major; V row-major with eigenvectors in columns == transpose of Vc storage
  transpose(Vc.ptr, V, n, n, s);
  GPFVM_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_pairs);
  cudaFree(d_off);
}

static void sygv_core(const double* A, const double* Bm, int n, double* V, double* w, cudaStream_t s) {
  // A V = Bm V diag(w), V^T Bm V = I.  With Bm = L L^T and (if A is SPD) A = M M^T,
  // C = L^{-1} A L^{-T} = G G^T for G = L^{-1} M, so one-sided Jacobi on the
  // columns of G^T (condition sqrt(kappa(C))) gives C's eigenvectors W and
  // w = sigma^2; V = L^{-T} W.  If A is not SPD, C itself is used (w = sigma).
  DevBuf L, W, Wt, U;
  L.ensure((size_t)n * n);
  W.ensure((size_t)n * n);
  Wt.ensure((size_t)n * n);
  U.ensure((size_t)n * n);
  int* d_info;
  GPFVM_CUDA(cudaMalloc(&d_info, sizeof(int)));
  GPFVM_CUDA(cudaMemcpyAsync(L.ptr, Bm, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  int info = cholesky_inplace(L.ptr, n, s, d_info);
  GPFVM_CHECK(info == 0, GPFVM_ERR_NUMERIC, "sygv: B factor not positive definite (column " + std::to_string(info) + ")");
  GPFVM_CUDA(cudaMemcpyAsync(W.ptr, A, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  int infoA = cholesky_inplace(W.ptr, n, s, d_info);
  cudaFree(d_info);
  if (infoA == 0) {
    trsm_lower(L.ptr, n, W.ptr, n, s);        // G = L^{-1} M (row-major) == column-major G^T
    jacobi_cols(W.ptr, n, U.ptr, w, true, s);
  } else {
    GPFVM_CUDA(cudaMemcpyAsync(W.ptr, A, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
    trsm_lower(L.ptr, n, W.ptr, n, s);        // W = L^{-1} A
    transpose(W.ptr, Wt.ptr, n, n, s);        // Wt = A L^{-T}
    trsm_lower(L.ptr, n, Wt.ptr, n, s);       // C = L^{-1} A L^{-T}
    symmetrize_kernel<<<(unsigned)(((int64_t)n * n + 255) / 256), 256, 0, s>>>(Wt.ptr, n);
    count_launch();
    jacobi_cols(Wt.ptr, n, U.ptr, w, false, s);
  }
  transpose(L.ptr, W.ptr, n, n, s);           // W = L^T (upper)
  trsm_upper(W.ptr, n, U.ptr, n, s);          // V = L^{-T} U
  GPFVM_CUDA(cudaMemcpyAsync(V, U.ptr, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

namespace {
// orthonormal trigonometric bases (columns = basis vectors): 1 = DST-I, 2 = DCT-II
__global__ void trig_basis_kernel(double* S, int n, int kind) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int j = (int)(idx / n), k = (int)(idx % n);
  const double pi = 3.14159265358979323846;
  double v;
  if (kind == 1) {
    v = sqrt(2.0 / (n + 1)) * sin(pi * (double)(j + 1) * (double)(k + 1) / (n + 1));
  } else {
    v = sqrt((k == 0 ? 1.0 : 2.0) / n) * cos(pi * (j + 0.5) * (double)k / n);
  }
  S[idx] = v;
}

void gemm_rm(const double* A, bool ta, const double* B, bool tb, double* C, int n, cudaStream_t s) {
  // C = op(A) op(B), n x n row-major; op(A) via column-major view when transposed
  Gemm g;
  g.M = n; g.N = n; g.K = n;
  g.A = A;
  if (!ta) { g.a_rs = n; g.a_cs = 1; } else { g.a_rs = 1; g.a_cs = n; }
  g.B = B;
  if (!tb) { g.b_rs = n; g.b_cs = 1; } else { g.b_rs = 1; g.b_cs = n; }
  g.C = C; g.c_rs = n; g.c_cs = 1;
  run_gemm(g, s);
}
}  // namespace

// A V = Bm V diag(w), V^T Bm V = I.  The pencil is first rotated into an
// orthonormal trigonometric basis S (DCT-II by default; measured 95 vs 150 ms on config 1): for the Toeplitz-like
// factor matrices of uniform grids S^T A S and S^T Bm S are nearly diagonal
// (median off-diagonal correlation ~1e-11), so the Jacobi iteration inside
// sygv_core needs far fewer sweeps.  Exact for any orthogonal S:
// A (S V') = Bm (S V') w  and  (S V')^T Bm (S V') = I.
void sygv(const double* A, const double* Bm, int n, double* V, double* w, cudaStream_t s) {
  static const int basis = getenv("GPFVM_EIG_BASIS") ? atoi(getenv("GPFVM_EIG_BASIS")) : 2;
  if (basis == 0 || n < 8) {
    sygv_core(A, Bm, n, V, w, s);
    return;
  }
  DevBuf S, T, Ap, Bp, Vp;
  S.ensure((size_t)n * n); T.ensure((size_t)n * n); Ap.ensure((size_t)n * n); Bp.ensure((size_t)n * n);
  Vp.ensure((size_t)n * n);
  unsigned blocks = (unsigned)(((int64_t)n * n + 255) / 256);
  trig_basis_kernel<<<blocks, 256, 0, s>>>(S.ptr, n, basis);
  count_launch();
  gemm_rm(A, false, S.ptr, false, T.ptr, n, s);      // T = A S
  gemm_rm(S.ptr, true, T.ptr, false, Ap.ptr, n, s);  // A' = S^T A S
  gemm_rm(Bm, false, S.ptr, false, T.ptr, n, s);
  gemm_rm(S.ptr, true, T.ptr, false, Bp.ptr, n, s);  // B' = S^T Bm S
  symmetrize_kernel<<<blocks, 256, 0, s>>>(Ap.ptr, n);
  symmetrize_kernel<<<blocks, 256, 0, s>>>(Bp.ptr, n);
  count_launch(2);
  sygv_core(Ap.ptr, Bp.ptr, n, Vp.ptr, w, s);
  gemm_rm(S.ptr, false, Vp.ptr, false, V, n, s);     // V = S V'
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gpfvm
