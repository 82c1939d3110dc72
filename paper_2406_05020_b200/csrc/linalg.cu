// Small dense FP64 linear algebra for the preconditioner:
//   * blocked right-looking Cholesky (panel in one CTA, trailing update on DMMA GEMM)
//   * blocked triangular solves (diagonal block per column thread, GEMM updates)
//   * symmetric eigensolver: block one-sided (Hestenes) Jacobi — each CTA
//     orthogonalises a pair of 16-column blocks held in shared memory
//     (Gram -> in-smem parallel cyclic Jacobi -> rotate columns), tournament
//     ordering across CTAs; converged columns X = C V = V diag(lambda).
//   * generalised symmetric-definite eigenproblem via Cholesky reduction.
#include <mutex>
#include <thread>
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
  __shared__ double inv_s;
  for (int j = 0; j < kb; j++) {
    if (t == 0) {
      double d = s[j][j];
      if (!(d > 0.0)) {
        if (*info == 0) *info = k + j + 1;
        d = NAN;
      }
      const double r = rsqrt(d);  // one reciprocal square root instead of sqrt + divisions
      s[j][j] = d * r;
      inv_s = r;
    }
    __syncthreads();
    const double inv = inv_s;
    for (int r = j + 1 + t; r < kb; r += blockDim.x) s[r][j] *= inv;
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
  __shared__ double dinv[PB];
  for (int i = threadIdx.x; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    L[r][c] = A[(int64_t)(k + r) * n + k + c];
  }
  __syncthreads();
  if (threadIdx.x < kb) dinv[threadIdx.x] = 1.0 / L[threadIdx.x][threadIdx.x];
  __syncthreads();
  int r = k + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[PB];
  double* row = A + (int64_t)r * n + k;
#pragma unroll
  for (int j = 0; j < PB; j++)
    if (j < kb) x[j] = row[j];
#pragma unroll
  for (int j = 0; j < PB; j++) {
    if (j < kb) {
      double v = x[j];
#pragma unroll
      for (int i = 0; i < PB; i++)
        if (i < j) v -= x[i] * L[j][i];
      x[j] = v * dinv[j];
    }
  }
#pragma unroll
  for (int j = 0; j < PB; j++)
    if (j < kb) row[j] = x[j];
}

// Forward substitution on a diagonal block: B[k:k+kb, c] <- L11^{-1} B[k:k+kb, c]
__global__ void trsm_lower_diag_kernel(const double* L, int n, double* B, int nrhs, int k, int kb) {
  __shared__ double s[PB][PB + 1];
  for (int i = threadIdx.x; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    s[r][c] = L[(int64_t)(k + r) * n + k + c];
  }
  __shared__ double dinv[PB];
  __syncthreads();
  if (threadIdx.x < kb) dinv[threadIdx.x] = 1.0 / s[threadIdx.x][threadIdx.x];
  __syncthreads();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  double x[PB];
#pragma unroll
  for (int i = 0; i < PB; i++)
    if (i < kb) x[i] = B[(int64_t)(k + i) * nrhs + c];
#pragma unroll
  for (int i = 0; i < PB; i++) {
    if (i < kb) {
      double v = x[i];
#pragma unroll
      for (int j = 0; j < PB; j++)
        if (j < i) v -= s[i][j] * x[j];
      x[i] = v * dinv[i];
    }
  }
#pragma unroll
  for (int i = 0; i < PB; i++)
    if (i < kb) B[(int64_t)(k + i) * nrhs + c] = x[i];
}

// Backward substitution with U = L^T (U upper, row-major): B[k:k+kb] <- U11^{-1} B[k:k+kb]
__global__ void trsm_upper_diag_kernel(const double* U, int n, double* B, int nrhs, int k, int kb) {
  __shared__ double s[PB][PB + 1];
  for (int i = threadIdx.x; i < kb * kb; i += blockDim.x) {
    int r = i / kb, c = i % kb;
    s[r][c] = U[(int64_t)(k + r) * n + k + c];
  }
  __shared__ double dinv[PB];
  __syncthreads();
  if (threadIdx.x < kb) dinv[threadIdx.x] = 1.0 / s[threadIdx.x][threadIdx.x];
  __syncthreads();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  // compile-time indices (guards on kb) keep x in registers
  double x[PB];
#pragma unroll
  for (int i = 0; i < PB; i++)
    if (i < kb) x[i] = B[(int64_t)(k + i) * nrhs + c];
#pragma unroll
  for (int i = PB - 1; i >= 0; i--) {
    if (i < kb) {
      double v = x[i];
#pragma unroll
      for (int j = 0; j < PB; j++)
        if (j > i && j < kb) v -= s[i][j] * x[j];
      x[i] = v * dinv[i];
    }
  }
#pragma unroll
  for (int i = 0; i < PB; i++)
    if (i < kb) B[(int64_t)(k + i) * nrhs + c] = x[i];
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

__global__ void scale_scalar_kernel(double* x, double a) { *x *= a; }
void scale_scalar(double* x, double a, cudaStream_t s) {
  scale_scalar_kernel<<<1, 1, 0, s>>>(x, a);
  count_launch();
}

__global__ void eye_kernel(double* A, int n) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  A[idx] = ((idx / n) == (idx % n)) ? 1.0 : 0.0;
}

// ---- block one-sided Jacobi ----------------------------------------------------
constexpr int JT = 256;         // threads per CTA (<= 255 registers: no spills in the X.Q update)
__constant__ int c_inner_sweeps = 1;

// Copy `cnt` columns (ids col_of) of a column-major n-row matrix into shared
// memory, 4 independent 16-byte loads in flight per thread (n even) so the
// copy is bandwidth- rather than latency-bound.
__device__ __forceinline__ void load_cols(double* __restrict__ Xs, const double* __restrict__ G, int n, int cnt,
                                          const int* col_of) {
  const int t = threadIdx.x;
  if ((n & 1) == 0) {
    const int h = n >> 1, total = cnt * h;
    for (int base = t; base < total; base += 4 * (int)blockDim.x) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        int i = base + u * (int)blockDim.x;
        if (i < total) {
          int c = i / h, r2 = i - c * h;
          v[u] = __ldg(reinterpret_cast<const double2*>(G + (size_t)col_of[c] * n) + r2);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        int i = base + u * (int)blockDim.x;
        if (i < total) {
          int c = i / h, r2 = i - c * h;
          reinterpret_cast<double2*>(Xs + (size_t)c * n)[r2] = v[u];
        }
      }
    }
  } else {
    for (int i = t; i < cnt * n; i += blockDim.x) {
      int c = i / n, r = i % n;
      Xs[(size_t)c * n + r] = G[(size_t)col_of[c] * n + r];
    }
  }
}

// Xc, Vc: column-major n x n (column j at Xc + j*n).  pairs: (blk_a, blk_b) per CTA.
template <int JB>
__global__ void __launch_bounds__(JB <= 8 ? 512 : 256) jacobi_round_kernel(double* Xc, double* Vc, int n, int nblk,
                                                          const int* __restrict__ pairs,
                                                          unsigned long long* offmax,
                                                          const double* __restrict__ floor_ptr, double skip_tol,
                                                          int dual) {
  constexpr int JC = 2 * JB;      // columns per CTA (pair of blocks)
  extern __shared__ double sm[];
  double* Xs = sm;                  // [JC][n] column-major (column c at Xs + c*n)
  double* Vs = dual ? Xs + (size_t)JC * n : Xs;  // V columns (dual: own buffer, loaded up front)
  double* H = Vs + (size_t)JC * n;  // [JC][JC+1]
  double* Q = H + JC * (JC + 1);    // [JC][JC+1]
  __shared__ double cs[JC / 2], sn[JC / 2];
  __shared__ int col_of[JC];
  __shared__ int pair_ab[JC / 2][2];
  __shared__ unsigned char ent_a[JC * (JC + 1) / 2], ent_b[JC * (JC + 1) / 2];
  const int t = threadIdx.x;
  const int pa = pairs[2 * blockIdx.x], pb = pairs[2 * blockIdx.x + 1];
  // column ids and the upper-triangle (a, b) table, computed in parallel
  const int na = (pa >= 0) ? min(JB, n - pa * JB) : 0;
  const int nbb = (pb >= 0) ? min(JB, n - pb * JB) : 0;
  const int cnt = na + nbb;
  if (cnt < 2) return;
  if (t < cnt) col_of[t] = (t < na) ? pa * JB + t : pb * JB + (t - na);
  for (int e = t; e < cnt * (cnt + 1) / 2; e += blockDim.x) {
    int a = 0, rem = e;
    while (rem >= cnt - a) { rem -= cnt - a; a++; }
    ent_a[e] = (unsigned char)a;
    ent_b[e] = (unsigned char)(a + rem);
  }
  __syncthreads();
  for (int i = t; i < JC * (JC + 1); i += blockDim.x) H[i] = 0.0;  // unused indices stay 0
  load_cols(Xs, Xc, n, cnt, col_of);
  if (dual) load_cols(Vs, Vc, n, cnt, col_of);
  __syncthreads();
  // Gram H = Xs^T Xs: one warp per (a, b) entry, lanes stride the rows
  // (consecutive lanes -> consecutive banks), 4 independent partial sums,
  // shuffle reduction.
  {
    const int warp = t >> 5, lane = t & 31, nw = blockDim.x / 32;
    const int npair = cnt * (cnt + 1) / 2;
    for (int e = warp; e < npair; e += nw) {
      const int a = ent_a[e], b = ent_b[e];
      const double* xa = Xs + (size_t)a * n;
      const double* xb = Xs + (size_t)b * n;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int r = lane;
      for (; r + 96 < n; r += 128) {
        s0 = fma(xa[r], xb[r], s0);
        s1 = fma(xa[r + 32], xb[r + 32], s1);
        s2 = fma(xa[r + 64], xb[r + 64], s2);
        s3 = fma(xa[r + 96], xb[r + 96], s3);
      }
      for (; r < n; r += 32) s0 = fma(xa[r], xb[r], s0);
      double s = (s0 + s1) + (s2 + s3);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        H[a * (JC + 1) + b] = s;
        H[b * (JC + 1) + a] = s;
      }
    }
  }
  for (int i = t; i < JC * (JC + 1); i += blockDim.x) Q[i] = 0.0;
  __syncthreads();
  for (int i = t; i < cnt; i += blockDim.x) Q[i * (JC + 1) + i] = 1.0;
  // Convergence measure over all column pairs held by this CTA:
  // |h_ab| / max(sqrt(h_aa h_bb), floor).  floor = tau ||X||_F^2 (0: the
  // classical relative measure) treats pairs of columns that are both below
  // the rounding level of the pencil as converged.  A CTA whose pairs are all
  // below skip_tol leaves its columns untouched.
  const double flo = floor_ptr ? *floor_ptr : 0.0;
  __shared__ unsigned long long mcta_bits;
  if (t == 0) mcta_bits = 0ull;
  __syncthreads();
  {
    // squared correlations over the upper-triangle table, all threads (one
    // reciprocal per pair; max of non-negative doubles via their bit patterns)
    double m = 0.0;
    const double flo2 = flo * flo;
    for (int e = t; e < cnt * (cnt + 1) / 2; e += blockDim.x) {
      const int a = ent_a[e], b = ent_b[e];
      if (b == a) continue;
      double d2 = fmax(fabs(H[a * (JC + 1) + a] * H[b * (JC + 1) + b]), flo2);
      double hab = H[a * (JC + 1) + b];
      double v = (d2 > 0.0) ? hab * hab * __drcp_rn(d2) : 0.0;
      m = fmax(m, v);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((t & 31) == 0 && m > 0.0) atomicMax(&mcta_bits, (unsigned long long)__double_as_longlong(m));
  }
  __syncthreads();
  const double mcta = sqrt(__longlong_as_double((long long)mcta_bits));
  if (t == 0) atomicMax(offmax, (unsigned long long)__double_as_longlong(mcta));
  if (mcta < skip_tol) return;
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
          // rotate unless |h_pq| <= 1e-16 sqrt(h_pp h_qq) (compared squared);
          // rotation from reciprocals and one rsqrt: only orthogonality
          // (c^2 + s^2 = 1 to rounding) matters, not correctly rounded c, s
          if (fabs(hpq) > 1e-300 && hpq * hpq > 1e-32 * fabs(hpp * hqq) && fabs(hpq) > 1e-16 * flo) {
            double zeta = (hqq - hpp) * 0.5 * __drcp_rn(hpq);
            double tt = copysign(__drcp_rn(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0))), zeta);
            c = rsqrt(fma(tt, tt, 1.0));
            s = c * tt;
            done = 0;
          }
        }
        cs[t] = c;
        sn[t] = s;
        pair_ab[t][0] = p;
        pair_ab[t][1] = q;
      }
      __syncthreads();
      // H <- J^T H J and Q <- Q J in one phase: thread per 2x2 block
      // H[{p1,q1},{p2,q2}] of a pair of pairs (disjoint, no races) plus the Q
      // column pairs.  Entries of unused indices (>= cnt) are zero and pairs
      // touching them rotate by the identity.
      {
        const int np2 = m / 2;
        const int nblk2 = np2 * np2;
        for (int i = t; i < nblk2 + np2 * cnt; i += blockDim.x) {
          if (i < nblk2) {
            const int i1 = i / np2, i2 = i - i1 * np2;
            const int p1 = pair_ab[i1][0], q1 = pair_ab[i1][1], p2 = pair_ab[i2][0], q2 = pair_ab[i2][1];
            const double c1 = cs[i1], s1 = sn[i1], c2 = cs[i2], s2 = sn[i2];
            const double hpp = H[p1 * (JC + 1) + p2], hpq = H[p1 * (JC + 1) + q2];
            const double hqp = H[q1 * (JC + 1) + p2], hqq = H[q1 * (JC + 1) + q2];
            // columns (right J2), then rows (left J1^T)
            const double ap = c2 * hpp - s2 * hpq, aq = s2 * hpp + c2 * hpq;  // row p1
            const double bp = c2 * hqp - s2 * hqq, bq = s2 * hqp + c2 * hqq;  // row q1
            H[p1 * (JC + 1) + p2] = c1 * ap - s1 * bp;
            H[q1 * (JC + 1) + p2] = s1 * ap + c1 * bp;
            H[p1 * (JC + 1) + q2] = c1 * aq - s1 * bq;
            H[q1 * (JC + 1) + q2] = s1 * aq + c1 * bq;
          } else {
            const int k = i - nblk2;
            const int pr = k / cnt, r = k - pr * cnt;
            const int p = pair_ab[pr][0], q = pair_ab[pr][1];
            if (q >= cnt) continue;
            const double c = cs[pr], sv = sn[pr];
            const double qp = Q[r * (JC + 1) + p], qq = Q[r * (JC + 1) + q];
            Q[r * (JC + 1) + p] = c * qp - sv * qq;
            Q[r * (JC + 1) + q] = sv * qp + c * qq;
          }
        }
      }
      __syncthreads();
    }
    if (done) break;
  }
  // X <- X Q and V <- V Q.  dual: both column sets are resident, all threads
  // work (thread w < n: row w of X, n <= w < 2n: row w - n of V); otherwise V
  // is staged through the X buffer in a second pass.  Per row JC independent
  // register accumulators (fully unrolled), operands from shared memory (column
  // major: consecutive rows -> consecutive banks; Q broadcast).  Unused
  // columns (cnt < JC) carry zeros in Q.
  const int passes = dual ? 1 : 2;
#pragma unroll 1
  for (int pass = 0; pass < passes; pass++) {
    if (pass == 1) {
      __syncthreads();
      load_cols(Xs, Vc, n, cnt, col_of);
      __syncthreads();
    }
    const int rows = dual ? 2 * n : n;
#pragma unroll 1
    for (int w = t; w < rows; w += blockDim.x) {
      const bool isV = dual ? (w >= n) : (pass == 1);
      const int r = (dual && w >= n) ? w - n : w;
      const double* src = (dual && isV) ? Vs : Xs;
      double* dst = isV ? Vc : Xc;
      double acc[JC];
#pragma unroll
      for (int j = 0; j < JC; j++) acc[j] = 0.0;
#pragma unroll 2
      for (int c = 0; c < JC; c++) {
        const double xv = (c < cnt) ? src[(size_t)c * n + r] : 0.0;
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
template <int JB>
static int jacobi_sweeps(double* Xc, double* Vc, int n, cudaStream_t s) {
  constexpr int JC = 2 * JB;
  int nblk = (n + JB - 1) / JB;
  int players = nblk + (nblk & 1);
  std::vector<int> rounds;  // (players - 1) rounds x players entries
  for (int r = 0; r < players - 1; r++) {
    for (int i = 0; i < players / 2; i++) {
      int a = (i == 0) ? 0 : 1 + ((i - 1 + r) % (players - 1));
      int b = 1 + ((players - 2 - i + r) % (players - 1));
      rounds.push_back(a < nblk ? a : -1);
      rounds.push_back(b < nblk ? b : -1);
    }
  }
  DevBuf pairs_buf, off_buf;
  pairs_buf.ensure((rounds.size() + 1) / 2 + 1);
  off_buf.ensure(1);
  int* d_pairs = reinterpret_cast<int*>(pairs_buf.ptr);
  unsigned long long* d_off = reinterpret_cast<unsigned long long*>(off_buf.ptr);
  GPFVM_CUDA(cudaMemcpyAsync(d_pairs, rounds.data(), sizeof(int) * rounds.size(), cudaMemcpyHostToDevice, s));
  size_t smem = sizeof(double) * ((size_t)JC * n + 2 * JC * (JC + 1));
  const size_t smem_dual = smem + sizeof(double) * (size_t)JC * n;
  static const bool no_dual = getenv("GPFVM_NO_DUAL") != nullptr;
  const int dual = (!no_dual && smem_dual <= 200 * 1024) ? 1 : 0;
  if (dual) smem = smem_dual;
  GPFVM_CHECK(smem <= 220 * 1024, GPFVM_ERR_UNSUPPORTED, "eigensolver: dimension too large");
  {
    // The attribute is per function and device, and sygv runs on several host
    // threads at once with different n: set it once to the maximum (under a
    // lock) instead of per call, so no thread lowers it under another's launch.
    static std::mutex mu;
    static unsigned long long done_mask = 0;
    int dev = 0;
    GPFVM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!(done_mask >> dev & 1ull)) {
      int optin = 0;
      GPFVM_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      cudaFuncAttributes fa;
      GPFVM_CUDA(cudaFuncGetAttributes(&fa, jacobi_round_kernel<JB>));
      GPFVM_CUDA(cudaFuncSetAttribute(jacobi_round_kernel<JB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      optin - (int)fa.sharedSizeBytes));
      done_mask |= 1ull << dev;
    }
  }
  // absolute floor tau ||X||_F^2 (GPFVM_JAC_TAU, default 0 = relative measure)
  static const double tau = getenv("GPFVM_JAC_TAU") ? atof(getenv("GPFVM_JAC_TAU")) : 0.0;
  DevBuf fro;
  const double* d_floor = nullptr;
  if (tau > 0.0) {
    fro.ensure(1);
    dot_many(Xc, (int64_t)n * n, Xc, (int64_t)n * n, 1, fro.ptr, s);
    scale_scalar(fro.ptr, tau, s);
    d_floor = fro.ptr;
  }
  const double conv_tol = std::max(4e-15, 2e-16 * n);
  // 512 threads for the 8-column blocks (measured 36 vs 38 ms on config 1), 256 above (registers)
  static const int jt_env = getenv("GPFVM_JT") ? atoi(getenv("GPFVM_JT")) : 0;
  const int jt = jt_env ? std::min(jt_env, JB <= 8 ? 512 : 256) : (JB <= 8 ? 512 : JT);
  int sweeps = 0;
  double offd = 1.0;
  const bool dbg2 = getenv("GPFVM_DEBUG") && atoi(getenv("GPFVM_DEBUG")) > 1;
  for (int sweep = 0; sweep < 40; sweep++) {
    sweeps++;
    GPFVM_CUDA(cudaMemsetAsync(d_off, 0, sizeof(unsigned long long), s));
    for (int r = 0; r < players - 1; r++) {
      jacobi_round_kernel<JB><<<players / 2, jt, smem, s>>>(Xc, Vc, n, nblk, d_pairs + r * players, d_off,
                                                             d_floor, sweep > 0 ? conv_tol : 0.0, dual);
      count_launch();
    }
    check_launch("jacobi_round_kernel");
    unsigned long long off = 0;
    GPFVM_CUDA(cudaMemcpyAsync(&off, d_off, sizeof(off), cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
    memcpy(&offd, &off, sizeof(double));
    if (dbg2) fprintf(stderr, "[gpfvm]   sweep %d off %.3e\n", sweep, offd);
    // one-sided Jacobi orthogonality floor ~ n eps (rounding of the column dots)
    if (offd < conv_tol) break;
  }
  if (getenv("GPFVM_DEBUG")) fprintf(stderr, "[gpfvm] jacobi n=%d JB=%d sweeps=%d offmax=%.3e\n", n, JB, sweeps, offd);
  return sweeps;
}

// One-sided (Hestenes) block Jacobi on the columns of X (column-major n x n):
// X W = U Sigma.  Eigenvectors of X^T X are the columns of W (returned row-major
// in V, eigenvectors in columns); w = Sigma^2 (squared = true) or Sigma.
// Column-block width JB: 8 for n <= 512 (more CTAs per round: the round is
// latency-bound, not flop-bound), 16 above (shared memory holds 2*JB columns).
static void jacobi_cols(const double* X0, int n, double* V, double* w, bool squared, cudaStream_t s) {
  DevBuf Xc, Vc;
  Xc.ensure((size_t)n * n);
  Vc.ensure((size_t)n * n);
  GPFVM_CUDA(cudaMemcpyAsync(Xc.ptr, X0, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  eye_kernel<<<(unsigned)(((int64_t)n * n + 255) / 256), 256, 0, s>>>(Vc.ptr, n);
  count_launch();
  if (getenv("GPFVM_INNER")) { int v = atoi(getenv("GPFVM_INNER")); GPFVM_CUDA(cudaMemcpyToSymbol(c_inner_sweeps, &v, sizeof(int))); }
  static const int jb_env = getenv("GPFVM_JB") ? atoi(getenv("GPFVM_JB")) : 0;
  const int jb = jb_env ? jb_env : (n <= 512 ? 8 : 16);
  if (jb == 4) jacobi_sweeps<4>(Xc.ptr, Vc.ptr, n, s);
  else if (jb == 8) jacobi_sweeps<8>(Xc.ptr, Vc.ptr, n, s);
  else jacobi_sweeps<16>(Xc.ptr, Vc.ptr, n, s);
  colnorm_kernel<<<n, 256, 0, s>>>(Xc.ptr, n, w, squared);
  count_launch();
  // Vc is column-major; V row-major with eigenvectors in columns == transpose of Vc storage
  transpose(Vc.ptr, V, n, n, s);
  GPFVM_CUDA(cudaStreamSynchronize(s));
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
  DevBuf info_buf;  // pooled: cudaFree would synchronise the whole device
  info_buf.ensure(1);
  int* d_info = reinterpret_cast<int*>(info_buf.ptr);
  GPFVM_CUDA(cudaMemcpyAsync(L.ptr, Bm, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  int info = cholesky_inplace(L.ptr, n, s, d_info);
  GPFVM_CHECK(info == 0, GPFVM_ERR_NUMERIC, "sygv: B factor not positive definite (column " + std::to_string(info) + ")");
  GPFVM_CUDA(cudaMemcpyAsync(W.ptr, A, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  int infoA = cholesky_inplace(W.ptr, n, s, d_info);
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
// orthonormal trigonometric bases (columns = basis vectors): 1 = DST-I, 2 = DCT-II, 4 = DCT-IV
__global__ void trig_basis_kernel(double* S, int n, int kind) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int j = (int)(idx / n), k = (int)(idx % n);
  const double pi = 3.14159265358979323846;
  double v;
  if (kind == 1) {
    v = sqrt(2.0 / (n + 1)) * sin(pi * (double)(j + 1) * (double)(k + 1) / (n + 1));
  } else if (kind == 4) {
    v = sqrt(2.0 / n) * cos(pi * (j + 0.5) * (k + 0.5) / n);
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
// max |A[i][j] - A[n-1-i][n-1-j]| and max |A[i][j]| (as ordered bit patterns)
__global__ void centro_kernel(const double* A, int n, unsigned long long* out) {
  double dev = 0.0, mx = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(idx / n), j = (int)(idx % n);
    double a = A[idx];
    dev = fmax(dev, fabs(a - A[(int64_t)(n - 1 - i) * n + (n - 1 - j)]));
    mx = fmax(mx, fabs(a));
  }
  for (int o = 16; o > 0; o >>= 1) {
    dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, (unsigned long long)__double_as_longlong(dev));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(mx));
  }
}

// Even / odd blocks of a centrosymmetric n x n matrix (n = 2h):
// E = A11 + A12 J, O = A11 - A12 J  (P^T A P for P = [[I, I], [J, -J]] / sqrt 2).
__global__ void parity_split_kernel(const double* A, int h, double* E, double* O) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)h * h) return;
  int i = (int)(idx / h), j = (int)(idx % h);
  const int n = 2 * h;
  double a = A[(int64_t)i * n + j], b = A[(int64_t)i * n + (n - 1 - j)];
  E[idx] = a + b;
  O[idx] = a - b;
}

// V = P blockdiag(Ve, Vo): columns c < h symmetric, c >= h antisymmetric.
__global__ void parity_merge_kernel(const double* Ve, const double* Vo, int h, double* V) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)h * h) return;
  int i = (int)(idx / h), c = (int)(idx % h);
  const int n = 2 * h;
  const double r = 0.70710678118654752440;
  double e = Ve[idx] * r, o = Vo[idx] * r;
  V[(int64_t)i * n + c] = e;
  V[(int64_t)(n - 1 - i) * n + c] = e;
  V[(int64_t)i * n + h + c] = o;
  V[(int64_t)(n - 1 - i) * n + h + c] = -o;
}
}  // namespace

// Pencil rotated into the orthonormal trigonometric basis S (kind), solved by
// sygv_core, rotated back: exact for any orthogonal S.
static void sygv_rotated(const double* A, const double* Bm, int n, double* V, double* w, int kind,
                         cudaStream_t s) {
  static const bool no_rot = getenv("GPFVM_NO_ROT") != nullptr;
  if (kind == 0 || n < 8 || no_rot) {
    sygv_core(A, Bm, n, V, w, s);
    return;
  }
  DevBuf S, T, Ap, Bp, Vp;
  S.ensure((size_t)n * n); T.ensure((size_t)n * n); Ap.ensure((size_t)n * n); Bp.ensure((size_t)n * n);
  Vp.ensure((size_t)n * n);
  unsigned blocks = (unsigned)(((int64_t)n * n + 255) / 256);
  trig_basis_kernel<<<blocks, 256, 0, s>>>(S.ptr, n, kind);
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

static bool centrosymmetric(const double* A, const double* Bm, int n, cudaStream_t s) {
  DevBuf buf;
  buf.ensure(4);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(buf.ptr);
  GPFVM_CUDA(cudaMemsetAsync(d, 0, 4 * sizeof(unsigned long long), s));
  int grid = (int)std::min<int64_t>(296, ((int64_t)n * n + 255) / 256);
  centro_kernel<<<grid, 256, 0, s>>>(A, n, d);
  centro_kernel<<<grid, 256, 0, s>>>(Bm, n, d + 2);
  count_launch(2);
  unsigned long long h[4];
  GPFVM_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  GPFVM_CUDA(cudaStreamSynchronize(s));
  double v[4];
  memcpy(v, h, sizeof(v));
  return v[0] <= 1e-14 * v[1] && v[2] <= 1e-14 * v[3];
}

// A V = Bm V diag(w), V^T Bm V = I (generalised symmetric-definite eigenproblem
// of the FD preconditioner).  Each (sub)pencil is first rotated
// into an orthonormal trigonometric basis (measured: fewer Jacobi sweeps on the
// factor matrices of uniform grids, 95 vs 150 ms on config 1 before the parity
// split); exact for any orthogonal S: A (S V') = Bm (S V') w.
void sygv(const double* A, const double* Bm, int n, double* V, double* w, cudaStream_t s) {
  static const int basis = getenv("GPFVM_EIG_BASIS") ? atoi(getenv("GPFVM_EIG_BASIS")) : 2;
  static const bool no_parity = getenv("GPFVM_NO_PARITY") != nullptr;
  if (basis == 0 || n < 16 || (n & 1) || no_parity || !centrosymmetric(A, Bm, n, s)) {
    sygv_rotated(A, Bm, n, V, w, basis, s);
    return;
  }
  // Centrosymmetric pencil (uniform grid, stationary kernel: J A J = A): the
  // even and odd subspaces decouple exactly, two independent n/2 problems
  // (1/4 of the Jacobi work each, solved concurrently).  Their trigonometric
  // bases are the even (DCT-II, size n/2) and odd (DCT-IV, size n/2) halves
  // of the size-n DCT-II.
  const int h = n / 2;
  DevBuf Ae, Ao, Be, Bo, Ve, Vo;
  for (DevBuf* b : {&Ae, &Ao, &Be, &Bo, &Ve, &Vo}) b->ensure((size_t)h * h);
  unsigned blocks = (unsigned)(((int64_t)h * h + 255) / 256);
  parity_split_kernel<<<blocks, 256, 0, s>>>(A, h, Ae.ptr, Ao.ptr);
  parity_split_kernel<<<blocks, 256, 0, s>>>(Bm, h, Be.ptr, Bo.ptr);
  count_launch(2);
  GPFVM_CUDA(cudaStreamSynchronize(s));
  cudaStream_t so;
  GPFVM_CUDA(cudaStreamCreateWithFlags(&so, cudaStreamNonBlocking));
  int dev = 0;
  GPFVM_CUDA(cudaGetDevice(&dev));
  Error err{GPFVM_OK, ""};
  std::thread th([&] {
    try {
      cudaSetDevice(dev);
      sygv_rotated(Ao.ptr, Bo.ptr, h, Vo.ptr, w + h, basis == 2 ? 4 : basis, so);
    } catch (const Error& e) {
      err = e;
    }
  });
  try {
    sygv_rotated(Ae.ptr, Be.ptr, h, Ve.ptr, w, basis, s);
  } catch (...) {
    th.join();
    cudaStreamDestroy(so);
    throw;
  }
  th.join();
  cudaStreamDestroy(so);
  if (err.code != GPFVM_OK) throw err;
  parity_merge_kernel<<<blocks, 256, 0, s>>>(Ve.ptr, Vo.ptr, h, V);
  count_launch();
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gpfvm
