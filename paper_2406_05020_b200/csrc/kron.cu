// Fused Kronecker-sum operator  Y (+)= sum_p ((x)_i F_i^p) X.
//
// One block pair of the Gram (Eq. 20) with P surviving term pairs becomes d
// GEMM launches, independent of P.  Two contraction orders; the cheaper one
// (fewer flops: contract shrinking dimensions before expanding ones) is
// chosen when the plan is built.
// forward (dim 0 first):
//   stage 0   stacked-M GEMM   Z[r][p][j0][n'_1..]   = (c_p F_0^p) X_r            M = P*n0
//   stage i   batched GEMM     Z[r][p][j0..ji][n'..]  = F_i^p Z                    batch (o, p, r)
//   stage d-1 K-segment GEMM   Y_r[rows][l] += sum_p Z[r][p][rows][:] F_{d-1}^{pT}
// reverse (dim d-1 first):
//   stage 0   stacked-N GEMM   Z[r][rows'][p][l]     = X_r [c_p F_{d-1}^{pT}]_p   N = P*n_{d-1}
//   stage i   batched GEMM     Z[r][n'_0..n'_{i-1}][p][j_i..] = F_i^p Z             batch (o, p, r)
//   stage d-1 K-segment GEMM   Y_r[j0][rest] += sum_p F_0^p Z[r][:][p][rest]
// (the p-sum is the K-concatenation of the last contraction).  d = 1: a single
// K-segment GEMM  Y_r = sum_p X_r (c_p F^p)^T.  Coefficients are folded into
// the first-applied factor.
#include <algorithm>
#include <map>
#include <cstdlib>

#include "problem.h"

namespace gpfvm {

namespace {
__global__ void scaled_copy_kernel(double* dst, const double* __restrict__ src, double c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = c * src[i];
}
// dst = a A + b B
__global__ void lincomb2_kernel(double* dst, double a, const double* __restrict__ A, double b,
                                const double* __restrict__ B, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = a * A[i] + b * B[i];
}
unsigned gsz(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 2048)); }

// 2D restacking so that both stages are plain GEMMs (no K-segments):
//   mode 0: dst[(r*P + p)*cols + k] = c * src[r*cols + k]     rows interleaved by term
//   mode 1: dst[r*(P*cols) + p*cols + k] = c * src[r*cols + k] columns concatenated by term
//   mode 2: dst[r*(cols*P) + k*P + p] = c * src[r*cols + k]   columns interleaved by term
__global__ void restack_kernel(double* dst, const double* __restrict__ src, double c, int p, int P, int rows, int cols,
                               int mode) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, k = i % cols;
    int64_t o = (mode == 0) ? (r * P + p) * cols + k : (mode == 1 ? r * ((int64_t)P * cols) + (int64_t)p * cols + k
                                                                  : r * ((int64_t)cols * P) + k * P + p);
    dst[o] = c * src[i];
  }
}

// dst[p][r][i] = src[r][i][p]   (p-innermost -> p-outermost, R x n x P)
__global__ void p_outer_kernel(double* __restrict__ dst, const double* __restrict__ src, int R, int64_t n, int P) {
  const int64_t total = (int64_t)R * n * P;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = o / ((int64_t)R * n), rem = o - p * R * n;
    const int64_t r = rem / n, i = rem - r * n;
    dst[o] = src[(r * n + i) * P + p];
  }
}

// Reflection-parity split (KronSum::par).  Half blocks of one factor
// (n x n, h = n/2) for parity class c of the input (0: even part, 1: odd part):
//   H_c[j][k] = coef * (F[j][k] + (-1)^c F[j][n-1-k])   j, k < h
// mode 0: dst[c][(j*P + p)][k]   (rows interleaved by term, stage-0 A)
// mode 1: dst[c][j][p*h + k]     (columns concatenated by term, stage-1 B)
__global__ void half_restack_kernel(double* dst, const double* __restrict__ F, double coef, int p, int P, int n,
                                    int mode) {
  const int h = n / 2;
  const int64_t tot = 2LL * h * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / ((int64_t)h * h));
    const int j = (int)((e / h) % h), k = (int)(e % h);
    const double a = F[(int64_t)j * n + k], b = F[(int64_t)j * n + (n - 1 - k)];
    const double v = coef * (c ? a - b : a + b);
    const int64_t o = mode == 0 ? (int64_t)c * P * h * h + ((int64_t)j * P + p) * h + k
                                : (int64_t)c * h * P * h + (int64_t)j * P * h + (int64_t)p * h + k;
    dst[o] = v;
  }
}

// x (R vectors, n0 x n1 row-major, stride ldx) -> parity classes
// xt[a][r][b][i][j] (a: time class, b: space class, i < h0, j < h1):
//   u/v along dim 0 then along dim 1 (sums and differences, no scaling)
__global__ void parity_fwd2_kernel(const double* __restrict__ x, int64_t ldx, double* __restrict__ xt, int R, int n0,
                                   int n1) {
  const int h0 = n0 / 2, h1 = n1 / 2;
  const int64_t cls = (int64_t)h0 * h1, tot = (int64_t)R * cls;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cls, ij = e - r * cls;
    const int i = (int)(ij / h1), j = (int)(ij - (int64_t)i * h1);
    const double* xr = x + r * ldx;
    const double x00 = xr[(int64_t)i * n1 + j], x01 = xr[(int64_t)i * n1 + (n1 - 1 - j)];
    const double x10 = xr[(int64_t)(n0 - 1 - i) * n1 + j], x11 = xr[(int64_t)(n0 - 1 - i) * n1 + (n1 - 1 - j)];
    const double u0 = x00 + x10, u1 = x01 + x11, v0 = x00 - x10, v1 = x01 - x11;
    xt[((0 * (int64_t)R + r) * 2 + 0) * cls + ij] = u0 + u1;
    xt[((0 * (int64_t)R + r) * 2 + 1) * cls + ij] = u0 - u1;
    xt[((1 * (int64_t)R + r) * 2 + 0) * cls + ij] = v0 + v1;
    xt[((1 * (int64_t)R + r) * 2 + 1) * cls + ij] = v0 - v1;
  }
}

// Inverse: y = beta y + (1/4) recombined classes + sum_k U[r][row][k] V[r][col][k]
// (the optional low-rank IC/BC coupling update).  The class of
// output parity (a, b) sits at position (a ^ sg0, b ^ sg1) (positions are
// input classes; a skew factor maps even to odd).
__global__ void parity_inv2_kernel(const double* __restrict__ yt, double* __restrict__ y, int64_t ldy, int R, int n0,
                                   int n1, int sg0, int sg1, double beta, const double* __restrict__ U,
                                   int64_t u_rs, int64_t u_b1, const double* __restrict__ V, int64_t v_rs,
                                   int64_t v_b1, int rk) {
  const int h0 = n0 / 2, h1 = n1 / 2;
  const int64_t cls = (int64_t)h0 * h1, tot = (int64_t)R * cls;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cls, ij = e - r * cls;
    const int i = (int)(ij / h1), j = (int)(ij - (int64_t)i * h1);
    auto at = [&](int a, int b) { return yt[(((int64_t)(a ^ sg0) * R + r) * 2 + (b ^ sg1)) * cls + ij]; };
    const double Y00 = at(0, 0), Y01 = at(0, 1), Y10 = at(1, 0), Y11 = at(1, 1);
    const int i1 = n0 - 1 - i, j1 = n1 - 1 - j;
    double o[4] = {0.25 * ((Y00 + Y01) + (Y10 + Y11)), 0.25 * ((Y00 - Y01) + (Y10 - Y11)),
                   0.25 * ((Y00 + Y01) - (Y10 + Y11)), 0.25 * ((Y00 - Y01) - (Y10 - Y11))};
    const int rows[4] = {i, i, i1, i1}, cols[4] = {j, j1, j, j1};
    double* yr = y + r * ldy;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      double v = o[q];
      if (rk > 0) {
        const double* u = U + r * u_b1 + (int64_t)rows[q] * u_rs;
        const double* w = V + r * v_b1 + (int64_t)cols[q] * v_rs;
        for (int k = 0; k < rk; k++) v = fma(u[k], w[k], v);
      }
      double* yp = yr + (int64_t)rows[q] * n1 + cols[q];
      *yp = (beta != 0.0) ? fma(beta, *yp, v) : v;
    }
  }
}

// Vectorised variant (h1 even, 16-byte aligned rows): one thread per column
// pair (j, j+1) of one half row; grid (column chunks, h0, R), no integer
// division.  The mirrored columns n1-1-j, n1-2-j are one reversed double2.
__global__ void __launch_bounds__(128)
    parity_inv2v_kernel(const double* __restrict__ yt, double* __restrict__ y, int64_t ldy, int R, int n0, int n1,
                        int sg0, int sg1, double beta, const double* __restrict__ U, int64_t u_rs, int64_t u_b1,
                        const double* __restrict__ V, int64_t v_rs, int64_t v_b1, int rk) {
  const int h0 = n0 >> 1, h1 = n1 >> 1;
  const int j = 2 * (blockIdx.x * blockDim.x + threadIdx.x), i = blockIdx.y, r = blockIdx.z;
  if (j >= h1) return;
  const int64_t cls = (int64_t)h0 * h1, ij = (int64_t)i * h1 + j;
  const double2 Y00 = *reinterpret_cast<const double2*>(yt + (((int64_t)(0 ^ sg0) * R + r) * 2 + (0 ^ sg1)) * cls + ij);
  const double2 Y01 = *reinterpret_cast<const double2*>(yt + (((int64_t)(0 ^ sg0) * R + r) * 2 + (1 ^ sg1)) * cls + ij);
  const double2 Y10 = *reinterpret_cast<const double2*>(yt + (((int64_t)(1 ^ sg0) * R + r) * 2 + (0 ^ sg1)) * cls + ij);
  const double2 Y11 = *reinterpret_cast<const double2*>(yt + (((int64_t)(1 ^ sg0) * R + r) * 2 + (1 ^ sg1)) * cls + ij);
  const int i1 = n0 - 1 - i, j1 = n1 - 2 - j;  // columns j1, j1 + 1 mirror j + 1, j
  // o[row half][col half][column of the pair]
  double oa[2] = {0.25 * ((Y00.x + Y01.x) + (Y10.x + Y11.x)), 0.25 * ((Y00.y + Y01.y) + (Y10.y + Y11.y))};  // (i, j..)
  double ob[2] = {0.25 * ((Y00.x - Y01.x) + (Y10.x - Y11.x)), 0.25 * ((Y00.y - Y01.y) + (Y10.y - Y11.y))};  // (i, mirror)
  double oc[2] = {0.25 * ((Y00.x + Y01.x) - (Y10.x + Y11.x)), 0.25 * ((Y00.y + Y01.y) - (Y10.y + Y11.y))};  // (i1, j..)
  double od[2] = {0.25 * ((Y00.x - Y01.x) - (Y10.x - Y11.x)), 0.25 * ((Y00.y - Y01.y) - (Y10.y - Y11.y))};  // (i1, mirror)
  if (rk > 0) {
    const double* u0 = U + r * u_b1 + (int64_t)i * u_rs;
    const double* u1 = U + r * u_b1 + (int64_t)i1 * u_rs;
    const double* Vr = V + r * v_b1;
    const double* wa0 = Vr + (int64_t)j * v_rs;
    const double* wa1 = Vr + (int64_t)(j + 1) * v_rs;
    const double* wb0 = Vr + (int64_t)(n1 - 1 - j) * v_rs;
    const double* wb1 = Vr + (int64_t)(n1 - 2 - j) * v_rs;
    for (int k = 0; k < rk; k++) {
      const double a = u0[k], b = u1[k], p0 = wa0[k], p1 = wa1[k], q0 = wb0[k], q1 = wb1[k];
      oa[0] = fma(a, p0, oa[0]); oa[1] = fma(a, p1, oa[1]);
      ob[0] = fma(a, q0, ob[0]); ob[1] = fma(a, q1, ob[1]);
      oc[0] = fma(b, p0, oc[0]); oc[1] = fma(b, p1, oc[1]);
      od[0] = fma(b, q0, od[0]); od[1] = fma(b, q1, od[1]);
    }
  }
  double* yr = y + r * ldy;
  double2* pa = reinterpret_cast<double2*>(yr + (int64_t)i * n1 + j);
  double2* pb = reinterpret_cast<double2*>(yr + (int64_t)i * n1 + j1);
  double2* pc = reinterpret_cast<double2*>(yr + (int64_t)i1 * n1 + j);
  double2* pd = reinterpret_cast<double2*>(yr + (int64_t)i1 * n1 + j1);
  double2 va = make_double2(oa[0], oa[1]), vb = make_double2(ob[1], ob[0]);
  double2 vc = make_double2(oc[0], oc[1]), vd = make_double2(od[1], od[0]);
  if (beta != 0.0) {
    const double2 a = *pa, b = *pb, c = *pc, d = *pd;
    va.x = fma(beta, a.x, va.x); va.y = fma(beta, a.y, va.y);
    vb.x = fma(beta, b.x, vb.x); vb.y = fma(beta, b.y, vb.y);
    vc.x = fma(beta, c.x, vc.x); vc.y = fma(beta, c.y, vc.y);
    vd.x = fma(beta, d.x, vd.x); vd.y = fma(beta, d.y, vd.y);
  }
  *pa = va; *pb = vb; *pc = vc; *pd = vd;
}

// ---- 3D reflection-parity split (KronSum::par3) ------------------------------------
// Half blocks of one factor, both classes back to back: dst[c][j][k] (h x h)
//   = coef (F[j][k] + (-1)^c F[j][n-1-k]);  rows optionally interleaved over a
// group of G factors (row (j, g) of a [c][(j, g)][k] stack).
__global__ void half_block_kernel(double* dst, const double* __restrict__ F, double coef, int n, int g, int G) {
  const int h = n / 2;
  const int64_t tot = 2LL * h * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / ((int64_t)h * h));
    const int j = (int)((e / h) % h), k = (int)(e % h);
    const double a = F[(int64_t)j * n + k], b = F[(int64_t)j * n + (n - 1 - k)];
    dst[(int64_t)c * G * h * h + ((int64_t)j * G + g) * h + k] = coef * (c ? a - b : a + b);
  }
}

// x (n0 x n1 x n2) -> xt, same shape, index (class, half index) per dimension:
// class 0 = x_k + x_{n-1-k}, class 1 = x_k - x_{n-1-k} (no scaling).
// grid (ceil(h2 / 128), h1, h0 * Rc); one thread per (r, i, j, k), 8 in, 8 out.
__global__ void __launch_bounds__(128)
    parity_fwd3_kernel(const double* __restrict__ x, int64_t ldx, double* __restrict__ xt, int64_t ldt, int n0,
                       int n1, int n2) {
  const int h0 = n0 >> 1, h1 = n1 >> 1, h2 = n2 >> 1;
  const int k = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  const int i = blockIdx.z % h0, r = blockIdx.z / h0;
  if (k >= h2) return;
  const double* xr = x + (int64_t)r * ldx;
  double v[8];
#pragma unroll
  for (int m = 0; m < 8; m++) {
    const int ii = (m & 4) ? n0 - 1 - i : i, jj = (m & 2) ? n1 - 1 - j : j, kk = (m & 1) ? n2 - 1 - k : k;
    v[m] = xr[((int64_t)ii * n1 + jj) * n2 + kk];
  }
#pragma unroll
  for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
    for (int m = 0; m < 8; m++)
      if (!(m & bit)) {
        const double a = v[m], b = v[m | bit];
        v[m] = a + b;
        v[m | bit] = a - b;
      }
  double* tr = xt + (int64_t)r * ldt;
#pragma unroll
  for (int m = 0; m < 8; m++) {
    const int ii = ((m & 4) ? h0 : 0) + i, jj = ((m & 2) ? h1 : 0) + j, kk = ((m & 1) ? h2 : 0) + k;
    tr[((int64_t)ii * n1 + jj) * n2 + kk] = v[m];
  }
}

// y = beta y + (1/8) inverse transform of yt + the mode-s updates of the block
// (ModeTerms: couplings from IC planes and boundary faces), all in the one
// pass that writes y.  Each thread owns the 8 mirror images of (i, j, k), so
// every W value it loads serves two outputs.
__global__ void __launch_bounds__(128)
    parity_inv3_kernel(const double* __restrict__ yt, int64_t ldt, double* __restrict__ y, int64_t ldy, int n0, int n1,
                       int n2, double beta, ModeTerms mt) {
  const int h0 = n0 >> 1, h1 = n1 >> 1, h2 = n2 >> 1;
  const int k = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  const int i = blockIdx.z % h0, r = blockIdx.z / h0;
  if (k >= h2) return;
  const double* tr = yt + (int64_t)r * ldt;
  double v[8];
#pragma unroll
  for (int m = 0; m < 8; m++) {
    const int ii = ((m & 4) ? h0 : 0) + i, jj = ((m & 2) ? h1 : 0) + j, kk = ((m & 1) ? h2 : 0) + k;
    v[m] = tr[((int64_t)ii * n1 + jj) * n2 + kk];
  }
#pragma unroll
  for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
    for (int m = 0; m < 8; m++)
      if (!(m & bit)) {
        const double a = v[m], b = v[m | bit];
        v[m] = a + b;
        v[m | bit] = a - b;
      }
#pragma unroll
  for (int m = 0; m < 8; m++) v[m] *= 0.125;
  const int I2[2] = {i, n0 - 1 - i}, J2[2] = {j, n1 - 1 - j}, K2[2] = {k, n2 - 1 - k};
  for (int e = 0; e < mt.n; e++) {
    const int P = mt.m[e].P, sd = mt.m[e].s;
    const double* U = mt.m[e].U;
    // a: index into U (the updated dimension); (b, c): the two indices of W
    const int ia[2] = {sd == 0 ? I2[0] : (sd == 1 ? J2[0] : K2[0]), sd == 0 ? I2[1] : (sd == 1 ? J2[1] : K2[1])};
    const int ib[2] = {sd == 0 ? J2[0] : I2[0], sd == 0 ? J2[1] : I2[1]};
    const int ic[2] = {sd == 2 ? J2[0] : K2[0], sd == 2 ? J2[1] : K2[1]};
    const int64_t nc = sd == 2 ? n1 : n2, AB = (sd == 0 ? (int64_t)n1 : (int64_t)n0) * nc;
    const double* W = mt.m[e].W + (int64_t)r * P * AB;
    for (int p = 0; p < P; p++) {
      const double u0 = U[(int64_t)ia[0] * P + p], u1 = U[(int64_t)ia[1] * P + p];
      const double* Wp = W + (int64_t)p * AB;
      const double w00 = Wp[ib[0] * nc + ic[0]], w01 = Wp[ib[0] * nc + ic[1]];
      const double w10 = Wp[ib[1] * nc + ic[0]], w11 = Wp[ib[1] * nc + ic[1]];
      // output m = (mi, mj, mk) bits 4, 2, 1
      if (sd == 0) {        // a = i, (b, c) = (j, k)
        v[0] = fma(u0, w00, v[0]); v[1] = fma(u0, w01, v[1]); v[2] = fma(u0, w10, v[2]); v[3] = fma(u0, w11, v[3]);
        v[4] = fma(u1, w00, v[4]); v[5] = fma(u1, w01, v[5]); v[6] = fma(u1, w10, v[6]); v[7] = fma(u1, w11, v[7]);
      } else if (sd == 1) { // a = j, (b, c) = (i, k)
        v[0] = fma(u0, w00, v[0]); v[1] = fma(u0, w01, v[1]); v[2] = fma(u1, w00, v[2]); v[3] = fma(u1, w01, v[3]);
        v[4] = fma(u0, w10, v[4]); v[5] = fma(u0, w11, v[5]); v[6] = fma(u1, w10, v[6]); v[7] = fma(u1, w11, v[7]);
      } else {              // a = k, (b, c) = (i, j)
        v[0] = fma(u0, w00, v[0]); v[1] = fma(u1, w00, v[1]); v[2] = fma(u0, w01, v[2]); v[3] = fma(u1, w01, v[3]);
        v[4] = fma(u0, w10, v[4]); v[5] = fma(u1, w10, v[5]); v[6] = fma(u0, w11, v[6]); v[7] = fma(u1, w11, v[7]);
      }
    }
  }
  double* yr = y + (int64_t)r * ldy;
#pragma unroll
  for (int m = 0; m < 8; m++) {
    double* yp = yr + ((int64_t)I2[m >> 2] * n1 + J2[(m >> 1) & 1]) * n2 + K2[m & 1];
    *yp = (beta != 0.0) ? fma(beta, *yp, v[m]) : v[m];
  }
}

// Vectorised variant of parity_inv3_kernel: two consecutive k per thread
// (16-byte loads and stores; the mirrored pair n2-1-k, n2-2-k is one reversed
// double2), so every W / U value fetched serves four outputs.  Needs 16-byte
// aligned y, yt, W and even leading dimensions (checked by the caller).
__global__ void __launch_bounds__(128)
    parity_inv3v_kernel(const double* __restrict__ yt, int64_t ldt, double* __restrict__ y, int64_t ldy, int n0, int n1,
                        int n2, double beta, ModeTerms mt) {
  const int h0 = n0 >> 1, h1 = n1 >> 1, h2 = n2 >> 1;
  const int k = 2 * (blockIdx.x * blockDim.x + threadIdx.x), j = blockIdx.y;
  const int i = blockIdx.z % h0, r = blockIdx.z / h0;
  if (k >= h2) return;
  const double* tr = yt + (int64_t)r * ldt;
  double2 v[8];
#pragma unroll
  for (int m = 0; m < 8; m++) {
    const int ii = ((m & 4) ? h0 : 0) + i, jj = ((m & 2) ? h1 : 0) + j, kk = ((m & 1) ? h2 : 0) + k;
    v[m] = *reinterpret_cast<const double2*>(tr + ((int64_t)ii * n1 + jj) * n2 + kk);
  }
#pragma unroll
  for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
    for (int m = 0; m < 8; m++)
      if (!(m & bit)) {
        const double2 a = v[m], b = v[m | bit];
        v[m] = make_double2(a.x + b.x, a.y + b.y);
        v[m | bit] = make_double2(a.x - b.x, a.y - b.y);
      }
  // v[m].x belongs to k (mirror n2-1-k), v[m].y to k+1 (mirror n2-2-k)
#pragma unroll
  for (int m = 0; m < 8; m++) { v[m].x *= 0.125; v[m].y *= 0.125; }
  const int I2[2] = {i, n0 - 1 - i}, J2[2] = {j, n1 - 1 - j};
  const int km = n2 - 2 - k;  // mirrored pair starts here: (km, km+1) mirror (k+1, k)
  for (int e = 0; e < mt.n; e++) {
    const int P = mt.m[e].P, sd = mt.m[e].s;
    const double* U = mt.m[e].U;
    if (sd == 2) {
      // y[i][j][k] += U[k][p] W[p][i][j]: W broadcast over the lanes, U per k
      const int64_t AB = (int64_t)n0 * n1;
      const double* W = mt.m[e].W + (int64_t)r * P * AB;
      for (int p = 0; p < P; p++) {
        const double ua = U[(int64_t)k * P + p], ub = U[(int64_t)(k + 1) * P + p];
        const double uc = U[(int64_t)(km + 1) * P + p], ud = U[(int64_t)km * P + p];  // mirrors of k, k+1
        const double* Wp = W + (int64_t)p * AB;
#pragma unroll
        for (int q = 0; q < 4; q++) {  // q = (mi, mj)
          const double w = Wp[(int64_t)I2[q >> 1] * n1 + J2[q & 1]];
          v[2 * q].x = fma(ua, w, v[2 * q].x);
          v[2 * q].y = fma(ub, w, v[2 * q].y);
          v[2 * q + 1].x = fma(uc, w, v[2 * q + 1].x);
          v[2 * q + 1].y = fma(ud, w, v[2 * q + 1].y);
        }
      }
    } else {
      // sd == 0: y[i][j][k] += U[i][p] W[p][j][k];  sd == 1: y[i][j][k] += U[j][p] W[p][i][k]
      const int64_t AB = (sd == 0 ? (int64_t)n1 : (int64_t)n0) * n2;
      const double* W = mt.m[e].W + (int64_t)r * P * AB;
      const int a0 = sd == 0 ? I2[0] : J2[0], a1 = sd == 0 ? I2[1] : J2[1];
      const int b0 = sd == 0 ? J2[0] : I2[0], b1 = sd == 0 ? J2[1] : I2[1];
      for (int p = 0; p < P; p++) {
        const double u0 = U[(int64_t)a0 * P + p], u1 = U[(int64_t)a1 * P + p];
        const double* Wp = W + (int64_t)p * AB;
        const double2 w00 = *reinterpret_cast<const double2*>(Wp + (int64_t)b0 * n2 + k);
        const double2 w01 = *reinterpret_cast<const double2*>(Wp + (int64_t)b0 * n2 + km);  // (.y, .x) mirror (k, k+1)
        const double2 w10 = *reinterpret_cast<const double2*>(Wp + (int64_t)b1 * n2 + k);
        const double2 w11 = *reinterpret_cast<const double2*>(Wp + (int64_t)b1 * n2 + km);
        // output m = (mi, mj, mk); the W row index b follows mj (sd == 0) or mi (sd == 1),
        // the U index a follows mi (sd == 0) or mj (sd == 1)
#pragma unroll
        for (int m = 0; m < 8; m++) {
          const int mi = m >> 2, mj = (m >> 1) & 1, mk = m & 1;
          const double u = (sd == 0 ? mi : mj) ? u1 : u0;
          const bool brow1 = (sd == 0 ? mj : mi) != 0;
          const double2 w = brow1 ? (mk ? w11 : w10) : (mk ? w01 : w00);
          // mk = 0: (.x, .y) are k, k+1; mk = 1: the mirrored pair, stored reversed
          v[m].x = fma(u, mk ? w.y : w.x, v[m].x);
          v[m].y = fma(u, mk ? w.x : w.y, v[m].y);
        }
      }
    }
  }
  double* yr = y + (int64_t)r * ldy;
#pragma unroll
  for (int m = 0; m < 8; m++) {
    const int64_t row = ((int64_t)I2[m >> 2] * n1 + J2[(m >> 1) & 1]) * n2;
    double2* yp = reinterpret_cast<double2*>(yr + row + ((m & 1) ? km : k));
    double2 o = (m & 1) ? make_double2(v[m].y, v[m].x) : v[m];
    if (beta != 0.0) {
      const double2 old = *yp;
      o.x = fma(beta, old.x, o.x);
      o.y = fma(beta, old.y, o.y);
    }
    *yp = o;
  }
}

double order_flops(int d, int P, const int* nin, const int* nout, bool rev) {
  int cur[GPFVM_MAX_DIMS];
  for (int i = 0; i < d; i++) cur[i] = nin[i];
  double fl = 0.0;
  for (int s = 0; s < d; s++) {
    int i = rev ? d - 1 - s : s;
    double v = 2.0 * P * nout[i] * (double)nin[i];
    for (int k = 0; k < d; k++)
      if (k != i) v *= cur[k];
    fl += v;
    cur[i] = nout[i];
  }
  return fl;
}
}  // namespace

void KronSum::build(int d_, const int* in_shape, const int* out_shape, const std::vector<double>& coefs_in,
                    const std::vector<std::vector<const double*>>& factors_in, cudaStream_t s,
                    const std::vector<std::vector<int>>* signs_in) {
  d = d_;
  for (int i = 0; i < GPFVM_MAX_DIMS; i++) {
    nin[i] = (i < d) ? in_shape[i] : 1;
    nout[i] = (i < d) ? out_shape[i] : 1;
  }
  // Terms that share every factor but one merge exactly (bilinearity):
  //   c_p (x)F_p + c_q (x)F_q = (x)F with F_e = c_p F_p,e + c_q F_q,e
  // e.g. advection-diffusion: (y,y) + (yy,yy) share T00 (x) X00, (x,x) +
  // (xx,xx) share T00 (.) Y00: 9 -> 7 Kronecker terms.
  std::vector<double> coefs = coefs_in;
  std::vector<std::vector<const double*>> factors = factors_in;
  std::vector<std::vector<int>> signs = signs_in ? *signs_in
                                                 : std::vector<std::vector<int>>(coefs.size(), std::vector<int>(d, 0));
  merged.clear();
  static const bool no_merge = getenv("GPFVM_NO_MERGE") != nullptr;
  for (bool again = !no_merge; again;) {
    again = false;
    for (size_t a = 0; a < coefs.size() && !again; a++)
      for (size_t b = a + 1; b < coefs.size() && !again; b++) {
        int e = -1, ndiff = 0;
        for (int i = 0; i < d; i++)
          if (factors[a][i] != factors[b][i]) { e = i; ndiff++; }
        if (ndiff != 1) continue;
        const int64_t fs = (int64_t)nout[e] * nin[e];
        merged.emplace_back();
        DevBuf& m = merged.back();
        m.ensure((size_t)fs);
        lincomb2_kernel<<<gsz(fs), 256, 0, s>>>(m.ptr, coefs[a], factors[a][e], coefs[b], factors[b][e], fs);
        count_launch();
        factors[a][e] = m.ptr;
        coefs[a] = 1.0;
        if (signs[a][e] != signs[b][e]) signs[a][e] = 0;  // mixed parity: no split
        coefs.erase(coefs.begin() + b);
        factors.erase(factors.begin() + b);
        signs.erase(signs.begin() + b);
        again = true;
      }
  }
  P = (int)coefs.size();
  if (P == 0) return;
  // reflection-parity split: every factor of a dimension has the same
  // nonzero sign, square even-length dimensions
  static const bool no_par = getenv("GPFVM_NO_KRON_PARITY") != nullptr;
  par = (d == 2) && !no_par;
  for (int i = 0; i < d && par; i++) {
    par = nin[i] == nout[i] && nin[i] >= 2 && nin[i] % 2 == 0 && signs[0][i] != 0;
    for (int p = 0; p < P && par; p++) par = signs[p][i] == signs[0][i];
    sg[i] = par ? (signs[0][i] < 0 ? 1 : 0) : 0;
  }
  if (par) {
    rev = false;
    mid_thin = last_thin = false;
    const int h0 = nin[0] / 2, h1 = nin[1] / 2;
    stk[0].ensure((size_t)2 * P * h0 * h0);
    stk[1].ensure((size_t)2 * h1 * P * h1);
    for (int p = 0; p < P; p++) {
      half_restack_kernel<<<gsz(2LL * h0 * h0), 256, 0, s>>>(stk[0].ptr, factors[p][0], coefs[p], p, P, nin[0], 0);
      half_restack_kernel<<<gsz(2LL * h1 * h1), 256, 0, s>>>(stk[1].ptr, factors[p][1], 1.0, p, P, nin[1], 1);
      count_launch(2);
    }
    check_launch("KronSum::build (parity)");
    return;
  }
  // 3D reflection-parity split: every factor is centrosymmetric
  // or skew on an even-length mirror-symmetric site list.  The transformed
  // vector keeps its shape with index (class, half index) per dimension; a
  // factor maps input class c to class c ^ skew through its half block H_c, so
  // every contraction of the forward plan becomes a class-batched GEMM with
  // half M and half K: half the flops of every stage.
  // smallest half size worth splitting (read per build: tests lower it)
  const int par3_minh = getenv("GPFVM_PAR3_MINH") ? atoi(getenv("GPFVM_PAR3_MINH")) : 32;
  par3 = (d == 3) && !no_par;
  for (int i = 0; i < d && par3; i++) {
    par3 = nin[i] == nout[i] && nin[i] % 4 == 0 && nin[i] / 2 >= par3_minh;
    for (int p = 0; p < P && par3; p++) par3 = signs[p][i] != 0;
  }
  if (par3) {
    rev = mid_thin = last_thin = false;
    const int h0 = nin[0] / 2, h1 = nin[1] / 2, h2 = nin[2] / 2;
    // distinct dim-0 / dim-2 factors, centrosymmetric ones first
    std::vector<const double*> d0, d2;
    std::vector<int> s0, s2;
    for (int pass = 0; pass < 2; pass++)
      for (int p = 0; p < P; p++) {
        if ((signs[p][0] < 0) == (pass == 1) && std::find(d0.begin(), d0.end(), factors[p][0]) == d0.end()) {
          d0.push_back(factors[p][0]);
          s0.push_back(pass);
        }
        if ((signs[p][2] < 0) == (pass == 1) && std::find(d2.begin(), d2.end(), factors[p][2]) == d2.end()) {
          d2.push_back(factors[p][2]);
          s2.push_back(pass);
        }
      }
    Q0 = (int)d0.size();
    Q2 = (int)d2.size();
    Qs0 = (int)std::count(s0.begin(), s0.end(), 0);
    Qs2 = (int)std::count(s2.begin(), s2.end(), 0);
    u0.assign(P, 0);
    u2.assign(P, 0);
    sk1.assign(P, 0);
    for (int p = 0; p < P; p++) {
      u0[p] = (int)(std::find(d0.begin(), d0.end(), factors[p][0]) - d0.begin());
      u2[p] = (int)(std::find(d2.begin(), d2.end(), factors[p][2]) - d2.begin());
      sk1[p] = signs[p][1] < 0;
    }
    stk[0].ensure((size_t)2 * Q0 * h0 * h0);
    stk[1].ensure((size_t)2 * P * h1 * h1);
    stk[2].ensure((size_t)2 * Q2 * h2 * h2);
    // stk[0]: group (centrosymmetric | skew) stacks [c][(j, qg)][k]
    for (int q = 0; q < Q0; q++) {
      const bool skew = q >= Qs0;
      const int G = skew ? Q0 - Qs0 : Qs0, g = skew ? q - Qs0 : q;
      half_block_kernel<<<gsz(2LL * h0 * h0), 256, 0, s>>>(stk[0].ptr + (skew ? (int64_t)2 * Qs0 * h0 * h0 : 0), d0[q], 1.0,
                                                           nin[0], g, G);
      count_launch();
    }
    for (int p = 0; p < P; p++) {
      half_block_kernel<<<gsz(2LL * h1 * h1), 256, 0, s>>>(stk[1].ptr + (int64_t)p * 2 * h1 * h1, factors[p][1], coefs[p],
                                                           nin[1], 0, 1);
      count_launch();
    }
    for (int q = 0; q < Q2; q++) {
      half_block_kernel<<<gsz(2LL * h2 * h2), 256, 0, s>>>(stk[2].ptr + (int64_t)q * 2 * h2 * h2, d2[q], 1.0, nin[2], 0, 1);
      count_launch();
    }
    check_launch("KronSum::build (3D parity)");
    return;
  }
  rev = (d > 1) && order_flops(d, P, nin, nout, true) < order_flops(d, P, nin, nout, false);
  const int first = rev ? d - 1 : 0;
  mid_thin = (d == 3 && nout[1] == 1 && nin[1] > 1 && P <= 8 && !getenv("GPFVM_NO_MIDTHIN"));
  last_thin = (!mid_thin && d == 3 && nout[2] == 1 && nin[2] > 1 && nout[1] > 1 && P <= 8 && !getenv("GPFVM_NO_MIDTHIN"));
  if (last_thin) {
    // stk[2]: P functionals (1 x n'_2) as a column-major B (P x n'_2); stk[1]:
    // P factors F1^p back to back; stk[0]: c_p F0^p back to back (K-segments)
    stk[0].ensure((size_t)P * nout[0] * nin[0]);
    stk[1].ensure((size_t)P * nout[1] * nin[1]);
    stk[2].ensure((size_t)P * nin[2]);
    for (int p = 0; p < P; p++) {
      scaled_copy_kernel<<<gsz((int64_t)nout[0] * nin[0]), 256, 0, s>>>(stk[0].ptr + (int64_t)p * nout[0] * nin[0],
                                                                         factors[p][0], coefs[p],
                                                                         (int64_t)nout[0] * nin[0]);
      scaled_copy_kernel<<<gsz((int64_t)nout[1] * nin[1]), 256, 0, s>>>(stk[1].ptr + (int64_t)p * nout[1] * nin[1],
                                                                         factors[p][1], 1.0, (int64_t)nout[1] * nin[1]);
      scaled_copy_kernel<<<gsz(nin[2]), 256, 0, s>>>(stk[2].ptr + (int64_t)p * nin[2], factors[p][2], 1.0, nin[2]);
      count_launch(3);
    }
    check_launch("KronSum::build (last-thin)");
    return;
  }
  if (mid_thin) {
    // stk[1]: P functionals (1 x n'_1) stacked as P x n'_1; stk[0]: P time
    // factors c_p F0^p back to back; stk[2]: F2^p columns concatenated (p, k2)
    stk[0].ensure((size_t)P * nout[0] * nin[0]);
    stk[1].ensure((size_t)P * nin[1]);
    stk[2].ensure((size_t)nout[2] * nin[2] * P);
    for (int p = 0; p < P; p++) {
      scaled_copy_kernel<<<gsz((int64_t)nout[0] * nin[0]), 256, 0, s>>>(stk[0].ptr + (int64_t)p * nout[0] * nin[0],
                                                                         factors[p][0], coefs[p],
                                                                         (int64_t)nout[0] * nin[0]);
      scaled_copy_kernel<<<gsz(nin[1]), 256, 0, s>>>(stk[1].ptr + (int64_t)p * nin[1], factors[p][1], 1.0, nin[1]);
      restack_kernel<<<gsz((int64_t)nout[2] * nin[2]), 256, 0, s>>>(stk[2].ptr, factors[p][2], 1.0, p, P, nout[2],
                                                                     nin[2], 1);
      count_launch(3);
    }
    check_launch("KronSum::build (mid-thin)");
    return;
  }
  if (d == 2) {
    // plain-GEMM layouts: forward: stk0 rows interleaved (j0,p) with c_p,
    // stk1 columns concatenated (p,k); reverse: stk1 blocks (p,j1) with c_p, stk0 columns
    // interleaved (k,p).
    for (int i = 0; i < 2; i++) stk[i].ensure((size_t)std::max<int64_t>(1, (int64_t)nout[i] * nin[i] * P));
    for (int p = 0; p < P; p++) {
      if (!rev) {
        restack_kernel<<<gsz((int64_t)nout[0] * nin[0]), 256, 0, s>>>(stk[0].ptr, factors[p][0], coefs[p], p, P,
                                                                       nout[0], nin[0], 0);
        restack_kernel<<<gsz((int64_t)nout[1] * nin[1]), 256, 0, s>>>(stk[1].ptr, factors[p][1], 1.0, p, P, nout[1],
                                                                       nin[1], 1);
      } else {
        scaled_copy_kernel<<<gsz((int64_t)nout[1] * nin[1]), 256, 0, s>>>(stk[1].ptr + (int64_t)p * nout[1] * nin[1],
                                                                           factors[p][1], coefs[p],
                                                                           (int64_t)nout[1] * nin[1]);
        restack_kernel<<<gsz((int64_t)nout[0] * nin[0]), 256, 0, s>>>(stk[0].ptr, factors[p][0], 1.0, p, P, nout[0],
                                                                       nin[0], 2);
      }
      count_launch(2);
    }
    check_launch("KronSum::build (2D)");
    return;
  }
  if (d == 3 && !rev) {
    // 3D forward plain layout: stk0 rows interleaved (j0,q) over the Q0 distinct
    // dim-0 factors, stk1 P plain blocks with c_p, stk2 columns concatenated
    // (q,k2) over the Q2 distinct dim-2 factors.  Terms sharing a factor share
    // its stage-0 slice / stage-2 K-segment (e.g. the 6 wave-operator term pairs
    // use 3 time and 3 y factors: stage 0 and stage 2 flops halve).  Dedup only
    // where the middle stage runs per term (the layout it needs).
    const bool per_term = P > 1 && nout[1] >= 64 && nin[2] >= 32 && !getenv("GPFVM_NO_DEDUP");
    u0.assign(P, 0);
    u2.assign(P, 0);
    std::vector<const double*> d0, d2;
    for (int p = 0; p < P; p++) {
      int q0 = per_term ? (int)(std::find(d0.begin(), d0.end(), factors[p][0]) - d0.begin()) : (int)d0.size();
      if (q0 == (int)d0.size()) d0.push_back(factors[p][0]);
      int q2 = per_term ? (int)(std::find(d2.begin(), d2.end(), factors[p][2]) - d2.begin()) : (int)d2.size();
      if (q2 == (int)d2.size()) d2.push_back(factors[p][2]);
      u0[p] = q0;
      u2[p] = q2;
    }
    Q0 = (int)d0.size();
    Q2 = (int)d2.size();
    // without dedup the coefficient stays on the dim-0 factor (identity maps)
    stk[0].ensure((size_t)std::max<int64_t>(1, (int64_t)nout[0] * nin[0] * Q0));
    stk[1].ensure((size_t)std::max<int64_t>(1, (int64_t)nout[1] * nin[1] * P));
    stk[2].ensure((size_t)std::max<int64_t>(1, (int64_t)nout[2] * nin[2] * Q2));
    for (int q = 0; q < Q0; q++) {
      restack_kernel<<<gsz((int64_t)nout[0] * nin[0]), 256, 0, s>>>(stk[0].ptr, d0[q], per_term ? 1.0 : coefs[q], q,
                                                                     Q0, nout[0], nin[0], 0);
      count_launch();
    }
    for (int p = 0; p < P; p++) {
      scaled_copy_kernel<<<gsz((int64_t)nout[1] * nin[1]), 256, 0, s>>>(stk[1].ptr + (int64_t)p * nout[1] * nin[1],
                                                                         factors[p][1], per_term ? coefs[p] : 1.0,
                                                                         (int64_t)nout[1] * nin[1]);
      count_launch();
    }
    for (int q = 0; q < Q2; q++) {
      restack_kernel<<<gsz((int64_t)nout[2] * nin[2]), 256, 0, s>>>(stk[2].ptr, d2[q], 1.0, q, Q2, nout[2], nin[2], 1);
      count_launch();
    }
    check_launch("KronSum::build (3D)");
    return;
  }
  for (int i = 0; i < d; i++) {
    int64_t fs = (int64_t)nout[i] * nin[i];
    stk[i].ensure((size_t)std::max<int64_t>(1, fs * P));
    for (int p = 0; p < P; p++) {
      double c = (i == first) ? coefs[p] : 1.0;
      scaled_copy_kernel<<<gsz(fs), 256, 0, s>>>(stk[i].ptr + p * fs, factors[p][i], c, fs);
      count_launch();
    }
  }
  check_launch("KronSum::build");
}

int64_t KronSum::workspace_per_rhs() const {
  if (P == 0 || d == 1) return 0;
  if (par3) return (int64_t)std::max(std::max(Q0, Q2), 1) * nin[0] * nin[1] * nin[2];
  if (mid_thin) return (int64_t)std::max(nin[0], nout[0]) * P * nin[2];
  if (last_thin) return (int64_t)nin[0] * P * std::max(nin[1], nout[1]);
  int64_t mx = 0;
  for (int s = 0; s <= d - 2; s++) {
    int64_t sz = P;
    for (int k = 0; k < d; k++) {
      bool done = rev ? (k >= d - 1 - s) : (k <= s);
      sz *= done ? nout[k] : nin[k];
    }
    mx = std::max(mx, sz);
  }
  return mx;
}

double KronSum::flops_per_rhs() const {
  if (P == 0) return 0.0;
  if (par) return order_flops(d, P, nin, nout, false) / 2.0;
  if (par3)
    return ((double)Q0 * nout[0] * nin[0] * nin[1] * nin[2] + (double)P * nout[0] * nout[1] * nin[1] * nin[2] +
            (double)Q2 * nout[0] * nout[1] * nout[2] * nin[2]);
  if (mid_thin)
    return 2.0 * P * ((double)nin[0] * nin[1] * nin[2] + (double)nout[0] * nin[0] * nin[2] +
                      (double)nout[0] * nout[2] * nin[2]);
  if (last_thin)
    return 2.0 * P * ((double)nin[0] * nin[1] * nin[2] + (double)nin[0] * nout[1] * nin[1] +
                      (double)nout[0] * nin[0] * nout[1]);
  if (d == 3 && !rev && Q0 > 0)
    return 2.0 * ((double)Q0 * nout[0] * nin[0] * nin[1] * nin[2] + (double)P * nout[0] * nout[1] * nin[1] * nin[2] +
                  (double)Q2 * nout[0] * nout[1] * nout[2] * nin[2]);
  return order_flops(d, P, nin, nout, rev);
}

void KronSum::apply(const double* x, int64_t ldx, double* y, int64_t ldy, int R, double beta, double* w0, double* w1,
                    cudaStream_t s, const Gemm* extra, cudaEvent_t extra_ready, const double* stage0,
                    const ModeTerms* modes) const {
  GPFVM_CHECK(!modes || par3, GPFVM_ERR_STATE, "mode terms need the 3D parity-split plan");
  if (extra_ready && !par && !par3) {  // only the parity path defers the wait to the kernel that reads the extra term
    GPFVM_CUDA(cudaStreamWaitEvent(s, extra_ready, 0));
    extra_ready = nullptr;
  }
  if (extra && extra->K2 > 0 && !(d == 2 && !rev && P > 0)) {
    // not fusable here: the Kronecker sum, then the low-rank term as its own GEMM
    apply(x, ldx, y, ldy, R, beta, w0, w1, s, nullptr, nullptr, stage0, modes);
    Gemm e;
    e.M = d == 2 ? nout[0] : 1; e.N = nout[d - 1];
    for (int k = 1; k < d - 1; k++) e.M *= nout[k];
    e.K = extra->K2; e.batch1 = R;
    e.A = extra->A2; e.a_rs = extra->a2_rs; e.a_cs = 1; e.a_b1 = extra->a2_b1;
    e.B = extra->B2; e.b_rs = 1; e.b_cs = extra->b2_rs; e.b_b1 = extra->b2_b1;
    e.C = y; e.c_rs = nout[d - 1]; e.c_cs = 1; e.c_b1 = ldy;
    e.beta = 1.0;
    run_gemm(e, s);
    return;
  }
  if (P == 0) {
    if (beta == 0.0) {
      int64_t osz = 1;
      for (int k = 0; k < d; k++) osz *= nout[k];
      for (int r = 0; r < R; r++) fill(y + r * ldy, 0.0, osz, s);
    }
    return;
  }
  if (d == 1) {
    Gemm g;
    g.M = R; g.N = nout[0]; g.K = nin[0]; g.nseg = P;
    g.A = x; g.a_rs = ldx; g.a_cs = 1; g.a_sg = 0;
    g.B = stk[0].ptr; g.b_rs = 1; g.b_cs = nin[0]; g.b_sg = (int64_t)nout[0] * nin[0];
    g.C = y; g.c_rs = ldy; g.c_cs = 1;
    g.beta = beta;
    run_gemm(g, s);
    return;
  }
  const int l = d - 1;
  if (par) {
    // X -> parity classes (w1), stage 0 over the time classes, stage 1 over the
    // space classes, classes -> Y (+ low-rank term, beta)
    const int h0 = nin[0] / 2, h1 = nin[1] / 2;
    const int64_t cls = (int64_t)h0 * h1, zc = (int64_t)P * cls;
    parity_fwd2_kernel<<<(unsigned)std::min<int64_t>((R * cls + 255) / 256, 148 * 16), 256, 0, s>>>(x, ldx, w1, R,
                                                                                                   nin[0], nin[1]);
    count_launch();
    Gemm g0, g1;
    // Z[a][(r,b)][(j0,p)][k1] = sum_k0 H0_a[(j0,p)][k0] Xt[a][(r,b)][k0][k1]
    g0.M = P * h0; g0.N = h1; g0.K = h0;
    g0.A = stk[0].ptr; g0.a_rs = h0; g0.a_cs = 1; g0.a_b1 = 0; g0.a_b2 = (int64_t)P * h0 * h0;
    g0.B = w1; g0.b_rs = h1; g0.b_cs = 1; g0.b_b1 = cls; g0.b_b2 = 2LL * R * cls;
    g0.C = w0; g0.c_rs = h1; g0.c_cs = 1; g0.c_b1 = zc; g0.c_b2 = 2LL * R * zc;
    g0.batch1 = 2 * R; g0.batch2 = 2;
    run_gemm(g0, s);
    // Yt[(a,r)][b][j0][j1] = sum_(p,k1) Z[(a,r)][b][j0][(p,k1)] H1_b[j1][(p,k1)]
    g1.M = h0; g1.N = h1; g1.K = P * h1;
    g1.A = w0; g1.a_rs = (int64_t)P * h1; g1.a_cs = 1; g1.a_b1 = 2 * zc; g1.a_b2 = zc;
    g1.B = stk[1].ptr; g1.b_rs = 1; g1.b_cs = (int64_t)P * h1; g1.b_b1 = 0; g1.b_b2 = (int64_t)h1 * P * h1;
    g1.C = w1; g1.c_rs = h1; g1.c_cs = 1; g1.c_b1 = 2 * cls; g1.c_b2 = cls;
    g1.batch1 = 2 * R; g1.batch2 = 2;
    run_gemm(g1, s);
    const bool lr = extra && extra->K2 > 0;
    if (extra_ready) GPFVM_CUDA(cudaStreamWaitEvent(s, extra_ready, 0));  // U, V prepared on a side stream
    const double* Ue = lr ? extra->A2 : nullptr;
    const double* Ve = lr ? extra->B2 : nullptr;
    const bool vec = (h1 % 2 == 0) && ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(w1)) & 15) == 0 &&
                     (ldy % 2 == 0) && h0 <= 65535 && R <= 65535;
    if (vec) {
      const dim3 grid((unsigned)((h1 / 2 + 127) / 128), (unsigned)h0, (unsigned)R);
      parity_inv2v_kernel<<<grid, 128, 0, s>>>(w1, y, ldy, R, nin[0], nin[1], sg[0], sg[1], beta, Ue, lr ? extra->a2_rs : 0,
                                               lr ? extra->a2_b1 : 0, Ve, lr ? extra->b2_rs : 0, lr ? extra->b2_b1 : 0,
                                               lr ? extra->K2 : 0);
    } else {
      parity_inv2_kernel<<<(unsigned)std::min<int64_t>((R * cls + 255) / 256, 148 * 16), 256, 0, s>>>(
          w1, y, ldy, R, nin[0], nin[1], sg[0], sg[1], beta, Ue, lr ? extra->a2_rs : 0, lr ? extra->a2_b1 : 0, Ve,
          lr ? extra->b2_rs : 0, lr ? extra->b2_b1 : 0, lr ? extra->K2 : 0);
    }
    count_launch();
    check_launch("KronSum::apply (parity)");
    return;
  }
  if (par3) {
    const int64_t n0 = nin[0], n1 = nin[1], n2 = nin[2], h0 = n0 / 2, h1 = n1 / 2, h2 = n2 / 2;
    const int64_t rest = n1 * n2, n = n0 * rest;
    // X -> Xt (w1)
    const int rc = (int)std::max<int64_t>(1, std::min<int64_t>(R, 65535 / h0));
    for (int r0 = 0; r0 < R; r0 += rc) {
      const int rn = std::min(rc, R - r0);
      parity_fwd3_kernel<<<dim3((unsigned)((h2 + 127) / 128), (unsigned)h1, (unsigned)(h0 * rn)), 128, 0, s>>>(
          x + (int64_t)r0 * ldx, ldx, w1 + (int64_t)r0 * n, n, (int)n0, (int)n1, (int)n2);
      count_launch();
    }
    // stage 0 per group: Z0_g[r][(c0', i')][qg][rest] = H0_(qg, c0) Xt_r[(c0, i)][rest]
    const int64_t G[2] = {Qs0, Q0 - Qs0};
    const int64_t zbase[2] = {0, (int64_t)R * n0 * Qs0 * rest};
    for (int g = 0; g < 2; g++) {
      if (G[g] == 0) continue;
      Gemm g0;
      g0.M = (int)(G[g] * h0); g0.N = (int)rest; g0.K = (int)h0;
      g0.A = stk[0].ptr + (g ? 2 * Qs0 * h0 * h0 : 0); g0.a_rs = h0; g0.a_cs = 1; g0.a_b1 = 0; g0.a_b2 = G[g] * h0 * h0;
      g0.B = w1; g0.b_rs = rest; g0.b_cs = 1; g0.b_b1 = n; g0.b_b2 = h0 * rest;
      g0.C = w0 + zbase[g] + (g ? h0 * G[g] * rest : 0); g0.c_rs = rest; g0.c_cs = 1; g0.c_b1 = n0 * G[g] * rest;
      g0.c_b2 = (g ? -1 : 1) * h0 * G[g] * rest;
      g0.batch1 = R; g0.batch2 = 2;
      run_gemm(g0, s);
    }
    // stage 1 per term over the combined (r, j0) batch and the dim-1 class:
    //   Z1[(r, j0)][(c1', j1')][slot][n2] (+)= c_p H1_(p, c1) Z0[(r, j0)][(c1, k1)][n2]
    const int64_t z1row = (int64_t)Q2 * n2;
    std::vector<char> seen(Q2, 0);
    for (int p = 0; p < P; p++) {
      const int g = u0[p] >= Qs0, qg = g ? u0[p] - Qs0 : u0[p];
      Gemm g1;
      g1.M = (int)h1; g1.N = (int)n2; g1.K = (int)h1;
      g1.A = stk[1].ptr + (int64_t)p * 2 * h1 * h1; g1.a_rs = h1; g1.a_cs = 1; g1.a_b1 = 0; g1.a_b2 = h1 * h1;
      g1.B = w0 + zbase[g] + qg * rest; g1.b_rs = n2; g1.b_cs = 1; g1.b_b1 = G[g] * rest; g1.b_b2 = h1 * n2;
      g1.C = w1 + (int64_t)u2[p] * n2 + (sk1[p] ? h1 * z1row : 0); g1.c_rs = z1row; g1.c_cs = 1; g1.c_b1 = n1 * z1row;
      g1.c_b2 = (sk1[p] ? -1 : 1) * h1 * z1row;
      g1.batch1 = (int)(R * n0); g1.batch2 = 2;
      g1.beta = seen[u2[p]] ? 1.0 : 0.0;
      seen[u2[p]] = 1;
      run_gemm(g1, s);
    }
    // stage 2 per group of dim-2 factors (K segments over its slots):
    //   Yt_r[(j0, j1)][(c2', k')] (+)= sum_(slot, k) Z1_r[(j0, j1)][slot][(c2, k)] H2_(slot, c2)[k'][k]
    bool first = true;
    for (int g = 0; g < 2; g++) {
      const int64_t ns = g ? Q2 - Qs2 : Qs2, s0 = g ? Qs2 : 0;
      if (ns == 0) continue;
      Gemm g2;
      g2.M = (int)(n0 * n1); g2.N = (int)h2; g2.K = (int)h2; g2.nseg = (int)ns;
      g2.A = w1 + s0 * n2; g2.a_rs = z1row; g2.a_cs = 1; g2.a_sg = n2; g2.a_b1 = n0 * n1 * z1row; g2.a_b2 = h2;
      g2.B = stk[2].ptr + s0 * 2 * h2 * h2; g2.b_rs = 1; g2.b_cs = h2; g2.b_sg = 2 * h2 * h2; g2.b_b1 = 0; g2.b_b2 = h2 * h2;
      g2.C = w0 + (g ? h2 : 0); g2.c_rs = n2; g2.c_cs = 1; g2.c_b1 = n; g2.c_b2 = (g ? -1 : 1) * h2;
      g2.batch1 = R; g2.batch2 = 2;
      g2.beta = first ? 0.0 : 1.0;
      first = false;
      run_gemm(g2, s);
    }
    if (extra_ready) GPFVM_CUDA(cudaStreamWaitEvent(s, extra_ready, 0));  // mode operands prepared on a side stream
    for (int r0 = 0; r0 < R; r0 += rc) {
      const int rn = std::min(rc, R - r0);
      ModeTerms mt;
      if (modes) {
        mt = *modes;
        for (int e = 0; e < mt.n; e++) mt.m[e].W += (int64_t)r0 * mt.m[e].P * (n / nin[mt.m[e].s]);
      }
      static const bool no_vec = getenv("GPFVM_NO_INV3V") != nullptr;
      bool vec = !no_vec && ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(w0)) & 15) == 0 && (ldy & 1) == 0;
      for (int e = 0; e < mt.n; e++) vec = vec && (reinterpret_cast<uintptr_t>(mt.m[e].W) & 15) == 0;
      if (vec)
        parity_inv3v_kernel<<<dim3((unsigned)((h2 / 2 + 127) / 128), (unsigned)h1, (unsigned)(h0 * rn)), 128, 0, s>>>(
            w0 + (int64_t)r0 * n, n, y + (int64_t)r0 * ldy, ldy, (int)n0, (int)n1, (int)n2, beta, mt);
      else
        parity_inv3_kernel<<<dim3((unsigned)((h2 + 127) / 128), (unsigned)h1, (unsigned)(h0 * rn)), 128, 0, s>>>(
            w0 + (int64_t)r0 * n, n, y + (int64_t)r0 * ldy, ldy, (int)n0, (int)n1, (int)n2, beta, mt);
      count_launch();
    }
    check_launch("KronSum::apply (3D parity)");
    return;
  }
  if (mid_thin) {
    // A: R[r][a][p][k2] = sum_k1 f_p[k1] X_r[a][k1][k2]   (few-row GEMM over row-major slices)
    const int64_t rsz = (int64_t)nin[0] * P * nin[2], zsz = (int64_t)nout[0] * P * nin[2];
    Gemm ga;
    ga.M = P; ga.N = nin[2]; ga.K = nin[1];
    ga.A = stk[1].ptr; ga.a_rs = nin[1]; ga.a_cs = 1;
    ga.B = x; ga.b_rs = nin[2]; ga.b_cs = 1; ga.b_b1 = (int64_t)nin[1] * nin[2]; ga.b_b2 = ldx;
    ga.C = w0; ga.c_rs = nin[2]; ga.c_cs = 1; ga.c_b1 = (int64_t)P * nin[2]; ga.c_b2 = rsz;
    ga.batch1 = nin[0]; ga.batch2 = R;
    run_gemm(ga, s);
    // B: Z[r][j0][p][k2] = sum_a c_p F0^p[j0][a] R[r][a][p][k2]   (per term)
    for (int p = 0; p < P; p++) {
      Gemm gb;
      gb.M = nout[0]; gb.N = nin[2]; gb.K = nin[0];
      gb.A = stk[0].ptr + (int64_t)p * nout[0] * nin[0]; gb.a_rs = nin[0]; gb.a_cs = 1;
      gb.B = w0 + (int64_t)p * nin[2]; gb.b_rs = (int64_t)P * nin[2]; gb.b_cs = 1; gb.b_b1 = rsz;
      gb.C = w1 + (int64_t)p * nin[2]; gb.c_rs = (int64_t)P * nin[2]; gb.c_cs = 1; gb.c_b1 = zsz;
      gb.batch1 = R;
      run_gemm(gb, s);
    }
    // C: Y_r[j0][j2] = beta Y + sum_(p,k2) Z[r][j0][(p,k2)] F2^p[j2][k2]
    Gemm gc;
    gc.M = nout[0]; gc.N = nout[2]; gc.K = P * nin[2];
    gc.A = w1; gc.a_rs = (int64_t)P * nin[2]; gc.a_cs = 1; gc.a_b1 = zsz;
    gc.B = stk[2].ptr; gc.b_rs = 1; gc.b_cs = (int64_t)P * nin[2];
    gc.C = y; gc.c_rs = nout[2]; gc.c_cs = 1; gc.c_b1 = ldy;
    gc.batch1 = R;
    gc.beta = beta;
    run_gemm(gc, s);
    return;
  }
  if (last_thin) {
    const int64_t rows = (int64_t)nin[0] * nin[1];
    // A: T[r][(a,k1)][p] = sum_k2 X_r[(a,k1)][k2] f_p[k2]   (few-column GEMM, X read once)
    Gemm ga;
    ga.M = (int)rows; ga.N = P; ga.K = nin[2];
    ga.A = x; ga.a_rs = nin[2]; ga.a_cs = 1; ga.a_b1 = ldx;
    ga.B = stk[2].ptr; ga.b_rs = 1; ga.b_cs = nin[2];
    ga.C = w1; ga.c_rs = P; ga.c_cs = 1; ga.c_b1 = rows * P;
    ga.batch1 = R;
    run_gemm(ga, s);
    // p outermost: T'[p][r][(a,k1)]
    p_outer_kernel<<<gsz(rows * R * P), 256, 0, s>>>(w0, w1, R, rows, P);
    count_launch();
    // B: U[p][(r,a)][j1] = sum_k1 T'[p][(r,a)][k1] F1^p[j1][k1]   (per term)
    const int64_t usz = (int64_t)R * nin[0] * nout[1];
    for (int p = 0; p < P; p++) {
      Gemm gb;
      gb.M = R * nin[0]; gb.N = nout[1]; gb.K = nin[1];
      gb.A = w0 + (int64_t)p * R * rows; gb.a_rs = nin[1]; gb.a_cs = 1;
      gb.B = stk[1].ptr + (int64_t)p * nout[1] * nin[1]; gb.b_rs = 1; gb.b_cs = nin[1];
      gb.C = w1 + (int64_t)p * usz; gb.c_rs = nout[1]; gb.c_cs = 1;
      run_gemm(gb, s);
    }
    // C: Y_r[j0][j1] = beta Y + sum_(p,a) c_p F0^p[j0][a] U[p][r][a][j1]   (K-segments over p)
    Gemm gc;
    gc.M = nout[0]; gc.N = nout[1]; gc.K = nin[0]; gc.nseg = P;
    gc.A = stk[0].ptr; gc.a_rs = nin[0]; gc.a_cs = 1; gc.a_sg = (int64_t)nout[0] * nin[0];
    gc.B = w1; gc.b_rs = nout[1]; gc.b_cs = 1; gc.b_sg = usz; gc.b_b1 = (int64_t)nin[0] * nout[1];
    gc.C = y; gc.c_rs = nout[1]; gc.c_cs = 1; gc.c_b1 = ldy;
    gc.batch1 = R;
    gc.beta = beta;
    run_gemm(gc, s);
    return;
  }
  if (d == 2) {
    const int64_t z0 = (int64_t)P * (rev ? nin[0] * nout[1] : nout[0] * nin[1]);
    Gemm g0, g1;
    if (!rev) {
      // Z_r[(j0,p)][k1] = sum_k0 c_p F0^p[j0][k0] X_r[k0][k1]
      g0.M = P * nout[0]; g0.N = nin[1]; g0.K = nin[0];
      g0.A = stk[0].ptr; g0.a_rs = nin[0]; g0.a_cs = 1;
      g0.B = x; g0.b_rs = nin[1]; g0.b_cs = 1; g0.b_b1 = ldx;
      g0.C = w0; g0.c_rs = nin[1]; g0.c_cs = 1; g0.c_b1 = z0;
      // Y_r[j0][j1] = sum_(p,k1) Z_r[j0][(p,k1)] F1^p[j1][k1]
      g1.M = nout[0]; g1.N = nout[1]; g1.K = P * nin[1];
      g1.A = w0; g1.a_rs = (int64_t)P * nin[1]; g1.a_cs = 1; g1.a_b1 = z0;
      g1.B = stk[1].ptr; g1.b_rs = 1; g1.b_cs = (int64_t)P * nin[1];
    } else {
      // Z_r[k0][(p,j1)] = sum_k1 X_r[k0][k1] c_p F1^p[j1][k1]
      g0.M = nin[0]; g0.N = P * nout[1]; g0.K = nin[1];
      g0.A = x; g0.a_rs = nin[1]; g0.a_cs = 1; g0.a_b1 = ldx;
      g0.B = stk[1].ptr; g0.b_rs = 1; g0.b_cs = nin[1];
      g0.C = w0; g0.c_rs = (int64_t)P * nout[1]; g0.c_cs = 1; g0.c_b1 = z0;
      // Y_r[j0][j1] = sum_(k0,p) F0^p[j0][k0] Z_r[(k0,p)][j1]
      g1.M = nout[0]; g1.N = nout[1]; g1.K = nin[0] * P;
      g1.A = stk[0].ptr; g1.a_rs = (int64_t)nin[0] * P; g1.a_cs = 1;
      g1.B = w0; g1.b_rs = nout[1]; g1.b_cs = 1; g1.b_b1 = z0;
    }
    g0.batch1 = R;
    g1.C = y; g1.c_rs = nout[1]; g1.c_cs = 1; g1.c_b1 = ldy;
    g1.batch1 = R;
    g1.beta = beta;
    if (extra && extra->K2 > 0) {
      g1.K2 = extra->K2;
      g1.A2 = extra->A2; g1.a2_rs = extra->a2_rs; g1.a2_b1 = extra->a2_b1;
      g1.B2 = extra->B2; g1.b2_rs = extra->b2_rs; g1.b2_b1 = extra->b2_b1;
    }
    if (stage0) {
      (rev ? g1.B : g1.A) = stage0;
    } else {
      run_gemm(g0, s);
    }
    run_gemm(g1, s);
    return;
  }
  if (d == 3 && !rev) {
    const int64_t n0 = nout[0], n1 = nout[1], n2 = nout[2], m0 = nin[0], m1 = nin[1], m2 = nin[2];
    const bool per_term = P > 1 && n1 >= 64 && m2 >= 32 && Q0 > 0;
    const int64_t q0 = per_term ? Q0 : P, q2 = per_term ? Q2 : P;
    const int64_t z0 = q0 * n0 * m1 * m2;  // [r][(j0,q0)][k1][k2]
    const int64_t z1 = n0 * n1 * q2 * m2;  // [r][j0][j1][q2][k2]
    Gemm g0, g1, g2;
    // stage 0: Z0_r[(j0,q)][(k1,k2)] = sum_k0 F0^q[j0][k0] X_r[k0][(k1,k2)]
    g0.M = (int)(q0 * n0); g0.N = (int)(m1 * m2); g0.K = (int)m0;
    g0.A = stk[0].ptr; g0.a_rs = m0; g0.a_cs = 1;
    g0.B = x; g0.b_rs = m1 * m2; g0.b_cs = 1; g0.b_b1 = ldx;
    g0.C = w0; g0.c_rs = m1 * m2; g0.c_cs = 1; g0.c_b1 = z0;
    g0.batch1 = R;
    run_gemm(g0, s);
    // stage 1 per (j0, p, r): Z1[j1][k2] = F1^p[j1][:] Z0[j0][p][:][k2], written as [j0][j1][p][k2]
    g1.M = (int)n1; g1.N = (int)m2; g1.K = (int)m1;
    g1.A = stk[1].ptr; g1.a_rs = m1; g1.a_cs = 1; g1.a_b2 = n1 * m1;
    g1.B = w0; g1.b_rs = m2; g1.b_cs = 1;
    g1.b_b1 = (int64_t)P * m1 * m2; g1.b_b2 = m1 * m2; g1.b_b3 = z0;
    g1.C = w1; g1.c_rs = (int64_t)P * m2; g1.c_cs = 1;
    g1.c_b1 = n1 * P * m2; g1.c_b2 = m2; g1.c_b3 = z1;
    g1.batch1 = (int)n0; g1.batch2 = P; g1.batch3 = R;
    if (per_term) {
      // one plain batched GEMM per term over the combined (r, j0) batch (uniform
      // strides) so the tensor-op template applies; terms with the same dim-2
      // factor accumulate into the same K-segment
      std::vector<char> seen(q2, 0);
      for (int p = 0; p < P; p++) {
        Gemm gp = g1;
        gp.A = stk[1].ptr + (int64_t)p * n1 * m1; gp.a_b2 = 0;
        gp.B = w0 + (int64_t)u0[p] * m1 * m2; gp.b_b1 = q0 * m1 * m2; gp.b_b2 = gp.b_b3 = 0;
        gp.C = w1 + (int64_t)u2[p] * m2; gp.c_rs = q2 * m2; gp.c_b1 = n1 * q2 * m2; gp.c_b2 = gp.c_b3 = 0;
        gp.batch1 = (int)(n0 * R); gp.batch2 = gp.batch3 = 1;
        gp.beta = seen[u2[p]] ? 1.0 : 0.0;
        seen[u2[p]] = 1;
        run_gemm(gp, s);
      }
    } else {
      run_gemm(g1, s);
    }
    // stage 2: Y_r[(j0,j1)][j2] = sum_(q,k2) Z1_r[(j0,j1)][(q,k2)] F2^q[j2][k2]
    g2.M = (int)(n0 * n1); g2.N = (int)n2; g2.K = (int)(q2 * m2);
    g2.A = w1; g2.a_rs = q2 * m2; g2.a_cs = 1; g2.a_b1 = z1;
    g2.B = stk[2].ptr; g2.b_rs = 1; g2.b_cs = q2 * m2;
    g2.C = y; g2.c_rs = n2; g2.c_cs = 1; g2.c_b1 = ldy;
    g2.batch1 = R;
    g2.beta = beta;
    run_gemm(g2, s);
    return;
  }
  if (!rev) {
    // stage 0: stacked M over p
    int64_t rest = 1;
    for (int k = 1; k < d; k++) rest *= nin[k];
    const int64_t z0 = (int64_t)P * nout[0] * rest;
    {
      Gemm g;
      g.M = P * nout[0]; g.N = (int)rest; g.K = nin[0];
      g.A = stk[0].ptr; g.a_rs = nin[0]; g.a_cs = 1;
      g.B = x; g.b_rs = rest; g.b_cs = 1; g.b_b1 = ldx;
      g.C = w0; g.c_rs = rest; g.c_cs = 1; g.c_b1 = z0;
      g.batch1 = R;
      run_gemm(g, s);
    }
    const double* cur = w0;
    int64_t cur_sz = z0;
    double* other = w1;
    for (int i = 1; i <= d - 2; i++) {
      int64_t outer = 1, inner = 1;
      for (int k = 0; k < i; k++) outer *= nout[k];
      for (int k = i + 1; k < d; k++) inner *= nin[k];
      const int64_t nsz = (int64_t)P * outer * nout[i] * inner;
      Gemm g;
      g.M = nout[i]; g.N = (int)inner; g.K = nin[i];
      g.A = stk[i].ptr; g.a_rs = nin[i]; g.a_cs = 1; g.a_b2 = (int64_t)nout[i] * nin[i];
      g.B = cur; g.b_rs = inner; g.b_cs = 1;
      g.b_b1 = (int64_t)nin[i] * inner; g.b_b2 = outer * nin[i] * inner; g.b_b3 = cur_sz;
      g.C = other; g.c_rs = inner; g.c_cs = 1;
      g.c_b1 = (int64_t)nout[i] * inner; g.c_b2 = outer * nout[i] * inner; g.c_b3 = nsz;
      g.batch1 = (int)outer; g.batch2 = P; g.batch3 = R;
      run_gemm(g, s);
      cur = other;
      other = (other == w1) ? w0 : w1;
      cur_sz = nsz;
    }
    int64_t rows = 1;
    for (int k = 0; k < l; k++) rows *= nout[k];
    Gemm g;
    g.M = (int)rows; g.N = nout[l]; g.K = nin[l]; g.nseg = P;
    g.A = cur; g.a_rs = nin[l]; g.a_cs = 1; g.a_sg = rows * nin[l]; g.a_b1 = cur_sz;
    g.B = stk[l].ptr; g.b_rs = 1; g.b_cs = nin[l]; g.b_sg = (int64_t)nout[l] * nin[l];
    g.C = y; g.c_rs = nout[l]; g.c_cs = 1; g.c_b1 = ldy;
    g.batch1 = R;
    g.beta = beta;
    run_gemm(g, s);
    return;
  }
  // ---- reverse order ----
  int64_t rows0 = 1;
  for (int k = 0; k < l; k++) rows0 *= nin[k];
  const int64_t z0 = rows0 * P * nout[l];
  {
    // Z[r][rows'][(p, j_l)] = X_r[rows'][:] . stk_l[(p, j_l)][:]   (B column-major, b_cs = n'_l)
    Gemm g;
    g.M = (int)rows0; g.N = P * nout[l]; g.K = nin[l];
    g.A = x; g.a_rs = nin[l]; g.a_cs = 1; g.a_b1 = ldx;
    g.B = stk[l].ptr; g.b_rs = 1; g.b_cs = nin[l];
    g.C = w0; g.c_rs = (int64_t)P * nout[l]; g.c_cs = 1; g.c_b1 = z0;
    g.batch1 = R;
    run_gemm(g, s);
  }
  const double* cur = w0;
  int64_t cur_sz = z0;
  double* other = w1;
  for (int i = l - 1; i >= 1; i--) {
    // Zin[r][o][j'][p][inner] -> Zout[r][o][p][j_i][inner]
    int64_t outer = 1, inner = 1;
    for (int k = 0; k < i; k++) outer *= nin[k];
    for (int k = i + 1; k < d; k++) inner *= nout[k];
    const int64_t nsz = outer * P * nout[i] * inner;
    Gemm g;
    g.M = nout[i]; g.N = (int)inner; g.K = nin[i];
    g.A = stk[i].ptr; g.a_rs = nin[i]; g.a_cs = 1; g.a_b2 = (int64_t)nout[i] * nin[i];
    g.B = cur; g.b_rs = (int64_t)P * inner; g.b_cs = 1;
    g.b_b1 = (int64_t)nin[i] * P * inner; g.b_b2 = inner; g.b_b3 = cur_sz;
    g.C = other; g.c_rs = inner; g.c_cs = 1;
    g.c_b1 = (int64_t)P * nout[i] * inner; g.c_b2 = (int64_t)nout[i] * inner; g.c_b3 = nsz;
    g.batch1 = (int)outer; g.batch2 = P; g.batch3 = R;
    run_gemm(g, s);
    cur = other;
    other = (other == w1) ? w0 : w1;
    cur_sz = nsz;
  }
  // final: Y_r[j0][rest] += sum_p F_0^p Z[r][:, p, :]
  int64_t rest = 1;
  for (int k = 1; k < d; k++) rest *= nout[k];
  Gemm g;
  g.M = nout[0]; g.N = (int)rest; g.K = nin[0]; g.nseg = P;
  g.A = stk[0].ptr; g.a_rs = nin[0]; g.a_cs = 1; g.a_sg = (int64_t)nout[0] * nin[0];
  g.B = cur; g.b_rs = (int64_t)P * rest; g.b_cs = 1; g.b_sg = rest; g.b_b1 = cur_sz;
  g.C = y; g.c_rs = rest; g.c_cs = 1; g.c_b1 = ldy;
  g.batch1 = R;
  g.beta = beta;
  run_gemm(g, s);
}

}  // namespace gpfvm

// ---- C ABI: standalone Kronecker-sum matvec ------------------------------------
namespace gpfvm {
int guarded_kron(int ndim, const int* in_shape, const int* out_shape, int P, const double* coefs,
                 const double* const* factors, const double* x, int64_t ldx, double* y, int64_t ldy, int R,
                 double beta, cudaStream_t s) {
  try {
    GPFVM_CHECK(ndim >= 1 && ndim <= GPFVM_MAX_DIMS && P >= 0 && R >= 1, GPFVM_ERR_INVALID, "bad kron_matvec sizes");
    GPFVM_CHECK(in_shape && out_shape && (P == 0 || (coefs && factors)) && x && y, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(x != y, GPFVM_ERR_INVALID, "x and y must not alias");
    int64_t nin = 1, nout = 1;
    for (int i = 0; i < ndim; i++) {
      GPFVM_CHECK(in_shape[i] >= 1 && out_shape[i] >= 1, GPFVM_ERR_INVALID, "empty dimension");
      nin *= in_shape[i];
      nout *= out_shape[i];
    }
    GPFVM_CHECK(ldx >= nin && ldy >= nout, GPFVM_ERR_INVALID, "ld smaller than the tensor size");
    std::vector<double> c(coefs, coefs + P);
    std::vector<std::vector<const double*>> fs(P);
    for (int p = 0; p < P; p++) fs[p].assign(factors + p * ndim, factors + (p + 1) * ndim);
    // cached plan + workspace keyed on the factor pointers (thread-local, small LRU)
    struct Entry {
      std::vector<int> key_shape;
      std::vector<double> key_c;
      std::vector<const double*> key_f;
      std::unique_ptr<KronSum> ks;
    };
    static thread_local std::map<int, std::vector<Entry>> caches;  // per device
    std::vector<Entry>& cache = caches[current_device()];
    DevBuf& w0 = scratch(s, 1);
    DevBuf& w1 = scratch(s, 2);
    std::vector<int> ks_shape(in_shape, in_shape + ndim);
    ks_shape.insert(ks_shape.end(), out_shape, out_shape + ndim);
    std::vector<const double*> kf(factors, factors + (size_t)P * ndim);
    KronSum* ks = nullptr;
    for (auto& e : cache)
      if (e.key_shape == ks_shape && e.key_c == c && e.key_f == kf) ks = e.ks.get();
    if (!ks) {
      if (cache.size() >= 8) cache.erase(cache.begin());
      Entry e{ks_shape, c, kf, std::make_unique<KronSum>()};
      e.ks->build(ndim, in_shape, out_shape, c, fs, s);
      ks = e.ks.get();
      cache.push_back(std::move(e));
    } else {
      ks->build(ndim, in_shape, out_shape, c, fs, s);  // refresh contents (factors may have changed)
    }
    size_t need = (size_t)std::max<int64_t>(1, ks->workspace_per_rhs() * R);
    w0.ensure(need);
    w1.ensure(need);
    ks->apply(x, ldx, y, ldy, R, beta, w0.ptr, w1.ptr, s);
    return GPFVM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GPFVM_ERR_INVALID;
  }
}
}  // namespace gpfvm

extern "C" int gpfvm_kron_matvec(int ndim, const int* in_shape, const int* out_shape, int n_terms, const double* coefs,
                                 const double* const* factors, const double* x, int64_t ldx, double* y, int64_t ldy,
                                 int nrhs, double beta, void* stream) {
  return gpfvm::guarded_kron(ndim, in_shape, out_shape, n_terms, coefs, factors, x, ldx, y, ldy, nrhs, beta,
                             (cudaStream_t)stream);
}
