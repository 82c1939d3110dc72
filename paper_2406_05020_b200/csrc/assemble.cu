// §8 row 1 — 1D factor-matrix assembly.
//
// F[j,j'] = L_{left_j; m} k L'_{right_j'; m'}   (Eq. 16, l.246)
//
// Every 1D functional is reduced to weighted evaluations at endpoints
// (Eq. 10, l.206-207: the fundamental theorem of calculus turns an
// integral of a derivative into an endpoint difference):
//   point p, order m       -> (+1 at p),               generalised order o = m
//   interval [a,b], m = 0  -> (+1 at b, -1 at a),       o = -1 (antiderivative K1)
//   interval [a,b], m >= 1 -> (+1 at b, -1 at a),       o = m - 1
// and  d^o/dx^o d^o'/dy^o' k(x - y) = (-1)^o' g_{o+o'}(x - y)  with
//   g_n = k^{(n)} (n >= 0),  g_{-1} = K1 = int_0^d k,  g_{-2} = K2 = int_0^d K1.
// For d >= 0 each g is exp(-lam d) times a polynomial:
//   k^{(n)}:  P_{n+1} = P_n' - lam P_n,
//   K1 = B(0) - e^{-lam d} B(d),   K2 = B(0) d - C(0) + e^{-lam d} C(d),
//   with int e^{-lam s}A(s) ds = -e^{-lam s}B(s)  (lam b_k - (k+1) b_{k+1} = a_k),
// extended to d < 0 by parity g_n(-d) = (-1)^n g_n(d).
//
// The lag d = e - e' is formed exactly (two_sum) and everything after it is
// double-double; one rounding at the end.  One thread per entry.
#include <vector>

#include "internal.h"

namespace gpfvm {

static void pq_rational(int q, double* num, double* den) {
  // p_q(s) = q!/(2q)! sum_i (q+i)!/(i!(q-i)!) (2s)^(q-i)   (Rasmussen & Williams 4.16)
  static const double N[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 1, 1, 0}, {1, 1, 2, 1}};
  static const double D[4][4] = {{1, 1, 1, 1}, {1, 1, 1, 1}, {1, 1, 3, 1}, {1, 1, 5, 15}};
  for (int k = 0; k < 4; k++) {
    num[k] = N[q][k];
    den[k] = D[q][k];
  }
}

MaternDD matern_dd(int q, double lengthscale, double variance) {
  MaternDD K;
  K.q = q;
  K.lam = dd_div(dd_sqrt(dd_make((double)(2 * q + 1))), dd_make(lengthscale));
  double num[4], den[4];
  pq_rational(q, num, den);
  dd lp = dd_make(variance);
  for (int k = 0; k < 4; k++) {
    if (k <= q) {
      K.a[k] = dd_mul(lp, dd_div(dd_make(num[k]), dd_make(den[k])));
      lp = dd_mul(lp, K.lam);
    } else {
      K.a[k] = dd_make(0.0);
    }
  }
  return K;
}

// polynomial coefficients (length q+1) of g_o for d >= 0, o in [-2, 2q]
__device__ static void g_poly(const MaternDD& K, int o, dd* c) {
  const int n = K.q + 1;
  for (int k = 0; k < n; k++) c[k] = K.a[k];
  if (o >= 0) {
    for (int it = 0; it < o; it++) {
      for (int k = 0; k < n; k++) {
        dd t = dd_mul(K.lam, c[k]);
        dd up = (k + 1 < n) ? dd_mul_d(c[k + 1], (double)(k + 1)) : dd_make(0.0);
        c[k] = dd_sub(up, t);
      }
    }
    return;
  }
  // antiderivatives: o = -1 -> B, o = -2 -> C
  int reps = -o;
  for (int it = 0; it < reps; it++) {
    dd b[4];
    b[n - 1] = dd_div(c[n - 1], K.lam);
    for (int k = n - 2; k >= 0; k--) b[k] = dd_div(dd_add(c[k], dd_mul_d(b[k + 1], (double)(k + 1))), K.lam);
    for (int k = 0; k < n; k++) c[k] = b[k];
  }
}

__device__ static dd horner(const dd* c, int n, dd x) {
  dd acc = c[n - 1];
  for (int k = n - 2; k >= 0; k--) acc = dd_add(dd_mul(acc, x), c[k]);
  return acc;
}

// g_o(d) with d given exactly as a dd lag; poly = g_poly(o) (for o<0: B or C) and
// c0 = B(0) (o = -1, -2), cc0 = C(0) (o = -2)
__device__ static dd g_eval(const MaternDD& K, int o, const dd* poly, dd B0, dd C0, dd d) {
  const int n = K.q + 1;
  double sgn = (d.hi > 0.0) ? 1.0 : ((d.hi < 0.0) ? -1.0 : 0.0);
  dd ad = (d.hi < 0.0) ? dd_neg(d) : d;
  dd e = dd_exp(dd_neg(dd_mul(K.lam, ad)));
  dd p = horner(poly, n, ad);
  if (o >= 0) {
    dd v = dd_mul(e, p);
    if (o & 1) v = dd_mul_d(v, sgn);
    return v;
  }
  if (o == -1) {
    dd v = dd_sub(B0, dd_mul(e, p));
    return dd_mul_d(v, sgn);
  }
  // o == -2
  return dd_add(dd_sub(dd_mul(B0, ad), C0), dd_mul(e, p));
}

struct FactorArgs {
  MaternDD K;
  int kindL, nL, mL, kindR, nR, mR;
  const double *loL, *hiL, *loR, *hiR;
};

// per-(K, o) constants: the polynomial of g_o and B(0), C(0) (dd divisions),
// computed once per CTA into shared memory
__device__ __forceinline__ void factor_consts(const FactorArgs& a, dd* s_poly, dd& s_B0, dd& s_C0) {
  const int o_blk = (a.kindL == GPFVM_SITE_POINT ? a.mL : a.mL - 1) + (a.kindR == GPFVM_SITE_POINT ? a.mR : a.mR - 1);
  if (threadIdx.x == 0) {
    dd pl[4];
    g_poly(a.K, o_blk, pl);
    for (int k = 0; k < 4; k++) s_poly[k] = pl[k];
    s_B0 = dd_make(0.0);
    s_C0 = dd_make(0.0);
    if (o_blk < 0) {
      dd t[4];
      g_poly(a.K, -1, t);
      s_B0 = t[0];
      g_poly(a.K, -2, t);
      s_C0 = t[0];
    }
  }
  __syncthreads();
}

// F[j][jj]: the 1D functional pair of Eq. 16 as endpoint sums of g_o (R2)
__device__ double factor_entry(const FactorArgs& a, const dd* s_poly, dd B0, dd C0, int j, int jj) {
  double eL[2], wL[2], eR[2], wR[2];
  int cL, cR, oL, oR;
  if (a.kindL == GPFVM_SITE_POINT) {
    eL[0] = a.loL[j]; wL[0] = 1.0; cL = 1; oL = a.mL;
  } else {
    eL[0] = a.hiL[j]; wL[0] = 1.0; eL[1] = a.loL[j]; wL[1] = -1.0; cL = 2; oL = a.mL - 1;
  }
  if (a.kindR == GPFVM_SITE_POINT) {
    eR[0] = a.loR[jj]; wR[0] = 1.0; cR = 1; oR = a.mR;
  } else {
    eR[0] = a.hiR[jj]; wR[0] = 1.0; eR[1] = a.loR[jj]; wR[1] = -1.0; cR = 2; oR = a.mR - 1;
  }
  const int o = oL + oR;
  dd poly[4];
  for (int k = 0; k < 4; k++) poly[k] = s_poly[k];
  dd acc = dd_make(0.0);
  for (int x = 0; x < cL; x++)
    for (int y = 0; y < cR; y++) {
      dd d = two_sum(eL[x], -eR[y]);
      dd v = g_eval(a.K, o, poly, B0, C0, d);
      acc = dd_add(acc, dd_mul_d(v, wL[x] * wR[y]));
    }
  double r = dd_to_double(acc);
  if (oR & 1) r = -r;  // (-1)^{o'} (o' = -1 is odd)
  return r;
}

__global__ void factor_kernel(FactorArgs a, double* __restrict__ out, int64_t ld) {
  __shared__ dd s_poly[4], s_B0, s_C0;
  factor_consts(a, s_poly, s_B0, s_C0);
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)a.nL * a.nR) return;
  const int j = (int)(idx / a.nR), jj = (int)(idx % a.nR);
  out[(int64_t)j * ld + jj] = factor_entry(a, s_poly, s_B0, s_C0, j, jj);
}

// Uniform site lists (every endpoint sequence arithmetic with one common step,
// checked exactly on the host): the entry depends only on the lag j - jj — the
// exact endpoint differences, hence the double-double inputs of g_o, are the
// same — so one evaluation per lag (nL + nR - 1 instead of nL nR), bitwise
// equal to the per-entry kernel.
__global__ void factor_lag_kernel(FactorArgs a, double* __restrict__ lagv) {
  __shared__ dd s_poly[4], s_B0, s_C0;
  factor_consts(a, s_poly, s_B0, s_C0);
  const int l = blockIdx.x * blockDim.x + threadIdx.x;  // lag + nR - 1
  if (l >= a.nL + a.nR - 1) return;
  const int lag = l - (a.nR - 1);
  const int j = lag > 0 ? lag : 0, jj = j - lag;
  lagv[l] = factor_entry(a, s_poly, s_B0, s_C0, j, jj);
}

__global__ void lag_fill_kernel(const double* __restrict__ lagv, int nL, int nR, double* __restrict__ out, int64_t ld) {
  const int64_t total = (int64_t)nL * nR;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx / nR), jj = (int)(idx % nR);
    out[(int64_t)j * ld + jj] = lagv[j - jj + nR - 1];
  }
}

// exact arithmetic-progression test of a site list's endpoints with step h
bool arithmetic(const std::vector<double>& v, double h) {
  for (size_t j = 1; j < v.size(); j++)
    if (v[j] - v[j - 1] != h || v[0] + (double)j * h != v[j]) return false;
  return true;
}
bool uniform_pair(const Sites& L, const Sites& R) {
  double h = 0.0;
  if (L.n >= 2) h = L.lo[1] - L.lo[0];
  else if (R.n >= 2) h = R.lo[1] - R.lo[0];
  else return false;
  if (!(h > 0.0)) return false;
  for (const Sites* S : {&L, &R}) {
    if (!arithmetic(S->lo, h)) return false;
    if (S->kind != GPFVM_SITE_POINT && !arithmetic(S->hi, h)) return false;
  }
  return true;
}

void launch_factor(const MaternDD& K, const Sites& L, int mL, const Sites& R, int mR, double* out,
                   int64_t ld, cudaStream_t s) {
  int64_t n = (int64_t)L.n * R.n;
  if (n == 0) return;
  FactorArgs a{K, L.kind, L.n, mL, R.kind, R.n, mR, L.d_lo.ptr, L.d_hi.ptr, R.d_lo.ptr, R.d_hi.ptr};
  static const bool no_lag = getenv("GPFVM_NO_LAG") != nullptr;
  if (!no_lag && n >= 256 && uniform_pair(L, R)) {
    const int nl = L.n + R.n - 1;
    DevBuf& lagv = scratch(s, 6);
    lagv.ensure((size_t)nl);
    factor_lag_kernel<<<(nl + 127) / 128, 128, 0, s>>>(a, lagv.ptr);
    lag_fill_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(lagv.ptr, L.n, R.n, out, ld);
    count_launch(2);
    check_launch("factor_lag_kernel");
    return;
  }
  int threads = 128;
  int64_t blocks = (n + threads - 1) / threads;
  factor_kernel<<<(unsigned)blocks, threads, 0, s>>>(a, out, ld);
  count_launch();
  check_launch("factor_kernel");
}

}  // namespace gpfvm
