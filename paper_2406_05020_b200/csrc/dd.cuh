// Double-double (~106-bit) arithmetic for the factor-assembly kernel.
//
// The closed forms of DESIGN.md §4.1 evaluate antiderivatives of the Matérn
// kernel at cell endpoints and take 2nd differences of them; in plain FP64
// that loses ~(l/h)^2 of relative accuracy (R2).  Evaluating the
// endpoint formula in double-double and rounding once gives entries within
// ~1 ulp of the exact value, which is what the 1e-12 parity bar needs.
// Algorithms: Dekker/Knuth two-sum, FMA two-product, Newton division/sqrt.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

struct dd {
  double hi, lo;
};

__host__ __device__ __forceinline__ dd dd_make(double a) { return {a, 0.0}; }

__host__ __device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}

__host__ __device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  double e = b - (s - a);
  return {s, e};
}

__host__ __device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  double e = fma(a, b, -p);
  return {p, e};
}

__host__ __device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}

__host__ __device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__host__ __device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

__host__ __device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}

__host__ __device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}

__host__ __device__ __forceinline__ dd dd_div(dd a, dd b) {
  double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul_d(b, q1));
  double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd_make(q3));
}

__host__ __device__ __forceinline__ dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return dd_make(0.0);
  double x = sqrt(a.hi);
  // one Newton step in dd: x + (a - x^2) / (2x)
  dd xx = two_prod(x, x);
  dd r = dd_sub(a, xx);
  double corr = r.hi / (2.0 * x);
  return quick_two_sum(x, corr);
}

__host__ __device__ __forceinline__ dd dd_ldexp(dd a, int e) { return {ldexp(a.hi, e), ldexp(a.lo, e)}; }

// exp(a) for a <= ~700, relative error ~1e-31.
__host__ __device__ inline dd dd_exp(dd a) {
  const dd LN2 = {6.931471805599452862e-01, 2.319046813846299558e-17};
  if (a.hi < -745.0) return dd_make(0.0);
  double k = nearbyint(a.hi / LN2.hi);
  dd r = dd_sub(a, dd_mul_d(LN2, k));
  // scale down by 2^-10 so the Taylor series converges in ~12 terms
  r = dd_ldexp(r, -10);
  // s = exp(r) - 1 = r + r^2/2! + ...
  dd term = r;
  dd s = r;
#pragma unroll 1
  for (int i = 2; i <= 14; i++) {
    term = dd_mul(term, r);
    term = dd_div(term, dd_make((double)i));
    s = dd_add(s, term);
    if (fabs(term.hi) < 1e-36) break;
  }
  // (1+s)^2 - 1 = 2s + s^2, ten times
#pragma unroll 1
  for (int i = 0; i < 10; i++) s = dd_add(dd_ldexp(s, 1), dd_mul(s, s));
  dd e = dd_add(s, dd_make(1.0));
  return dd_ldexp(e, (int)k);
}

__host__ __device__ __forceinline__ double dd_to_double(dd a) { return a.hi + a.lo; }
