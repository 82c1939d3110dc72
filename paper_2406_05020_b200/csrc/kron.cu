// Fused Kronecker-sum operator  Y (+)= sum_p ((x)_i F_i^p) X.
//
// One block pair of the Gram (Eq. 20) with P surviving term pairs becomes d
// GEMM launches, independent of P:
//   stage 0   stacked-M GEMM  Z0[r][p][j0][rest'] = (c_p F_0^p) X_r      M = P*n0
//   stage i   batched GEMM    Z_i[r][p][..][j_i][..] = F_i^p  Z_{i-1}   batch (o, p, r)
//   stage d-1 K-segment GEMM  Y_r[rows][l] += sum_p Z[r][p][rows][:] F_{d-1}^{pT}
// (the p-sum is the K-concatenation of the last contraction).  For d = 1 a
// single K-segment GEMM  Y_r = sum_p X_r (c_p F^p)^T.  The stacked factors are
// built once per plan by device copies (coefficients folded into stage 0).
#include "problem.h"

namespace gpfvm {

namespace {
__global__ void scaled_copy_kernel(double* dst, const double* __restrict__ src, double c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = c * src[i];
}
unsigned gsz(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 2048)); }
}  // namespace

void KronSum::build(int d_, const int* in_shape, const int* out_shape, const std::vector<double>& coefs,
                    const std::vector<std::vector<const double*>>& factors, cudaStream_t s) {
  d = d_;
  P = (int)coefs.size();
  for (int i = 0; i < GPFVM_MAX_DIMS; i++) {
    nin[i] = (i < d) ? in_shape[i] : 1;
    nout[i] = (i < d) ? out_shape[i] : 1;
  }
  if (P == 0) return;
  for (int i = 0; i < d; i++) {
    int64_t fs = (int64_t)nout[i] * nin[i];
    stk[i].ensure((size_t)std::max<int64_t>(1, fs * P));
    for (int p = 0; p < P; p++) {
      double c = (i == 0) ? coefs[p] : 1.0;
      scaled_copy_kernel<<<gsz(fs), 256, 0, s>>>(stk[i].ptr + p * fs, factors[p][i], c, fs);
      count_launch();
    }
  }
  check_launch("KronSum::build");
}

int64_t KronSum::workspace_per_rhs() const {
  if (P == 0 || d == 1) return 0;
  int64_t mx = 0;
  for (int i = 0; i <= d - 2; i++) {
    int64_t sz = P;
    for (int k = 0; k <= i; k++) sz *= nout[k];
    for (int k = i + 1; k < d; k++) sz *= nin[k];
    mx = std::max(mx, sz);
  }
  return mx;
}

double KronSum::flops_per_rhs() const {
  if (P == 0) return 0.0;
  double fl = 0.0;
  for (int i = 0; i < d; i++) {
    double v = 2.0 * P * nout[i] * (double)nin[i];
    for (int k = 0; k < i; k++) v *= nout[k];
    for (int k = i + 1; k < d; k++) v *= nin[k];
    fl += v;
  }
  return fl;
}

void KronSum::apply(const double* x, int64_t ldx, double* y, int64_t ldy, int R, double beta, double* w0, double* w1,
                    cudaStream_t s) const {
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
  // stage 0: stacked M
  int64_t rest = 1;
  for (int k = 1; k < d; k++) rest *= nin[k];
  const int64_t z0 = (int64_t)P * nout[0] * rest;  // per-rhs size
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
  // middle stages
  for (int i = 1; i <= d - 2; i++) {
    int64_t outer = 1, inner = 1;
    for (int k = 0; k < i; k++) outer *= nout[k];
    for (int k = i + 1; k < d; k++) inner *= nin[k];
    const int64_t nsz = (int64_t)P * outer * nout[i] * inner;
    Gemm g;
    g.M = nout[i]; g.N = (int)inner; g.K = nin[i];
    g.A = stk[i].ptr; g.a_rs = nin[i]; g.a_cs = 1;
    g.a_b2 = (int64_t)nout[i] * nin[i];
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
  // last stage: K-segments over p
  {
    const int l = d - 1;
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
  }
}

}  // namespace gpfvm
