// §8 row 3 — gpfvm_solve: preconditioned CG in IterGP form.
//
// Preconditioner (built once per assembly, cached on the handle):
//   FD for the single non-deflated 2D block P whose Gram keeps
//       two Kronecker terms  c_a A0(x)A1 + c_b B0(x)B1  (exact for the heat
//       operator, R6).  Generalised eigenproblems on the GPU (block Jacobi):
//         B0 V = A0 V Lam (V^T A0 V = I),   A1 W = B1 W M (W^T B1 W = I)
//       P^{-1}_PP = (V(x)W) D^{-1} (V(x)W)^T,  D_ij = c_a M_j + c_b Lam_i
//       (+ block noise * |v_i|^2 |w_j|^2).
//   block LDL (§5.2) over the deflated IC/BC blocks b (§4.2):
//       Y = FD(G_pb), S = G_bb - G_pb^T Y (shifted only if Cholesky fails),
//       P^{-1} r = [S^{-1}(r_b - G_pb^T FD r_p) ;  FD r_p - Y z_b].
// Iteration (§4.1, Wenger et al. 2022 Alg. 1, CG policy, full
// reorthogonalisation §6 l.475):
//   s = P^{-1} r ; z = G s ; c_j = d_j.z / eta_j ; d = s - sum c_j d_j ;
//   Gd = z - sum c_j Gd_j ; eta = z.d ; a = d.r / eta ; x += a d ; r -= a Gd
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "problem.h"

namespace gpfvm {

void destroy_precond(Precond* pc) { delete pc; }

namespace {

__global__ void scale_cols_kernel(double* X, const double* __restrict__ d, int64_t n, int R, int64_t ld) {
  const int r = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    X[r * ld + i] *= d[i];
}

__global__ void colsumsq_kernel(const double* __restrict__ V, int n, double* out) {
  // out[j] = sum_r V[r][j]^2  (V row-major n x n)
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int r = 0; r < n; r++) s = fma(V[(int64_t)r * n + j], V[(int64_t)r * n + j], s);
  out[j] = s;
}

__global__ void dinv_kernel(double* D, const double* __restrict__ lam, const double* __restrict__ mu,
                            const double* __restrict__ vv, const double* __restrict__ ww, int n0, int n1,
                            double ca, double cb, double noise) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n0 * n1) return;
  int i = (int)(idx / n1), j = (int)(idx % n1);
  double d = ca * mu[j] + cb * lam[i] + noise * vv[i] * ww[j];
  D[idx] = 1.0 / d;
}

// Dense expansion of one Kronecker term of a Gram block (Eq. 20):
//   S[(c) * ld + r] += coef * prod_i F_i[r_i][c_i],  r / c the row-major
// multi-indices of the output / input block (S holds G_{I,J}[r][c] at row c,
// column r; G_bb is symmetric).  One thread per entry.
struct KronDenseArgs {
  int d;
  int nr[GPFVM_MAX_DIMS], nc[GPFVM_MAX_DIMS];
  const double* F[GPFVM_MAX_DIMS];
};
__global__ void kron_dense_kernel(double* S, int64_t ld, KronDenseArgs a, int64_t R, int64_t Cn, double coef) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < R * Cn; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / R, r = e - c * R;
    int64_t rr = r, cc = c;
    double v = coef;
    for (int i = a.d - 1; i >= 0; i--) {
      const int ri = (int)(rr % a.nr[i]), ci = (int)(cc % a.nc[i]);
      rr /= a.nr[i];
      cc /= a.nc[i];
      v *= a.F[i][(int64_t)ri * a.nc[i] + ci];
    }
    S[c * ld + r] += v;
  }
}

__global__ void set_identity_kernel(double* X, int n, int64_t ld) {
  // X: n vectors of length n at stride ld
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int r = (int)(idx / n), c = (int)(idx % n);
  X[r * ld + c] = (r == c) ? 1.0 : 0.0;
}

__global__ void add_diag_kernel(double* A, int n, const double* __restrict__ d, double shift) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[(int64_t)i * n + i] += (d ? d[i] : 0.0) + shift;
}

__global__ void sub_kernel(double* a, const double* __restrict__ b, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] -= b[i];
}

// X[i][c] = v[i] * M[i][c]  (rows x cols)
__global__ void row_scale_kernel(double* X, const double* __restrict__ v, const double* __restrict__ M, int rows,
                                 int cols) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    X[k] = v[k / cols] * M[k];
}
__global__ void vec_mul_kernel(double* z, const double* __restrict__ a, const double* __restrict__ b, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) z[i] = a[i] * b[i];
}

__global__ void symm_kernel(double* A, int n) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int r = (int)(idx / n), c = (int)(idx % n);
  if (c <= r) return;
  double v = 0.5 * (A[(int64_t)r * n + c] + A[(int64_t)c * n + r]);
  A[(int64_t)r * n + c] = v;
  A[(int64_t)c * n + r] = v;
}

struct PhaseTimer {
  cudaStream_t s;
  bool on;
  double t0;
  explicit PhaseTimer(cudaStream_t st) : s(st), on(getenv("GPFVM_DEBUG") != nullptr), t0(0) { mark(nullptr); }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    double t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (what) fprintf(stderr, "[gpfvm] %-28s %8.2f ms\n", what, t - t0);
    t0 = t;
  }
};

unsigned g1(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// FD apply on R vectors (stride ldx in, ldy out), x != y
// Second half of FD: y_r = (V (x) W) D^{-1} t_r for R vectors t_r stored in
// pc.t2 (stride Np, overwritten).
static void fd_backward(Precond& pc, double* y, int64_t ldy, int R, cudaStream_t s) {
  const int n0 = pc.n0, n1 = pc.n1;
  const int64_t np = pc.Np;
  scale_cols_kernel<<<dim3(std::min<unsigned>(g1(np), 1184), R), 256, 0, s>>>(pc.t2.ptr, pc.Dinv.ptr, np, R, np);
  count_launch();
  Gemm g;
  // T1_r = V T2_r
  g.M = n0; g.N = n1; g.K = n0; g.batch1 = R;
  g.A = pc.V.ptr; g.a_rs = n0; g.a_cs = 1;
  g.B = pc.t2.ptr; g.b_rs = n1; g.b_cs = 1; g.b_b1 = np;
  g.C = pc.t1.ptr; g.c_rs = n1; g.c_cs = 1; g.c_b1 = np;
  run_gemm(g, s);
  // Y_r = T1_r W^T
  g = Gemm();
  g.M = n0; g.N = n1; g.K = n1; g.batch1 = R;
  g.A = pc.t1.ptr; g.a_rs = n1; g.a_cs = 1; g.a_b1 = np;
  g.B = pc.W.ptr; g.b_rs = 1; g.b_cs = n1;
  g.C = y; g.c_rs = n1; g.c_cs = 1; g.c_b1 = ldy;
  run_gemm(g, s);
}

// y_r = FD x_r = (V (x) W) D^{-1} (V (x) W)^T x_r
static void fd_apply(Precond& pc, const double* x, int64_t ldx, double* y, int64_t ldy, int R, cudaStream_t s) {
  const int n0 = pc.n0, n1 = pc.n1;
  const int64_t np = pc.Np;
  pc.t1.ensure((size_t)np * R);
  pc.t2.ensure((size_t)np * R);
  Gemm g;
  // T1_r = X_r W
  g.M = n0; g.N = n1; g.K = n1; g.batch1 = R;
  g.A = x; g.a_rs = n1; g.a_cs = 1; g.a_b1 = ldx;
  g.B = pc.W.ptr; g.b_rs = n1; g.b_cs = 1;
  g.C = pc.t1.ptr; g.c_rs = n1; g.c_cs = 1; g.c_b1 = np;
  run_gemm(g, s);
  // T2_r = V^T T1_r
  g = Gemm();
  g.M = n0; g.N = n1; g.K = n0; g.batch1 = R;
  g.A = pc.Vt.ptr; g.a_rs = n0; g.a_cs = 1;
  g.B = pc.t1.ptr; g.b_rs = n1; g.b_cs = 1; g.b_b1 = np;
  g.C = pc.t2.ptr; g.c_rs = n1; g.c_cs = 1; g.c_b1 = np;
  run_gemm(g, s);
  fd_backward(pc, y, ldy, R, s);
}

static const KronTerm* find_term(gpfvm_problem* p, int I, int J, int fid0, int fid1) {
  for (const auto& t : p->terms)
    if (t.I == I && t.J == J && t.fid[0] == fid0 && t.fid[1] == fid1) return &t;
  return nullptr;
}

// The exact FD path needs G_PP to be exactly c_a A0 (x) A1 + c_b B0 (x) B1: two
// Kronecker terms on the block, both diagonal pairs (a,a), (b,b).  When the R6
// cross pair survives (even total derivative order, e.g. u_t + a u_x or the 1D
// wave operator) a third term exists and FD would silently drop it.
static bool exact_fd_ok(gpfvm_problem* p, int P) {
  const BlockInt& B = p->blocks[P];
  if (p->ndim != 2 || B.terms.size() != 2 || B.terms[0].output != B.terms[1].output) return false;
  auto lookup = [&](int dim, int m) {
    auto it = p->factor_index.find(FactorKey{B.terms[0].output, dim, P, m, P, m});
    return it == p->factor_index.end() ? -1 : it->second;
  };
  int nPP = 0;
  for (const auto& t : p->terms) nPP += (t.I == P && t.J == P);
  if (nPP != 2) return false;
  for (const auto& tm : B.terms) {
    const int f0 = lookup(0, tm.order[0]), f1 = lookup(1, tm.order[1]);
    if (f0 < 0 || f1 < 0 || !find_term(p, P, P, f0, f1)) return false;
  }
  return true;
}

static void build_fd(gpfvm_problem* p, Precond& pc, cudaStream_t s) {
  const BlockInt& B = p->blocks[pc.P];
  GPFVM_CHECK(p->ndim == 2 && B.terms.size() == 2, GPFVM_ERR_UNSUPPORTED,
              "BLOCK_FD preconditioner needs a 2D non-deflated block with a two-term operator");
  gpfvm_term ta = B.terms[0], tb = B.terms[1];
  if (ta.order[0] < tb.order[0]) std::swap(ta, tb);
  GPFVM_CHECK(ta.output == tb.output, GPFVM_ERR_UNSUPPORTED, "BLOCK_FD: terms on different outputs");
  const int out = ta.output;
  int fA0 = get_factor(p, out, 0, pc.P, ta.order[0], pc.P, ta.order[0]);
  int fA1 = get_factor(p, out, 1, pc.P, ta.order[1], pc.P, ta.order[1]);
  int fB0 = get_factor(p, out, 0, pc.P, tb.order[0], pc.P, tb.order[0]);
  int fB1 = get_factor(p, out, 1, pc.P, tb.order[1], pc.P, tb.order[1]);
  GPFVM_CHECK(find_term(p, pc.P, pc.P, fA0, fA1) && find_term(p, pc.P, pc.P, fB0, fB1), GPFVM_ERR_STATE,
              "BLOCK_FD: diagonal term pairs missing");
  pc.n0 = B.shape[0];
  pc.n1 = B.shape[1];
  pc.Np = B.size;
  const int n0 = pc.n0, n1 = pc.n1;
  DevBuf lam, mu, vv, ww;
  lam.ensure(n0); mu.ensure(n1); vv.ensure(n0); ww.ensure(n1);
  pc.V.ensure((size_t)n0 * n0);
  pc.Vt.ensure((size_t)n0 * n0);
  pc.W.ensure((size_t)n1 * n1);
  pc.Dinv.ensure((size_t)n0 * n1);
  // the two generalised eigenproblems are independent and each keeps only
  // n/32 CTAs busy per Jacobi round: run them concurrently (two host threads,
  // two streams; sygv synchronises its own stream)
  GPFVM_CUDA(cudaStreamSynchronize(s));
  {
    cudaStream_t s2[2];
    for (auto& st : s2) GPFVM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int dev = 0;
    GPFVM_CUDA(cudaGetDevice(&dev));
    Error err{GPFVM_OK, ""};
    std::thread th([&] {
      try {
        cudaSetDevice(dev);
        sygv(p->factors[fA1].data.ptr, p->factors[fB1].data.ptr, n1, pc.W.ptr, mu.ptr, s2[1]);
      } catch (const Error& e) {
        err = e;
      }
    });
    try {
      sygv(p->factors[fB0].data.ptr, p->factors[fA0].data.ptr, n0, pc.V.ptr, lam.ptr, s2[0]);
    } catch (...) {
      th.join();
      for (auto st : s2) cudaStreamDestroy(st);
      throw;
    }
    th.join();
    for (auto st : s2) cudaStreamDestroy(st);
    if (err.code != GPFVM_OK) throw err;
  }
  transpose(pc.V.ptr, pc.Vt.ptr, n0, n0, s);
  colsumsq_kernel<<<g1(n0, 128), 128, 0, s>>>(pc.V.ptr, n0, vv.ptr);
  colsumsq_kernel<<<g1(n1, 128), 128, 0, s>>>(pc.W.ptr, n1, ww.ptr);
  dinv_kernel<<<g1((int64_t)n0 * n1), 256, 0, s>>>(pc.Dinv.ptr, lam.ptr, mu.ptr, vv.ptr, ww.ptr, n0, n1,
                                                   ta.coeff * ta.coeff, tb.coeff * tb.coeff, B.noise);
  count_launch(3);
  check_launch("build_fd");
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

// Rotated couplings Z_J (see Precond::RotTerm) and their Kronecker sums.
static void build_rot(gpfvm_problem* p, Precond& pc, cudaStream_t s) {
  const int n0 = pc.n0, n1 = pc.n1;
  pc.WT.ensure((size_t)n1 * n1);
  transpose(pc.W.ptr, pc.WT.ptr, n1, n1, s);
  pc.rot.clear();
  pc.rot.resize(pc.bblocks.size());
  pc.rot_ks.clear();
  pc.rot_ks.resize(pc.bblocks.size());
  pc.structured = getenv("GPFVM_LDL_DENSE") == nullptr;
  for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
    const int J = pc.bblocks[jb];
    const BlockInt& BJ = p->blocks[J];
    const bool ic = BJ.shape[0] == 1, bc = !ic && BJ.shape[1] == 1;
    if (!ic && !bc) pc.structured = false;
    std::vector<double> coefs;
    std::vector<std::vector<const double*>> fs;
    for (const auto& t : p->terms) {
      if (t.I != pc.P || t.J != J) continue;
      const Factor& F0 = p->factors[t.fid[0]];
      const Factor& F1 = p->factors[t.fid[1]];
      Precond::RotTerm rt;
      rt.c = t.coef;
      rt.m0 = F0.cols;
      rt.m1 = F1.cols;
      rt.R0.ensure((size_t)n0 * rt.m0);
      rt.R1.ensure((size_t)n1 * rt.m1);
      Gemm g;  // R0 = V^T F0
      g.M = n0; g.N = rt.m0; g.K = n0;
      g.A = pc.Vt.ptr; g.a_rs = n0; g.a_cs = 1;
      g.B = F0.data.ptr; g.b_rs = rt.m0; g.b_cs = 1;
      g.C = rt.R0.ptr; g.c_rs = rt.m0; g.c_cs = 1;
      run_gemm(g, s);
      g = Gemm();  // R1 = W^T F1
      g.M = n1; g.N = rt.m1; g.K = n1;
      g.A = pc.WT.ptr; g.a_rs = n1; g.a_cs = 1;
      g.B = F1.data.ptr; g.b_rs = rt.m1; g.b_cs = 1;
      g.C = rt.R1.ptr; g.c_rs = rt.m1; g.c_cs = 1;
      run_gemm(g, s);
      if (ic || bc) {  // transposed long factor: IC-like R1 (n1 x nJ), BC-like R0 (n0 x nJ)
        const int rows = ic ? n1 : n0, cols = ic ? rt.m1 : rt.m0;
        rt.LT.ensure((size_t)rows * cols);
        transpose(ic ? rt.R1.ptr : rt.R0.ptr, rt.LT.ptr, rows, cols, s);
      }
      coefs.push_back(t.coef);
      fs.push_back({rt.R0.ptr, rt.R1.ptr});
      pc.rot[jb].push_back(std::move(rt));
    }
    pc.rot_ks[jb].build(p->ndim, BJ.shape, p->blocks[pc.P].shape, coefs, fs, s);
  }
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

// S -= Z^T D^{-1} Z block by block from the rotated thin factors (no Y): for
// IC-like J (a = R0 column, L = R1) and BC-like J (b = R1 column, L = R0)
//   IC-IC  L^T diag(D^{-T}(a o a')) L'          BC-BC  L^T diag(D^{-1}(b o b')) L'
//   IC-BC  L^T diag(b') D^{-T} diag(a) L'       BC-IC  L^T diag(a') D^{-1} diag(b) L'
// (all n x n x nJ GEMMs, ~1e3 x fewer flops than S = G_bb - G_pb^T Y).
static void structured_schur(gpfvm_problem* p, Precond& pc, double* S, cudaStream_t s) {
  const int n0 = pc.n0, n1 = pc.n1, nb = (int)pc.nb;
  pc.DinvT.ensure((size_t)n1 * n0);
  transpose(pc.Dinv.ptr, pc.DinvT.ptr, n0, n1, s);
  DevBuf v, e, Mx, T;
  const int nmax = std::max(n0, n1);
  v.ensure(nmax);
  e.ensure(nmax);
  int64_t big = 0;
  for (size_t jb = 0; jb < pc.bblocks.size(); jb++) big = std::max<int64_t>(big, p->blocks[pc.bblocks[jb]].size);
  Mx.ensure((size_t)nmax * big);
  T.ensure((size_t)nmax * big);
  for (size_t jb = 0; jb < pc.bblocks.size(); jb++)
    for (size_t kb = 0; kb < pc.bblocks.size(); kb++) {
      const bool icJ = p->blocks[pc.bblocks[jb]].shape[0] == 1, icK = p->blocks[pc.bblocks[kb]].shape[0] == 1;
      const int nJ = (int)p->blocks[pc.bblocks[jb]].size, nK = (int)p->blocks[pc.bblocks[kb]].size;
      for (const auto& ra : pc.rot[jb])
        for (const auto& rb : pc.rot[kb]) {
          const double w = -ra.c * rb.c;
          int inner = 0;      // length of the contracted long dimension
          const double* Tp = nullptr;
          if (icJ && icK) {
            // e = D^{-T} (a o a'), T = diag(e) L'
            vec_mul_kernel<<<g1(n0), 256, 0, s>>>(v.ptr, ra.R0.ptr, rb.R0.ptr, n0);
            count_launch();
            Gemm g;
            g.M = 1; g.N = n1; g.K = n0;
            g.A = v.ptr; g.a_rs = n0; g.a_cs = 1;
            g.B = pc.Dinv.ptr; g.b_rs = n1; g.b_cs = 1;
            g.C = e.ptr; g.c_rs = n1; g.c_cs = 1;
            run_gemm(g, s);
            row_scale_kernel<<<g1((int64_t)n1 * nK), 256, 0, s>>>(T.ptr, e.ptr, rb.R1.ptr, n1, nK);
            count_launch();
            inner = n1;
          } else if (!icJ && !icK) {
            // f = D^{-1} (b o b'), T = diag(f) L'
            vec_mul_kernel<<<g1(n1), 256, 0, s>>>(v.ptr, ra.R1.ptr, rb.R1.ptr, n1);
            count_launch();
            Gemm g;
            g.M = 1; g.N = n0; g.K = n1;
            g.A = v.ptr; g.a_rs = n1; g.a_cs = 1;
            g.B = pc.DinvT.ptr; g.b_rs = n0; g.b_cs = 1;
            g.C = e.ptr; g.c_rs = n0; g.c_cs = 1;
            run_gemm(g, s);
            row_scale_kernel<<<g1((int64_t)n0 * nK), 256, 0, s>>>(T.ptr, e.ptr, rb.R0.ptr, n0, nK);
            count_launch();
            inner = n0;
          } else if (icJ && !icK) {
            // Mx = D^{-T} diag(a) L'  (n1 x nK), T = diag(b') Mx
            row_scale_kernel<<<g1((int64_t)n0 * nK), 256, 0, s>>>(T.ptr, ra.R0.ptr, rb.R0.ptr, n0, nK);
            count_launch();
            Gemm g;
            g.M = n1; g.N = nK; g.K = n0;
            g.A = pc.DinvT.ptr; g.a_rs = n0; g.a_cs = 1;
            g.B = T.ptr; g.b_rs = nK; g.b_cs = 1;
            g.C = Mx.ptr; g.c_rs = nK; g.c_cs = 1;
            run_gemm(g, s);
            row_scale_kernel<<<g1((int64_t)n1 * nK), 256, 0, s>>>(T.ptr, rb.R1.ptr, Mx.ptr, n1, nK);
            count_launch();
            inner = n1;
          } else {
            // My = D^{-1} diag(b) L'  (n0 x nK), T = diag(a') My
            row_scale_kernel<<<g1((int64_t)n1 * nK), 256, 0, s>>>(T.ptr, ra.R1.ptr, rb.R1.ptr, n1, nK);
            count_launch();
            Gemm g;
            g.M = n0; g.N = nK; g.K = n1;
            g.A = pc.Dinv.ptr; g.a_rs = n1; g.a_cs = 1;
            g.B = T.ptr; g.b_rs = nK; g.b_cs = 1;
            g.C = Mx.ptr; g.c_rs = nK; g.c_cs = 1;
            run_gemm(g, s);
            row_scale_kernel<<<g1((int64_t)n0 * nK), 256, 0, s>>>(T.ptr, rb.R0.ptr, Mx.ptr, n0, nK);
            count_launch();
            inner = n0;
          }
          Tp = T.ptr;
          // S[J rows][K cols] += w * LT_J (nJ x inner) T (inner x nK)
          Gemm g;
          g.M = nJ; g.N = nK; g.K = inner;
          g.A = ra.LT.ptr; g.a_rs = inner; g.a_cs = 1;
          g.B = Tp; g.b_rs = nK; g.b_cs = 1;
          g.C = S + pc.boff[jb] * nb + pc.boff[kb]; g.c_rs = nb; g.c_cs = 1;
          g.alpha = w; g.beta = 1.0;
          run_gemm(g, s);
        }
    }
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

static void build_ldl(gpfvm_problem* p, Precond& pc, cudaStream_t s) {
  const int nblk = (int)p->blocks.size();
  pc.nb = 0;
  for (int b = 0; b < nblk; b++)
    if (p->blocks[b].deflate) {
      pc.bblocks.push_back(b);
      pc.boff.push_back(pc.nb);
      pc.nb += p->blocks[b].size;
    }
  if (pc.nb == 0) return;
  GPFVM_CHECK(pc.nb <= 16384, GPFVM_ERR_UNSUPPORTED, "block-LDL: more than 16384 deflated observations");
  const int nb = (int)pc.nb;
  const int64_t np = pc.Np;
  DevBuf S, S0, eye, Lf;
  PhaseTimer pt(s);
  build_rot(p, pc, s);
  pt.mark("ldl: rotated couplings");
  if (!pc.structured) pc.YT.ensure((size_t)nb * np);
  S.ensure((size_t)nb * nb);
  fill(S.ptr, 0.0, (int64_t)nb * nb, s);
  // G_bb entry by entry from its Kronecker terms (the deflated blocks are small:
  // one kernel per term instead of identity blocks pushed through mode products)
  for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
    const int J = pc.bblocks[jb];
    for (size_t ib = 0; ib < pc.bblocks.size(); ib++) {
      const int I = pc.bblocks[ib];
      for (const auto& t : p->terms) {
        if (t.I != I || t.J != J) continue;
        KronDenseArgs a;
        a.d = p->ndim;
        for (int i = 0; i < p->ndim; i++) {
          a.nr[i] = p->blocks[I].shape[i];
          a.nc[i] = p->blocks[J].shape[i];
          a.F[i] = p->factors[t.fid[i]].data.ptr;
        }
        const int64_t Rn = p->blocks[I].size, Cn = p->blocks[J].size;
        kron_dense_kernel<<<g1(Rn * Cn), 256, 0, s>>>(S.ptr + pc.boff[jb] * nb + pc.boff[ib], nb, a, Rn, Cn, t.coef);
        count_launch();
      }
    }
  }
  check_launch("kron_dense_kernel");
  pt.mark("ldl: Gbb from its Kronecker terms");
  // noise on the diagonal of G_bb
  {
    std::vector<double> nz(nb);
    for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
      const BlockInt& B = p->blocks[pc.bblocks[jb]];
      for (int64_t i = 0; i < B.size; i++) nz[pc.boff[jb] + i] = B.noise;
    }
    DevBuf dn;
    dn.ensure(nb);
    GPFVM_CUDA(cudaMemcpyAsync(dn.ptr, nz.data(), nb * sizeof(double), cudaMemcpyHostToDevice, s));
    add_diag_kernel<<<g1(nb), 256, 0, s>>>(S.ptr, nb, dn.ptr, 0.0);
    count_launch();
    GPFVM_CUDA(cudaStreamSynchronize(s));
  }
  if (!pc.structured) {
  // Y^T = FD(G_pb) rows without forming G_pb: per deflated block J,
  // (V (x) W)^T G_{P,J} = sum_tau c_tau (V^T F0_tau) (x) (W^T F1_tau) is again a
  // Kronecker sum with small factors, applied to the identity of block J; then
  // the D^{-1} scale and the (V (x) W) half of FD.
  {
    const int n0 = pc.n0, n1 = pc.n1;
    std::vector<DevBuf> rot;
    DevBuf w0, w1;
    for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
      const int J = pc.bblocks[jb];
      const int nJ = (int)p->blocks[J].size;
      std::vector<double> coefs;
      std::vector<std::vector<const double*>> fs;
      for (const auto& t : p->terms) {
        if (t.I != pc.P || t.J != J) continue;
        const Factor& F0 = p->factors[t.fid[0]];
        const Factor& F1 = p->factors[t.fid[1]];
        DevBuf R0, R1;
        R0.ensure((size_t)n0 * F0.cols);
        R1.ensure((size_t)n1 * F1.cols);
        Gemm g;  // R0 = V^T F0
        g.M = n0; g.N = F0.cols; g.K = n0;
        g.A = pc.Vt.ptr; g.a_rs = n0; g.a_cs = 1;
        g.B = F0.data.ptr; g.b_rs = F0.cols; g.b_cs = 1;
        g.C = R0.ptr; g.c_rs = F0.cols; g.c_cs = 1;
        run_gemm(g, s);
        g = Gemm();  // R1 = W^T F1
        g.M = n1; g.N = F1.cols; g.K = n1;
        g.A = pc.W.ptr; g.a_rs = 1; g.a_cs = n1;
        g.B = F1.data.ptr; g.b_rs = F1.cols; g.b_cs = 1;
        g.C = R1.ptr; g.c_rs = F1.cols; g.c_cs = 1;
        run_gemm(g, s);
        coefs.push_back(t.coef);
        fs.push_back({R0.ptr, R1.ptr});
        rot.push_back(std::move(R0));
        rot.push_back(std::move(R1));
      }
      pc.t1.ensure((size_t)np * nJ);
      pc.t2.ensure((size_t)np * nJ);
      if (coefs.empty()) {
        fill(pc.YT.ptr + pc.boff[jb] * np, 0.0, (int64_t)nJ * np, s);
        continue;
      }
      eye.ensure((size_t)nJ * nJ);
      set_identity_kernel<<<g1((int64_t)nJ * nJ), 256, 0, s>>>(eye.ptr, nJ, nJ);
      count_launch();
      KronSum ks;
      ks.build(p->ndim, p->blocks[J].shape, p->blocks[pc.P].shape, coefs, fs, s);
      const int64_t wsz = std::max<int64_t>(1, ks.workspace_per_rhs()) * nJ;
      w0.ensure((size_t)wsz);
      w1.ensure((size_t)wsz);
      ks.apply(eye.ptr, nJ, pc.t2.ptr, np, nJ, 0.0, w0.ptr, w1.ptr, s);
      fd_backward(pc, pc.YT.ptr + pc.boff[jb] * np, np, nJ, s);
    }
    GPFVM_CUDA(cudaStreamSynchronize(s));
  }
  pt.mark("ldl: Y = FD(Gpb)");
  }  // !structured
  // G_{I,P} Kronecker sums (used by P^{-1})
  pc.ks_bp.clear();
  pc.ks_bp.resize(pc.bblocks.size());
  {
    int64_t wmax = 1;
    for (size_t ib = 0; ib < pc.bblocks.size(); ib++) {
      const int I = pc.bblocks[ib];
      std::vector<double> coefs;
      std::vector<std::vector<const double*>> fs;
      for (const auto& t : p->terms) {
        if (t.I != I || t.J != pc.P) continue;
        coefs.push_back(t.coef);
        std::vector<const double*> f;
        for (int i = 0; i < p->ndim; i++) f.push_back(p->factors[t.fid[i]].data.ptr);
        fs.push_back(f);
      }
      pc.ks_bp[ib].build(p->ndim, p->blocks[pc.P].shape, p->blocks[I].shape, coefs, fs, s);
      wmax = std::max(wmax, pc.ks_bp[ib].workspace_per_rhs());
    }
    for (const auto& k : pc.rot_ks) wmax = std::max(wmax, k.workspace_per_rhs());
    pc.kw0.ensure((size_t)wmax);
    pc.kw1.ensure((size_t)wmax);
  }
  if (pc.structured) {
    structured_schur(p, pc, S.ptr, s);
  } else {
  // S = G_bb - G_bp Y: instead of the dense GEMM with G_pb^T (nb x nb x N_PDE
  // flops) apply each Kronecker sum -G_{I,P} to the nb columns of Y, contracted
  // in its cheapest mode order (IC/BC blocks are thin in one dimension: ~100x
  // fewer flops on config 1).  Row c of S receives (G_{I,P} y_c)^T; S is
  // symmetrised below.
  {
    DevBuf w0, w1;
    for (size_t ib = 0; ib < pc.bblocks.size(); ib++) {
      const int I = pc.bblocks[ib];
      std::vector<double> coefs;
      std::vector<std::vector<const double*>> fs;
      for (const auto& t : p->terms) {
        if (t.I != I || t.J != pc.P) continue;
        coefs.push_back(-t.coef);
        std::vector<const double*> f;
        for (int i = 0; i < p->ndim; i++) f.push_back(p->factors[t.fid[i]].data.ptr);
        fs.push_back(f);
      }
      if (coefs.empty()) continue;
      KronSum ks;
      ks.build(p->ndim, p->blocks[pc.P].shape, p->blocks[I].shape, coefs, fs, s);
      const int64_t wsz = std::max<int64_t>(1, ks.workspace_per_rhs()) * nb;
      w0.ensure((size_t)wsz);
      w1.ensure((size_t)wsz);
      ks.apply(pc.YT.ptr, np, S.ptr + pc.boff[ib], nb, nb, 1.0, w0.ptr, w1.ptr, s);
    }
    GPFVM_CUDA(cudaStreamSynchronize(s));
  }
  }  // structured / dense Schur
  symm_kernel<<<g1((int64_t)nb * nb), 256, 0, s>>>(S.ptr, nb);
  count_launch();
  pt.mark("ldl: S = Gbb - Gpb^T Y");
  // Cholesky with shift-on-failure
  S0.ensure((size_t)nb * nb);
  Lf.ensure((size_t)nb * nb);
  copy(S0.ptr, S.ptr, (int64_t)nb * nb, s);
  std::vector<double> diag(nb);
  // fetch the diagonal only (strided copy) for the shift scale
  GPFVM_CUDA(cudaMemcpy2DAsync(diag.data(), sizeof(double), S0.ptr, sizeof(double) * (nb + 1), sizeof(double), nb,
                               cudaMemcpyDeviceToHost, s));
  GPFVM_CUDA(cudaStreamSynchronize(s));
  double dmax = 0.0;
  for (double v : diag) dmax = std::max(dmax, v);
  DevBuf info_buf;  // pooled: cudaFree would synchronise the whole device
  info_buf.ensure(1);
  int* d_info = reinterpret_cast<int*>(info_buf.ptr);
  double shift = 0.0;
  for (int attempt = 0; attempt < 30; attempt++) {
    copy(Lf.ptr, S0.ptr, (int64_t)nb * nb, s);
    if (shift > 0.0) {
      add_diag_kernel<<<g1(nb), 256, 0, s>>>(Lf.ptr, nb, nullptr, shift);
      count_launch();
    }
    int info = cholesky_inplace(Lf.ptr, nb, s, d_info);
    if (info == 0) break;
    shift = (shift == 0.0) ? 1e-14 * dmax : shift * 10.0;
    GPFVM_CHECK(attempt < 29, GPFVM_ERR_NUMERIC, "block-LDL: Schur complement not SPD even after shifting");
  }
  pc.shift = shift;
  // explicit L^{-1} (lower triangular; the PRECOND variance uses ||L^{-1} z||^2)
  // and S^{-1} = L^{-T} L^{-1} (nb x nb) so each application is one multi-dot
  pt.mark("ldl: cholesky(S)");
  pc.Linv.ensure((size_t)nb * nb);
  set_identity_kernel<<<g1((int64_t)nb * nb), 256, 0, s>>>(pc.Linv.ptr, nb, nb);
  count_launch();
  trsm_lower(Lf.ptr, nb, pc.Linv.ptr, nb, s);
  pc.Sinv.ensure((size_t)nb * nb);
  {
    Gemm g;
    g.M = nb; g.N = nb; g.K = nb;
    g.A = pc.Linv.ptr; g.a_rs = 1; g.a_cs = nb;  // L^{-T}
    g.B = pc.Linv.ptr; g.b_rs = nb; g.b_cs = 1;
    g.C = pc.Sinv.ptr; g.c_rs = nb; g.c_cs = 1;
    run_gemm(g, s);
  }
  pt.mark("ldl: S^{-1}");
  symm_kernel<<<g1((int64_t)nb * nb), 256, 0, s>>>(pc.Sinv.ptr, nb);
  count_launch();
  pc.rb.ensure(nb);
  pc.zb.ensure(nb);
  pc.cvec.ensure(nb);
  pc.yb.ensure((size_t)np);
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

static void build_precond(gpfvm_problem* p, int type, cudaStream_t s) {
  if (p->pc && p->pc->type == type) return;
  // validate before dropping the cached preconditioner (a failed request must
  // not invalidate a later COV_PRECOND predict)
  GPFVM_CHECK(type == GPFVM_PRECOND_NONE || type == GPFVM_PRECOND_BLOCK_FD, GPFVM_ERR_UNSUPPORTED,
              "unsupported preconditioner");
  destroy_precond(p->pc);
  p->pc = nullptr;
  if (type == GPFVM_PRECOND_NONE) return;
  double t0 = now_ms();
  auto pc = new Precond();
  try {
    pc->type = type;
    int ndefl = 0, nfree = 0;
    int64_t nb = 0;
    for (int b = 0; b < (int)p->blocks.size(); b++) {
      if (!p->blocks[b].deflate) {
        pc->P = b;
        nfree++;
      } else {
        ndefl++;
        nb += p->blocks[b].size;
      }
    }
    // exact path: one 2D two-term PDE block + a dense IC/BC Schur
    // complement; otherwise block-Jacobi fast diagonalisation (§5.4)
    const bool exact = nfree == 1 && exact_fd_ok(p, pc->P) && nb <= 16384 && getenv("GPFVM_FORCE_BJFD") == nullptr;
    PhaseTimer pt(s);
    if (exact) {
      build_fd(p, *pc, s);
      pt.mark("fd: 2 x sygv");
      build_ldl(p, *pc, s);
    } else {
      pc->blockjacobi = true;
      pc->bj.resize(p->blocks.size());
      PencilCache cache;
      static const bool no_cache = getenv("GPFVM_NO_PENCIL_CACHE") != nullptr;
      for (int b = 0; b < (int)p->blocks.size(); b++) build_block_fd(p, b, pc->bj[b], s, no_cache ? nullptr : &cache);
      pt.mark("block-Jacobi FD");
    }
  } catch (...) {
    delete pc;
    throw;
  }
  pc->setup_ms = now_ms() - t0;
  p->pc = pc;
}

// z = P^{-1} r (single vector, z != r)
void precond_apply(gpfvm_problem* p, const double* r, double* z, cudaStream_t s) {
  Precond& pc = *p->pc;
  if (pc.blockjacobi) {
    for (const auto& bf : pc.bj) {
      const BlockInt& B = p->blocks[bf.J];
      apply_block_fd(bf, r + B.offset, z + B.offset, B.size, s);
    }
    return;
  }
  const BlockInt& BP = p->blocks[pc.P];
  const double* rp = r + BP.offset;
  double* zp = z + BP.offset;
  fd_apply(pc, rp, pc.Np, zp, pc.Np, 1, s);
  if (pc.nb == 0) return;
  const int nb = (int)pc.nb;
  for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
    const BlockInt& B = p->blocks[pc.bblocks[jb]];
    copy(pc.rb.ptr + pc.boff[jb], r + B.offset, B.size, s);
  }
  for (size_t ib = 0; ib < pc.bblocks.size(); ib++)  // c = G_bp FD r_p
    pc.ks_bp[ib].apply(zp, pc.Np, pc.cvec.ptr + pc.boff[ib], p->blocks[pc.bblocks[ib]].size, 1, 0.0,
                       pc.kw0.ptr, pc.kw1.ptr, s);
  sub_kernel<<<g1(nb), 256, 0, s>>>(pc.rb.ptr, pc.cvec.ptr, nb);
  count_launch();
  dot_many(pc.Sinv.ptr, nb, pc.rb.ptr, nb, nb, pc.zb.ptr, s);    // z_b = S^{-1} t
  for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
    const BlockInt& B = p->blocks[pc.bblocks[jb]];
    copy(z + B.offset, pc.zb.ptr + pc.boff[jb], B.size, s);
  }
  if (pc.structured) {
    // z_p -= FD G_pb z_b = (V (x) W) D^{-1} sum_J Z_J z_b,J
    for (size_t jb = 0; jb < pc.bblocks.size(); jb++)
      pc.rot_ks[jb].apply(pc.zb.ptr + pc.boff[jb], p->blocks[pc.bblocks[jb]].size, pc.t2.ptr, pc.Np, 1,
                          jb == 0 ? 0.0 : 1.0, pc.kw0.ptr, pc.kw1.ptr, s);
    fd_backward(pc, pc.yb.ptr, pc.Np, 1, s);
    sub_kernel<<<g1(pc.Np), 256, 0, s>>>(zp, pc.yb.ptr, pc.Np);
    count_launch();
  } else {
    axpy_many(zp, pc.YT.ptr, pc.Np, pc.zb.ptr, -1.0, pc.Np, nb, s);  // z_p -= Y z_b
  }
}

// grow a Krylov store to `need` slots, keeping the first `valid` ones
static void ensure_krylov_K(Krylov& K, int64_t N, int need, int valid, cudaStream_t s) {
  if (need <= K.cap) return;
  int cap = std::max(need, std::max(8, K.cap * 2));
  DevBuf d, gd;
  d.ensure((size_t)cap * N);
  gd.ensure((size_t)cap * N);
  if (valid > 0) {
    copy(d.ptr, K.d.ptr, (int64_t)valid * N, s);
    copy(gd.ptr, K.gd.ptr, (int64_t)valid * N, s);
  }
  K.d = std::move(d);
  K.gd = std::move(gd);
  K.cap = cap;
}
static void ensure_krylov(gpfvm_problem* p, int need, int valid, cudaStream_t s) {
  ensure_krylov_K(p->kry, p->N, need, valid, s);
}

static double norm2(const double* v, int64_t n, double* dtmp, cudaStream_t s) {
  dot_many(v, n, v, n, 1, dtmp, s);
  double h;
  GPFVM_CUDA(cudaMemcpyAsync(&h, dtmp, sizeof(double), cudaMemcpyDeviceToHost, s));
  GPFVM_CUDA(cudaStreamSynchronize(s));
  return std::sqrt(h);
}

void solve_impl(gpfvm_problem* p, const double* y, double* x, const gpfvm_solve_opts& o, gpfvm_solve_report& rep,
                cudaStream_t s) {
  const int64_t N = p->N;
  double t_setup0 = now_ms();
  bool had = p->pc != nullptr && p->pc->type == o.precond;
  build_precond(p, o.precond, s);
  rep.setup_ms = had ? 0.0 : (now_ms() - t_setup0);
  rep.precond_shift = p->pc ? p->pc->shift : 0.0;
  double t0 = now_ms();
  Krylov& K = p->kry;
  K.k = 0;
  K.eta.clear();
  // keep_actions = 0: only a ring of W = max(1, reorth_window) actions is kept
  // (memory O(W N) for long budgeted solves); the IterGP covariance then
  // covers those W actions only
  const bool keep = o.keep_actions != 0;
  const int W = keep ? 0 : std::max(1, o.reorth_window);
  const int neta = keep ? std::max(1, o.max_iter) : W;
  DevBuf r, sc;
  r.ensure(N);
  // device scalars: [state (ST_SIZE)] [c: reorthogonalisation coefficients] [eta_j]
  sc.ensure((size_t)ST_SIZE + 2 * (size_t)neta + 8);
  double* state = sc.ptr;
  double* cdev = sc.ptr + ST_SIZE;
  double* etad = cdev + neta;
  copy(r.ptr, y, N, s);
  fill(x, 0.0, N, s);
  itergp_init(y, N, o.rtol, state, s);
  // host view of the state: read only at the periodic checks (iterations 1-4,
  // then every 4th) — the kernels themselves stop once converged
  double hst[ST_SIZE];
  auto read_state = [&]() {
    GPFVM_CUDA(cudaMemcpyAsync(hst, state, sizeof(hst), cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
  };
  read_state();
  const double ny = hst[ST_NY];
  int it = 0;  // host-issued iterations (>= the device count)
  while (it < o.max_iter) {
    if (it > 0 && (it <= 4 || it % 4 == 0)) {
      read_state();
      if (hst[ST_DONE] != 0.0) break;
    } else if (it == 0 && hst[ST_DONE] != 0.0) {
      break;
    }
    const int stored = keep ? it : std::min(it, W);
    const int slot = keep ? it : it % W;
    ensure_krylov(p, keep ? it + 1 : std::min(it + 1, W), stored, s);
    // s = P^{-1} r ; z = G s  on fixed operands (graph-replayed matvec)
    p->pcg_s.ensure(N);
    p->pcg_z.ensure(N);
    double* d = p->pcg_s.ptr;
    double* gd = p->pcg_z.ptr;
    if (p->pc) precond_apply(p, r.ptr, d, s);
    else copy(d, r.ptr, N, s);
    matvec_device(p, d, gd, 1, N, s);
    // G-orthogonalise against the last w kept directions (w = k: full
    // reorthogonalisation, §6 l.475; w = 1: the PCG recurrence), store the
    // action in its Krylov slot, eta = d.Gd, a = d.r / eta: two fused passes
    const int w = stored == 0 ? 0 : (keep && o.reorth_window > 0 ? std::min(o.reorth_window, stored) : stored);
    const int j0 = stored - w;
    itergp_reorth_coefs(K.d.ptr + (int64_t)j0 * N, N, w, gd, N, etad + j0, cdev, state, s);
    double* dslot = K.d.ptr + (int64_t)slot * N;
    double* gslot = K.gd.ptr + (int64_t)slot * N;
    itergp_update(d, gd, K.d.ptr + (int64_t)j0 * N, K.gd.ptr + (int64_t)j0 * N, N, w, cdev, r.ptr, dslot, gslot, N,
                  state, etad + slot, s);
    itergp_step(x, r.ptr, dslot, gslot, N, state, s);
    it++;
  }
  read_state();
  const int done_it = (int)hst[ST_COUNT];
  const bool breakdown = hst[ST_DONE] == 2.0;
  // the kept actions: every completed iteration (ring: the last min(done, W))
  K.k = keep ? done_it : std::min(done_it, W);
  K.eta.assign(K.k, 0.0);
  if (K.k > 0) {
    GPFVM_CUDA(cudaMemcpyAsync(K.eta.data(), etad, sizeof(double) * K.k, cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
  }
  const double nr = hst[ST_NR];
  rep.converged = (hst[ST_DONE] == 1.0 || (ny > 0 && nr <= o.rtol * ny) || ny == 0.0) ? 1 : 0;
  rep.breakdown = breakdown ? 1 : 0;
  rep.iterations = done_it;
  rep.rel_residual = ny > 0 ? nr / ny : 0.0;
  rep.iterate_ms = now_ms() - t0;
  // true residual ||G x - y||
  matvec_device(p, x, r.ptr, 1, N, s);
  double one = 1.0;
  GPFVM_CUDA(cudaMemcpyAsync(cdev, &one, sizeof(double), cudaMemcpyHostToDevice, s));
  axpy_many(r.ptr, y, N, cdev, -1.0, N, 1, s);  // r = Gx - y
  double tr = norm2(r.ptr, N, cdev + 1, s);
  rep.true_rel_residual = ny > 0 ? tr / ny : 0.0;
}

// nrhs > 1: one IterGP run per right-hand side, sharing every batched
// operation: the preconditioner (block-Jacobi FD, R vectors per Kronecker
// product) and the graph-replayed Gram matvec on R vectors.
// The per-RHS vector steps run on per-RHS device states, each stopping on its
// own convergence.  The exact 2D preconditioner is single-vector: those solves
// run one after the other.  The Krylov store of RHS 0 is the one gpfvm_predict
// uses for the ITERGP variance.
void solve_many_impl(gpfvm_problem* p, const double* Y, int64_t ldy, double* X, int64_t ldx, int R,
                     const gpfvm_solve_opts& o, gpfvm_solve_report* reps, cudaStream_t s) {
  if (R == 1) {
    solve_impl(p, Y, X, o, reps[0], s);
    return;
  }
  double t_setup0 = now_ms();
  const bool had = p->pc != nullptr && p->pc->type == o.precond;
  build_precond(p, o.precond, s);
  const double setup_ms = had ? 0.0 : (now_ms() - t_setup0);
  if (p->pc && !p->pc->blockjacobi) {
    for (int r = R - 1; r >= 0; r--) {
      solve_impl(p, Y + r * ldy, X + r * ldx, o, reps[r], s);
      if (r == R - 1) reps[r].setup_ms = setup_ms;
    }
    return;
  }
  const int64_t N = p->N;
  double t0 = now_ms();
  const bool keep = o.keep_actions != 0;
  const int W = keep ? 0 : std::max(1, o.reorth_window);
  const int neta = keep ? std::max(1, o.max_iter) : W;
  const int64_t sc_per = ST_SIZE + 2 * (int64_t)neta + 8;
  std::vector<Krylov> extra(R - 1);
  auto Kr = [&](int r) -> Krylov& { return r == 0 ? p->kry : extra[r - 1]; };
  p->kry.k = 0;
  p->kry.eta.clear();
  DevBuf rv, sc;
  rv.ensure((size_t)R * N);
  sc.ensure((size_t)R * sc_per);
  auto state = [&](int r) { return sc.ptr + r * sc_per; };
  auto cdev = [&](int r) { return sc.ptr + r * sc_per + ST_SIZE; };
  auto etad = [&](int r) { return sc.ptr + r * sc_per + ST_SIZE + neta; };
  for (int r = 0; r < R; r++) {
    copy(rv.ptr + r * N, Y + r * ldy, N, s);
    fill(X + r * ldx, 0.0, N, s);
    itergp_init(Y + r * ldy, N, o.rtol, state(r), s);
  }
  std::vector<double> hst((size_t)R * ST_SIZE);
  auto read_states = [&]() {
    for (int r = 0; r < R; r++)
      GPFVM_CUDA(cudaMemcpyAsync(hst.data() + r * ST_SIZE, state(r), ST_SIZE * sizeof(double), cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
  };
  auto all_done = [&]() {
    for (int r = 0; r < R; r++)
      if (hst[r * ST_SIZE + ST_DONE] == 0.0) return false;
    return true;
  };
  read_states();
  // batched preconditioner workspaces
  DevBuf ptmp, pw0, pw1;
  if (p->pc) {
    int64_t mx = 1, mw = 1;
    for (const auto& bf : p->pc->bj) {
      mx = std::max<int64_t>(mx, p->blocks[bf.J].size);
      mw = std::max<int64_t>(mw, std::max(bf.fwd.workspace_per_rhs(), bf.bwd.workspace_per_rhs()));
    }
    ptmp.ensure((size_t)R * mx);
    pw0.ensure((size_t)R * mw);
    pw1.ensure((size_t)R * mw);
  }
  p->pcg_s.ensure((size_t)R * N);
  p->pcg_z.ensure((size_t)R * N);
  double* d = p->pcg_s.ptr;
  double* gd = p->pcg_z.ptr;
  int it = 0;
  while (it < o.max_iter) {
    if (it > 0 && (it <= 4 || it % 4 == 0)) {
      read_states();
      if (all_done()) break;
    } else if (it == 0 && all_done()) {
      break;
    }
    const int stored = keep ? it : std::min(it, W);
    const int slot = keep ? it : it % W;
    for (int r = 0; r < R; r++) ensure_krylov_K(Kr(r), N, keep ? it + 1 : std::min(it + 1, W), stored, s);
    if (p->pc) {
      for (const auto& bf : p->pc->bj) {
        const BlockInt& B = p->blocks[bf.J];
        apply_block_fd_many(bf, rv.ptr + B.offset, N, d + B.offset, N, B.size, R, ptmp.ptr, pw0.ptr, pw1.ptr, s);
      }
    } else {
      copy(d, rv.ptr, (int64_t)R * N, s);
    }
    matvec_device(p, d, gd, R, N, s);
    const int w = stored == 0 ? 0 : (keep && o.reorth_window > 0 ? std::min(o.reorth_window, stored) : stored);
    const int j0 = stored - w;
    for (int r = 0; r < R; r++) {
      Krylov& K = Kr(r);
      double* dr = d + r * N;
      double* gr = gd + r * N;
      itergp_reorth_coefs(K.d.ptr + (int64_t)j0 * N, N, w, gr, N, etad(r) + j0, cdev(r), state(r), s);
      double* dslot = K.d.ptr + (int64_t)slot * N;
      double* gslot = K.gd.ptr + (int64_t)slot * N;
      itergp_update(dr, gr, K.d.ptr + (int64_t)j0 * N, K.gd.ptr + (int64_t)j0 * N, N, w, cdev(r), rv.ptr + r * N,
                    dslot, gslot, N, state(r), etad(r) + slot, s);
      itergp_step(X + r * ldx, rv.ptr + r * N, dslot, gslot, N, state(r), s);
    }
    it++;
  }
  read_states();
  const double iterate_ms = now_ms() - t0;
  // true residuals: one batched matvec
  DevBuf res, one;
  res.ensure((size_t)R * ldx);
  matvec_device(p, X, res.ptr, R, ldx, s);
  one.ensure(2);
  fill(one.ptr, 1.0, 1, s);
  for (int r = 0; r < R; r++) {
    axpy_many(res.ptr + r * ldx, Y + r * ldy, N, one.ptr, -1.0, N, 1, s);
    dot_many(res.ptr + r * ldx, N, res.ptr + r * ldx, N, 1, one.ptr + 1, s);
    double tr2 = 0.0;
    GPFVM_CUDA(cudaMemcpyAsync(&tr2, one.ptr + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
    const double* h = hst.data() + r * ST_SIZE;
    Krylov& K = Kr(r);
    const int done_it = (int)h[ST_COUNT];
    K.k = keep ? done_it : std::min(done_it, W);
    K.eta.assign(K.k, 0.0);
    if (K.k > 0) {
      GPFVM_CUDA(cudaMemcpyAsync(K.eta.data(), etad(r), sizeof(double) * K.k, cudaMemcpyDeviceToHost, s));
      GPFVM_CUDA(cudaStreamSynchronize(s));
    }
    const double ny = h[ST_NY], nr = h[ST_NR];
    gpfvm_solve_report& rep = reps[r];
    rep = gpfvm_solve_report{};
    rep.iterations = done_it;
    rep.converged = (h[ST_DONE] == 1.0 || ny == 0.0 || (ny > 0 && nr <= o.rtol * ny)) ? 1 : 0;
    rep.breakdown = h[ST_DONE] == 2.0 ? 1 : 0;
    rep.rel_residual = ny > 0 ? nr / ny : 0.0;
    rep.true_rel_residual = ny > 0 ? std::sqrt(tr2) / ny : 0.0;
    rep.precond_shift = p->pc ? p->pc->shift : 0.0;
    rep.setup_ms = r == 0 ? setup_ms : 0.0;
    rep.iterate_ms = iterate_ms;
  }
}

}  // namespace gpfvm

// ---- C ABI: standalone FD setup and elementwise product (sharded path) ----------
namespace gpfvm {
namespace {
__global__ void vmul_kernel(double* x, const double* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= d[i];
}
}  // namespace
}  // namespace gpfvm

extern "C" int gpfvm_fd_setup(int n0, int n1, const double* A0, const double* A1, const double* B0, const double* B1,
                              double ca, double cb, double noise, double* V, double* W, double* Dinv, void* stream) {
  using namespace gpfvm;
  try {
    GPFVM_CHECK(n0 >= 1 && n1 >= 1 && A0 && A1 && B0 && B1 && V && W && Dinv, GPFVM_ERR_INVALID, "bad fd_setup args");
    cudaStream_t s = (cudaStream_t)stream;
    DevBuf lam, mu, vv, ww;
    lam.ensure(n0); mu.ensure(n1); vv.ensure(n0); ww.ensure(n1);
    sygv(B0, A0, n0, V, lam.ptr, s);
    sygv(A1, B1, n1, W, mu.ptr, s);
    colsumsq_kernel<<<g1(n0, 128), 128, 0, s>>>(V, n0, vv.ptr);
    colsumsq_kernel<<<g1(n1, 128), 128, 0, s>>>(W, n1, ww.ptr);
    dinv_kernel<<<g1((int64_t)n0 * n1), 256, 0, s>>>(Dinv, lam.ptr, mu.ptr, vv.ptr, ww.ptr, n0, n1, ca, cb, noise);
    count_launch(3);
    check_launch("gpfvm_fd_setup");
    GPFVM_CUDA(cudaStreamSynchronize(s));
    return GPFVM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  }
}

extern "C" int gpfvm_vmul(double* x, const double* d, int64_t n, void* stream) {
  using namespace gpfvm;
  try {
    GPFVM_CHECK(x && d && n >= 0, GPFVM_ERR_INVALID, "bad vmul args");
    if (n == 0) return GPFVM_OK;
    vmul_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 2048), 256, 0, (cudaStream_t)stream>>>(x, d, n);
    count_launch();
    check_launch("vmul_kernel");
    return GPFVM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  }
}
