// §8 row 4 — gpfvm_predict: posterior mean / variance on a tensor grid
// (Eq. 5-6, l.113-114).
//
// The grid is a pseudo-block of point functionals of order 0 on output
// `out`.  Its cross-covariance with block J is a sum of Kronecker products
// of 1D cross factors  F(grid_i, 0; sites_J,i, alpha_i)  (Eq. 14, l.244),
// assembled by the same double-double kernel as the Gram factors and applied
// with the same DMMA mode products:
//   mean = sum_J K_{*J} alpha_J
//   var  = k(x,x) - k_x^T C k_x
//     ITERGP : C = sum_i d_i d_i^T / eta_i        (rows of W = K_* D, downdate)
//     PRECOND: C = P^{-1}, evaluated for the whole grid without a per-point
//              solve: with (V(x)W)^T k_p = sum_tau c_tau (A_tau V)[t,:] (x) (B_tau W)[x,:]
//              the FD part is  sum_{tau,tau'} c c' [(Â_tau o Â_tau') D^{-1} (B̂_tau o B̂_tau')^T]
//              (three GEMMs per pair), and the IC/BC Schur part is
//              z^T S^{-1} z with z = k_b - Y^T k_p, processed in grid slabs.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "problem.h"

namespace gpfvm {


namespace {

__global__ void downdate_kernel(double* var, const double* __restrict__ W, const double* __restrict__ inv_eta,
                                int k, int64_t ng, bool init, double prior) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    double v = init ? prior : var[g];
    for (int j = 0; j < k; j++) {
      double w = W[j * ng + g];
      v -= w * w * inv_eta[j];
    }
    var[g] = v;
  }
}

__global__ void hadamard_kernel(double* out, const double* __restrict__ a, const double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

// var[g] -= sum_c Z[c][g] T[c][g]
__global__ void coldot_sub_kernel(double* var, const double* __restrict__ Z, const double* __restrict__ T, int nb,
                                  int64_t ng) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nb; c++) s = fma(Z[(int64_t)c * ng + g], T[(int64_t)c * ng + g], s);
    var[g] -= s;
  }
}

// X[r][k] *= d[k] for r = blockIdx.y (rows of length n)
__global__ void scale_rows_by_kernel(double* X, const double* __restrict__ d, int64_t n) {
  double* xr = X + (int64_t)blockIdx.y * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    xr[k] *= d[k];
}

unsigned gs(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

}  // namespace

// cross factors between a grid (points, order 0) and every block with a term on `out`
struct CrossPlan {
  DevBuf w0, w1;  // KronSum workspaces
  std::vector<Factor> factors;
  std::vector<std::vector<KronTerm>> terms;  // per block J
  int gshape[GPFVM_MAX_DIMS] = {1, 1, 1, 1};
  Sites gsites[GPFVM_MAX_DIMS];
};

static void build_cross(gpfvm_problem* p, const gpfvm_grid& g, int row0, int rows, CrossPlan& cp, cudaStream_t s) {
  const int d = p->ndim;
  for (int i = 0; i < d; i++) {
    Sites& S = cp.gsites[i];
    S.kind = GPFVM_SITE_POINT;
    int off = (i == 0) ? row0 : 0;
    S.n = (i == 0) ? rows : g.n[i];
    S.lo.assign(g.pts[i] + off, g.pts[i] + off + S.n);
    S.hi = S.lo;
    S.d_lo.ensure(S.n);
    S.d_hi.ensure(S.n);
    GPFVM_CUDA(cudaMemcpyAsync(S.d_lo.ptr, S.lo.data(), S.n * sizeof(double), cudaMemcpyHostToDevice, s));
    GPFVM_CUDA(cudaMemcpyAsync(S.d_hi.ptr, S.lo.data(), S.n * sizeof(double), cudaMemcpyHostToDevice, s));
    cp.gshape[i] = S.n;
  }
  std::map<std::tuple<int, int, int>, int> idx;  // (dim, block, order) -> factor
  cp.terms.assign(p->blocks.size(), {});
  for (int J = 0; J < (int)p->blocks.size(); J++) {
    const BlockInt& B = p->blocks[J];
    for (const auto& t : B.terms) {
      if (t.output != g.output) continue;
      KronTerm kt;
      kt.I = -1;
      kt.J = J;
      kt.coef = t.coeff;
      for (int i = 0; i < d; i++) {
        auto key = std::make_tuple(i, J, t.order[i]);
        auto it = idx.find(key);
        if (it == idx.end()) {
          Factor F;
          F.rows = cp.gsites[i].n;
          F.cols = B.sites[i].n;
          F.data.ensure((size_t)std::max(1, F.rows * F.cols));
          const gpfvm_kernel1d& k = p->kernels[g.output * d + i];
          launch_factor(matern_dd(k.q, k.lengthscale, k.variance), cp.gsites[i], 0, B.sites[i], t.order[i],
                        F.data.ptr, F.cols, s);
          cp.factors.push_back(std::move(F));
          it = idx.emplace(key, (int)cp.factors.size() - 1).first;
        }
        kt.fid[i] = it->second;
      }
      cp.terms[J].push_back(kt);
    }
  }
}

// Y_r = beta Y_r + scale * K_{*J} X_r for R vectors through the fused KronSum plan
static void cross_apply(gpfvm_problem* p, CrossPlan& cp, int J, double scale, const double* X, int64_t ldx, double* Y,
                        int64_t ldy, int R, double beta, cudaStream_t s) {
  std::vector<double> coefs;
  std::vector<std::vector<const double*>> fs;
  for (const auto& t : cp.terms[J]) {
    coefs.push_back(scale * t.coef);
    std::vector<const double*> f;
    for (int i = 0; i < p->ndim; i++) f.push_back(cp.factors[t.fid[i]].data.ptr);
    fs.push_back(f);
  }
  KronSum ks;
  ks.build(p->ndim, p->blocks[J].shape, cp.gshape, coefs, fs, s);
  size_t need = (size_t)std::max<int64_t>(1, ks.workspace_per_rhs() * R);
  cp.w0.ensure(need);
  cp.w1.ensure(need);
  ks.apply(X, ldx, Y, ldy, R, beta, cp.w0.ptr, cp.w1.ptr, s);
  GPFVM_CUDA(cudaStreamSynchronize(s));  // ks (stacked factors) is freed on return
}

// out[r] (grid slab) = sum_J K_{*J} X_J[r]  (overwrite), R vectors of stride ldx
static void apply_cross(gpfvm_problem* p, CrossPlan& cp, const double* X, int64_t ldx, double* out, int64_t ldo, int R,
                        double scale, bool overwrite, cudaStream_t s) {
  bool first = overwrite;
  for (int J = 0; J < (int)p->blocks.size(); J++) {
    if (cp.terms[J].empty()) continue;
    cross_apply(p, cp, J, scale, X + p->blocks[J].offset, ldx, out, ldo, R, first ? 0.0 : 1.0, s);
    first = false;
  }
  if (first) {
    int64_t ng = 1;
    for (int i = 0; i < p->ndim; i++) ng *= cp.gshape[i];
    for (int r = 0; r < R; r++) fill(out + r * ldo, 0.0, ng, s);
  }
}

static double prior_var(gpfvm_problem* p, int out) {
  double v = 1.0;
  for (int i = 0; i < p->ndim; i++) v *= p->kernels[out * p->ndim + i].variance;
  return v;
}

static void var_precond_slab(gpfvm_problem* p, CrossPlan& cp, double* var, int64_t ng, cudaStream_t s) {
  GPFVM_CHECK(p->pc && p->pc->type == GPFVM_PRECOND_BLOCK_FD, GPFVM_ERR_STATE,
              "GPFVM_COV_PRECOND needs a preceding gpfvm_solve with the BLOCK_FD preconditioner");
  Precond& pc = *p->pc;
  GPFVM_CHECK(!pc.blockjacobi, GPFVM_ERR_UNSUPPORTED,
              "GPFVM_COV_PRECOND needs the exact (2D two-term, block-LDL) preconditioner; use GPFVM_COV_ITERGP");
  const int n0 = pc.n0, n1 = pc.n1;
  const int g0 = cp.gshape[0], g1 = cp.gshape[1];
  // --- FD part -------------------------------------------------------------
  const auto& tP = cp.terms[pc.P];
  std::vector<DevBuf> Ah(tP.size()), Bh(tP.size());
  for (size_t a = 0; a < tP.size(); a++) {
    const Factor& A = cp.factors[tP[a].fid[0]];  // g0 x n0
    const Factor& B = cp.factors[tP[a].fid[1]];  // g1 x n1
    Ah[a].ensure((size_t)g0 * n0);
    Bh[a].ensure((size_t)g1 * n1);
    Gemm g;
    g.M = g0; g.N = n0; g.K = n0;
    g.A = A.data.ptr; g.a_rs = n0; g.a_cs = 1;
    g.B = pc.V.ptr; g.b_rs = n0; g.b_cs = 1;
    g.C = Ah[a].ptr; g.c_rs = n0; g.c_cs = 1;
    run_gemm(g, s);
    g = Gemm();
    g.M = g1; g.N = n1; g.K = n1;
    g.A = B.data.ptr; g.a_rs = n1; g.a_cs = 1;
    g.B = pc.W.ptr; g.b_rs = n1; g.b_cs = 1;
    g.C = Bh[a].ptr; g.c_rs = n1; g.c_cs = 1;
    run_gemm(g, s);
  }
  DevBuf Pm, Qm, M1;
  Pm.ensure((size_t)g0 * n0);
  Qm.ensure((size_t)g1 * n1);
  M1.ensure((size_t)g0 * n1);
  for (size_t a = 0; a < tP.size(); a++)
    for (size_t b = a; b < tP.size(); b++) {
      double w = tP[a].coef * tP[b].coef * (a == b ? 1.0 : 2.0);
      hadamard_kernel<<<gs((int64_t)g0 * n0), 256, 0, s>>>(Pm.ptr, Ah[a].ptr, Ah[b].ptr, (int64_t)g0 * n0);
      hadamard_kernel<<<gs((int64_t)g1 * n1), 256, 0, s>>>(Qm.ptr, Bh[a].ptr, Bh[b].ptr, (int64_t)g1 * n1);
      count_launch(2);
      Gemm g;
      g.M = g0; g.N = n1; g.K = n0;
      g.A = Pm.ptr; g.a_rs = n0; g.a_cs = 1;
      g.B = pc.Dinv.ptr; g.b_rs = n1; g.b_cs = 1;
      g.C = M1.ptr; g.c_rs = n1; g.c_cs = 1;
      run_gemm(g, s);
      g = Gemm();
      g.M = g0; g.N = g1; g.K = n1;
      g.A = M1.ptr; g.a_rs = n1; g.a_cs = 1;
      g.B = Qm.ptr; g.b_rs = 1; g.b_cs = n1;
      g.C = var; g.c_rs = g1; g.c_cs = 1;
      g.alpha = -w; g.beta = 1.0;
      run_gemm(g, s);
    }
  // --- IC/BC Schur part ----------------------------------------------------
  // z(x) = k_b(x) - Y^T k_p(x), var -= z^T S^{-1} z = ||L^{-1} z||^2.  By
  // linearity L^{-1} Z = K_{*b} L^{-T} - K_{*P} (L^{-1} Y^T)^T: push the rows of
  // L^{-1} (per deflated block) and of L^{-1} Y^T (cached per preconditioner)
  // through the cross-covariance Kronecker sums, then column sums of squares.
  if (pc.nb == 0) return;
  const int nb = (int)pc.nb;
  if (pc.structured) {
    // K_{*P} Y L^{-T} = K_{*P} (V (x) W) D^{-1} Z L^{-T} = Khat M with
    // Khat = sum_a c_a (A_a V) (x) (B_a W) (the Ah, Bh above) and the nb rows of
    // M = D^{-1} (sum_J Z_J L^{-T}[J rows, :]) cached per preconditioner.
    if (!pc.LYT.ptr) {
      pc.LYT.ensure((size_t)nb * pc.Np);
      DevBuf w0, w1;
      for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
        const int64_t wsz = std::max<int64_t>(1, pc.rot_ks[jb].workspace_per_rhs()) * nb;
        w0.ensure((size_t)wsz);
        w1.ensure((size_t)wsz);
        pc.rot_ks[jb].apply(pc.Linv.ptr + pc.boff[jb], nb, pc.LYT.ptr, pc.Np, nb, jb == 0 ? 0.0 : 1.0, w0.ptr, w1.ptr,
                            s);
      }
      scale_rows_by_kernel<<<dim3(gs(pc.Np), nb), 256, 0, s>>>(pc.LYT.ptr, pc.Dinv.ptr, pc.Np);
      count_launch();
      GPFVM_CUDA(cudaStreamSynchronize(s));
    }
    DevBuf Z;
    Z.ensure((size_t)nb * ng);
    bool first = true;
    // K_{*b} L^{-T}: every thin deflated block couples to the 2D grid as a
    // rank-P update, so all of them go into one rank-r GEMM that writes Z once
    // (instead of one K = 1 expansion pass over Z per block)
    {
      LowRank lr;
      lr.n0 = g0;
      lr.n1 = g1;
      std::vector<int64_t> boff(p->blocks.size(), 0);
      for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
        const int J = pc.bblocks[jb];
        boff[J] = pc.boff[jb];
        if (cp.terms[J].empty()) continue;
        std::vector<LowRankTerm> lt;
        for (const auto& t : cp.terms[J])
          lt.push_back({t.coef, cp.factors[t.fid[0]].data.ptr, cp.factors[t.fid[1]].data.ptr});
        add_lowrank_part(lr, J, p->blocks[J].shape, lt, s);
      }
      if (lr.rk > 0) {
        lr.ensure(nb);
        lr.apply(pc.Linv.ptr, nb, Z.ptr, ng, nb, 0.0, boff.data(), s);
        first = false;
      }
      GPFVM_CUDA(cudaStreamSynchronize(s));
    }
    std::vector<double> coefs;
    std::vector<std::vector<const double*>> fs;
    for (size_t a = 0; a < tP.size(); a++) {
      coefs.push_back(-tP[a].coef);
      fs.push_back({Ah[a].ptr, Bh[a].ptr});
    }
    KronSum ks;
    ks.build(p->ndim, p->blocks[pc.P].shape, cp.gshape, coefs, fs, s);
    size_t need = (size_t)std::max<int64_t>(1, ks.workspace_per_rhs() * nb);
    cp.w0.ensure(need);
    cp.w1.ensure(need);
    ks.apply(pc.LYT.ptr, pc.Np, Z.ptr, ng, nb, first ? 0.0 : 1.0, cp.w0.ptr, cp.w1.ptr, s);
    coldot_sub_kernel<<<gs(ng), 256, 0, s>>>(var, Z.ptr, Z.ptr, nb, ng);
    count_launch();
    GPFVM_CUDA(cudaStreamSynchronize(s));
    return;
  }
  if (!pc.LYT.ptr) {
    // L^{-1} Y^T with L^{-1} lower triangular: row panels touch only the
    // nonzero columns
    pc.LYT.ensure((size_t)nb * pc.Np);
    constexpr int RB = 128;
    for (int i0 = 0; i0 < nb; i0 += RB) {
      const int rb = std::min(RB, nb - i0);
      Gemm g;
      g.M = rb; g.N = (int)pc.Np; g.K = i0 + rb;
      g.A = pc.Linv.ptr + (int64_t)i0 * nb; g.a_rs = nb; g.a_cs = 1;
      g.B = pc.YT.ptr; g.b_rs = pc.Np; g.b_cs = 1;
      g.C = pc.LYT.ptr + (int64_t)i0 * pc.Np; g.c_rs = pc.Np; g.c_cs = 1;
      run_gemm(g, s);
    }
  }
  DevBuf Z;
  Z.ensure((size_t)nb * ng);
  bool first = true;
  for (size_t jb = 0; jb < pc.bblocks.size(); jb++) {
    const int J = pc.bblocks[jb];
    if (cp.terms[J].empty()) continue;
    cross_apply(p, cp, J, 1.0, pc.Linv.ptr + pc.boff[jb], nb, Z.ptr, ng, nb, first ? 0.0 : 1.0, s);
    first = false;
  }
  cross_apply(p, cp, pc.P, -1.0, pc.LYT.ptr, pc.Np, Z.ptr, ng, nb, first ? 0.0 : 1.0, s);
  coldot_sub_kernel<<<gs(ng), 256, 0, s>>>(var, Z.ptr, Z.ptr, nb, ng);
  count_launch();
}

// Time-sharded posterior mean: this rank's share
//   mean_partial = sum_J K_{*J}[:, owned rows of J] alpha_J,local
// — the time cross factor restricted to the owned columns; the sum over the
// ranks (all_reduce by the caller) is the posterior mean of Eq. 5 (l.113).
// loc_off/row0/rows: the shard layout of every block.
void predict_mean_shard(gpfvm_problem* p, const gpfvm_grid& g, const double* alpha_local, const int64_t* loc_off,
                        const int* row0, const int* rows, double* mean, cudaStream_t s) {
  const int d = p->ndim;
  int64_t ng = 1;
  for (int i = 0; i < d; i++) ng *= g.n[i];
  fill(mean, 0.0, ng, s);
  CrossPlan cp;
  build_cross(p, g, 0, g.n[0], cp, s);
  for (int J = 0; J < (int)p->blocks.size(); J++) {
    if (cp.terms[J].empty() || rows[J] == 0) continue;
    const BlockInt& B = p->blocks[J];
    int in_shape[GPFVM_MAX_DIMS];
    for (int i = 0; i < d; i++) in_shape[i] = B.shape[i];
    in_shape[0] = rows[J];
    std::vector<double> coefs;
    std::vector<std::vector<const double*>> fs;
    std::vector<DevBuf> sub(cp.terms[J].size());
    for (size_t k = 0; k < cp.terms[J].size(); k++) {
      const KronTerm& t = cp.terms[J][k];
      const Factor& F0 = cp.factors[t.fid[0]];  // grid_t x n0_J
      sub[k].ensure((size_t)F0.rows * rows[J]);
      GPFVM_CUDA(cudaMemcpy2DAsync(sub[k].ptr, rows[J] * sizeof(double), F0.data.ptr + row0[J], F0.cols * sizeof(double),
                                   rows[J] * sizeof(double), F0.rows, cudaMemcpyDeviceToDevice, s));
      coefs.push_back(t.coef);
      std::vector<const double*> f{sub[k].ptr};
      for (int i = 1; i < d; i++) f.push_back(cp.factors[t.fid[i]].data.ptr);
      fs.push_back(f);
    }
    KronSum ks;
    ks.build(d, in_shape, cp.gshape, coefs, fs, s);
    size_t need = (size_t)std::max<int64_t>(1, ks.workspace_per_rhs());
    cp.w0.ensure(need);
    cp.w1.ensure(need);
    ks.apply(alpha_local + loc_off[J], 1, mean, ng, 1, 1.0, cp.w0.ptr, cp.w1.ptr, s);
    GPFVM_CUDA(cudaStreamSynchronize(s));  // sub / ks freed on scope exit
  }
}

void predict_impl(gpfvm_problem* p, const gpfvm_grid& g, const double* alpha, double* mean, double* var, int cov_mode,
                  cudaStream_t s) {
  const int d = p->ndim;
  int64_t ng = 1;
  for (int i = 0; i < d; i++) ng *= g.n[i];
  const double prior = prior_var(p, g.output);
  if (mean) {
    CrossPlan cp;
    build_cross(p, g, 0, g.n[0], cp, s);
    apply_cross(p, cp, alpha, p->N, mean, ng, 1, 1.0, true, s);
  }
  if (!var) return;
  if (cov_mode == GPFVM_COV_ITERGP) {
    CrossPlan cp;
    build_cross(p, g, 0, g.n[0], cp, s);
    Krylov& K = p->kry;
    if (K.k == 0) {
      fill(var, prior, ng, s);
      return;
    }
    const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(64, (int64_t)(2e9 / 8 / std::max<int64_t>(ng, 1))));
    DevBuf Wb, ie;
    Wb.ensure((size_t)chunk * ng);
    ie.ensure(K.k);
    std::vector<double> inv(K.k);
    for (int j = 0; j < K.k; j++) inv[j] = 1.0 / K.eta[j];
    GPFVM_CUDA(cudaMemcpyAsync(ie.ptr, inv.data(), K.k * sizeof(double), cudaMemcpyHostToDevice, s));
    for (int j0 = 0; j0 < K.k; j0 += chunk) {
      int kc = std::min(chunk, K.k - j0);
      apply_cross(p, cp, K.d.ptr + (int64_t)j0 * p->N, p->N, Wb.ptr, ng, kc, 1.0, true, s);
      downdate_kernel<<<gs(ng), 256, 0, s>>>(var, Wb.ptr, ie.ptr + j0, kc, ng, j0 == 0, prior);
      count_launch();
    }
    return;
  }
  // PRECOND: slabs along grid dim 0 to bound the nb x slab workspace
  GPFVM_CHECK(d == 2, GPFVM_ERR_UNSUPPORTED, "GPFVM_COV_PRECOND: 2D problems only");
  const int64_t per_row = g.n[1];
  const int64_t nbv = p->pc ? std::max<int64_t>(1, p->pc->nb) : 1;
  // slab budget from free device memory (up to 48 GB): the first mode product
  // of the Schur part does not depend on the grid rows, so every extra slab
  // repeats it — one slab covers config 1's 512 x 1024 grid on a B200
  size_t free_b = 0, total_b = 0;
  GPFVM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  // from the device size (the same plan on every B200), then clamped to what
  // is free (fewer rows per slab rather than an out-of-memory failure);
  // GPFVM_PREDICT_SLAB_ROWS overrides (tests force the multi-slab path)
  const double budget = std::min(std::min(48e9, 0.3 * (double)total_b), 0.9 * (double)free_b);
  int rows = (int)std::max<int64_t>(1, std::min<int64_t>(g.n[0], (int64_t)(budget / 8 / (4 * nbv * per_row))));
  if (const char* e = getenv("GPFVM_PREDICT_SLAB_ROWS")) rows = std::max(1, std::min(g.n[0], atoi(e)));
  if (getenv("GPFVM_DEBUG"))
    fprintf(stderr, "[gpfvm] predict PRECOND: free %.1f GB, budget %.1f GB, %d rows per slab\n", free_b / 1e9,
            budget / 1e9, rows);
  for (int r0 = 0; r0 < g.n[0]; r0 += rows) {
    int rr = std::min(rows, g.n[0] - r0);
    CrossPlan cp;
    build_cross(p, g, r0, rr, cp, s);
    double* vslab = var + (int64_t)r0 * per_row;
    fill(vslab, prior, (int64_t)rr * per_row, s);
    var_precond_slab(p, cp, vslab, (int64_t)rr * per_row, s);
  }
}

}  // namespace gpfvm
