// Low-rank couplings of a 2D output block fused into one rank-rk update
// y = U V (see LowRank in problem.h).
#include "problem.h"

namespace gpfvm {

namespace {
unsigned gb(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096)); }

// fixed[m*P + p] = c * src[m]
__global__ void set_col_kernel(double* fixed, int P, int p, const double* __restrict__ src, int n, double c) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) fixed[(int64_t)m * P + p] = c * src[m];
}
// U[r][m][k0+p] = fixed[m][p]   (rk = row stride)
__global__ void bcast_cols_kernel(double* U, int R, int n0, int rk, int k0, int P, const double* __restrict__ fixed) {
  int64_t total = (int64_t)R * n0 * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int p = (int)(i % P);
    int64_t rm = i / P;
    int m = (int)(rm % n0);
    U[rm * rk + k0 + p] = fixed[(int64_t)m * P + p];
  }
}
// U[r][m][k0+p] = T[r][p][m]
__global__ void scatter_cols_kernel(double* U, const double* __restrict__ T, int R, int n0, int rk, int k0, int P) {
  int64_t total = (int64_t)R * P * n0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int m = (int)(i % n0);
    int64_t rp = i / n0;
    int p = (int)(rp % P);
    int64_t r = rp / P;
    U[(r * n0 + m) * rk + k0 + p] = T[i];
  }
}
// Vt[r][n][k0+p] = fixed[p][n]   (V stored transposed, row stride rk)
__global__ void bcast_vt_kernel(double* Vt, int R, int rk, int n1, int k0, int P, const double* __restrict__ fixed) {
  int64_t total = (int64_t)R * n1 * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int p = (int)(i % P);
    int64_t rn = i / P;
    int n = (int)(rn % n1);
    Vt[rn * rk + k0 + p] = fixed[(int64_t)p * n1 + n];
  }
}
__global__ void scaled_copy2(double* dst, const double* __restrict__ src, double c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = c * src[i];
}
}  // namespace

// y[r][a][i][b] = beta y[r][a][i][b] + sum_p U[i][p] W[r][p][a][b]   (P <= 16).
// blockIdx.y walks the (r, a) slabs (each ns*B contiguous doubles of y), the
// x-dimension the slab: coalesced y and W, 32-bit index math.  U (ns x P) is
// staged in shared memory once per CTA; for B = 1 (s = last dimension) the P
// values W[r][:][a] of a slab are broadcast from shared memory too.
__global__ void mode_update_kernel(double* __restrict__ y, int64_t ldy, const double* __restrict__ U,
                                   const double* __restrict__ W, int R, int A, int ns, int B, int P, double beta) {
  extern __shared__ double us[];  // [ns][P], then [P] slab values (B = 1)
  for (int k = threadIdx.x; k < ns * P; k += blockDim.x) us[k] = U[k];
  double* wsl = us + (size_t)ns * P;
  __syncthreads();
  const int slab = ns * B;
  const int64_t AB = (int64_t)A * B;
  for (int ra = blockIdx.y; ra < R * A; ra += gridDim.y) {
    const int r = ra / A, a = ra - r * A;
    double* yr = y + (int64_t)r * ldy + (int64_t)a * slab;
    const double* Wr = W + (int64_t)r * P * AB + (int64_t)a * B;
    if (B == 1) {
      __syncthreads();
      if (threadIdx.x < P) wsl[threadIdx.x] = Wr[(int64_t)threadIdx.x * AB];
      __syncthreads();
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < slab; e += gridDim.x * blockDim.x) {
      const int i = e / B, b = e - i * B;
      const double* Ui = us + (size_t)i * P;
      double acc = 0.0;
      if (B == 1) {
        for (int q = 0; q < P; q++) acc = fma(Ui[q], wsl[q], acc);
      } else {
        for (int q = 0; q < P; q++) acc = fma(Ui[q], __ldg(Wr + (int64_t)q * AB + b), acc);
      }
      yr[e] = (beta != 0.0) ? fma(beta, yr[e], acc) : acc;
    }
  }
}

int64_t ModeUpdate::workspace_per_rhs() const {
  int64_t w = 0;
  for (const auto& part : parts)
    for (const auto& k : part.ks) w = std::max(w, k.workspace_per_rhs());
  return w;
}

void ModeUpdate::prepare(const double* x, int64_t ldx, int R, const int64_t* block_off, double* w0, double* w1,
                         cudaStream_t st) const {
  const int64_t AB = (int64_t)A * B;
  for (const auto& part : parts)
    for (size_t q = 0; q < part.ks.size(); q++)
      part.ks[q].apply(x + block_off[part.J], ldx, W.ptr + (part.p0 + (int64_t)q) * AB, (int64_t)P * AB, R, 0.0, w0,
                       w1, st);
}

void ModeUpdate::apply(const double* x, int64_t ldx, double* y, int64_t ldy, int R, double beta,
                       const int64_t* block_off, double* w0, double* w1, cudaStream_t st) const {
  prepare(x, ldx, R, block_off, w0, w1, st);
  update(y, ldy, R, beta, st);
}

void ModeUpdate::update(double* y, int64_t ldy, int R, double beta, cudaStream_t st) const {
  const int slab = ns * B;
  const int bx = slab >= 256 ? 256 : 128;
  // ~16 CTAs per SM in total, split between slab chunks (x) and slabs (y)
  const int64_t nslab = (int64_t)R * A;
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((slab + bx - 1) / bx, (148 * 16 + nslab - 1) / nslab));
  const int64_t gy = std::min<int64_t>(nslab, std::max<int64_t>(1, 148 * 16 / gx));
  const size_t smem = sizeof(double) * ((size_t)ns * P + P);
  if (smem > 48 * 1024) {
    static bool attr = false;  // per process; the pencil sizes here are small
    if (!attr) {
      GPFVM_CUDA(cudaFuncSetAttribute(mode_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    GPFVM_CHECK(smem <= 200 * 1024, GPFVM_ERR_UNSUPPORTED, "mode update: ns * P too large");
  }
  mode_update_kernel<<<dim3((unsigned)gx, (unsigned)std::min<int64_t>(gy, 65535)), bx, smem, st>>>(
      y, ldy, U.ptr, W.ptr, R, A, ns, B, P, beta);
  count_launch();
}

// Mode updates of every d >= 3 output block (see ModeUpdate in problem.h).
static void build_modes(gpfvm_problem* p, MatvecPlan& pl, cudaStream_t s) {
  const int nb = (int)p->blocks.size(), d = p->ndim;
  pl.modes.clear();
  pl.modes.resize(nb);
  if (d < 3 || getenv("GPFVM_NO_MODEUPDATE")) return;
  for (int I = 0; I < nb; I++) {
    const BlockInt& BI = p->blocks[I];
    for (int k : pl.by_out[I]) {
      PairOp& op = pl.pairs[k];
      if (op.J == I) continue;
      const BlockInt& BJ = p->blocks[op.J];
      int sdim = -1, nsing = 0;
      for (int i = 0; i < d; i++)
        if (BJ.shape[i] == 1 && BI.shape[i] > 1) { sdim = i; nsing++; }
      if (nsing != 1) continue;
      std::vector<const KronTerm*> ts;
      for (const auto& t : p->terms)
        if (t.I == I && t.J == op.J) ts.push_back(&t);
      if (ts.empty()) continue;
      // find / create the mode-s update of this output block
      ModeUpdate* mu = nullptr;
      for (auto& m : pl.modes[I])
        if (m.s == sdim) mu = &m;
      if (!mu) {
        pl.modes[I].emplace_back();
        mu = &pl.modes[I].back();
        mu->s = sdim;
        mu->A = 1; mu->B = 1;
        for (int i = 0; i < sdim; i++) mu->A *= BI.shape[i];
        for (int i = sdim + 1; i < d; i++) mu->B *= BI.shape[i];
        mu->ns = BI.shape[sdim];
      }
      if (mu->P + (int)ts.size() > 16) continue;  // kernel bound: keep the plain pair
      ModeUpdate::Part part;
      part.J = op.J;
      part.p0 = mu->P;
      int in_r[GPFVM_MAX_DIMS], out_r[GPFVM_MAX_DIMS], dr = 0;
      for (int i = 0; i < d; i++)
        if (i != sdim) { in_r[dr] = BJ.shape[i]; out_r[dr] = BI.shape[i]; dr++; }
      for (const KronTerm* t : ts) {
        std::vector<std::vector<const double*>> fs(1);
        for (int i = 0; i < d; i++)
          if (i != sdim) fs[0].push_back(p->factors[t->fid[i]].data.ptr);
        part.ks.emplace_back();
        part.ks.back().build(dr, in_r, out_r, {1.0}, fs, s);
      }
      mu->P += (int)ts.size();
      mu->parts.push_back(std::move(part));
      op.lowrank = true;  // served by the mode update, skipped as a plain pair
    }
    // fixed columns U[:, p] = c_p F_s^p[:, 0]
    for (auto& m : pl.modes[I]) {
      m.U.ensure((size_t)m.ns * std::max(1, m.P));
      for (const auto& part : m.parts) {
        int q = 0;
        for (const auto& t : p->terms) {
          if (t.I != I || t.J != part.J) continue;
          set_col_kernel<<<gb(m.ns), 256, 0, s>>>(m.U.ptr, m.P, part.p0 + q, p->factors[t.fid[m.s]].data.ptr, m.ns,
                                                  t.coef);
          count_launch();
          q++;
        }
      }
    }
  }
  check_launch("build_modes");
}

// Append one coupling (input block J of shape shJ, thin in dim 0 or 1) to the
// rank-r update of a 2D output block of shape (lr.n0, lr.n1).
void add_lowrank_part(LowRank& lr, int J, const int* shJ, const std::vector<LowRankTerm>& ts, cudaStream_t s) {
  LowRank::Part part;
  part.J = J;
  part.type = (shJ[0] == 1) ? 0 : 1;
  part.k0 = lr.rk;
  part.nin = part.type == 0 ? shJ[1] : shJ[0];
  part.P = (int)ts.size();
  const int P = part.P;
  if (part.type == 0) {
    part.stk.ensure((size_t)P * lr.n1 * part.nin);
    part.fixed.ensure((size_t)lr.n0 * P);
    for (int q = 0; q < P; q++) {  // F0: n0 x 1, F1: n1 x n'_1
      scaled_copy2<<<gb((int64_t)lr.n1 * part.nin), 256, 0, s>>>(part.stk.ptr + (int64_t)q * lr.n1 * part.nin,
                                                                 ts[q].F1, 1.0, (int64_t)lr.n1 * part.nin);
      set_col_kernel<<<gb(lr.n0), 256, 0, s>>>(part.fixed.ptr, P, q, ts[q].F0, lr.n0, ts[q].coef);
      count_launch(2);
    }
  } else {
    part.stk.ensure((size_t)P * lr.n0 * part.nin);
    part.fixed.ensure((size_t)P * lr.n1);
    for (int q = 0; q < P; q++) {  // F0: n0 x n'_0, F1: n1 x 1
      scaled_copy2<<<gb((int64_t)lr.n0 * part.nin), 256, 0, s>>>(part.stk.ptr + (int64_t)q * lr.n0 * part.nin,
                                                                 ts[q].F0, ts[q].coef, (int64_t)lr.n0 * part.nin);
      scaled_copy2<<<gb(lr.n1), 256, 0, s>>>(part.fixed.ptr + (int64_t)q * lr.n1, ts[q].F1, 1.0, lr.n1);
      count_launch(2);
    }
  }
  lr.rk += P;
  lr.parts.push_back(std::move(part));
}

void LowRank::ensure(int Rn) {
  int pmax = 1;
  for (const auto& part : parts) pmax = std::max(pmax, part.P);
  const int kp = std::max(2, rkp());
  U.ensure((size_t)Rn * n0 * kp);
  V.ensure((size_t)Rn * n1 * kp);
  T.ensure((size_t)Rn * pmax * std::max(n0, n1));
}

// Mark and build the low-rank parts of every 2D output block (and the mode
// updates of d >= 3 output blocks).
void build_lowrank(gpfvm_problem* p, MatvecPlan& pl, cudaStream_t s) {
  const int nb = (int)p->blocks.size();
  pl.lowrank.clear();
  pl.lowrank.resize(nb);
  pl.block_off.resize(nb);
  for (int b = 0; b < nb; b++) pl.block_off[b] = p->blocks[b].offset;
  build_modes(p, pl, s);
  if (p->ndim != 2 || getenv("GPFVM_NO_LOWRANK")) return;
  for (int I = 0; I < nb; I++) {
    LowRank& lr = pl.lowrank[I];
    lr.n0 = p->blocks[I].shape[0];
    lr.n1 = p->blocks[I].shape[1];
    for (int k : pl.by_out[I]) {
      PairOp& op = pl.pairs[k];
      const BlockInt& BJ = p->blocks[op.J];
      if (op.J == I || !(BJ.shape[0] == 1 || BJ.shape[1] == 1)) continue;
      std::vector<const KronTerm*> ts;
      for (const auto& t : p->terms)
        if (t.I == I && t.J == op.J) ts.push_back(&t);
      if (ts.empty()) continue;
      std::vector<LowRankTerm> lt;
      for (const KronTerm* t : ts)
        lt.push_back({t->coef, p->factors[t->fid[0]].data.ptr, p->factors[t->fid[1]].data.ptr});
      add_lowrank_part(lr, op.J, BJ.shape, lt, s);
      op.lowrank = true;
    }
  }
  check_launch("build_lowrank");
}

void LowRank::prepare(const double* x, int64_t ldx, int Rn, const int64_t* block_off, cudaStream_t s) {
  const int kp = rkp();
  for (const Part& part : parts) {
    const double* xJ = x + block_off[part.J];
    const int P = part.P;
    Gemm g;
    g.M = Rn; g.K = part.nin;
    g.A = xJ; g.a_rs = ldx; g.a_cs = 1;
    g.B = part.stk.ptr; g.b_rs = 1; g.b_cs = part.nin;
    g.C = T.ptr; g.c_cs = 1;
    if (part.type == 0) {
      g.N = P * n1;  // T[r][p][:] = F1^p x_J  ->  Vt[r][:][k0+p]
      g.c_rs = (int64_t)P * n1;
      run_gemm(g, s);
      scatter_cols_kernel<<<gb((int64_t)Rn * P * n1), 256, 0, s>>>(V.ptr, T.ptr, Rn, n1, kp, part.k0, P);
      bcast_cols_kernel<<<gb((int64_t)Rn * n0 * P), 256, 0, s>>>(U.ptr, Rn, n0, kp, part.k0, P, part.fixed.ptr);
    } else {
      g.N = P * n0;  // T[r][p][:] = c_p F0^p x_J  ->  U[r][:][k0+p]
      g.c_rs = (int64_t)P * n0;
      run_gemm(g, s);
      scatter_cols_kernel<<<gb((int64_t)Rn * P * n0), 256, 0, s>>>(U.ptr, T.ptr, Rn, n0, kp, part.k0, P);
      bcast_vt_kernel<<<gb((int64_t)Rn * P * n1), 256, 0, s>>>(V.ptr, Rn, kp, n1, part.k0, P, part.fixed.ptr);
    }
    count_launch(2);
  }
  check_launch("LowRank::prepare");
}

void LowRank::as_extra(Gemm& g, int Rn) const {
  const int kp = rkp();
  g.K2 = rk;
  g.A2 = U.ptr; g.a2_rs = kp; g.a2_b1 = (int64_t)n0 * kp;
  g.B2 = V.ptr; g.b2_rs = kp; g.b2_b1 = (int64_t)n1 * kp;
  (void)Rn;
}

void LowRank::apply(const double* x, int64_t ldx, double* y, int64_t ldy, int Rn, double beta, const int64_t* block_off,
                    cudaStream_t s) {
  prepare(x, ldx, Rn, block_off, s);
  // y_r = beta y_r + U_r V_r^T   (n0 x rk) (rk x n1)
  const int kp = rkp();
  Gemm g;
  g.M = n0; g.N = n1; g.K = rk;
  g.A = U.ptr; g.a_rs = kp; g.a_cs = 1; g.a_b1 = (int64_t)n0 * kp;
  g.B = V.ptr; g.b_rs = 1; g.b_cs = kp; g.b_b1 = (int64_t)n1 * kp;
  g.C = y; g.c_rs = n1; g.c_cs = 1; g.c_b1 = ldy;
  g.batch1 = Rn;
  g.beta = beta;
  run_gemm(g, s);
  check_launch("LowRank::apply");
}

}  // namespace gpfvm
