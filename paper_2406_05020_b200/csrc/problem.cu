// C ABI: handle lifetime, factor assembly (§8 row 1) and the Kronecker Gram
// matvec (§8 row 2).  See include/gpfvm.h for the contract and DESIGN.md §4.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "problem.h"

namespace gpfvm {

static thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error{GPFVM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

bool is_device_ptr(const void* ptr) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return GPFVM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GPFVM_ERR_INVALID;
  }
}

static void upload_sites(Sites& s, cudaStream_t st) {
  s.d_lo.ensure(std::max(1, s.n));
  s.d_hi.ensure(std::max(1, s.n));
  if (s.n > 0) {
    GPFVM_CUDA(cudaMemcpyAsync(s.d_lo.ptr, s.lo.data(), s.n * sizeof(double), cudaMemcpyHostToDevice, st));
    GPFVM_CUDA(cudaMemcpyAsync(s.d_hi.ptr, s.hi.data(), s.n * sizeof(double), cudaMemcpyHostToDevice, st));
  }
}

static void copy_sites(Sites& dst, const gpfvm_sites1d& src, int q_max_order_check) {
  (void)q_max_order_check;
  GPFVM_CHECK(src.kind == GPFVM_SITE_POINT || src.kind == GPFVM_SITE_INTERVAL, GPFVM_ERR_INVALID, "bad site kind");
  GPFVM_CHECK(src.n >= 0, GPFVM_ERR_INVALID, "negative site count");
  GPFVM_CHECK(src.n == 0 || src.lo != nullptr, GPFVM_ERR_INVALID, "sites.lo is NULL");
  dst.kind = src.kind;
  dst.n = src.n;
  dst.lo.assign(src.lo, src.lo + src.n);
  if (src.kind == GPFVM_SITE_INTERVAL) {
    GPFVM_CHECK(src.n == 0 || src.hi != nullptr, GPFVM_ERR_INVALID, "sites.hi is NULL");
    dst.hi.assign(src.hi, src.hi + src.n);
    for (int j = 0; j < src.n; j++)
      GPFVM_CHECK(dst.lo[j] < dst.hi[j], GPFVM_ERR_INVALID, "interval with lo >= hi");
  } else {
    dst.hi = dst.lo;
  }
}

// Even-length site list invariant under the reflection x -> c - x about its
// centre (site i <-> site n-1-i), to 1e-14 of its extent.
static bool mirror_symmetric(const Sites& S) {
  if (S.n < 2 || S.n % 2) return false;
  const int n = S.n;
  const double c = S.lo[0] + S.hi[n - 1];
  const double tol = 1e-14 * (std::fabs(S.lo[0]) + std::fabs(S.hi[n - 1]) + (S.hi[n - 1] - S.lo[0]));
  for (int i = 0; i < n; i++)
    if (!(std::fabs(S.lo[i] + S.hi[n - 1 - i] - c) <= tol)) return false;
  return true;
}

int get_factor(gpfvm_problem* p, int out, int dim, int bl, int ml, int br, int mr) {
  FactorKey key{out, dim, bl, ml, br, mr};
  auto it = p->factor_index.find(key);
  if (it != p->factor_index.end()) return it->second;
  Factor f;
  f.rows = p->blocks[bl].sites[dim].n;
  f.cols = p->blocks[br].sites[dim].n;
  // a stationary kernel k(x - y) on one mirror-symmetric site list: the
  // reflection maps cell i to n-1-i and each derivative flips sign, so
  // F[n-1-i][n-1-j] = (-1)^(ml + mr) F[i][j]  (KronSum parity split)
  // (two blocks with the same site list, e.g. the PDE rows of a multi-output
  // system, share the property: the kernel depends on x - y only)
  const Sites& SL = p->blocks[bl].sites[dim];
  const Sites& SR = p->blocks[br].sites[dim];
  const bool same = bl == br || (SL.kind == SR.kind && SL.n == SR.n && SL.lo == SR.lo && SL.hi == SR.hi);
  if (same && mirror_symmetric(SL)) f.psign = ((ml + mr) & 1) ? -1 : 1;
  p->factors.push_back(std::move(f));
  int id = (int)p->factors.size() - 1;
  p->factor_index[key] = id;
  return id;
}

// Kronecker terms of all block pairs (Eq. 15/20 double sum), with the exact
// algebraic cancellation of DESIGN.md R6 on diagonal blocks: for tau != tau'
// the pair (tau', tau) equals prod_i s_i times the pair (tau, tau'),
// s_i = (-1)^(alpha_i + alpha'_i), so the two merge into one term with
// coefficient (1 + prod s_i) c c'.
static void build_terms(gpfvm_problem* p) {
  p->terms.clear();
  const int nb = (int)p->blocks.size();
  for (int I = 0; I < nb; I++)
    for (int J = 0; J < nb; J++) {
      const auto& TI = p->blocks[I].terms;
      const auto& TJ = p->blocks[J].terms;
      for (size_t a = 0; a < TI.size(); a++)
        for (size_t b = 0; b < TJ.size(); b++) {
          const gpfvm_term& t1 = TI[a];
          const gpfvm_term& t2 = TJ[b];
          if (t1.output != t2.output) continue;
          double coef = t1.coeff * t2.coeff;
          if (I == J && a != b) {
            if (b < a) continue;
            int par = 0;
            for (int i = 0; i < p->ndim; i++) par += t1.order[i] + t2.order[i];
            if (par & 1) continue;  // cancels against (b, a)
            coef *= 2.0;
          }
          if (coef == 0.0) continue;
          KronTerm kt;
          kt.I = I;
          kt.J = J;
          kt.coef = coef;
          for (int i = 0; i < p->ndim; i++) kt.fid[i] = get_factor(p, t1.output, i, I, t1.order[i], J, t2.order[i]);
          p->terms.push_back(kt);
        }
    }
}

double term_flops(const gpfvm_problem* p, const KronTerm& t, const int* in_shape, const int* out_shape) {
  (void)p;
  (void)t;
  double fl = 0.0;
  const int d = p->ndim;
  for (int i = d - 1; i >= 0; i--) {
    double outer = 1, inner = 1;
    for (int k = 0; k < i; k++) outer *= in_shape[k];
    for (int k = i + 1; k < d; k++) inner *= out_shape[k];
    fl += 2.0 * outer * inner * in_shape[i] * (double)out_shape[i];
  }
  return fl;
}

void apply_terms(gpfvm_problem* p, const std::vector<Factor>& factors, const std::vector<const KronTerm*>& terms, const int* in_shape,
                 const int* out_shape, const double* x, int64_t ldx, double* y, int64_t ldy, int R,
                 bool overwrite, cudaStream_t s, Workspace& ws) {
  const int d = p->ndim;
  // temp sizes: per vector, after stage i (dims i..d-1 converted)
  int64_t maxsz = 0;
  for (int i = d - 1; i >= 1; i--) {
    int64_t sz = 1;
    for (int k = 0; k < i; k++) sz *= in_shape[k];
    for (int k = i; k < d; k++) sz *= out_shape[k];
    maxsz = std::max(maxsz, sz);
  }
  if (d > 1) {
    ws.t0.ensure((size_t)maxsz * R);
    ws.t1.ensure((size_t)maxsz * R);
  }
  bool first_term = true;
  for (const KronTerm* t : terms) {
    const double* cur = x;
    int64_t cur_ld = ldx;
    for (int i = d - 1; i >= 0; i--) {
      const Factor& F = factors[t->fid[i]];
      int64_t outer = 1, inner = 1;
      for (int k = 0; k < i; k++) outer *= in_shape[k];
      for (int k = i + 1; k < d; k++) inner *= out_shape[k];
      const int nin = in_shape[i], nout = out_shape[i];
      double* dst;
      int64_t dst_ld;
      double alpha = 1.0, beta = 0.0;
      if (i == 0) {
        dst = y;
        dst_ld = ldy;
        alpha = t->coef;
        beta = (overwrite && first_term) ? 0.0 : 1.0;
      } else {
        dst = ((d - 1 - i) % 2 == 0) ? ws.t0.ptr : ws.t1.ptr;
        dst_ld = outer * nout * inner;
      }
      Gemm g;
      g.alpha = alpha;
      g.beta = beta;
      if (inner == 1) {
        // Y (outer x nout) = X (outer x nin) F^T
        g.M = (int)outer; g.N = nout; g.K = nin;
        g.A = cur; g.a_rs = nin; g.a_cs = 1; g.a_b1 = cur_ld;
        g.B = F.data.ptr; g.b_rs = 1; g.b_cs = nin; g.b_b1 = 0;
        g.C = dst; g.c_rs = nout; g.c_cs = 1; g.c_b1 = dst_ld;
        g.batch1 = R; g.batch2 = 1;
      } else {
        // per (rhs, o): Y_o (nout x inner) = F (nout x nin) X_o (nin x inner)
        g.M = nout; g.N = (int)inner; g.K = nin;
        g.A = F.data.ptr; g.a_rs = nin; g.a_cs = 1; g.a_b1 = 0; g.a_b2 = 0;
        g.B = cur; g.b_rs = inner; g.b_cs = 1; g.b_b1 = (int64_t)nin * inner; g.b_b2 = cur_ld;
        g.C = dst; g.c_rs = inner; g.c_cs = 1; g.c_b1 = (int64_t)nout * inner; g.c_b2 = dst_ld;
        g.batch1 = (int)outer; g.batch2 = R;
      }
      run_gemm(g, s);
      cur = dst;
      cur_ld = dst_ld;
    }
    first_term = false;
  }
  if (overwrite && first_term) {
    // no terms: zero the output
    int64_t osz = 1;
    for (int k = 0; k < d; k++) osz *= out_shape[k];
    for (int r = 0; r < R; r++) fill(y + r * ldy, 0.0, osz, s);
  }
}

MatvecPlan::~MatvecPlan() {
  release_graphs();
  for (auto st : branch) cudaStreamDestroy(st);
  if (cap) cudaStreamDestroy(cap);
  for (auto e : ev) cudaEventDestroy(e);
  for (auto& ff : fused)
    if (ff.ev) cudaEventDestroy(ff.ev);
  for (auto st : side)
    if (st) cudaStreamDestroy(st);
  for (auto e : side_fork)
    if (e) cudaEventDestroy(e);
  for (auto e : side_ready)
    if (e) cudaEventDestroy(e);
  for (auto& lr : lowrank) {
    if (lr.side) cudaStreamDestroy(lr.side);
    if (lr.ev_fork) cudaEventDestroy(lr.ev_fork);
    if (lr.ev_ready) cudaEventDestroy(lr.ev_ready);
  }
}

void MatvecPlan::release_graphs() {
  for (auto& g : graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  graphs.clear();
}

// One KronSum per nonzero block pair (built after the factors exist).
void build_plan(gpfvm_problem* p, cudaStream_t s) {
  if (p->plan) {
    // re-assembly of the same problem: refresh the stacked factors in place
    // (same shapes -> same buffers), so captured matvec graphs stay valid
    for (auto& op : p->plan->pairs) {
      std::vector<double> coefs;
      std::vector<std::vector<const double*>> fs;
      std::vector<std::vector<int>> sgn;
      for (const auto& t : p->terms) {
        if (t.I != op.I || t.J != op.J) continue;
        coefs.push_back(t.coef);
        std::vector<const double*> f;
        std::vector<int> sv;
        for (int i = 0; i < p->ndim; i++) {
          f.push_back(p->factors[t.fid[i]].data.ptr);
          sv.push_back(p->factors[t.fid[i]].psign);
        }
        fs.push_back(f);
        sgn.push_back(sv);
      }
      op.ks.build(p->ndim, p->blocks[op.J].shape, p->blocks[op.I].shape, coefs, fs, s, &sgn);
    }
    refresh_fused_func(*p->plan, s);
    return;
  }
  auto plan = std::make_unique<MatvecPlan>();
  const int nb = (int)p->blocks.size();
  plan->by_out.assign(nb, {});
  for (int I = 0; I < nb; I++)
    for (int J = 0; J < nb; J++) {
      std::vector<double> coefs;
      std::vector<std::vector<const double*>> fs;
      std::vector<std::vector<int>> sgn;
      for (const auto& t : p->terms) {
        if (t.I != I || t.J != J) continue;
        coefs.push_back(t.coef);
        std::vector<const double*> f;
        std::vector<int> sv;
        for (int i = 0; i < p->ndim; i++) {
          f.push_back(p->factors[t.fid[i]].data.ptr);
          sv.push_back(p->factors[t.fid[i]].psign);
        }
        fs.push_back(f);
        sgn.push_back(sv);
      }
      if (coefs.empty()) continue;
      PairOp op;
      op.I = I;
      op.J = J;
      op.ks.build(p->ndim, p->blocks[J].shape, p->blocks[I].shape, coefs, fs, s, &sgn);
      plan->flops_per_rhs += op.ks.flops_per_rhs();
      plan->by_out[I].push_back((int)plan->pairs.size());
      plan->pairs.push_back(std::move(op));
    }
  plan->w0.resize(nb);
  plan->w1.resize(nb);
  build_lowrank(p, *plan, s);
  build_fused_func(p, *plan, s);
  // executed flops per right-hand side: plain pairs + low-rank / mode updates
  plan->flops_per_rhs = 0.0;
  plan->flops_split_saved = 0.0;
  for (const auto& op : plan->pairs)
    if (!op.lowrank) {
      plan->flops_per_rhs += op.ks.flops_per_rhs();
      // a parity-split pair executes exactly half the flops of its unsplit plan
      if (op.ks.par || op.ks.par3) plan->flops_split_saved += op.ks.flops_per_rhs();
    }
  for (const auto& lr : plan->lowrank) {
    for (const auto& part : lr.parts)
      plan->flops_per_rhs += 2.0 * part.nin * part.P * (part.type == 0 ? lr.n1 : lr.n0);
    plan->flops_per_rhs += 2.0 * lr.n0 * lr.n1 * lr.rk;
  }
  for (const auto& ms : plan->modes)
    for (const auto& mu : ms) {
      for (const auto& part : mu.parts)
        for (const auto& k : part.ks) plan->flops_per_rhs += k.flops_per_rhs();
      plan->flops_per_rhs += 2.0 * mu.A * mu.ns * mu.B * mu.P;
    }
  p->plan = std::move(plan);
}

static int only_branch() {
  static const int only = getenv("GPFVM_TIMING_ONLY_BRANCH") ? atoi(getenv("GPFVM_TIMING_ONLY_BRANCH")) : -1;
  return only;
}

// the block's mode updates can ride on its own 3D parity-split Kronecker sum
static bool mode_fusable(const MatvecPlan& pl, int I, const PairOp* diag) {
  static const bool off = getenv("GPFVM_NO_MODEFUSE") != nullptr;
  if (off || !diag || !diag->ks.par3) return false;
  int n = 0;
  for (const auto& mu : pl.modes[I]) n += mu.P > 0;
  return n >= 1 && n <= 3;
}

static void matvec_branch(gpfvm_problem* p, int I, const double* x, double* y, int nrhs, int64_t ld, cudaStream_t s) {
  MatvecPlan& pl = *p->plan;
  const int only = only_branch();
  if (only >= 0 && I != only) return;  // timing experiments only: wrong results
  const BlockInt& B = p->blocks[I];
  // noise-free block: the first pair overwrites (beta = 0), saving one read-modify-write pass
  bool overwrite = (B.noise == 0.0) && !pl.by_out[I].empty();
  if (!overwrite) vec_scale_add(y + B.offset, x + B.offset, p->noise.ptr + B.offset, B.size, nrhs, ld, s);
  LowRank& lr = pl.lowrank[I];
  // the rank-rk IC/BC coupling update is fused into the last contraction of
  // the block's own (diagonal) Kronecker sum when there is one
  const PairOp* diag = nullptr;
  for (int k : pl.by_out[I])
    if (pl.pairs[k].J == I && !pl.pairs[k].lowrank) diag = &pl.pairs[k];
  static const bool no_fuse = getenv("GPFVM_NO_LRFUSE") != nullptr;
  Gemm lr_extra;
  cudaEvent_t lr_ready = nullptr;
  if (lr.rk > 0) {
    if (diag && !no_fuse) {
      // parity-split Kronecker sum: U, V are read only by its last kernel, so
      // they are prepared on a side stream beside the two mode products
      static const bool no_fork = getenv("GPFVM_NO_LRFORK") != nullptr;
      if (diag->ks.par && !no_fork) {
        if (!lr.side) {
          int lo = 0, hi = 0;
          GPFVM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
          GPFVM_CUDA(cudaStreamCreateWithPriority(&lr.side, cudaStreamNonBlocking, lo));
          GPFVM_CUDA(cudaEventCreateWithFlags(&lr.ev_fork, cudaEventDisableTiming));
          GPFVM_CUDA(cudaEventCreateWithFlags(&lr.ev_ready, cudaEventDisableTiming));
        }
        if (!pl.serial_now) {
          GPFVM_CUDA(cudaEventRecord(lr.ev_fork, s));
          GPFVM_CUDA(cudaStreamWaitEvent(lr.side, lr.ev_fork, 0));
          lr.prepare(x, ld, nrhs, pl.block_off.data(), lr.side);
          GPFVM_CUDA(cudaEventRecord(lr.ev_ready, lr.side));
          lr_ready = lr.ev_ready;
        } else {
          lr.prepare(x, ld, nrhs, pl.block_off.data(), s);
        }
      } else {
        lr.prepare(x, ld, nrhs, pl.block_off.data(), s);
      }
      lr.as_extra(lr_extra, nrhs);
    } else {
      lr.apply(x, ld, y + B.offset, ld, nrhs, overwrite ? 0.0 : 1.0, pl.block_off.data(), s);
      overwrite = false;
    }
  }
  // 3D parity-split diagonal pair: the mode-s updates (IC planes, faces) are
  // added by its last kernel in the pass that writes y; their operands W are
  // prepared on a side stream beside the mode products
  ModeTerms mt;
  const bool fuse_modes = mode_fusable(pl, I, diag);
  if (fuse_modes) {
    if (pl.side.empty()) {
      pl.side.assign(p->blocks.size(), nullptr);
      pl.side_fork.assign(p->blocks.size(), nullptr);
      pl.side_ready.assign(p->blocks.size(), nullptr);
    }
    if (!pl.side[I]) {
      int lo = 0, hi = 0;
      GPFVM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      GPFVM_CUDA(cudaStreamCreateWithPriority(&pl.side[I], cudaStreamNonBlocking, lo));
      GPFVM_CUDA(cudaEventCreateWithFlags(&pl.side_fork[I], cudaEventDisableTiming));
      GPFVM_CUDA(cudaEventCreateWithFlags(&pl.side_ready[I], cudaEventDisableTiming));
    }
    static const bool noside = getenv("GPFVM_MODE_NOSIDE") != nullptr;
    const bool fork = !noside && !pl.serial_now;
    cudaStream_t ps = fork ? pl.side[I] : s;
    if (fork) {
      GPFVM_CUDA(cudaEventRecord(pl.side_fork[I], s));
      GPFVM_CUDA(cudaStreamWaitEvent(pl.side[I], pl.side_fork[I], 0));
    }
    for (const auto& mu : pl.modes[I]) {
      if (mu.P == 0) continue;
      mu.prepare(x, ld, nrhs, pl.block_off.data(), mu.mw0.ptr, mu.mw1.ptr, ps);
      mt.m[mt.n++] = {mu.U.ptr, mu.W.ptr, mu.P, mu.s};
    }
    if (fork) GPFVM_CUDA(cudaEventRecord(pl.side_ready[I], pl.side[I]));
    diag->ks.apply(x + B.offset, ld, y + B.offset, ld, nrhs, overwrite ? 0.0 : 1.0, pl.w0[I].ptr, pl.w1[I].ptr, s, nullptr,
                   fork ? pl.side_ready[I] : nullptr, nullptr, &mt);
    overwrite = false;
  } else {
    for (const auto& mu : pl.modes[I]) {
      if (mu.P == 0) continue;
      mu.apply(x, ld, y + B.offset, ld, nrhs, overwrite ? 0.0 : 1.0, pl.block_off.data(), pl.w0[I].ptr, pl.w1[I].ptr, s);
      overwrite = false;
    }
  }
  for (int k : pl.by_out[I]) {
    const PairOp& op = pl.pairs[k];
    if (op.lowrank || (fuse_modes && &op == diag)) continue;
    const double* stage0 = nullptr;
    if (pl.fused_on && pl.fused_of[k] >= 0) {
      const FusedFunc& ff = pl.fused[pl.fused_of[k]];
      GPFVM_CUDA(cudaStreamWaitEvent(s, ff.ev, 0));
      stage0 = ff.stage0_of(k, nrhs);
    }
    op.ks.apply(x + p->blocks[op.J].offset, ld, y + B.offset, ld, nrhs, overwrite ? 0.0 : 1.0, pl.w0[I].ptr,
                pl.w1[I].ptr, s, (&op == diag && lr_extra.K2 > 0) ? &lr_extra : nullptr,
                (&op == diag && lr_extra.K2 > 0) ? lr_ready : nullptr, stage0);
    overwrite = false;
  }
}

static void ensure_plan_workspace(gpfvm_problem* p, int nrhs) {
  MatvecPlan& pl = *p->plan;
  for (size_t I = 0; I < pl.by_out.size(); I++) {
    int64_t need = 0;
    for (int k : pl.by_out[I]) need = std::max(need, pl.pairs[k].ks.workspace_per_rhs());
    for (auto& mu : pl.modes[I]) {
      need = std::max(need, mu.workspace_per_rhs());
      const size_t nw = (size_t)nrhs * std::max(1, mu.P) * mu.A * mu.B;
      const size_t nm = (size_t)std::max<int64_t>(1, mu.workspace_per_rhs() * nrhs);
      if (mu.W.n < nw || mu.mw0.n < nm) {
        pl.release_graphs();
        mu.W.ensure(nw);
        mu.mw0.ensure(nm);
        mu.mw1.ensure(nm);
      }
    }
    size_t n = (size_t)std::max<int64_t>(1, need * nrhs);
    if (pl.w0[I].n < n) {
      pl.release_graphs();  // captured graphs reference the old buffers
      pl.w0[I].ensure(n);
      pl.w1[I].ensure(n);
    }
    if (I == 0)
      for (auto& ff : pl.fused) {
        const size_t nz = (size_t)ff.zper * nrhs, nc = (size_t)nrhs * ff.tiles() * 4 * ff.n1;
        if (ff.zbuf.n < nz || ff.colpart.n < nc) {
          pl.release_graphs();
          ff.ensure(nrhs);
        }
      }
    LowRank& lr = pl.lowrank[I];
    if (lr.rk > 0) {
      int pmax = 1;
      for (const auto& part : lr.parts) pmax = std::max(pmax, part.P);
      const size_t kp = std::max(2, lr.rkp());
      size_t nu = (size_t)nrhs * lr.n0 * kp, nv = (size_t)nrhs * lr.n1 * kp,
             nt = (size_t)nrhs * pmax * std::max(lr.n0, lr.n1);
      if (lr.U.n < nu || lr.V.n < nv || lr.T.n < nt) {
        pl.release_graphs();
        lr.U.ensure(nu);
        lr.V.ensure(nv);
        lr.T.ensure(nt);
      }
    }
  }
}

// Y = G X (+ Sigma X).  Direct launch the first time a (x, y, nrhs, ld) key is
// seen; from the second time on the whole matvec is a CUDA graph (one branch
// per output block, joined) replayed on `s`.
void matvec_device(gpfvm_problem* p, const double* x, double* y, int nrhs, int64_t ld, cudaStream_t s) {
  GPFVM_CHECK(p->assembled && p->plan, GPFVM_ERR_STATE, "gpfvm_gram_matvec: call gpfvm_assemble_factors first");
  MatvecPlan& pl = *p->plan;
  ensure_plan_workspace(p, nrhs);
  const int nb = (int)p->blocks.size();
  static const bool no_graph = getenv("GPFVM_NO_GRAPH") != nullptr;
  MatvecPlan::G* hit = nullptr;
  for (auto& g : pl.graphs)
    if (g.x == x && g.y == y && g.nrhs == nrhs && g.ld == ld) hit = &g;
  if (hit && hit->exec) {
    GPFVM_CUDA(cudaGraphLaunch(hit->exec, s));
    count_launch(hit->nodes);
    return;
  }
  if (!pl.cap) {
    GPFVM_CUDA(cudaStreamCreateWithFlags(&pl.cap, cudaStreamNonBlocking));
    pl.branch.resize(nb);
    // The heaviest output block (the PDE-PDE mode products) gets the highest
    // stream priority: its GEMM waves take the SMs first and the light IC/BC
    // branches fill the gaps instead of competing for every wave.
    int lo = 0, hi = 0;
    GPFVM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    static const bool no_prio = getenv("GPFVM_NO_PRIO") != nullptr;
    int heavy = 0;
    double best = -1.0;
    for (int I = 0; I < nb; I++) {
      double f = 0.0;
      for (int k : pl.by_out[I]) f += pl.pairs[k].ks.flops_per_rhs();
      if (f > best) { best = f; heavy = I; }
    }
    for (int I = 0; I < nb; I++)
      GPFVM_CUDA(cudaStreamCreateWithPriority(&pl.branch[I], cudaStreamNonBlocking, (!no_prio && I == heavy) ? hi : lo));
    pl.ev.resize(nb + 1);
    for (auto& e : pl.ev) GPFVM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // one branch per output block on its own stream, forked from and joined
  // into `s` (direct launch) or the capture stream (graph)
  // the fused functional passes need 16-byte aligned rows of x
  pl.fused_on = !pl.fused.empty() && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (ld & 1) == 0 && only_branch() < 0 &&
                (int64_t)nrhs * pl.fused[0].tiles() >= 64;  // few vectors: too few CTAs for one pass to pay
  auto run_branches = [&](cudaStream_t origin, bool serial) {
    pl.serial_now = serial;
    if (serial) {
      // every branch on the caller's stream, one kernel at a time
      if (pl.fused_on)
        for (auto& ff : pl.fused) {
          ff.run(x + p->blocks[ff.J].offset, ld, nrhs, origin);
          GPFVM_CUDA(cudaEventRecord(ff.ev, origin));
        }
      for (int I = 0; I < nb; I++) matvec_branch(p, I, x, y, nrhs, ld, origin);
      return;
    }
    GPFVM_CUDA(cudaEventRecord(pl.ev[nb], origin));
    std::vector<char> waited(nb, 0);
    if (pl.fused_on)
      for (auto& ff : pl.fused) {
        // first on the input block's own branch stream (measured: 1.024 ms against
        // 1.052 ms on a consumer's stream beside the parity transform); the
        // consumers wait on ff.ev
        const int sb = ff.J;
        cudaStream_t fs = pl.branch[sb];
        if (!waited[sb]) GPFVM_CUDA(cudaStreamWaitEvent(fs, pl.ev[nb], 0));
        waited[sb] = 1;
        ff.run(x + p->blocks[ff.J].offset, ld, nrhs, fs);
        GPFVM_CUDA(cudaEventRecord(ff.ev, fs));
      }
    for (int I = 0; I < nb; I++) {
      if (!waited[I]) GPFVM_CUDA(cudaStreamWaitEvent(pl.branch[I], pl.ev[nb], 0));
      matvec_branch(p, I, x, y, nrhs, ld, pl.branch[I]);
      GPFVM_CUDA(cudaEventRecord(pl.ev[I], pl.branch[I]));
      GPFVM_CUDA(cudaStreamWaitEvent(origin, pl.ev[I], 0));
    }
  };
  if (no_graph || !hit) {
    if (!no_graph) {
      if (pl.graphs.size() >= 16) {
        if (pl.graphs.front().exec) cudaGraphExecDestroy(pl.graphs.front().exec);
        pl.graphs.erase(pl.graphs.begin());
      }
      pl.graphs.push_back({x, y, nrhs, ld, nullptr, 0, 1});
    }
    // Direct launches (first sighting of a key, GPFVM_NO_GRAPH) run serially on
    // the caller's stream: the cold first call of a process is where kernels
    // of different branches overlapped in ever-changing ways and the TMA GEMM
    // was seen to produce wrong tiles; the concurrent schedule is
    // the captured graph's.  GPFVM_DIRECT_CONCURRENT restores branch streams.
    static const bool direct_conc = getenv("GPFVM_DIRECT_CONCURRENT") != nullptr;
    run_branches(s, !direct_conc);
    return;
  }
  // second sighting: capture
  const int64_t l0 = g_launches.load();
  cudaGraph_t graph;
  GPFVM_CUDA(cudaStreamBeginCapture(pl.cap, cudaStreamCaptureModeThreadLocal));
  try {
    run_branches(pl.cap, false);
  } catch (...) {
    cudaStreamEndCapture(pl.cap, &graph);
    throw;
  }
  GPFVM_CUDA(cudaStreamEndCapture(pl.cap, &graph));
  cudaGraphExec_t exec;
  GPFVM_CUDA(cudaGraphInstantiate(&exec, graph, cudaGraphInstantiateFlagUseNodePriority));
  cudaGraphDestroy(graph);
  const int64_t nodes = g_launches.load() - l0;
  g_launches.fetch_sub(nodes);
  hit->exec = exec;
  hit->nodes = nodes;
  GPFVM_CUDA(cudaGraphLaunch(exec, s));
  count_launch(nodes);
}

}  // namespace gpfvm

using namespace gpfvm;

gpfvm_problem::~gpfvm_problem() {
  destroy_precond(pc);
  plan.reset();
  for (auto st : pipe)
    if (st) cudaStreamDestroy(st);
}

extern "C" {

const char* gpfvm_last_error(void) { return g_err.c_str(); }
const char* gpfvm_version(void) { return "gpfvm 0.1 (sm_100a, FP64 DMMA)"; }
int64_t gpfvm_launch_count(void) { return g_launches.load(); }

int gpfvm_problem_create(const gpfvm_problem_desc* desc, int device, gpfvm_problem** out) {
  return guarded([&] {
    GPFVM_CHECK(desc && out, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(desc->ndim >= 1 && desc->ndim <= GPFVM_MAX_DIMS, GPFVM_ERR_INVALID, "ndim out of range");
    GPFVM_CHECK(desc->n_outputs >= 1, GPFVM_ERR_INVALID, "n_outputs < 1");
    GPFVM_CHECK(desc->n_blocks >= 1 && desc->blocks, GPFVM_ERR_INVALID, "no blocks");
    GPFVM_CHECK(desc->kernels != nullptr, GPFVM_ERR_INVALID, "kernels is NULL");
    auto p = std::make_unique<gpfvm_problem>();
    p->device = device;
    p->ndim = desc->ndim;
    p->nout = desc->n_outputs;
    p->kernels.assign(desc->kernels, desc->kernels + desc->ndim * desc->n_outputs);
    for (const auto& k : p->kernels) {
      GPFVM_CHECK(k.q >= 0 && k.q <= 3, GPFVM_ERR_UNSUPPORTED, "Matérn q must be in [0,3]");
      GPFVM_CHECK(k.lengthscale > 0 && k.variance > 0, GPFVM_ERR_INVALID, "lengthscale/variance must be > 0");
    }
    int64_t off = 0;
    p->blocks.resize(desc->n_blocks);
    for (int b = 0; b < desc->n_blocks; b++) {
      const gpfvm_block& src = desc->blocks[b];
      BlockInt& B = p->blocks[b];
      GPFVM_CHECK(src.n_terms >= 1 && src.n_terms <= GPFVM_MAX_TERMS, GPFVM_ERR_INVALID, "block needs 1..16 terms");
      GPFVM_CHECK(src.noise >= 0.0, GPFVM_ERR_INVALID, "negative noise");
      B.size = 1;
      for (int i = 0; i < desc->ndim; i++) {
        copy_sites(B.sites[i], src.sites[i], 0);
        B.shape[i] = B.sites[i].n;
        B.size *= B.sites[i].n;
      }
      for (int t = 0; t < src.n_terms; t++) {
        const gpfvm_term& tm = src.terms[t];
        GPFVM_CHECK(tm.output >= 0 && tm.output < desc->n_outputs, GPFVM_ERR_INVALID, "term output out of range");
        for (int i = 0; i < desc->ndim; i++) {
          int q = p->kernels[tm.output * desc->ndim + i].q;
          int m = tm.order[i];
          GPFVM_CHECK(m >= 0, GPFVM_ERR_INVALID, "negative derivative order");
          int o = (B.sites[i].kind == GPFVM_SITE_POINT) ? m : m - 1;
          GPFVM_CHECK(o <= q, GPFVM_ERR_INVALID,
                      "derivative order exceeds kernel smoothness (point order <= q, interval order <= q+1)");
        }
        B.terms.push_back(tm);
      }
      B.noise = src.noise;
      B.deflate = src.deflate;
      B.offset = off;
      off += B.size;
    }
    p->N = off;
    build_terms(p.get());
    *out = p.release();
  });
}

int gpfvm_problem_destroy(gpfvm_problem* p) {
  return guarded([&] {
    if (!p) return;
    cudaSetDevice(p->device);
    delete p;
    pool_trim();
  });
}

int64_t gpfvm_problem_size(const gpfvm_problem* p) { return p ? p->N : -1; }

int gpfvm_assemble_factors(gpfvm_problem* p, void* stream) {
  return guarded([&] {
    GPFVM_CHECK(p, GPFVM_ERR_INVALID, "null problem");
    GPFVM_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = (cudaStream_t)stream;
    for (auto& B : p->blocks)
      for (int i = 0; i < p->ndim; i++) upload_sites(B.sites[i], s);
    for (const auto& kv : p->factor_index) {
      int out, dim, bl, ml, br, mr;
      std::tie(out, dim, bl, ml, br, mr) = kv.first;
      Factor& F = p->factors[kv.second];
      F.data.ensure((size_t)std::max(1, F.rows * F.cols));
      const gpfvm_kernel1d& k = p->kernels[out * p->ndim + dim];
      MaternDD K = matern_dd(k.q, k.lengthscale, k.variance);
      launch_factor(K, p->blocks[bl].sites[dim], ml, p->blocks[br].sites[dim], mr, F.data.ptr, F.cols, s);
    }
    p->noise.ensure(std::max<int64_t>(1, p->N));
    for (const auto& B : p->blocks) fill(p->noise.ptr + B.offset, B.noise, B.size, s);
    build_plan(p, s);
    p->assembled = true;
    destroy_precond(p->pc);  // factors changed: rebuild lazily
    p->pc = nullptr;
    GPFVM_CUDA(cudaStreamSynchronize(s));
  });
}

int gpfvm_factor_matrix(const gpfvm_kernel1d* k, const gpfvm_sites1d* left, int m_left, const gpfvm_sites1d* right,
                        int m_right, double* out, int64_t ld, void* stream) {
  return guarded([&] {
    GPFVM_CHECK(k && left && right && out, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(k->q >= 0 && k->q <= 3, GPFVM_ERR_UNSUPPORTED, "Matérn q must be in [0,3]");
    GPFVM_CHECK(ld >= right->n, GPFVM_ERR_INVALID, "ld < right->n");
    cudaStream_t s = (cudaStream_t)stream;
    Sites L, R;
    copy_sites(L, *left, 0);
    copy_sites(R, *right, 0);
    int oL = (L.kind == GPFVM_SITE_POINT) ? m_left : m_left - 1;
    int oR = (R.kind == GPFVM_SITE_POINT) ? m_right : m_right - 1;
    GPFVM_CHECK(m_left >= 0 && m_right >= 0 && oL <= k->q && oR <= k->q, GPFVM_ERR_INVALID,
                "derivative order exceeds kernel smoothness");
    upload_sites(L, s);
    upload_sites(R, s);
    launch_factor(matern_dd(k->q, k->lengthscale, k->variance), L, m_left, R, m_right, out, ld, s);
    GPFVM_CUDA(cudaStreamSynchronize(s));
  });
}

int gpfvm_gram_matvec(gpfvm_problem* p, const double* x, double* y, int nrhs, int64_t ld, void* stream) {
  return guarded([&] {
    GPFVM_CHECK(p && x && y, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(nrhs >= 1 && ld >= p->N, GPFVM_ERR_INVALID, "nrhs < 1 or ld < N");
    GPFVM_CHECK(x != y, GPFVM_ERR_INVALID, "x and y must not alias");
    GPFVM_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = (cudaStream_t)stream;
    const bool dx = is_device_ptr(x), dy = is_device_ptr(y);
    const double* xd = x;
    double* yd = y;
    size_t n = (size_t)ld * (nrhs - 1) + p->N;
    if (!dx && !dy && nrhs >= 8) {
      // host -> device -> host pipeline over RHS chunks on three internal
      // streams: H2D of chunk c+1 and D2H of chunk c-1 overlap the matvec of c
      GPFVM_CHECK(p->assembled && p->plan, GPFVM_ERR_STATE, "gpfvm_gram_matvec: call gpfvm_assemble_factors first");
      if (!p->pipe[0])
        for (int i = 0; i < 3; i++) GPFVM_CUDA(cudaStreamCreateWithFlags(&p->pipe[i], cudaStreamNonBlocking));
      // enough chunks that the pipeline tail (last compute + last D2H) is short;
      // each chunk keeps >= 8 vectors so the DMMA GEMMs stay efficient
      static const int nch_env = getenv("GPFVM_PIPE_CHUNKS") ? atoi(getenv("GPFVM_PIPE_CHUNKS")) : 0;
      const int nch = nch_env > 0 ? nch_env : std::max(1, std::min(8, nrhs / 8)), csz = (nrhs + nch - 1) / nch;
      p->stage_in.ensure(n);
      p->stage_out.ensure(n);
      std::vector<cudaEvent_t> evs(2 * nch + 1);
      for (auto& e : evs) GPFVM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      GPFVM_CUDA(cudaEventRecord(evs[2 * nch], s));  // prior work on the caller's stream (assembly)
      for (int i = 0; i < 3; i++) GPFVM_CUDA(cudaStreamWaitEvent(p->pipe[i], evs[2 * nch], 0));
      for (int c = 0; c < nch; c++) {
        const int r0 = c * csz, rc = std::min(csz, nrhs - r0);
        if (rc <= 0) break;
        const size_t off = (size_t)r0 * ld, cnt = (size_t)ld * (rc - 1) + p->N;
        GPFVM_CUDA(cudaMemcpyAsync(p->stage_in.ptr + off, x + off, cnt * sizeof(double), cudaMemcpyHostToDevice,
                                   p->pipe[0]));
        GPFVM_CUDA(cudaEventRecord(evs[c], p->pipe[0]));
        GPFVM_CUDA(cudaStreamWaitEvent(p->pipe[1], evs[c], 0));
        matvec_device(p, p->stage_in.ptr + off, p->stage_out.ptr + off, rc, ld, p->pipe[1]);
        GPFVM_CUDA(cudaEventRecord(evs[nch + c], p->pipe[1]));
        GPFVM_CUDA(cudaStreamWaitEvent(p->pipe[2], evs[nch + c], 0));
        GPFVM_CUDA(cudaMemcpyAsync(y + off, p->stage_out.ptr + off, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                   p->pipe[2]));
      }
      GPFVM_CUDA(cudaStreamSynchronize(p->pipe[2]));
      GPFVM_CUDA(cudaStreamSynchronize(p->pipe[1]));
      for (auto& e : evs) cudaEventDestroy(e);
      return;
    }
    if (!dx) {
      p->stage_in.ensure(n);
      GPFVM_CUDA(cudaMemcpyAsync(p->stage_in.ptr, x, n * sizeof(double), cudaMemcpyHostToDevice, s));
      xd = p->stage_in.ptr;
    }
    if (!dy) {
      p->stage_out.ensure(n);
      yd = p->stage_out.ptr;
    }
    matvec_device(p, xd, yd, nrhs, ld, s);
    if (!dy) {
      GPFVM_CUDA(cudaMemcpyAsync(y, yd, n * sizeof(double), cudaMemcpyDeviceToHost, s));
      GPFVM_CUDA(cudaStreamSynchronize(s));
    } else if (!dx) {
      GPFVM_CUDA(cudaStreamSynchronize(s));
    }
  });
}

double gpfvm_matvec_flops_unsplit(const gpfvm_problem* p) {
  if (!p) return 0.0;
  return gpfvm_matvec_flops(p) + (p->plan ? p->plan->flops_split_saved : 0.0);
}

double gpfvm_matvec_flops(const gpfvm_problem* p) {
  if (!p) return 0.0;
  if (p->plan) return p->plan->flops_per_rhs;
  double fl = 0.0;
  for (const auto& t : p->terms) fl += term_flops(p, t, p->blocks[t.J].shape, p->blocks[t.I].shape);
  return fl;
}

int gpfvm_solve(gpfvm_problem* p, const double* y, double* alpha, const gpfvm_solve_opts* opts,
                gpfvm_solve_report* report, void* stream) {
  return guarded([&] {
    GPFVM_CHECK(p && y && alpha, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(p->assembled, GPFVM_ERR_STATE, "gpfvm_solve: call gpfvm_assemble_factors first");
    GPFVM_CUDA(cudaSetDevice(p->device));
    gpfvm_solve_opts o{1e-8, 1000, GPFVM_PRECOND_BLOCK_FD, 0, 1};
    if (opts) o = *opts;
    GPFVM_CHECK(o.rtol >= 0 && o.max_iter >= 0 && o.reorth_window >= 0, GPFVM_ERR_INVALID, "bad solve options");
    gpfvm_solve_report rep{};
    cudaStream_t s = (cudaStream_t)stream;
    const bool dy = is_device_ptr(y), da = is_device_ptr(alpha);
    DevBuf ybuf, abuf;
    const double* yd = y;
    double* ad = alpha;
    if (!dy) {
      ybuf.ensure(p->N);
      GPFVM_CUDA(cudaMemcpyAsync(ybuf.ptr, y, p->N * sizeof(double), cudaMemcpyHostToDevice, s));
      yd = ybuf.ptr;
    }
    if (!da) {
      abuf.ensure(p->N);
      ad = abuf.ptr;
    }
    solve_impl(p, yd, ad, o, rep, s);
    if (!da) GPFVM_CUDA(cudaMemcpyAsync(alpha, ad, p->N * sizeof(double), cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
    if (report) *report = rep;
  });
}

int gpfvm_solve_many(gpfvm_problem* p, const double* y, double* alpha, int nrhs, int64_t ld,
                     const gpfvm_solve_opts* opts, gpfvm_solve_report* reports, void* stream) {
  return guarded([&] {
    GPFVM_CHECK(p && y && alpha && reports, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(nrhs >= 1 && ld >= p->N, GPFVM_ERR_INVALID, "nrhs < 1 or ld < N");
    GPFVM_CHECK(p->assembled, GPFVM_ERR_STATE, "gpfvm_solve_many: call gpfvm_assemble_factors first");
    GPFVM_CHECK(is_device_ptr(y) && is_device_ptr(alpha), GPFVM_ERR_INVALID, "gpfvm_solve_many: device pointers only");
    GPFVM_CHECK(y != alpha, GPFVM_ERR_INVALID, "y and alpha must not alias");
    GPFVM_CUDA(cudaSetDevice(p->device));
    gpfvm_solve_opts o{1e-8, 1000, GPFVM_PRECOND_BLOCK_FD, 0, 1};
    if (opts) o = *opts;
    GPFVM_CHECK(o.rtol >= 0 && o.max_iter >= 0 && o.reorth_window >= 0, GPFVM_ERR_INVALID, "bad solve options");
    cudaStream_t s = (cudaStream_t)stream;
    solve_many_impl(p, y, ld, alpha, ld, nrhs, o, reports, s);
    GPFVM_CUDA(cudaStreamSynchronize(s));
  });
}

int gpfvm_predict(gpfvm_problem* p, const gpfvm_grid* grid, const double* alpha, double* mean, double* var,
                  int cov_mode, void* stream) {
  return guarded([&] {
    GPFVM_CHECK(p && grid && alpha, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(p->assembled, GPFVM_ERR_STATE, "gpfvm_predict: call gpfvm_assemble_factors first");
    GPFVM_CHECK(grid->output >= 0 && grid->output < p->nout, GPFVM_ERR_INVALID, "grid output out of range");
    GPFVM_CHECK(cov_mode == GPFVM_COV_ITERGP || cov_mode == GPFVM_COV_PRECOND, GPFVM_ERR_INVALID, "bad cov_mode");
    GPFVM_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = (cudaStream_t)stream;
    int64_t ng = 1;
    for (int i = 0; i < p->ndim; i++) {
      GPFVM_CHECK(grid->n[i] >= 1 && grid->pts[i], GPFVM_ERR_INVALID, "empty grid dimension");
      ng *= grid->n[i];
    }
    const bool da = is_device_ptr(alpha);
    DevBuf abuf, mbuf, vbuf;
    const double* ad = alpha;
    if (!da) {
      abuf.ensure(p->N);
      GPFVM_CUDA(cudaMemcpyAsync(abuf.ptr, alpha, p->N * sizeof(double), cudaMemcpyHostToDevice, s));
      ad = abuf.ptr;
    }
    double* md = mean;
    double* vd = var;
    if (mean && !is_device_ptr(mean)) { mbuf.ensure(ng); md = mbuf.ptr; }
    if (var && !is_device_ptr(var)) { vbuf.ensure(ng); vd = vbuf.ptr; }
    predict_impl(p, *grid, ad, md, vd, cov_mode, s);
    if (mean && md != mean) GPFVM_CUDA(cudaMemcpyAsync(mean, md, ng * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (var && vd != var) GPFVM_CUDA(cudaMemcpyAsync(var, vd, ng * sizeof(double), cudaMemcpyDeviceToHost, s));
    GPFVM_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
