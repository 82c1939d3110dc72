// The opaque gpfvm_problem handle and the Kronecker-term plan.
#pragma once
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "internal.h"

namespace gpfvm {

struct BlockInt {
  Sites sites[GPFVM_MAX_DIMS];
  std::vector<gpfvm_term> terms;
  double noise = 0.0;
  int deflate = 0;
  int64_t size = 0, offset = 0;
  int shape[GPFVM_MAX_DIMS] = {1, 1, 1, 1};
};

// factor identity: (output, dim, left block, left order, right block, right order)
using FactorKey = std::tuple<int, int, int, int, int, int>;

struct Factor {
  int rows = 0, cols = 0;
  // reflection parity of a square factor on a mirror-symmetric site list:
  // F[n-1-i][n-1-j] = psign * F[i][j] (+1 centrosymmetric, -1 skew; 0: none)
  int psign = 0;
  DevBuf data;  // row-major rows x cols
};

// coef * ((x)_i F_i) applied from block J (input) to block I (output)
struct KronTerm {
  int I = 0, J = 0;
  double coef = 0.0;
  int fid[GPFVM_MAX_DIMS] = {-1, -1, -1, -1};
};

// Mode-s updates (ModeUpdate below) handed to the 3D parity-split KronSum,
// whose last kernel adds them while it writes y:
//   y[i0][i1][i2] += sum_p U_s[i_s][p] W_s[r][p][the other two indices]
struct ModeTerms {
  int n = 0;
  struct T {
    const double* U;  // [n_s][P]
    const double* W;  // [R][P][A][B]
    int P, s;
  } m[3];
};

// Fused sum of Kronecker products of one block pair (kron.cu)
struct KronSum {
  int d = 0, P = 0;
  bool rev = false;  // contraction order: dim d-1 first (chosen by flop count)
  int nin[GPFVM_MAX_DIMS] = {1, 1, 1, 1}, nout[GPFVM_MAX_DIMS] = {1, 1, 1, 1};
  DevBuf stk[GPFVM_MAX_DIMS];  // stacked factors per dim (coefficients folded into dim 0)
  std::vector<DevBuf> merged;  // combined factors of merged terms (build)
  // 3D forward plain path: terms that share their dim-0 (dim-2) factor share
  // the stage-0 (stage-2) slice: Q0 / Q2 distinct factors, u0[p] / u2[p] map
  int Q0 = 0, Q2 = 0;
  std::vector<int> u0, u2;
  // 3D with a single output site in the middle dimension (e.g. a boundary face
  // y = const observed from the PDE block): contract that dimension first (the
  // cheap, shrinking point functional), then time, then the last dimension
  bool mid_thin = false;
  // 3D with a single output site in the last dimension (faces x = const of a
  // (t, y, x) layout): point functional first, then dimension 1, then time
  bool last_thin = false;
  // reflection-parity split (d = 2): every factor of dimension
  // i is centrosymmetric (sg[i] = 0) or skew-centrosymmetric (sg[i] = 1) on an
  // even-length mirror-symmetric site list.  X is transformed to its even/odd
  // parts per dimension (u = x_k + x_{n-1-k}, v = x_k - x_{n-1-k}), each factor
  // splits into two half-size blocks E = F_top-left + F_top-right J and
  // O = F_top-left - F_top-right J, and the Kronecker sum runs on the four
  // parity classes as two-level batched GEMMs: half the flops of every stage
  bool par = false;
  int sg[GPFVM_MAX_DIMS] = {0, 0, 0, 0};
  // 3D variant (kron.cu): per-term skews, class-batched forward plan; dim-0
  // and dim-2 factors ordered centrosymmetric first (Qs0 / Qs2 of Q0 / Q2)
  bool par3 = false;
  int Qs0 = 0, Qs2 = 0;
  std::vector<int> sk1;
  // signs (optional): per term, per dimension the factor's psign (0 = none)
  void build(int d, const int* in_shape, const int* out_shape, const std::vector<double>& coefs,
             const std::vector<std::vector<const double*>>& factors, cudaStream_t s,
             const std::vector<std::vector<int>>* signs = nullptr);
  int64_t workspace_per_rhs() const;
  double flops_per_rhs() const;
  // y = beta*y + sum_p (x)F^p x  for R vectors; w0/w1: R*workspace_per_rhs() doubles each
  // extra: optional low-rank term (Gemm::K2 fields) added to the result, fused
  // into the last contraction where its layout allows (2D forward order)
  // extra_ready: event after which the extra term's operands are valid (they
  // may be prepared on another stream while the contractions run)
  // stage0 (d = 2, plain path): the result of the first contraction, already
  // computed elsewhere (FusedFunc) in the layout this plan's stage 0 writes
  void apply(const double* x, int64_t ldx, double* y, int64_t ldy, int R, double beta, double* w0, double* w1,
             cudaStream_t s, const Gemm* extra = nullptr, cudaEvent_t extra_ready = nullptr,
             const double* stage0 = nullptr, const ModeTerms* modes = nullptr) const;
};

// Per-block fast-diagonalisation (bjfd.cu)
struct BlockFD {
  int J = 0, d = 0;
  int shape[GPFVM_MAX_DIMS] = {1, 1, 1, 1};
  DevBuf Q[GPFVM_MAX_DIMS], Qt[GPFVM_MAX_DIMS], Dinv, w0, w1, tmp;
  KronSum fwd, bwd;
};

// Block-LDL / fast-diagonalisation preconditioner state (solve.cu)
struct Precond {
  bool blockjacobi = false;      // general case: block-Jacobi FD (bj) instead of exact LDL
  std::vector<BlockFD> bj;
  int type = GPFVM_PRECOND_NONE;
  int P = -1;
  int n0 = 0, n1 = 0;
  int64_t Np = 0;
  DevBuf V, Vt, W, Dinv;
  std::vector<int> bblocks;
  std::vector<int64_t> boff;  // offset of each deflated block inside the b-vector
  int64_t nb = 0;
  DevBuf YT, Sinv, Linv;           // Y^T = (FD G_pb)^T (nb x Np), explicit S^{-1} = L^{-T} L^{-1}
  DevBuf LYT;                      // L^{-1} Y^T (nb x Np), built on the first PRECOND predict (dense path)
  // Rotated couplings Z_J = (V (x) W)^T G_{P,J} = sum_s c_s (V^T F0_s) (x) (W^T F1_s)
  // per deflated block.  structured: every deflated block is
  // thin (IC-like m0 = 1 or BC-like m1 = 1), Y is never formed.
  struct RotTerm {
    double c = 0.0;
    int m0 = 0, m1 = 0;
    DevBuf R0, R1, LT;  // R0 = V^T F0 (n0 x m0), R1 = W^T F1 (n1 x m1), LT = long factor transposed
  };
  std::vector<std::vector<RotTerm>> rot;
  std::vector<KronSum> rot_ks;
  bool structured = false;
  DevBuf yb, WT, DinvT;
  std::vector<KronSum> ks_bp;      // G_{I,P} per deflated block I (Kronecker sums)
  DevBuf kw0, kw1;                 // their workspaces (one vector)
  double shift = 0.0;
  DevBuf t1, t2, rb, zb, cvec;
  double setup_ms = 0.0;
};
struct Krylov {   // kept IterGP actions
  DevBuf d, gd;   // [cap][N]
  std::vector<double> eta;
  int k = 0, cap = 0;
};

struct Workspace {
  DevBuf t0, t1;
};

struct PairOp {
  int I = 0, J = 0;
  KronSum ks;
  bool lowrank = false;  // folded into the output block's LowRank update
};

// 2D output block: couplings from blocks with a singleton dimension are
// rank-P updates  sum_p u_p v_p^T  (u: n0, v: n1) — IC-like blocks (n'_0 = 1):
// u_p = c_p F0^p[:,0] fixed, v_p = F1^p x_J; BC-like blocks (n'_1 = 1):
// u_p = c_p F0^p x_J, v_p = F1^p[:,0] fixed.  All of them are evaluated into
// U (n0 x rk) and V (rk x n1) per vector and applied as ONE batched GEMM
// y = U V, replacing one read-modify-write pass per coupling.
struct LowRank {
  struct Part {
    int J = 0, type = 0, P = 0, k0 = 0, nin = 0;  // type 0: IC-like, 1: BC-like
    DevBuf stk;    // type 0: F1^p stacked (P*n1 x n'_1); type 1: c_p F0^p stacked (P*n0 x n'_0)
    DevBuf fixed;  // type 0: c_p F0^p[:,0] as [n0][P]; type 1: F1^p[:,0] as [P][n1]
  };
  int n0 = 0, n1 = 0, rk = 0;
  std::vector<Part> parts;
  DevBuf U, V, T;  // U [R][n0][rkp], V (transposed) [R][n1][rkp], scratch T
  int R = 0;
  // side stream on which prepare() runs beside the block's own Kronecker sum
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_ready = nullptr;
  int rkp() const { return (rk + 1) & ~1; }  // even row stride (16-byte TMA strides)
  // U and V of y += U V^T for the current input (the coupling GEMMs)
  void prepare(const double* x, int64_t ldx, int Rn, const int64_t* block_off, cudaStream_t s);
  // the update as the extra term of g (fused into g's k loop)
  void as_extra(Gemm& g, int Rn) const;
  void apply(const double* x, int64_t ldx, double* y, int64_t ldy, int R, double beta, const int64_t* block_off,
             cudaStream_t s);
  void ensure(int Rn);  // U, V, T for Rn right-hand sides
};
struct LowRankTerm {
  double coef;
  const double* F0;  // n0 x n'_0 (row-major)
  const double* F1;  // n1 x n'_1
};
void add_lowrank_part(LowRank& lr, int J, const int* shJ, const std::vector<LowRankTerm>& ts, cudaStream_t s);

// d >= 3 output block: couplings from blocks that are singleton in exactly one
// dimension s (IC planes, boundary faces) are mode-s updates
//   y[a, i, b] += sum_p U[i, p] W_p[a, b],   W_p = (x)_{k != s} F_k^p x_J,
// U[:, p] = c_p F_s^p[:, 0] (fixed).  The W_p are (d-1)-dimensional Kronecker
// products on the small input block (one single-term KronSum each); the update
// is one streaming pass over y instead of full-size mode products that expand
// the singleton dimension.
struct ModeUpdate {
  struct Part {
    int J = 0, p0 = 0;
    std::vector<KronSum> ks;  // one per term
  };
  int s = 0, A = 1, ns = 1, B = 1, P = 0;
  DevBuf U;    // [ns][P]
  DevBuf W;    // [R][P][A][B]
  DevBuf mw0, mw1;  // own workspaces (prepare() on a side stream)
  std::vector<Part> parts;
  int64_t workspace_per_rhs() const;
  // W for the current input (the small Kronecker products), then the update
  void prepare(const double* x, int64_t ldx, int R, const int64_t* block_off, double* w0, double* w1,
               cudaStream_t s) const;
  void update(double* y, int64_t ldy, int R, double beta, cudaStream_t s) const;
  void apply(const double* x, int64_t ldx, double* y, int64_t ldy, int R, double beta, const int64_t* block_off,
             double* w0, double* w1, cudaStream_t s) const;
};

// One read of a 2D input block J for every thin pair (I, J) (funcpass.cu): the
// first contraction of each such pair (a time-point or space-point functional
// of the whole block) evaluated together; the pairs' KronSums then start at
// their second contraction (KronSum::apply `stage0`).
struct FusedFunc {
  struct Out {
    int pair, type, P, first;  // type 0: column sums (IC-like), 1: row sums (BC-like); first slot of its P functionals
    int64_t off;               // per-RHS offset of the pair's stage-0 result inside zbuf
  };
  int J = 0, n0 = 0, n1 = 0, NC = 0, NR = 0;
  int64_t zper = 0;            // stage-0 doubles per RHS over all pairs
  std::vector<Out> outs;
  DevBuf wc, wr, zbuf, colpart;
  cudaEvent_t ev = nullptr;
  int tiles() const;
  void ensure(int R);
  void run(const double* xJ, int64_t ldx, int R, cudaStream_t s) const;
  const double* stage0_of(int pair, int R) const;
};

// Matvec plan: one KronSum per nonzero block pair, grouped by output block
// (graph branches), with CUDA-graph replay cached per (x, y, nrhs, ld).
struct MatvecPlan {
  std::vector<PairOp> pairs;
  std::vector<std::vector<int>> by_out;
  std::vector<LowRank> lowrank;  // per output block (rk = 0: unused)
  std::vector<std::vector<ModeUpdate>> modes;  // per output block (d >= 3)
  std::vector<FusedFunc> fused;  // per 2D input block with >= 2 thin pairs
  std::vector<int> fused_of;     // per pair: index into fused or -1
  bool fused_on = false;         // this launch uses the fused pass (alignment checked per call)
  bool serial_now = false;       // this launch runs every branch on one stream (direct launches)
  std::vector<int64_t> block_off;
  std::vector<DevBuf> w0, w1;  // per output-block branch
  std::vector<cudaStream_t> branch;
  // per output block: side stream on which the mode-update operands are
  // prepared beside the block's own Kronecker sum (created on first use)
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> side_fork, side_ready;
  cudaStream_t cap = nullptr;
  std::vector<cudaEvent_t> ev;
  struct G {
    const double* x;
    double* y;
    int nrhs;
    int64_t ld;
    cudaGraphExec_t exec;
    int64_t nodes;
    int seen;
  };
  std::vector<G> graphs;
  double flops_per_rhs = 0.0;
  double flops_split_saved = 0.0;  // flops the reflection-parity split removed (context for the roofline)
  ~MatvecPlan();
  void release_graphs();
};

}  // namespace gpfvm

struct gpfvm_problem {
  int device = 0;
  int ndim = 0, nout = 0;
  std::vector<gpfvm_kernel1d> kernels;  // [nout * ndim]
  std::vector<gpfvm::BlockInt> blocks;
  int64_t N = 0;
  std::map<gpfvm::FactorKey, int> factor_index;
  std::vector<gpfvm::Factor> factors;
  std::vector<gpfvm::KronTerm> terms;
  gpfvm::DevBuf noise;
  bool assembled = false;
  gpfvm::Workspace ws;
  gpfvm::Precond* pc = nullptr;
  gpfvm::Krylov kry;
  gpfvm::DevBuf stage_in, stage_out;  // host-pointer staging
  std::unique_ptr<gpfvm::MatvecPlan> plan;
  gpfvm::DevBuf pcg_s, pcg_z;           // fixed PCG operands (graph-replayable matvec)
  cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};  // host-pointer matvec pipeline (H2D, compute, D2H)
  ~gpfvm_problem();
};

namespace gpfvm {

// Apply the Kronecker terms of block pair (I, J) (or of the explicit term list)
// to R vectors: Y_I (+)= sum coef (x)F X_J.  x/y strides per vector: ldx, ldy;
// x and y point at the block starts.  beta_first = 0 overwrites Y on the first
// term when `overwrite` is true.
void apply_terms(gpfvm_problem* p, const std::vector<Factor>& factors, const std::vector<const KronTerm*>& terms, const int* in_shape,
                 const int* out_shape, const double* x, int64_t ldx, double* y, int64_t ldy, int R,
                 bool overwrite, cudaStream_t s, Workspace& ws);
void matvec_device(gpfvm_problem* p, const double* x, double* y, int nrhs, int64_t ld, cudaStream_t s);
void build_plan(gpfvm_problem* p, cudaStream_t s);
void build_lowrank(gpfvm_problem* p, MatvecPlan& pl, cudaStream_t s);
void build_fused_func(gpfvm_problem* p, MatvecPlan& pl, cudaStream_t s);
void refresh_fused_func(MatvecPlan& pl, cudaStream_t s);
double term_flops(const gpfvm_problem* p, const KronTerm& t, const int* in_shape, const int* out_shape);
int get_factor(gpfvm_problem* p, int out, int dim, int bl, int ml, int br, int mr);

bool is_device_ptr(const void* ptr);

// solve.cu / predict.cu
void solve_impl(gpfvm_problem* p, const double* y, double* alpha, const gpfvm_solve_opts& o,
                gpfvm_solve_report& rep, cudaStream_t s);
void predict_impl(gpfvm_problem* p, const gpfvm_grid& g, const double* alpha, double* mean, double* var,
                  int cov_mode, cudaStream_t s);
void solve_many_impl(gpfvm_problem* p, const double* Y, int64_t ldy, double* X, int64_t ldx, int R,
                     const gpfvm_solve_opts& o, gpfvm_solve_report* reps, cudaStream_t s);
void apply_block_fd_many(const BlockFD& bf, const double* r, int64_t ldr, double* z, int64_t ldz, int64_t n, int R,
                         double* tmp, double* w0, double* w1, cudaStream_t s);
void destroy_precond(Precond* pc);
void predict_mean_shard(gpfvm_problem* p, const gpfvm_grid& g, const double* alpha_local, const int64_t* loc_off,
                        const int* row0, const int* rows, double* mean, cudaStream_t s);
// eigenbases already computed in this preconditioner build, keyed by the
// pencil's definition: (output, dim, lower order, higher order or -1 for the
// identity, site kind) and the site endpoints — blocks that share a site list
// (e.g. the time cells of the faces and of the PDE block) share the basis
using PencilKey = std::tuple<int, int, int, int, int, std::vector<double>, std::vector<double>>;
using PencilCache = std::map<PencilKey, const double*>;
void build_block_fd(gpfvm_problem* p, int J, BlockFD& bf, cudaStream_t s, PencilCache* cache = nullptr);
void apply_block_fd(const BlockFD& bf, const double* r, double* z, int64_t n, cudaStream_t s);

}  // namespace gpfvm
