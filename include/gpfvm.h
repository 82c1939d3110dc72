/*
 * gpfvm.h — C ABI of the B200-native GP-FVM hot path (libgpfvm.so).
 *
 * GP-FVM (arxiv 2406.05020, "PAPER.md") conditions a Gaussian-process prior
 * on finite-volume observations of a linear PDE.  With a product Matérn
 * kernel (Eq. 13) and factorized box schemes (§4
 * Definition, l.306-313) the Gram matrix is a sum of Kronecker products of
 * small 1D factor matrices (Eq. 20, l.316-318).  This library implements,
 * on one sm_100a GPU in FP64:
 *
 *   gpfvm_assemble_factors   1D closed-form functional pairs (Eq. 10/16)
 *   gpfvm_gram_matvec        Y = G X  for a block of vectors (Eq. 20)
 *   gpfvm_solve              preconditioned CG / IterGP (§4.1, §4.2)
 *   gpfvm_predict            posterior mean / variance on a grid (Eq. 5-6)
 *
 * Conventions (all entry points)
 *   - Return value: GPFVM_OK (0) on success, a negative gpfvm_status
 *     otherwise; gpfvm_last_error() returns a thread-local message.  Errors
 *     never abort the process; a failing call leaves its outputs undefined.
 *   - Memory: arrays inside *desc structs are HOST pointers, read during
 *     the call and not retained.  Vector arguments (x, y, alpha, mean, var)
 *     may be DEVICE pointers (fast path) or HOST pointers (pageable or
 *     pinned): the library detects host memory with cudaPointerGetAttributes
 *     and stages it through device buffers (host<->device copies are then
 *     part of the call).  The caller owns all arrays it passes; the library
 *     owns everything reachable from a gpfvm_problem handle.
 *   - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).
 *     Device-pointer calls are asynchronous w.r.t. the host unless stated;
 *     host-pointer calls synchronise the stream before returning.
 *   - Precision: every quantity is IEEE FP64.
 *   - Layout of the observation vector: blocks in the order given; inside a
 *     block, observations are the Cartesian product of the per-dimension
 *     sites flattened row-major (dimension 0 slowest).  A block of vectors
 *     is nrhs vectors of length N, vector r starting at x + r*ld (ld >= N).
 *   - Thread safety: calls on distinct handles are independent; calls on one
 *     handle must be serialised by the caller.
 */
#ifndef GPFVM_H
#define GPFVM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPFVM_MAX_DIMS 4
#define GPFVM_MAX_TERMS 16

typedef enum {
  GPFVM_OK = 0,
  GPFVM_ERR_INVALID = -1,     /* bad argument / description */
  GPFVM_ERR_CUDA = -2,        /* CUDA runtime error (message has details) */
  GPFVM_ERR_UNSUPPORTED = -3, /* valid input outside what is implemented */
  GPFVM_ERR_NUMERIC = -4,     /* breakdown (non-SPD, NaN) */
  GPFVM_ERR_STATE = -5        /* call order violated (e.g. solve before assemble) */
} gpfvm_status;

/* Site kinds of a 1D functional list (PAPER.md l.170 point functionals;
 * l.195-198 interval [a,b] functionals). */
enum { GPFVM_SITE_POINT = 0, GPFVM_SITE_INTERVAL = 1 };

/* One 1D Matérn factor, nu = q + 1/2 (Eq. 12, l.213-216):
 *   k(d) = variance * exp(-sqrt(2q+1)|d|/l) * p_q(sqrt(2q+1)|d|/l),  0 <= q <= 3. */
typedef struct {
  int q;
  double lengthscale;
  double variance;
} gpfvm_kernel1d;

/* 1D site list: n sites of one kind.  For intervals lo[j] < hi[j]; for
 * points lo[j] is the location (hi ignored).  Host pointers. */
typedef struct {
  int kind;
  int n;
  const double* lo;
  const double* hi;
} gpfvm_sites1d;

/* One operator term  coeff * D^order [u_output]  (Eq. 18 preamble, l.267). */
typedef struct {
  double coeff;
  int order[GPFVM_MAX_DIMS];
  int output;
} gpfvm_term;

/* One factorized observation block (§4 Definition): per-dimension sites,
 * the operator applied in every cell (Eq. 8/15), i.i.d. noise variance
 * (Sigma, l.108) and whether the block is eliminated exactly in the
 * preconditioner (IC/BC deflation, §4.2 l.331-339). */
typedef struct {
  gpfvm_sites1d sites[GPFVM_MAX_DIMS];
  int n_terms;
  gpfvm_term terms[GPFVM_MAX_TERMS];
  double noise;
  int deflate;
} gpfvm_block;

typedef struct {
  int ndim;                          /* 1..GPFVM_MAX_DIMS */
  int n_outputs;                     /* multi-output prior (Eq. 17) */
  const gpfvm_kernel1d* kernels;     /* [n_outputs * ndim], output-major */
  int n_blocks;
  const gpfvm_block* blocks;
} gpfvm_problem_desc;

typedef struct gpfvm_problem gpfvm_problem;  /* opaque */

/* ---- library / handle ------------------------------------------------- */
const char* gpfvm_last_error(void);
const char* gpfvm_version(void);

/* Validate `desc`, copy it, allocate device storage on `device`.  Checks:
 * ndim/q ranges, interval ordering, derivative orders (point order <= q,
 * interval order <= q+1: PAPER.md §3.2 l.250 smoothness).  No GPU work. */
int gpfvm_problem_create(const gpfvm_problem_desc* desc, int device, gpfvm_problem** out);
int gpfvm_problem_destroy(gpfvm_problem* p);
/* N (total number of observations). */
int64_t gpfvm_problem_size(const gpfvm_problem* p);

/* ---- §8 row 1: factor assembly ------------------------------------------
 * Compute every 1D factor matrix  F[j,j'] = L_{left_j; m} k L'_{right_j'; m'}
 * the Gram needs (Eq. 16, l.246; endpoint reduction Eq. 10, l.207) on the
 * device, in double-double arithmetic from closed-form antiderivatives at
 * the cell endpoints, rounded once to FP64.  Must precede
 * matvec/solve/predict; may be called again (idempotent, bitwise
 * reproducible). */
int gpfvm_assemble_factors(gpfvm_problem* p, void* stream);

/* Standalone single factor matrix into a caller DEVICE buffer `out`
 * (row-major, left->n rows, right->n columns, leading dimension ld). */
int gpfvm_factor_matrix(const gpfvm_kernel1d* k, const gpfvm_sites1d* left, int m_left,
                        const gpfvm_sites1d* right, int m_right, double* out, int64_t ld,
                        void* stream);

/* ---- §8 row 2: Gram matvec ------------------------------------------------
 * Y = G X + Sigma X for nrhs vectors (Eq. 20 + l.109), G never formed:
 * batched mode-n contractions on FP64 tensor cores (DMMA).  x and y must not
 * alias. */
int gpfvm_gram_matvec(gpfvm_problem* p, const double* x, double* y, int nrhs, int64_t ld,
                      void* stream);

/* General Kronecker-sum primitive (the local kernel of the sharded path,
 * DESIGN.md §7):  Y_r = beta*Y_r + sum_p c_p ((x)_{i<ndim} F_{p,i}) X_r  for
 * r < nrhs, with X_r/Y_r tensors of shape in_shape / out_shape flattened
 * row-major (dim 0 slowest).  factors[p*ndim + i] is a DEVICE pointer to the
 * row-major out_shape[i] x in_shape[i] matrix F_{p,i}.  x, y: DEVICE pointers,
 * must not alias.  Same fused plan as gpfvm_gram_matvec (d DMMA GEMMs). */
int gpfvm_kron_matvec(int ndim, const int* in_shape, const int* out_shape, int n_terms, const double* coefs,
                      const double* const* factors, const double* x, int64_t ldx, double* y, int64_t ldy,
                      int nrhs, double beta, void* stream);

/* Row-major DMMA GEMM  C = alpha A B + beta C  (A: M x K, B: K x N, C: M x N;
 * DEVICE pointers, leading dimensions in elements).  The time contraction of
 * the sharded path after its all-to-all. */
int gpfvm_gemm(int M, int N, int K, double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
               double beta, double* C, int64_t ldc, void* stream);

/* dst = permutation of the row-major tensor src (ndim <= 4): dst has shape
 * (shape[perm[0]], ..., shape[perm[ndim-1]]).  DEVICE pointers, no aliasing. */
int gpfvm_permute(int ndim, const int* shape, const int* perm, const double* src, double* dst, void* stream);

/* Generalised symmetric-definite eigenproblem  A V = B V diag(w),  V^T B V = I
 * (A symmetric, B SPD; n x n row-major DEVICE matrices; V row-major with the
 * eigenvectors in its columns).  Cholesky reduction + one-sided block Jacobi
 * (DESIGN.md §5.1).  Synchronises `stream`. */
int gpfvm_sygv(int n, const double* A, const double* B, double* V, double* w, void* stream);

/* Fused solver vector ops (DEVICE pointers; coef is a DEVICE array of k values):
 *   gpfvm_dot_many:  out[j] = X_j . v  for j < k (X_j = X + j*ldx), warp-shuffle
 *                    reductions, deterministic fixed-order second pass
 *   gpfvm_axpy_many: y += sign * sum_j coef[j] X_j  (one pass over y) */
int gpfvm_dot_many(const double* X, int64_t ldx, const double* v, int64_t n, int k, double* out, void* stream);
int gpfvm_axpy_many(double* y, const double* X, int64_t ldx, const double* coef, double sign, int64_t n, int k,
                    void* stream);

/* Fast-diagonalisation factors of a two-term 2D Kronecker block
 * ca A0(x)A1 + cb B0(x)B1 (+ noise I):  B0 V = A0 V Lam,
 * A1 W = B1 W M,  Dinv[i*n1+j] = 1/(ca M_j + cb Lam_i + noise |v_i|^2 |w_j|^2).
 * All DEVICE row-major; V n0 x n0, W n1 x n1, Dinv n0*n1.  Synchronises. */
int gpfvm_fd_setup(int n0, int n1, const double* A0, const double* A1, const double* B0, const double* B1,
                   double ca, double cb, double noise, double* V, double* W, double* Dinv, void* stream);
/* x[i] *= d[i]  (DEVICE pointers) */
int gpfvm_vmul(double* x, const double* d, int64_t n, void* stream);

/* ---- §8 row 3: solve -----------------------------------------------------
 * Solve G alpha = y with preconditioned CG in IterGP form (§4.1; Wenger et
 * al. 2022 Alg. 1, CG policy, full reorthogonalisation §6 l.475): actions
 * s_i = P^{-1} r_{i-1}, G-conjugate directions d_i and eta_i = d_i^T G d_i
 * are kept on the device for the computational-uncertainty downdate used by
 * gpfvm_predict.  P is built on the first call after assembly
 * and cached: for one 2D two-term PDE block with <= 16384 deflated IC/BC
 * cells, fast diagonalisation of the PDE block + exact block-LDL elimination
 * of the IC/BC cells (thin blocks: in closed Kronecker form); otherwise
 * block-Jacobi fast diagonalisation of every block.
 * Stops when ||r||_2 <= rtol ||y||_2 (recursive residual) or after
 * max_iter iterations; the report holds the final true residual too.
 * opts may be NULL (defaults below); y, alpha: N-vectors (device or host).
 * One right-hand side (several: gpfvm_solve_many).  Errors:
 * GPFVM_ERR_STATE before assembly, GPFVM_ERR_NUMERIC if the Schur complement
 * cannot be factorised even after shifting, GPFVM_ERR_CUDA on device errors
 * (e.g. out of memory for the Krylov store: see keep_actions). */
enum { GPFVM_PRECOND_NONE = 0, GPFVM_PRECOND_BLOCK_FD = 2 };  /* 1 is reserved */

typedef struct {
  double rtol;        /* default 1e-8 */
  int max_iter;       /* default 1000 */
  int precond;        /* GPFVM_PRECOND_* (default BLOCK_FD) */
  int reorth_window;  /* 0: full reorthogonalisation against every kept direction (default);
                         w > 0: only the last w (w = 1 is the PCG recurrence) */
  int keep_actions;   /* 1 (default): keep every action d_i, G d_i, eta_i for the IterGP
                         covariance; 0: keep only a ring of max(1, reorth_window) of them
                         (device memory O(w N) for long budgeted solves; the ITERGP
                         variance of gpfvm_predict then covers those actions only) */
} gpfvm_solve_opts;

typedef struct {
  int iterations;
  int converged;
  double rel_residual;       /* recursive ||r_i|| / ||y|| */
  double true_rel_residual;  /* ||y - G alpha|| / ||y||, recomputed */
  double precond_shift;      /* Schur-complement shift used (0 normally) */
  double setup_ms;           /* preconditioner build (first call) */
  double iterate_ms;
  int breakdown;             /* 1: stopped because eta_i = d_i^T G d_i <= 0 or non-finite
                                (loss of positive definiteness in rounding); alpha and the
                                kept actions are those of the completed iterations */
} gpfvm_solve_report;

int gpfvm_solve(gpfvm_problem* p, const double* y, double* alpha, const gpfvm_solve_opts* opts,
                gpfvm_solve_report* report, void* stream);
/* nrhs right-hand sides at once (y, alpha: nrhs vectors of stride ld >= N,
 * device pointers): one IterGP run per right-hand side sharing the batched
 * preconditioner and Gram matvec (e.g. BASELINE config 2's 4-RHS batch; the N*
 * solves of a covariance, P:l.288).  reports: nrhs entries.  With the exact 2D
 * preconditioner the solves run one after the other.  The Krylov store kept
 * for gpfvm_predict's ITERGP variance is that of right-hand side 0. */
int gpfvm_solve_many(gpfvm_problem* p, const double* y, double* alpha, int nrhs, int64_t ld,
                     const gpfvm_solve_opts* opts, gpfvm_solve_report* reports, void* stream);

/* ---- §8 row 4: predict -----------------------------------------------------
 * Posterior on the tensor grid  X_* = pts[0] x ... x pts[ndim-1]  for
 * output `output` (Eq. 5-6):
 *   mean[g] = sum_J K_{*J} alpha_J        (cross-covariance Kronecker products)
 *   var[g]  = k(x,x) - k_x^T C k_x        with C chosen by cov_mode:
 *     GPFVM_COV_ITERGP  C = sum_i d_i d_i^T / eta_i  (IterGP combined posterior,
 *                       the Krylov actions kept by the last gpfvm_solve)
 *     GPFVM_COV_PRECOND C = P^{-1} (the exact posterior when
 *                       P^{-1} = G^{-1}, e.g. the heat operator)
 * mean/var: n_grid = prod n[i] entries, row-major (dim 0 slowest); either
 * may be NULL to skip it.  alpha: the representer weights (length N).  Device
 * or host pointers as everywhere; grid points are host arrays read during the
 * call.  PRECOND variance is evaluated in grid slabs along dim 0 sized from
 * the device memory (one slab for config 1's 512 x 1024 grid on a B200).
 * Errors: GPFVM_ERR_STATE for GPFVM_COV_PRECOND without a preceding
 * gpfvm_solve with GPFVM_PRECOND_BLOCK_FD; GPFVM_ERR_UNSUPPORTED for
 * GPFVM_COV_PRECOND with the block-Jacobi (3D / multi-output) preconditioner
 * or ndim != 2; GPFVM_ERR_INVALID for a bad grid (output out of range). */
enum { GPFVM_COV_ITERGP = 0, GPFVM_COV_PRECOND = 1 };

typedef struct {
  int n[GPFVM_MAX_DIMS];
  const double* pts[GPFVM_MAX_DIMS];   /* host pointers */
  int output;
} gpfvm_grid;

int gpfvm_predict(gpfvm_problem* p, const gpfvm_grid* grid, const double* alpha, double* mean,
                  double* var, int cov_mode, void* stream);

/* ---- time-mode sharded operators (multi-GPU) ---------------
 * north_star: "the observation tensor is sharded along the time mode; NCCL
 * all-to-all re-partition for the time-mode contraction and an allreduce for
 * the CG inner products".  Every block whose dimension 0 is the common time
 * axis (n0 sites) is split into `world` contiguous time slabs (rank r owns
 * sites [r n0/world, (r+1) n0/world)); blocks with one time site (IC planes)
 * live on rank 0.  The local vector is the concatenation, block by block, of
 * the owned rows (row-major, dimension 0 slowest); gpfvm_shard_layout gives
 * the offsets.  One application of a sharded operator is three library calls
 * around two all-to-all exchanges done by the caller (NCCL
 * all_to_all_single with the per-rank counts of gpfvm_shard_counts):
 *   begin(x_local) -> send1  | all-to-all | mid(recv1) -> send2 |
 *   all-to-all | end(recv2) -> y_local.
 * GPFVM_SHARD_GRAM: y = G x (Eq. 20, noise included), one phase (0).
 * GPFVM_SHARD_PRECOND: block-Jacobi FD as phase 0 (Q^T),
 * gpfvm_shard_precond_scale (D^{-1}, local) and phase 1 (Q).
 * Every buffer is a device pointer owned by the caller; the handle owns its
 * workspaces and must be destroyed before the problem.  Errors:
 * GPFVM_ERR_STATE before assembly, GPFVM_ERR_UNSUPPORTED for d < 2 or blocks
 * whose time extent is neither n0 nor 1, GPFVM_ERR_INVALID for bad ranks. */
enum { GPFVM_SHARD_GRAM = 0, GPFVM_SHARD_PRECOND = 1 };
typedef struct gpfvm_shard gpfvm_shard;
int gpfvm_shard_create(gpfvm_problem* p, int rank, int world, int kind, gpfvm_shard** out, void* stream);
int gpfvm_shard_destroy(gpfvm_shard* sh);
/* local vector length on this rank */
int64_t gpfvm_shard_local_size(const gpfvm_shard* sh);
/* per block: offset in the local vector, first owned time row, owned rows,
 * spatial size (arrays of n_blocks entries; any may be NULL) */
int gpfvm_shard_layout(const gpfvm_shard* sh, int64_t* local_offset, int64_t* row0, int64_t* rows, int64_t* spatial);
/* element counts per peer rank (arrays of `world` entries) of the two exchanges */
int gpfvm_shard_counts(const gpfvm_shard* sh, int phase, int64_t* send1, int64_t* recv1, int64_t* send2,
                       int64_t* recv2);
int gpfvm_shard_apply_begin(gpfvm_shard* sh, int phase, const double* x_local, double* send1, void* stream);
int gpfvm_shard_apply_mid(gpfvm_shard* sh, int phase, const double* recv1, double* send2, void* stream);
/* y_local = (Gram: noise x_local; precond: 0) + the received contributions */
int gpfvm_shard_apply_end(gpfvm_shard* sh, int phase, const double* recv2, const double* x_local, double* y_local,
                          void* stream);
int gpfvm_shard_precond_scale(gpfvm_shard* sh, double* z_local, void* stream);
/* Host-only plan query (no device work; valid before assembly): the local
 * length and the Gram's exchange counts of `rank` — the layout logic of
 * gpfvm_shard_create, testable without a GPU. */
int gpfvm_shard_plan_counts(const gpfvm_problem* p, int rank, int world, int64_t* local_n, int64_t* send1,
                            int64_t* recv1, int64_t* send2, int64_t* recv2);
/* Sharded posterior mean (Eq. 5, l.113): this rank's partial sum
 * K_{*,local} alpha_local on the grid (prod(grid->n) doubles, device); the
 * sum over the ranks (all_reduce) is the mean. */
int gpfvm_shard_predict_mean(gpfvm_shard* sh, const gpfvm_grid* grid, const double* alpha_local, double* mean_partial,
                             void* stream);
/* the local slab of a full (block-concatenated, length N) device vector */
int gpfvm_shard_gather_local(const gpfvm_shard* sh, const double* full, double* local, void* stream);

/* ---- IterGP iteration steps with device-resident scalars (sharded solve) ---
 * The single-GPU gpfvm_solve fuses these; the sharded solve (dist.py) calls
 * them on local slabs and all_reduces (sum) the small `partial` arrays in
 * between — the only arithmetic outside the library is that sum.
 * state: GPFVM_ITER_STATE doubles (||y||, ||r||, threshold, a, eta, done flag
 * (0 running, 1 converged, 2 breakdown), iteration count); once done != 0
 * every step is a no-op.  Reference: PAPER.md §4.1 l.295-302 (IterGP, CG
 * policy), §6 l.475 (full reorthogonalisation). */
enum { GPFVM_ITER_STATE = 8 };
/* state from ||y||^2 (the all-reduced local dot of y) */
int gpfvm_iter_init(const double* yy, double rtol, double* state, void* stream);
/* c_j = dots[j] / eta[j]  (dots: all-reduced K_d[j] . G d, j < w) */
int gpfvm_iter_coefs(const double* dots, int w, const double* eta, double* c, const double* state, void* stream);
/* d' = d - sum c_j Kd_j, g' = g - sum c_j Kg_j into dout/gout; partial[0..1] =
 * local d'.g', d'.r */
int gpfvm_iter_update_local(const double* d, const double* g, const double* Kd, const double* Kg, int64_t ld, int w,
                            const double* c, const double* r, double* dout, double* gout, int64_t n, double* partial,
                            const double* state, void* stream);
/* eta = sums[0] -> *eta_slot, a = sums[1] / eta (breakdown flag if eta <= 0) */
int gpfvm_iter_update_final(const double* sums, double* state, double* eta_slot, void* stream);
/* x += a dn, r -= a gn; partial[0] = local r.r */
int gpfvm_iter_step_local(double* x, double* r, const double* dn, const double* gn, int64_t n, double* partial,
                          const double* state, void* stream);
/* ||r|| = sqrt(sum[0]), convergence flag, iteration count */
int gpfvm_iter_step_final(const double* sum, double* state, void* stream);

/* ---- instrumentation ------------------------------------------------------
 * Kernel-launch counter: every kernel this library launches increments it
 * (a replayed matvec graph counts its kernel nodes). */
int64_t gpfvm_launch_count(void);
/* Flops of one single-vector Gram matvec as executed (after the algebraic
 * term cancellation of DESIGN.md R6; low-rank and mode updates counted as
 * the GEMMs/streams actually run).  0 before assembly. */
double gpfvm_matvec_flops(const gpfvm_problem* p);
/* The same count for the plan without the reflection-parity split
 * (a split block pair executes exactly half the flops of its
 * unsplit plan): context for throughput figures, equal to
 * gpfvm_matvec_flops where no pair is split. */
double gpfvm_matvec_flops_unsplit(const gpfvm_problem* p);
/* FP64 tensor-core peak probe (the roofline denominator bench.py reports):
 * a register-only DMMA.8x8x4 (mma.sync.m8n8k4.f64) kernel, 4 CTAs x 8 warps
 * per SM, each warp issuing 8 independent accumulator chains; best of two
 * ~2 ms launches on `stream`, timed with CUDA events.  *tflops receives
 * TFLOP/s (2 x 256 flops per DMMA).  Synchronises the stream. */
int gpfvm_probe_fp64_peak(double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GPFVM_H */
