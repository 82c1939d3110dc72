"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same
seeded inputs.  Tolerances: factor entries and matvecs 1e-12
relative (normwise, plus element-wise above 1e-6 of the max); posterior mean
1e-8 relative; posterior variance 1e-8 x prior variance (absolute)."""
import numpy as np
import pytest

import gpfvm_inputs as gi
from gpfvm_inputs import Block, Kernel1D, Problem, Sites, Term

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.gram import KroneckerGram, dense_cross_cov, dense_gram, factor_matrix as ofm  # noqa: E402
from oracle.posterior import posterior_exact, variance_itergp  # noqa: E402
from oracle.solve import BlockLDLPreconditioner, itergp_cg  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem, factor_matrix, launch_count  # noqa: E402
from paper_2406_05020_b200._lib import GpfvmError  # noqa: E402

DEV = "cuda:0"


def _t(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def _close(got, ref, rtol, elem=True):
    got = np.asarray(got)
    ref = np.asarray(ref)
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= rtol * scale, np.abs(got - ref).max() / scale
    if elem:
        big = np.abs(ref) > 1e-6 * scale
        rel = np.abs(got - ref)[big] / np.abs(ref)[big]
        assert rel.max() <= rtol * 1e3 if rel.size else True


def _rand_sites(rng, n, kind):
    if kind == gi.POINT:
        return gi.points(np.sort(rng.uniform(-0.5, 1.5, n)))
    e = np.sort(np.concatenate([[0.0, 1.0], rng.uniform(0, 1, n - 1)]))
    e = np.unique(e)
    return Sites(gi.INTERVAL, e[:-1], e[1:])


@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_factor_matrices_match_oracle(q):
    rng = np.random.default_rng(q)
    k = Kernel1D(q, float(rng.uniform(0.05, 0.6)), float(rng.uniform(0.5, 2.0)))
    for kl, kr in [(gi.INTERVAL, gi.INTERVAL), (gi.POINT, gi.INTERVAL), (gi.INTERVAL, gi.POINT), (gi.POINT, gi.POINT)]:
        L = _rand_sites(rng, 37, kl)   # ragged sizes
        R = _rand_sites(rng, 13, kr)
        for ml in range(0, q + 2):
            for mr in range(0, q + 2):
                if (kl == gi.POINT and ml > q) or (kr == gi.POINT and mr > q):
                    continue
                got = factor_matrix(k, L, ml, R, mr).cpu().numpy()
                ref = ofm((k.q, k.lengthscale, k.variance), L, ml, R, mr)
                _close(got, ref, 1e-12)


def test_factor_uniform_fine_grid_bitwise_close():
    """Config-1 time factor (256 cells, l = 0.5): cancellation-heavy 2nd
    differences; the double-double kernel must still agree to ~1 ulp."""
    k = Kernel1D(2, 0.5, 1.0)
    T = gi.cells(256)
    for m in [(0, 0), (1, 1), (1, 0)]:
        got = factor_matrix(k, T, m[0], T, m[1]).cpu().numpy()
        ref = ofm((2, 0.5, 1.0), T, m[0], T, m[1])
        _close(got, ref, 1e-14)


def _random_problem(seed, ndim=3, nout=1):
    rng = np.random.default_rng(seed)
    kern = [[Kernel1D(int(rng.integers(2, 4)), float(rng.uniform(0.2, 0.8)), float(rng.uniform(0.5, 2)))
             for _ in range(ndim)] for _ in range(nout)]
    blocks = []
    for b in range(3):
        sites = []
        for i in range(ndim):
            n = int(rng.integers(3, 11))
            sites.append(gi.points(np.sort(rng.uniform(0, 1, 2))) if (b == 2 and i == 0) else _rand_sites(rng, n, gi.INTERVAL))
        terms = []
        for _ in range(int(rng.integers(1, 4))):
            order = tuple(int(rng.integers(0, 2)) if (b == 2 and i == 0) else int(rng.integers(0, 3)) for i in range(ndim))
            terms.append(Term(float(rng.standard_normal()), order, int(rng.integers(0, nout))))
        blk = Block(f"B{b}", sites, terms, float(rng.uniform(0, 1e-3)), b != 0, np.zeros(0))
        blk.rhs = np.zeros(blk.size)
        blocks.append(blk)
    return Problem(f"rand{seed}", ndim, kern, blocks)


@pytest.mark.parametrize("seed,ndim,nout", [(0, 3, 1), (1, 2, 1), (2, 3, 2), (3, 1, 1), (4, 3, 3), (5, 4, 1)])
def test_matvec_matches_dense_oracle(seed, ndim, nout):
    p = _random_problem(seed, ndim, nout)
    G = dense_gram(p)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, 3, seed)
    Y = gp.gpfvm_gram_matvec(_t(X)).cpu().numpy()
    _close(Y, X @ G.T, 1e-12, elem=False)


def test_matvec_config0_and_ld_stride():
    p = gi.config0()
    G = dense_gram(p)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, 5, 1)
    Y = gp.gpfvm_gram_matvec(_t(X)).cpu().numpy()
    _close(Y, X @ G.T, 1e-12)
    # host pointers (numpy): staged inside the library, same numbers
    Yh = gp.gpfvm_gram_matvec(np.ascontiguousarray(X))
    assert np.array_equal(Yh, Y)


def test_matvec_config1_fullsize_vs_oracle_kronecker():
    """BASELINE config 1 at full size (131,072 PDE cells + 1,024 IC/BC), in the
    launch configuration bench.py times (block of vectors)."""
    p = gi.config1()
    K = KroneckerGram(p)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    R = 128                                   # bench.py's block of vectors
    X = gi.random_vectors(p.size, R, 7)
    Xt = _t(X)
    Yt = torch.empty_like(Xt)
    ref = K.matvec(X)
    for call in range(3):                     # direct launch, graph capture, graph replay
        gp.gpfvm_gram_matvec(Xt, out=Yt)
        _close(Yt.cpu().numpy(), ref, 1e-12, elem=False)


def test_host_pointer_pipeline_config1():
    """nrhs >= 8 with host buffers runs the chunked H2D/compute/D2H pipeline;
    same numbers as the device-pointer path (up to GEMM-kernel choice)."""
    p = gi.config1()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    for R in (16, 128, 37):                   # 2 chunks, bench.py's 8 chunks, ragged chunks
        X = np.ascontiguousarray(gi.random_vectors(p.size, R, 3))
        Yd = gp.gpfvm_gram_matvec(_t(X)).cpu().numpy()
        Yh = gp.gpfvm_gram_matvec(X)
        assert np.abs(Yh - Yd).max() <= 1e-14 * np.abs(Yd).max(), R


def test_solve_and_predict_config0():
    p = gi.config0()
    G = dense_gram(p)
    y = p.rhs()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=1e-10)
    assert rep["converged"] and rep["iterations"] <= 3 and rep["true_rel_residual"] <= 1e-9
    grid = gi.heat_grid(64, 64)
    m_ref, v_ref, a_ref = posterior_exact(p, grid, G, y)
    mean, var = gp.gpfvm_predict(grid, alpha, cov_mode=1)
    _close(mean.cpu().numpy(), m_ref, 1e-8, elem=False)
    assert np.abs(var.cpu().numpy() - v_ref).max() <= 1e-8 * 1.0
    # IterGP combined variance with the kept Krylov actions vs the oracle's IterGP
    P = BlockLDLPreconditioner(p, G)
    tr = itergp_cg(lambda v: G @ v, y, P.apply, rtol=1e-10)
    assert tr.iterations == rep["iterations"]
    _, vi = gp.gpfvm_predict(grid, alpha, cov_mode=0, want_mean=False)
    assert np.abs(vi.cpu().numpy() - variance_itergp(p, grid, tr.directions, tr.etas)).max() <= 1e-8


def test_solve_unpreconditioned_matches_oracle_itergp():
    """Plain IterGP-CG (no preconditioner) on a small system: same iterates as
    the oracle step for step (full reorthogonalisation keeps them close)."""
    p = gi.heat_problem(6, 6)
    G = dense_gram(p)
    y = p.rhs()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=0.0, max_iter=10, precond=0)
    tr = itergp_cg(lambda v: G @ v, y, None, rtol=0.0, max_iter=10)
    assert rep["iterations"] == tr.iterations == 10
    _close(alpha.cpu().numpy(), tr.x, 1e-8, elem=False)


def test_cos_ode_1d():
    """PAPER.md Fig. 2 problem (1D, FVM cells + Dirichlet points)."""
    p = gi.cos_ode_problem(8)
    G = dense_gram(p)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(p.rhs()), rtol=1e-12, max_iter=200, precond=0)
    grid = gi.Grid([np.linspace(0, 2 * np.pi, 50)])
    m_ref, v_ref, _ = posterior_exact(p, grid, G, p.rhs())
    mean, _ = gp.gpfvm_predict(grid, alpha, want_var=False)
    _close(mean.cpu().numpy(), m_ref, 1e-8, elem=False)
    assert np.sqrt(np.mean((mean.cpu().numpy() - np.sin(grid.points[0])) ** 2)) < 0.05


def test_config1_fullsize_solve_properties():
    """Full-size config 1: PCG reaches 1e-8 (true residual recomputed by the
    oracle's Kronecker matvec), posterior mean agrees with the oracle's
    cross-covariance rows at sampled grid points and with the analytic heat
    solution; PRECOND variance non-negative and small everywhere."""
    p = gi.config1()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    y = p.rhs()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=1e-8)
    assert rep["converged"] and rep["iterations"] <= 10
    a = alpha.cpu().numpy()
    K = KroneckerGram(p)
    r = K.matvec(a) - y
    assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(y)
    grid = gi.heat_grid(512, 1024)
    mean, var = gp.gpfvm_predict(grid, alpha, cov_mode=1)
    mean = mean.cpu().numpy()
    rng = np.random.default_rng(0)
    it = rng.integers(0, 512, 6)
    ix = rng.integers(0, 1024, 6)
    sub = gi.Grid([grid.points[0][it], grid.points[1][ix]])
    Ks = dense_cross_cov(p, sub)                      # 36 sampled points (6 x 6 sub-grid)
    ref = (Ks @ a).reshape(6, 6)
    got = mean.reshape(512, 1024)[np.ix_(it, ix)]
    # K_* alpha cancels heavily (|alpha| ~ |G^{-1} y|): the summation-order
    # bound is eps * (|K_*| |alpha|) per point
    bound = 64 * np.finfo(float).eps * (np.abs(Ks) @ np.abs(a)).reshape(6, 6)
    assert np.all(np.abs(got - ref) <= bound), np.max(np.abs(got - ref) / bound)
    true = gi.heat_analytic(p.meta["amps"], 0.1, grid.points[0], grid.points[1]).ravel()
    assert np.sqrt(np.mean((mean - true) ** 2)) < 2e-4
    v = var.cpu().numpy()
    # ||L^{-1} z||^2 form: no cancellation below zero; the domain is observed
    # everywhere (PDE cells + IC/BC), so the posterior variance is tiny
    assert v.min() >= -1e-12 and v.max() <= 1e-6, (v.min(), v.max())


def test_errors_and_call_order():
    p = gi.config0()
    gp = GpfvmProblem(p)
    with pytest.raises(GpfvmError, match="assemble"):
        gp.gpfvm_gram_matvec(_t(np.zeros(p.size)))
    gp.gpfvm_assemble_factors()
    x = _t(np.zeros(p.size))
    with pytest.raises(GpfvmError, match="alias"):
        gp.gpfvm_gram_matvec(x, out=x)


def test_kernels_actually_launch():
    n0 = launch_count()
    p = gi.config0()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    gp.gpfvm_gram_matvec(_t(np.ones(p.size)))
    torch.cuda.synchronize()
    assert launch_count() - n0 > 5


def _gpu_sygv(A, B):
    import ctypes as C
    from paper_2406_05020_b200 import _lib as L
    lib = L.load()
    n = A.shape[0]
    tA, tB = _t(A), _t(B)
    V = torch.empty((n, n), dtype=torch.float64, device=DEV)
    w = torch.empty(n, dtype=torch.float64, device=DEV)
    L.check(lib.gpfvm_sygv(n, C.c_void_p(tA.data_ptr()), C.c_void_p(tB.data_ptr()), C.c_void_p(V.data_ptr()),
                           C.c_void_p(w.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return V.cpu().numpy(), w.cpu().numpy()


@pytest.mark.parametrize("n", [15, 64, 100, 257])
def test_sygv_random_pencil_vs_lapack(n):
    """gpfvm_sygv on a well-conditioned random SPD pencil (no centrosymmetry):
    eigenvalues match LAPACK's generalised eigh to 1e-12, A V = B V diag(w),
    V^T B V = I."""
    import scipy.linalg as sl
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, n))
    A = X @ X.T / n + 0.5 * np.eye(n)
    Y = rng.standard_normal((n, n))
    B = Y @ Y.T / n + np.eye(n)
    V, w = _gpu_sygv(A, B)
    ref = sl.eigh(A, B, eigvals_only=True)
    assert np.abs(np.sort(w) - ref).max() <= 1e-12 * ref.max()
    assert np.abs(A @ V - B @ V * w).max() <= 1e-12 * np.abs(A).max() * np.abs(V).max() * n
    assert np.abs(V.T @ B @ V - np.eye(n)).max() <= 1e-12 * n


@pytest.mark.parametrize("n,q,ell", [(64, 2, 0.5), (128, 3, 0.05), (256, 2, 0.2)])
def test_sygv_centrosymmetric_matern_pencil(n, q, ell):
    """The FD pencils of uniform grids (interval Matérn factors of orders 0 and
    1, oracle-assembled) are centrosymmetric: the parity-split path must give
    the same pencil diagonalisation as the unsplit definition (residuals at the
    rounding level of the pencil, B-orthonormality, eigenvalues vs LAPACK
    where the pencil is resolvable)."""
    import scipy.linalg as sl
    cells = gi.cells(n)
    kp = (q, ell, 1.0)
    A = ofm(kp, cells, 0, cells, 0)   # T00 (ill-conditioned)
    B = ofm(kp, cells, 1, cells, 1)   # T11
    assert np.abs(A - A[::-1, ::-1]).max() <= 1e-14 * np.abs(A).max()
    V, w = _gpu_sygv(A, B)
    # B-orthonormality and the eigen-residual, normwise at the rounding level
    VtBV = V.T @ B @ V
    assert np.abs(VtBV - np.eye(n)).max() <= 1e-8
    R = A @ V - B @ V * w
    assert np.linalg.norm(R) <= 1e-10 * np.linalg.norm(A) * np.linalg.norm(V)
    # eigenvalues: the resolvable part of the spectrum matches LAPACK
    ref = np.sort(sl.eigh(A, B, eigvals_only=True))
    got = np.sort(w)
    big = ref > 1e-8 * ref.max()
    assert np.abs(got[big] - ref[big]).max() <= 1e-9 * ref.max()


def test_degenerate_cases():
    """Edge cases: zero right-hand side (alpha = 0, converged at once), zero
    input block (y = 0), a one-cell problem with one IC point (2 x 2 Gram vs
    the oracle), predict before solve."""
    p = gi.config0()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    z = _t(np.zeros(p.size))
    alpha, rep = gp.gpfvm_solve(z, rtol=1e-10)
    assert rep["converged"] and rep["iterations"] == 0
    assert float(alpha.abs().max()) == 0.0
    y = gp.gpfvm_gram_matvec(z.reshape(1, -1).contiguous())
    assert float(y.abs().max()) == 0.0
    # one PDE cell + one IC point: 2 x 2 Gram
    k = Kernel1D(2, 0.5)
    cell = Sites(gi.INTERVAL, np.array([0.0]), np.array([0.3]))
    one = Problem("one_cell", 2, [[k, Kernel1D(2, 0.4)]],
                  [Block("IC", [gi.points([0.0]), cell], [Term(1.0, (0, 0))], 1e-8, True, np.array([0.2])),
                   Block("PDE", [cell, cell], [Term(1.0, (1, 0)), Term(-0.1, (0, 2))], 0.0, False, np.array([0.0]))])
    G = dense_gram(one)
    g1 = GpfvmProblem(one)
    g1.gpfvm_assemble_factors()
    X = gi.random_vectors(one.size, 3, 5)
    _close(g1.gpfvm_gram_matvec(_t(X)).cpu().numpy(), X @ G.T, 1e-12)
    grid = gi.Grid([np.array([0.1, 0.2]), np.array([0.15])])
    # before any solve: ITERGP variance is the prior, PRECOND is a call-order error
    _, v0 = g1.gpfvm_predict(grid, _t(np.zeros(one.size)), cov_mode=0)
    assert np.allclose(v0.cpu().numpy(), 1.0)
    with pytest.raises(GpfvmError, match="solve"):
        g1.gpfvm_predict(grid, _t(np.zeros(one.size)), cov_mode=1)
    a1, r1 = g1.gpfvm_solve(_t(one.rhs()), rtol=1e-12)
    assert r1["converged"]
    assert np.allclose(a1.cpu().numpy(), np.linalg.solve(G, one.rhs()), rtol=1e-8, atol=0)


def test_itergp_variance_monotone_in_iterations():
    """IterGP combined variance (Wenger et al. 2022, P:l.299-302) is
    non-increasing in the iteration count and bounded below by the exact
    posterior variance (each action is a PSD downdate)."""
    from oracle.posterior import posterior_exact
    p = gi.config0()
    G = dense_gram(p)
    y = p.rhs()
    grid = gi.heat_grid(9, 9)
    _, v_ref, _ = posterior_exact(p, grid, G, y)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    prev = None
    for k in (1, 2, 4, 8, 16, 32):
        alpha, _ = gp.gpfvm_solve(_t(y), rtol=0.0, max_iter=k, precond=0)
        _, var = gp.gpfvm_predict(grid, alpha, cov_mode=0)
        v = var.cpu().numpy()
        assert np.all(v >= v_ref - 1e-10)
        if prev is not None:
            assert np.all(v <= prev + 1e-12)
        prev = v
