"""Pins for the oracle's Gram assembly, Kronecker matvec, solvers and posterior (CPU only)."""
import mpmath as mp
import numpy as np
import pytest
import scipy.linalg as sl

import gpfvm_inputs as gi
from gpfvm_inputs import Block, Kernel1D, Problem, Sites, Term
from oracle.gram import KroneckerGram, dense_cross_cov, dense_gram, factor_matrix, prior_variance
from oracle.matern import matern_direct
from oracle.posterior import posterior_exact, variance_itergp, variance_precond
from oracle.solve import BlockLDLPreconditioner, FDPreconditioner, cholesky_solve, itergp_cg


def _random_problem(seed, ndim=3, n_outputs=1):
    """Small random factorized scheme: non-uniform cells, multi-term
    operators, point blocks, (optionally) several outputs."""
    rng = np.random.default_rng(seed)
    kern = [[Kernel1D(int(rng.integers(2, 4)), float(rng.uniform(0.2, 0.8)), float(rng.uniform(0.5, 2)))
             for _ in range(ndim)] for _ in range(n_outputs)]
    blocks = []
    for b in range(3):
        sites = []
        for i in range(ndim):
            n = int(rng.integers(2, 5))
            if b == 2 and i == 0:
                sites.append(gi.points(np.sort(rng.uniform(0, 1, 2))))
            else:
                e = np.sort(np.concatenate([[0.0, 1.0], rng.uniform(0, 1, n - 1)]))
                sites.append(Sites(gi.INTERVAL, e[:-1], e[1:]))
        nterm = int(rng.integers(1, 4))
        terms = []
        for _ in range(nterm):
            order = tuple(int(rng.integers(0, 3)) if not (b == 2 and i == 0) else int(rng.integers(0, 2))
                          for i in range(ndim))
            terms.append(Term(float(rng.standard_normal()), order, int(rng.integers(0, n_outputs))))
        blk = Block(f"B{b}", sites, terms, 0.0, b != 0, np.zeros(0))
        blk.rhs = np.zeros(blk.size)
        blocks.append(blk)
    return Problem(f"rand{seed}", ndim, kern, blocks)


@pytest.mark.parametrize("seed,ndim,nout", [(0, 3, 1), (1, 2, 1), (2, 3, 2), (3, 1, 1), (4, 3, 3)])
def test_kronecker_matvec_equals_dense(seed, ndim, nout):
    p = _random_problem(seed, ndim, nout)
    G = dense_gram(p)
    K = KroneckerGram(p)
    X = gi.random_vectors(p.size, 3, seed)
    Y = K.matvec(X)
    ref = X @ G.T
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("seed,ndim,nout", [(0, 3, 1), (2, 3, 2), (5, 2, 1)])
def test_gram_symmetric_psd(seed, ndim, nout):
    p = _random_problem(seed, ndim, nout)
    G = dense_gram(p)
    assert np.abs(G - G.T).max() <= 1e-14 * np.abs(G).max()
    w = np.linalg.eigvalsh(G)
    assert w[0] >= -1e-10 * w[-1]


def test_multioutput_zero_cross_covariance():
    """Eq. 17-19: functionals on different outputs are uncorrelated."""
    p = _random_problem(7, 2, 2)
    for b in p.blocks:
        for t in b.terms:
            t.output = 0
    p.blocks[1].terms = [Term(1.0, (0, 0), 1)]
    G = dense_gram(p)
    off = p.offsets
    assert np.all(G[off[1]:off[2], off[0]:off[1]] == 0.0)


def test_config0_gram_entry_bruteforce():
    """One PDE-cell x point-observation entry of config 0 against a 2D
    quadrature of (d_t - kappa d_xx) applied to the literal product kernel
    (Eq. 8 + Eq. 13): checks the multi-dimensional reduction of Eq. 15."""
    p = gi.config0()
    kt, kx = p.kernels[0]
    t0, x0 = 0.3, 0.55
    a_t, b_t = 2 / 16, 3 / 16
    a_x, b_x = 8 / 16, 9 / 16
    kap = p.meta["kappa"]
    ft = lambda d: matern_direct(kt.q, kt.lengthscale, 1.0, d)
    fx = lambda d: matern_direct(kx.q, kx.lengthscale, 1.0, d)
    with mp.workdps(25):
        def integrand(t, x):
            dk_t = mp.diff(ft, t - t0, 1)
            dk_xx = mp.diff(fx, x - x0, 2)
            return dk_t * fx(x - x0) - kap * ft(t - t0) * dk_xx
        ref = mp.quad(integrand, [a_t, b_t], [a_x, x0, b_x])
    T = Sites(gi.INTERVAL, np.array([a_t]), np.array([b_t]))
    X = Sites(gi.INTERVAL, np.array([a_x]), np.array([b_x]))
    PT = gi.points([t0])
    PX = gi.points([x0])
    got = (factor_matrix((kt.q, kt.lengthscale, 1.0), T, 1, PT, 0)[0, 0] *
           factor_matrix((kx.q, kx.lengthscale, 1.0), X, 0, PX, 0)[0, 0] -
           kap * factor_matrix((kt.q, kt.lengthscale, 1.0), T, 0, PT, 0)[0, 0] *
           factor_matrix((kx.q, kx.lengthscale, 1.0), X, 2, PX, 0)[0, 0])
    assert abs(got - float(ref)) <= 1e-10 * abs(float(ref))


def test_heat_posterior_converges_to_analytic_solution():
    """Posterior mean -> e^{-0.1 pi^2 t} sin(pi x) under grid refinement
    (BASELINE.json north_star oracle pin)."""
    g = gi.heat_grid(33, 33)
    true = gi.heat_analytic(np.array([1.0]), 0.1, g.points[0], g.points[1]).ravel()
    errs = []
    for n in [8, 16, 32]:
        p = gi.heat_problem(n, n)
        G = dense_gram(p)
        m, v, _ = posterior_exact(p, g, G, p.rhs())
        errs.append(np.sqrt(np.mean((m - true) ** 2)))
        assert v.min() >= -1e-8 and v.max() <= 1.0 + 1e-12
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 5e-4
    rate = np.log2(errs[1] / errs[2])
    assert rate > 1.5, errs


def test_wave_posterior_converges_to_analytic_solution():
    """2D wave equation u_tt = u_xx + u_yy (P:l.694) with the sine initial
    condition of the paper's wave benchmark (i = j = 1 mode, P:l.703),
    u_t(0) = 0 and Dirichlet-0 faces: the posterior mean converges to
    cos(sqrt2 pi t) sin(pi x) sin(pi y) under grid refinement.  Pins the 3D
    Kronecker Gram, the Matérn-7/2 order-2 functionals and the u_t(0) block."""
    pts = [np.array([0.2, 0.45, 0.7]), np.array([0.3, 0.5]), np.array([0.35, 0.6])]
    grid = gi.Grid(pts)
    true = gi.wave_analytic_sine(1.0, *pts).ravel()
    errs = []
    for n in [4, 6, 8, 10]:
        p = gi.wave_problem(n, n, n, ell=(0.5, 0.3, 0.3), q=3, ic="sine")
        G = dense_gram(p)
        m, v, _ = posterior_exact(p, grid, G, p.rhs())
        errs.append(np.abs(m - true).max())
        assert v.min() >= -1e-8
    assert errs[0] > errs[1] > errs[2] > errs[3], errs
    assert errs[3] < 1e-2, errs
    rate = np.log(errs[1] / errs[3]) / np.log(10 / 6)
    assert rate > 3.0, (rate, errs)


def test_ic_observations_reproduced():
    """The posterior mean integrated over the IC cells reproduces the IC data
    (noise 1e-8 h^2), i.e. the solve honours the information operator."""
    p = gi.config0()
    G = dense_gram(p)
    alpha = cholesky_solve(G, p.rhs())
    ic = G[:16] @ alpha
    assert np.abs(ic - p.blocks[0].rhs).max() <= 1e-6 * np.abs(p.blocks[0].rhs).max()


def test_cholesky_small_exact():
    G = np.array([[2.0, 1.0], [1.0, 2.0]])
    x = cholesky_solve(G, np.array([1.0, 0.0]))
    assert np.allclose(x, [2 / 3, -1 / 3], atol=1e-15)


def test_itergp_full_budget_equals_cholesky():
    """§4.1: IterGP-CG 'produces an exact posterior' at full budget."""
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((60, 60)))
    G = (Q * np.logspace(0, 4, 60)) @ Q.T
    b = rng.standard_normal(60)
    tr = itergp_cg(lambda v: G @ v, b, rtol=1e-13, max_iter=60)
    x = cholesky_solve(G, b)
    assert np.abs(tr.x - x).max() <= 1e-10 * np.abs(x).max()
    D = np.stack(tr.directions)
    GD = D @ G @ D.T
    off = GD - np.diag(np.diag(GD))
    assert np.abs(off).max() <= 1e-10 * np.abs(np.diag(GD)).max()
    C = sum(np.outer(d, d) / e for d, e in zip(tr.directions, tr.etas))
    # C_i is the G-orthogonal projector onto the explored Krylov space: C G d_j = d_j, x_i = C_i b
    assert np.abs(C @ G @ D.T - D.T).max() <= 1e-8 * np.abs(D).max()
    assert np.abs(C @ b - tr.x).max() <= 1e-12 * np.abs(x).max()


def test_itergp_variance_monotone_and_conservative():
    """Combined variance is non-increasing in the iteration count and never
    below the exact posterior variance (computational uncertainty >= 0)."""
    p = gi.heat_problem(8, 8)
    G = dense_gram(p)
    g = gi.heat_grid(9, 9)
    _, vex, _ = posterior_exact(p, g, G, p.rhs())
    tr = itergp_cg(lambda v: G @ v, p.rhs(), rtol=0.0, max_iter=40)
    prev = None
    for i in range(0, 41, 5):
        v = variance_itergp(p, g, tr.directions[:i], tr.etas[:i])
        assert np.all(v >= vex - 1e-10)
        if prev is not None:
            assert np.all(v <= prev + 1e-12)
        prev = v


def test_fd_preconditioner_exact_for_heat_block():
    """for the noise-free heat PDE block FD = G_pp^{-1}."""
    p = gi.config0()
    G = dense_gram(p)
    fd = FDPreconditioner(p, 3)
    o = p.offsets
    Gpp = G[o[3]:, o[3]:]
    x = gi.random_vectors(Gpp.shape[0], 1, 1)[0]
    assert np.abs(fd.apply(Gpp @ x) - x).max() <= 1e-6 * np.abs(x).max()


def test_block_ldl_preconditioner_and_pcg_config0():
    p = gi.config0()
    G = dense_gram(p)
    P = BlockLDLPreconditioner(p, G)
    y = p.rhs()
    tr = itergp_cg(lambda v: G @ v, y, P.apply, rtol=1e-10, max_iter=20)
    assert tr.converged and tr.iterations <= 3
    g = gi.heat_grid(16, 16)
    m, v, alpha = posterior_exact(p, g, G, y)
    Ks = dense_cross_cov(p, g)
    assert np.abs(Ks @ tr.x - m).max() <= 1e-9 * np.abs(m).max()
    vp = variance_precond(p, g, P.apply)
    assert np.abs(vp - v).max() <= 1e-10


def _sw_means(p):
    G = dense_gram(p)
    y = p.rhs()
    ts, xs, ys = np.array([0.2, 0.6]), np.array([0.1, 0.3, 0.7, 0.9]), np.array([0.2, 0.5, 0.8])
    out = []
    for o in (0, 1, 2):
        m, _, _ = posterior_exact(p, gi.Grid([ts, xs, ys], output=o), G, y)
        out.append(m.reshape(2, 4, 3))
    return out


def test_shallow_water_mirror_symmetry_locks_radiation_signs():
    """Linearised shallow water (P:l.746-761) with a centred, noise-free IC on a
    symmetric grid: the posterior mean of eta and v is mirror-symmetric in x and
    u antisymmetric (and eta, u symmetric / v antisymmetric in y).  This locks
    the per-face signs of the radiation conditions (the paper states only the
    x = 0 face, reading R5/SPEC): flipping one face's sign breaks the symmetry."""
    p = gi.shallow_water_problem(3, 4, 4, center=(0.5, 0.5), noise_frac=0.0)
    eta, u, v = _sw_means(p)
    scale = max(np.abs(eta).max(), np.abs(u).max(), np.abs(v).max())
    tol = 1e-10 * scale
    assert np.abs(eta - eta[:, ::-1, :]).max() <= tol and np.abs(eta - eta[:, :, ::-1]).max() <= tol
    assert np.abs(u + u[:, ::-1, :]).max() <= tol and np.abs(u - u[:, :, ::-1]).max() <= tol
    assert np.abs(v - v[:, ::-1, :]).max() <= tol and np.abs(v + v[:, :, ::-1]).max() <= tol
    # a wrong sign on the x = 1 face must be visible
    bad = gi.shallow_water_problem(3, 4, 4, center=(0.5, 0.5), noise_frac=0.0)
    for b in bad.blocks:
        if b.name == "BCx1":
            b.terms[1] = Term(-b.terms[1].coeff, b.terms[1].order, b.terms[1].output)
    eta_b, _, _ = _sw_means(bad)
    assert np.abs(eta_b - eta_b[:, ::-1, :]).max() > 1e3 * tol


def test_fvm_functional_tends_to_collocation():
    """FVM/collocation consistency: (1/h^2) x the interval-interval factor of
    cells of width h centred at x, y tends to the point-point kernel k(x - y)
    as h -> 0, at second order (midpoint rule)."""
    from oracle.gram import factor_matrix
    kp = (2, 0.3, 1.0)
    xs = np.array([0.2, 0.55])
    ref = factor_matrix(kp, gi.points(xs), 0, gi.points(xs), 0)
    errs = []
    for h in (0.1, 0.05, 0.025):
        cells = gi.Sites(gi.INTERVAL, xs - h / 2, xs + h / 2)
        F = factor_matrix(kp, cells, 0, cells, 0) / h ** 2
        errs.append(np.abs(F - ref).max())
    assert errs[0] > errs[1] > errs[2]
    assert np.log2(errs[1] / errs[2]) > 1.5, errs


def test_itergp_variance_full_budget_equals_exact():
    """At full budget (N iterations, full reorthogonalisation) IterGP's
    C_N = sum_j d_j d_j^T / eta_j is G^{-1} (its directions are a G-conjugate
    basis of R^N; Wenger et al. via PAPER.md §4.1 l.299-302), so the combined
    variance equals the exact posterior variance of Eq. 6 (l.114).  Dropping
    the last direction leaves a visible computational-uncertainty gap."""
    p = gi.heat_problem(4, 4)
    G = dense_gram(p)
    N = G.shape[0]
    g = gi.heat_grid(7, 7)
    _, vex, _ = posterior_exact(p, g, G, p.rhs())
    tr = itergp_cg(lambda v: G @ v, p.rhs(), rtol=0.0, max_iter=N)
    assert len(tr.etas) == N
    v = variance_itergp(p, g, tr.directions, tr.etas)
    prior = prior_variance(p, 0)
    assert np.abs(v - vex).max() <= 1e-9 * prior
    v_short = variance_itergp(p, g, tr.directions[:N - 4], tr.etas[:N - 4])
    assert np.abs(v_short - vex).max() >= 1e-7 * prior
