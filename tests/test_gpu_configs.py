"""BASELINE configs 2-4 (3D wave, advection-diffusion, multi-output shallow
water) through the C ABI: full-size config-2 matvec against the oracle's
Kronecker matvec (4-RHS batch, the bench launch configuration), reduced-size
configs 3/4 against the dense oracle, and full-size properties (symmetry of
G, linearity) for configs 3/4 where the oracle is too slow."""
import numpy as np
import pytest

import gpfvm_inputs as gi

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.gram import KroneckerGram, dense_gram  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem  # noqa: E402


def _t(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")


def test_config2_fullsize_matvec_4rhs_vs_oracle():
    p = gi.config2()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, 4, 21)
    Y = gp.gpfvm_gram_matvec(_t(X)).cpu().numpy()
    ref = KroneckerGram(p).matvec(X)
    assert np.abs(Y - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("builder", [
    lambda: gi.wave_problem(4, 6, 5),
    lambda: gi.advdiff_problem(4, 6, 6, n_modes=4),
    lambda: gi.shallow_water_problem(3, 4, 5),
])
def test_reduced_configs_vs_dense_oracle(builder):
    p = builder()
    G = dense_gram(p)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, 3, 4)
    Y = gp.gpfvm_gram_matvec(_t(X)).cpu().numpy()
    ref = X @ G.T
    assert np.abs(Y - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("cfg", [gi.config3, gi.config4])
def test_fullsize_3d_properties(cfg):
    p = cfg()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = _t(gi.random_vectors(p.size, 2, 9))
    Y = gp.gpfvm_gram_matvec(X)
    # symmetry: x^T G y = y^T G x
    a = float(torch.dot(X[0], Y[1]))
    b = float(torch.dot(X[1], Y[0]))
    assert abs(a - b) <= 1e-10 * (abs(a) + abs(b))
    # linearity of the batch: G(x0 + 2 x1) = G x0 + 2 G x1
    Z = gp.gpfvm_gram_matvec((X[0] + 2 * X[1]).reshape(1, -1).contiguous())
    ref = Y[0] + 2 * Y[1]
    assert float((Z[0] - ref).abs().max()) <= 1e-12 * float(ref.abs().max())
    # positive semi-definite in the sampled directions
    assert float(torch.dot(X[0], Y[0])) > 0


@pytest.mark.parametrize("builder", [
    lambda: gi.wave_problem(4, 6, 6),
    lambda: gi.advdiff_problem(4, 6, 6, n_modes=4),
    lambda: gi.shallow_water_problem(3, 4, 4),
])
def test_3d_solve_blockjacobi_fd_vs_cholesky(builder):
    """General-case preconditioner (block-Jacobi fast diagonalisation, DESIGN.md
    §5.4): PCG/IterGP converges and matches the oracle's Cholesky solution and
    posterior mean; ITERGP variance is within [exact, prior]."""
    from oracle.posterior import posterior_exact
    p = builder()
    G = dense_gram(p)
    y = p.rhs()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=1e-13, max_iter=4000)
    assert rep["converged"], rep
    a = alpha.cpu().numpy()
    assert np.linalg.norm(G @ a - y) <= 1e-12 * np.linalg.norm(y)
    grid = gi.Grid([np.linspace(0, 1, 5), np.linspace(0, 1, 4), np.linspace(0, 1, 3)])
    m_ref, v_ref, _ = posterior_exact(p, grid, G, y)
    mean, var = gp.gpfvm_predict(grid, alpha, cov_mode=0)
    mean = mean.cpu().numpy()
    # north_star: posterior mean within 1e-8 relative
    assert np.abs(mean - m_ref).max() <= 1e-8 * max(1e-12, np.abs(m_ref).max())
    v = var.cpu().numpy()
    assert np.all(v >= v_ref - 1e-8) and np.all(v <= 1.0 + 1e-12)


@pytest.mark.parametrize("window,keep", [(1, True), (8, True), (1, False), (4, False)])
def test_3d_solve_reorth_window(window, keep):
    """gpfvm_solve_opts.reorth_window (R7): windowed
    reorthogonalisation still converges to the Cholesky solution (w = 1 is the
    plain PCG recurrence, identical to full reorthogonalisation in exact
    arithmetic)."""
    p = gi.wave_problem(4, 6, 6)
    G = dense_gram(p)
    y = p.rhs()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=1e-10, max_iter=4000, reorth_window=window, keep_actions=keep)
    assert rep["converged"], rep
    a = alpha.cpu().numpy()
    assert np.linalg.norm(G @ a - y) <= 1e-9 * np.linalg.norm(y)
    a_ref = np.linalg.solve(G, y)
    assert np.linalg.norm(a - a_ref) <= 1e-6 * np.linalg.norm(a_ref)
    # the ITERGP variance of the kept actions is a valid (conservative) bound
    from oracle.posterior import posterior_exact
    grid = gi.Grid([np.linspace(0, 1, 4), np.linspace(0, 1, 3), np.linspace(0, 1, 3)])
    _, v_ref, _ = posterior_exact(p, grid, G, y)
    _, var = gp.gpfvm_predict(grid, alpha, cov_mode=0)
    v = var.cpu().numpy()
    assert np.all(v >= v_ref - 1e-8) and np.all(v <= 1.0 + 1e-12)


def test_wave_sine_solve_predict_vs_oracle_and_analytic():
    """GPU solve (block-Jacobi FD PCG) + predict on the sine-IC wave problem:
    posterior mean equals the oracle's Cholesky posterior (1e-8 relative) and
    the analytic solution within the oracle's own discretisation error."""
    from oracle.posterior import posterior_exact
    pts = [np.array([0.2, 0.45, 0.7]), np.array([0.3, 0.5]), np.array([0.35, 0.6])]
    grid = gi.Grid(pts)
    p = gi.wave_problem(8, 8, 8, ell=(0.5, 0.3, 0.3), q=3, ic="sine")
    G = dense_gram(p)
    y = p.rhs()
    m_ref, v_ref, _ = posterior_exact(p, grid, G, y)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=1e-12, max_iter=3000)
    assert rep["converged"], rep
    mean, var = gp.gpfvm_predict(grid, alpha, cov_mode=0)
    mean = mean.cpu().numpy()
    assert np.abs(mean - m_ref).max() <= 1e-8 * np.abs(m_ref).max()
    true = gi.wave_analytic_sine(1.0, *pts).ravel()
    assert np.abs(mean - true).max() < 2e-2


def test_shallow_water_mirror_symmetry_gpu():
    """GPU solve + predict of the centred shallow-water problem: eta is mirror
    symmetric in x, u antisymmetric (radiation-BC sign lock on the CUDA path),
    and the means equal the oracle posterior."""
    from oracle.posterior import posterior_exact
    p = gi.shallow_water_problem(3, 4, 4, center=(0.5, 0.5), noise_frac=0.0)
    G = dense_gram(p)
    y = p.rhs()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=1e-12, max_iter=3000)
    assert rep["converged"], rep
    ts, xs, ys = np.array([0.2, 0.6]), np.array([0.1, 0.3, 0.7, 0.9]), np.array([0.2, 0.5, 0.8])
    for out, sign in ((0, 1.0), (1, -1.0)):
        grid = gi.Grid([ts, xs, ys], output=out)
        m, _ = gp.gpfvm_predict(grid, alpha, cov_mode=0, want_var=False)
        m = m.cpu().numpy()
        m_ref, _, _ = posterior_exact(p, grid, G, y)
        scale = np.abs(m_ref).max()
        assert np.abs(m - m_ref).max() <= 1e-8 * scale
        m3 = m.reshape(2, 4, 3)
        assert np.abs(m3 - sign * m3[:, ::-1, :]).max() <= 1e-8 * scale
