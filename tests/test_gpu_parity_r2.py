"""Parity cases added in round 2 (VERDICT r1 "close the parity gaps"):

* 3D matvecs at sizes that reach the full-size plan (per-term factor sharing
  needs n_x >= 64 and n_y >= 32; the TMA tensor-core path needs >= 148 64x64
  tiles) against the oracle's plain Kronecker matvec, element by element at
  1e-12 of max|ref| (Eq. 20);
* the full-size config-3 and config-4 Grams against the oracle on one vector;
* cold processes (the first matvec of a fresh process, where a TMA pipeline
  race once showed up) against the oracle;
* the PRECOND posterior variance of a heat problem on the structured block-LDL
  path, forced through several ragged predict slabs, against the oracle's dense
  Cholesky posterior (Eq. 6, l.114) at 1e-8 x prior variance.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import gpfvm_inputs as gi

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.gram import KroneckerGram, dense_gram, prior_variance  # noqa: E402
from oracle.posterior import posterior_exact  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _t(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")


def _elementwise(Y, ref, tol=1e-12):
    err = np.abs(Y - ref).max()
    scale = np.abs(ref).max()
    assert err <= tol * scale, f"max |Y - ref| = {err:.3e} > {tol:g} x max|ref| = {tol * scale:.3e}"


@pytest.mark.parametrize("builder", [
    lambda: gi.advdiff_problem(16, 64, 64, n_modes=32),
    lambda: gi.shallow_water_problem(12, 64, 64),
    lambda: gi.wave_problem(16, 64, 64),
], ids=["advdiff-16x64x64", "shallow-water-12x64x64", "wave-16x64x64"])
def test_plan_size_3d_matvec_vs_oracle(builder):
    p = builder()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, 3, 31)
    ref = KroneckerGram(p).matvec(X)
    xt = _t(X)
    out = torch.empty_like(xt)
    for _ in range(3):  # direct launch, graph capture, graph replay
        gp.gpfvm_gram_matvec(xt, out=out)
        _elementwise(out.cpu().numpy(), ref)


@pytest.mark.parametrize("cfg", [gi.config3, gi.config4], ids=["config3", "config4"])
def test_fullsize_3d_matvec_vs_oracle(cfg):
    p = cfg()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, 1, 41)
    Y = gp.gpfvm_gram_matvec(_t(X)).cpu().numpy()
    ref = KroneckerGram(p).matvec(X)
    _elementwise(Y, ref)


_COLD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import gpfvm_inputs as gi
from paper_2406_05020_b200 import GpfvmProblem
p = gi.config2()
gp = GpfvmProblem(p); gp.gpfvm_assemble_factors()
X = gi.random_vectors(p.size, 4, 21)
Y = gp.gpfvm_gram_matvec(torch.tensor(X, device="cuda:0")).cpu().numpy()
np.save({out!r}, Y)
"""


def test_cold_process_config2_matvec_vs_oracle(tmp_path):
    p = gi.config2()
    ref = KroneckerGram(p).matvec(gi.random_vectors(p.size, 4, 21))
    for i in range(3):
        out = str(tmp_path / f"y{i}.npy")
        subprocess.run([sys.executable, "-c", _COLD.format(root=ROOT, out=out)], check=True, cwd=ROOT, timeout=600)
        _elementwise(np.load(out), ref)


def test_precond_variance_multislab_vs_oracle(monkeypatch):
    amps = np.random.default_rng(5).normal(size=4) / np.arange(1, 5)
    p = gi.heat_problem(32, 128, amps=amps)
    G = dense_gram(p)
    y = p.rhs()
    grid = gi.heat_grid(37, 96)
    m_ref, v_ref, _ = posterior_exact(p, grid, G, y)
    prior = prior_variance(p, 0)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    alpha, rep = gp.gpfvm_solve(_t(y), rtol=1e-12, max_iter=50)
    assert rep["converged"], rep
    monkeypatch.setenv("GPFVM_PREDICT_SLAB_ROWS", "8")  # 37 rows: 5 slabs, the last ragged
    mean, var = gp.gpfvm_predict(grid, alpha, cov_mode=1)
    mean, var = mean.cpu().numpy(), var.cpu().numpy()
    assert np.abs(mean - m_ref).max() <= 1e-8 * np.abs(m_ref).max()
    assert np.abs(var - v_ref).max() <= 1e-8 * prior
    monkeypatch.delenv("GPFVM_PREDICT_SLAB_ROWS")
    _, var1 = gp.gpfvm_predict(grid, alpha, cov_mode=1, want_mean=False)
    assert np.abs(var1.cpu().numpy() - var).max() <= 1e-11 * prior  # slab plans differ only in rounding


@pytest.mark.parametrize("builder,precond", [
    (lambda: gi.wave_problem(6, 8, 8, ell=(0.5, 0.3, 0.3), ic="sine"), 2),   # block-Jacobi FD: batched
    (lambda: gi.advdiff_problem(6, 8, 8, n_modes=4), 2),
    (lambda: gi.heat_problem(12, 16), 2),                                   # exact 2D path: sequential
    (lambda: gi.heat_problem(8, 8), 0),                                     # no preconditioner: batched
], ids=["wave-bjfd", "advdiff-bjfd", "heat-exact", "heat-none"])
def test_solve_many_vs_cholesky(builder, precond):
    """gpfvm_solve_many (several right-hand sides, one IterGP run each, shared
    batched preconditioner and matvec) against the dense Cholesky solutions;
    right-hand side 0 matches the single-RHS solve and its Krylov store drives
    the ITERGP variance."""
    p = builder()
    G = dense_gram(p)
    rng = np.random.default_rng(7)
    Y = np.stack([p.rhs(), G @ rng.normal(size=p.size), 0.5 * p.rhs() + G @ rng.normal(size=p.size)])
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    A, reps = gp.gpfvm_solve(_t(Y), rtol=1e-10, max_iter=3000, precond=precond)
    A = A.cpu().numpy()
    for r in range(3):
        assert reps[r]["converged"], (r, reps[r])
        res = np.linalg.norm(G @ A[r] - Y[r]) / np.linalg.norm(Y[r])
        assert res <= 2e-10 and abs(reps[r]["true_rel_residual"] - res) <= 1e-10 * max(1.0, res / 1e-10)
        if r == 0:  # the smooth physical right-hand side: solution to the north_star 1e-8
            ref = np.linalg.solve(G, Y[r])
            assert np.linalg.norm(A[r] - ref) <= 1e-6 * np.linalg.norm(ref)
    grid = gi.Grid([np.linspace(0, 1, 4) for _ in range(p.ndim)])
    _, v_many = gp.gpfvm_predict(grid, _t(A[0]), cov_mode=0)
    a0, rep0 = gp.gpfvm_solve(_t(Y[0]), rtol=1e-10, max_iter=3000, precond=precond)
    assert abs(rep0["iterations"] - reps[0]["iterations"]) <= 2
    _, v_one = gp.gpfvm_predict(grid, a0, cov_mode=0)
    assert np.abs(v_many.cpu().numpy() - v_one.cpu().numpy()).max() <= 1e-8
