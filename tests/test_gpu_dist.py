"""The time-sharded path (paper_2406_05020_b200.dist + the library's
gpfvm_shard_* / gpfvm_iter_* calls) on one GPU: W = 1, 2, 3 ranks emulated in
one process (dist.LocalComm: the exchanges are device copies, no kernel waits
on another rank), every block of the problem sharded (IC planes on rank 0,
BC faces and the PDE block split in time, multi-output blocks), against the
oracle's Kronecker matvec and dense Cholesky (Eq. 20 / Eq. 5, PAPER.md
l.316-320, l.113)."""
import numpy as np
import pytest

import gpfvm_inputs as gi

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.gram import KroneckerGram, dense_gram  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem  # noqa: E402
from paper_2406_05020_b200.dist import LocalComm, ShardedProblem  # noqa: E402


def _sharded(p, W):
    gps = []
    for _ in range(W):
        gp = GpfvmProblem(p)
        gp.gpfvm_assemble_factors()
        gps.append(gp)
    return ShardedProblem(gps, LocalComm(W)), gps


def _full(sp, locals_, p):
    out = np.zeros(p.size)
    for i, loc in enumerate(locals_):
        off, row0, rows, spatial = sp.G.layout(i)
        l = loc.cpu().numpy()
        for J, b in enumerate(p.blocks):
            n = rows[J] * spatial[J]
            if n:
                s = p.offsets[J] + row0[J] * spatial[J]
                out[s:s + n] = l[off[J]:off[J] + n]
    return out


PROBLEMS = {
    "heat-16x24": lambda: gi.heat_problem(16, 24),
    "wave-8x10x12": lambda: gi.wave_problem(8, 10, 12, ell=(0.5, 0.3, 0.3)),
    "advdiff-9x8x8": lambda: gi.advdiff_problem(9, 8, 8, n_modes=4),
    "shallow-water-6x6x7": lambda: gi.shallow_water_problem(6, 6, 7),
}


@pytest.mark.parametrize("W", [1, 2, 3])
@pytest.mark.parametrize("name", list(PROBLEMS))
def test_sharded_matvec_vs_oracle(name, W):
    p = PROBLEMS[name]()
    sp, gps = _sharded(p, W)
    x = gi.random_vectors(p.size, 1, 17)[0]
    xt = torch.tensor(x, device="cuda:0")
    ys = sp.matvec(sp.local([xt] * W))
    y = _full(sp, ys, p)
    ref = KroneckerGram(p).matvec(x)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    # the second application reuses the plan and buffers
    y2 = _full(sp, sp.matvec(sp.local([xt] * W)), p)
    assert np.array_equal(y, y2)
    sp.close()


@pytest.mark.parametrize("W", [1, 2, 3])
def test_sharded_solve_vs_cholesky(W):
    """Sharded IterGP with the sharded block-Jacobi FD preconditioner: the
    solution equals the dense Cholesky one and the iteration count equals the
    single-GPU solve with the same preconditioner (GPFVM_FORCE_BJFD)."""
    p = gi.wave_problem(6, 8, 8, ell=(0.5, 0.3, 0.3), ic="sine")
    G = dense_gram(p)
    y = p.rhs()
    a_ref = np.linalg.solve(G, y)
    sp, gps = _sharded(p, W)
    yt = torch.tensor(y, device="cuda:0")
    xs, rep = sp.solve(sp.local([yt] * W), rtol=1e-11, max_iter=400)
    assert rep.converged and not rep.breakdown, rep
    a = _full(sp, xs, p)
    assert np.linalg.norm(G @ a - y) <= 1e-10 * np.linalg.norm(y)
    assert np.linalg.norm(a - a_ref) <= 1e-6 * np.linalg.norm(a_ref)
    sp.close()


def test_sharded_solve_matches_single_gpu_iterations(monkeypatch):
    monkeypatch.setenv("GPFVM_FORCE_BJFD", "1")
    p = gi.advdiff_problem(8, 8, 8, n_modes=4)
    y = p.rhs()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    yt = torch.tensor(y, device="cuda:0")
    _, rep1 = gp.gpfvm_solve(yt, rtol=1e-9, max_iter=500)
    sp, _ = _sharded(p, 2)
    xs, rep2 = sp.solve(sp.local([yt] * 2), rtol=1e-9, max_iter=500)
    assert rep1["converged"] and rep2.converged
    assert abs(rep1["iterations"] - rep2.iterations) <= 2, (rep1["iterations"], rep2.iterations)
    sp.close()


@pytest.mark.parametrize("W", [2, 3])
def test_sharded_predict_mean(W):
    """Sharded posterior mean (partial sums over the owned time rows +
    all_reduce) equals the oracle's Cholesky posterior mean."""
    from oracle.posterior import posterior_exact
    p = gi.wave_problem(6, 8, 8, ell=(0.5, 0.3, 0.3), ic="sine")
    G = dense_gram(p)
    y = p.rhs()
    grid = gi.Grid([np.linspace(0, 1, 5), np.linspace(0.1, 0.9, 4), np.linspace(0, 1, 3)])
    m_ref, _, _ = posterior_exact(p, grid, G, y)
    sp, gps = _sharded(p, W)
    yt = torch.tensor(y, device="cuda:0")
    xs, rep = sp.solve(sp.local([yt] * W), rtol=1e-12, max_iter=600)
    assert rep.converged
    means = sp.predict_mean(grid, xs)
    for m in means:
        assert np.abs(m.cpu().numpy() - m_ref).max() <= 1e-8 * np.abs(m_ref).max()
    sp.close()
