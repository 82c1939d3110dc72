"""The sharded path (paper_2406_05020_b200.dist) on the GPU through the library
kernels (GpuOps), world size 1 (the collectives are identities; their host
logic is covered by tests/test_dist.py with gloo, world size 2)."""
import numpy as np
import pytest

import gpfvm_inputs as gi
from gpfvm_inputs import Problem

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.gram import KroneckerGram  # noqa: E402
from paper_2406_05020_b200 import factor_matrix  # noqa: E402
from paper_2406_05020_b200.dist import GpuOps, heat_pde_operator, sharded_pcg  # noqa: E402


def _factors(p):
    kt, kx = p.kernels[0]
    T, X = p.blocks[3].sites
    return {"T00": factor_matrix(kt, T, 0, T, 0), "T11": factor_matrix(kt, T, 1, T, 1),
            "X00": factor_matrix(kx, X, 0, X, 0), "X22": factor_matrix(kx, X, 2, X, 2)}


@pytest.mark.parametrize("nt,nx", [(16, 32), (256, 512)])
def test_gpu_sharded_heat_operator_and_pcg(nt, nx):
    p = gi.heat_problem(nt, nx)
    pde = Problem("pde", 2, p.kernels, [p.blocks[3]])
    ops = GpuOps("cuda:0")
    A, fd = heat_pde_operator(ops, _factors(p), 0.1)
    x = gi.random_vectors(nt * nx, 1, 3)[0]
    y = A.matvec(torch.tensor(x, device="cuda:0")).cpu().numpy()
    ref = KroneckerGram(pde).matvec(x)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    # FD-preconditioned IterGP on the PDE block with a smooth right-hand side
    b = KroneckerGram(pde).matvec(np.sin(np.arange(nt * nx) * 0.001))
    res = sharded_pcg(ops, A, torch.tensor(b, device="cuda:0"), fd, rtol=1e-8, max_iter=30)
    assert res.converged and res.iterations <= 10, (res.iterations, res.residual_norms)
    a = res.x.cpu().numpy()
    r = KroneckerGram(pde).matvec(a) - b
    assert np.linalg.norm(r) <= 1e-7 * np.linalg.norm(b)


def test_gpu_sharded_3d_pde_block_matches_library():
    """block_kron_terms (R6 cancellation rebuilt on the host) + ShardedKron on a
    3D advection-diffusion PDE block == the library's own Gram matvec restricted
    to that block (the bench's N>1 sharded measurement path, world size 1)."""
    from paper_2406_05020_b200 import GpfvmProblem
    from paper_2406_05020_b200.dist import ShardedKron, block_kron_terms
    p = gi.advdiff_problem(16, 24, 24, n_modes=4)
    P = len(p.blocks) - 1
    pde = Problem("pde", 3, p.kernels, [p.blocks[P]])
    ops = GpuOps("cuda:0")
    coefs, facs = block_kron_terms(pde, 0)
    A = ShardedKron(ops, pde.blocks[0].shape, coefs, facs)
    gp = GpfvmProblem(pde)
    gp.gpfvm_assemble_factors()
    x = torch.tensor(gi.random_vectors(pde.size, 1, 4)[0], device="cuda:0")
    y = A.matvec(x)
    ref = gp.gpfvm_gram_matvec(x.reshape(1, -1).contiguous())[0]
    assert float((y - ref).abs().max()) <= 1e-12 * float(ref.abs().max())
