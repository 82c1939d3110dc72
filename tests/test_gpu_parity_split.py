"""GPU parity of the reflection-parity split of the Kronecker-sum matvec
(KronSum::par): on a mirror-symmetric site list every factor of
a stationary kernel satisfies F[n-1-i][n-1-j] = (-1)^(m+m') F[i][j], so the
diagonal block pairs of Eq. 20 run on even/odd parts with
half-size factors.  The oracle knows nothing of this: it is compared through
the dense Gram / plain Kronecker matvec, element by element at 1e-12 of
max|ref|.  Cases: graded (non-uniform) mirror-symmetric cells, noisy PDE
block, three-term operator, R = 1 / ragged R, and problems where the split
must NOT apply (odd cell counts, asymmetric cells, mixed-parity advection)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import gpfvm_inputs as gi
from gpfvm_inputs import Block, Kernel1D, Problem, Sites, Term

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.gram import KroneckerGram, dense_gram  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _t(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")


def _elementwise(Y, ref, tol=1e-12):
    err = np.abs(Y - ref).max() / np.abs(ref).max()
    assert err <= tol, err


def _graded(n, beta=0.35):
    """n cells on [0, 1], graded towards both ends, mirror-symmetric."""
    s = np.linspace(-1.0, 1.0, n + 1)
    e = 0.5 + 0.5 * (s + beta * np.sin(np.pi * s) / np.pi) / (1.0 + 0.0)
    e = 0.5 * (e + (1.0 - e[::-1]))      # exact mirror symmetry up to rounding
    e[0], e[-1] = 0.0, 1.0
    return Sites(gi.INTERVAL, e[:-1].copy(), e[1:].copy())


def _heat_like(T, X, terms, pde_noise=0.0, q=2, ell=(0.4, 0.15)):
    nt, nx = T.n, X.n
    blocks = [
        Block("IC", [gi.point(0.0), X], [Term(1.0, (0, 0))], 1e-8 / nx ** 2, True, np.zeros(nx)),
        Block("BC0", [T, gi.point(0.0)], [Term(1.0, (0, 0))], 1e-8 / nt ** 2, True, np.zeros(nt)),
        Block("BC1", [T, gi.point(1.0)], [Term(1.0, (0, 0))], 1e-8 / nt ** 2, True, np.zeros(nt)),
        Block("PDE", [T, X], terms, pde_noise, False, np.zeros(nt * nx)),
    ]
    kern = [[Kernel1D(q, ell[0], 1.0), Kernel1D(q, ell[1], 1.3)]]
    return Problem(f"heatlike_{nt}x{nx}", 2, kern, blocks)


HEAT = [Term(1.0, (1, 0)), Term(-0.1, (0, 2))]
THREE = [Term(1.0, (1, 0)), Term(-0.05, (0, 2)), Term(0.7, (0, 0))]
ADV = [Term(1.0, (1, 0)), Term(0.8, (0, 1)), Term(-0.02, (0, 2))]


def _pde_pair_flops(nt, nx, P):
    return 2.0 * P * nt * nx * (nt + nx)


@pytest.mark.parametrize("case", ["graded", "graded_noise", "three_terms", "uniform_rect"])
def test_parity_split_vs_dense_oracle(case):
    if case == "graded":
        p, P = _heat_like(_graded(24), _graded(40), HEAT), 2
    elif case == "graded_noise":
        p, P = _heat_like(_graded(18), _graded(30), HEAT, pde_noise=1e-3), 2
    elif case == "three_terms":
        p, P = _heat_like(gi.cells(20), _graded(36), THREE), 3
    else:
        p, P = _heat_like(gi.cells(16), gi.cells(64), HEAT), 2
    nt, nx = p.blocks[3].shape
    G = dense_gram(p)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    # the split ran: the PDE pair costs half of its plain mode products
    assert gp.matvec_flops() < 0.6 * _pde_pair_flops(nt, nx, P) + 4.0 * p.size * 64
    for R in (1, 5, 16):
        X = gi.random_vectors(p.size, R, 11 + R)
        for _ in range(3):                       # direct, capture, replay
            Y = gp.gpfvm_gram_matvec(_t(X)).cpu().numpy()
            _elementwise(Y, X @ G.T)


@pytest.mark.parametrize("case", ["odd", "asymmetric", "advection"])
def test_no_split_where_it_does_not_hold(case):
    if case == "odd":
        p, P = _heat_like(gi.cells(15), gi.cells(33), HEAT), 2
    elif case == "asymmetric":
        X = gi.cells(32)
        X.lo = X.lo ** 1.1
        X.hi = X.hi ** 1.1
        p, P = _heat_like(gi.cells(16), X, HEAT), 2
    else:
        p, P = _heat_like(gi.cells(16), gi.cells(32), ADV), 3
    nt, nx = p.blocks[3].shape
    G = dense_gram(p)
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    # full mode-product flops of the PDE pair (R6 may merge terms: >= P - 1)
    assert gp.matvec_flops() >= _pde_pair_flops(nt, nx, P - 1)
    X = gi.random_vectors(p.size, 4, 3)
    _elementwise(gp.gpfvm_gram_matvec(_t(X)).cpu().numpy(), X @ G.T)


def test_config1_split_equals_plain_path():
    """Config 1 at full size in bench.py's launch configuration: the split path
    against the oracle's Kronecker matvec element by element, and against the
    plain (GPFVM_NO_KRON_PARITY) path run in a separate process."""
    p = gi.config1()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    assert gp.matvec_flops() < 0.55 * _pde_pair_flops(256, 512, 2) + 1e8
    R = 128
    X = gi.random_vectors(p.size, R, 5)
    Xt = _t(X)
    Yt = torch.empty_like(Xt)
    for _ in range(3):
        gp.gpfvm_gram_matvec(Xt, out=Yt)
    Y = Yt.cpu().numpy()
    ref = KroneckerGram(p).matvec(X[:6])
    _elementwise(Y[:6], ref)
    code = ("import sys, numpy as np, torch; sys.path.insert(0, %r); import gpfvm_inputs as gi;"
            "from paper_2406_05020_b200 import GpfvmProblem; p = gi.config1(); gp = GpfvmProblem(p);"
            "gp.gpfvm_assemble_factors(); X = torch.tensor(gi.random_vectors(p.size, 128, 5), device='cuda:0');"
            "print(gp.matvec_flops()); np.save(sys.argv[1], gp.gpfvm_gram_matvec(X)[:16].cpu().numpy())" % ROOT)
    out = os.path.join(ROOT, "gpurun_out") if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp"
    f = os.path.join(out, "plain_config1.npy")
    env = dict(os.environ, GPFVM_NO_KRON_PARITY="1")
    r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert float(r.stdout.split()[-1]) > 1.9 * gp.matvec_flops() * 0.9
    plain = np.load(f)
    _elementwise(Y[:16], plain, 1e-13)
