"""GPU parity of the 3D reflection-parity split (KronSum::par3, DESIGN.md
§4.3): on mirror-symmetric site lists every factor of Eq. 20 (PAPER.md
l.316-320) is centrosymmetric or skew-centrosymmetric, so the PDE-PDE block
pairs of the 2D-space problems run class by class with half-size factors
(terms with odd derivative orders map even parts to odd parts).  The oracle
knows nothing of this: dense Gram / plain Kronecker matvec, element by element
at 1e-12 of max|ref|; and the split path against the unsplit path of the same
library (GPFVM_PAR3_MINH raised).  The full-size configs 3 and 4 go through the
split by default (tests/test_gpu_parity_r2.py compares them with the oracle)."""
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


def _elementwise(Y, ref, tol=1e-12):
    err = np.abs(Y - ref).max() / np.abs(ref).max()
    assert err <= tol, err


def _build(p, monkeypatch, minh):
    monkeypatch.setenv("GPFVM_PAR3_MINH", str(minh))
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    return gp


SMALL = {
    "wave": lambda: gi.wave_problem(4, 8, 12),                    # even orders only
    "advdiff": lambda: gi.advdiff_problem(8, 4, 12, n_modes=4),   # skew time/space factors (odd orders)
    "shallow_water": lambda: gi.shallow_water_problem(4, 8, 4),   # 3 x 3 PDE block pairs, cross-output pairs
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_split3d_small_vs_dense_oracle(name, monkeypatch):
    p = SMALL[name]()
    G = dense_gram(p)
    plain = _build(p, monkeypatch, 1 << 20)
    split = _build(p, monkeypatch, 2)
    assert split.matvec_flops() < 0.8 * plain.matvec_flops(), (split.matvec_flops(), plain.matvec_flops())
    for R in (1, 3):
        X = gi.random_vectors(p.size, R, 5 + R)
        ref = X @ G.T
        for _ in range(3):                       # direct, capture, replay
            _elementwise(split.gpfvm_gram_matvec(_t(X)).cpu().numpy(), ref)
        _elementwise(plain.gpfvm_gram_matvec(_t(X)).cpu().numpy(), ref)


@pytest.mark.parametrize("name,builder", [
    ("advdiff", lambda: gi.advdiff_problem(16, 64, 64, n_modes=8)),
    ("shallow_water", lambda: gi.shallow_water_problem(16, 64, 64)),
    ("wave", lambda: gi.wave_problem(16, 64, 64)),
])
def test_split3d_plan_size_vs_oracle_and_plain(name, builder, monkeypatch):
    """Sizes that reach the TMA GEMMs of every stage (class-batched, negative
    class strides for skew factors): against the oracle's Kronecker matvec and
    the unsplit plan."""
    p = builder()
    plain = _build(p, monkeypatch, 1 << 20)
    split = _build(p, monkeypatch, 8)
    assert split.matvec_flops() < 0.8 * plain.matvec_flops()
    X = gi.random_vectors(p.size, 3, 17)
    ref = KroneckerGram(p).matvec(X)
    xt = _t(X)
    out = torch.empty_like(xt)
    for _ in range(3):
        split.gpfvm_gram_matvec(xt, out=out)
        _elementwise(out.cpu().numpy(), ref)
    _elementwise(split.gpfvm_gram_matvec(xt).cpu().numpy(), plain.gpfvm_gram_matvec(xt).cpu().numpy(), 1e-13)


def test_no_split3d_on_odd_or_asymmetric_cells(monkeypatch):
    p = gi.wave_problem(4, 6, 10)   # 6 and 10 are not multiples of 4: the class offsets would be misaligned
    G = dense_gram(p)
    plain = _build(p, monkeypatch, 1 << 20)
    split = _build(p, monkeypatch, 2)
    assert split.matvec_flops() == plain.matvec_flops()
    X = gi.random_vectors(p.size, 2, 9)
    _elementwise(split.gpfvm_gram_matvec(_t(X)).cpu().numpy(), X @ G.T)
