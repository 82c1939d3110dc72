"""Repeatability of the Gram matvec under the concurrency of its own graph
(one branch per output block plus the side streams that prepare the coupling
operands): every reduction in the path has a fixed order, so repeated calls
must agree bit for bit, and the first must agree with the oracle.  Guards the
failure found in round 2: the TMA GEMM's consumer warps
released a pipeline stage without a fence.proxy.async between their
generic-proxy reads and the TMA refill, and under shared-memory pressure from
co-resident CTAs about half of the config-4 matvecs had wrong warp tiles,
never in the same place twice."""
import numpy as np
import pytest

import gpfvm_inputs as gi

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.gram import KroneckerGram  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem  # noqa: E402


@pytest.mark.parametrize("cfg,R,calls", [(gi.config4, 2, 24), (gi.config2, 4, 24), (gi.config1, 32, 24)])
def test_matvec_bitwise_repeatable_and_equal_to_oracle(cfg, R, calls):
    p = cfg()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, R, 13)
    xt = torch.tensor(X, dtype=torch.float64, device="cuda:0")
    first = gp.gpfvm_gram_matvec(xt).clone()
    ref = KroneckerGram(p).matvec(X[:1])
    err = np.abs(first[:1].cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 1e-12, err
    out = torch.empty_like(xt)
    for c in range(calls):          # direct launch, graph capture, graph replays
        gp.gpfvm_gram_matvec(xt, out=out)
        assert torch.equal(out, first), f"call {c}: max diff {float((out - first).abs().max())}"
