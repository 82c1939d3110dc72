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


def test_tma_gemm_beside_cp_async_gemm_is_repeatable():
    """The two-stream situation of tools/gemm_race.cu through the C ABI: a TMA
    GEMM with 64x64 tiles (two CTAs per SM) repeated on one stream while the
    other stream runs GEMMs the TMA path rejects (odd leading dimension ->
    cp.async kernel).  Every repetition must equal the solitary result bit for
    bit (without the proxy fence about a third differed)."""
    import ctypes as C
    from paper_2406_05020_b200 import _lib
    lib = _lib.load()
    dev = torch.device("cuda:0")
    g = torch.Generator(device="cpu").manual_seed(5)
    M, N, K = 64, 64 * 1184, 96                     # one row of 64x64 tiles: the 2-CTA-per-SM variant
    A = torch.rand(M, K, generator=g, dtype=torch.float64).to(dev) - 0.5
    B = torch.rand(K, N, generator=g, dtype=torch.float64).to(dev) - 0.5
    Cm = torch.empty(M, N, dtype=torch.float64, device=dev)
    m2, k2 = 768, 191                               # odd lda: not TMA-eligible
    A2 = torch.rand(m2, k2, generator=g, dtype=torch.float64).to(dev)
    B2 = torch.rand(k2, m2, generator=g, dtype=torch.float64).to(dev)
    C2 = torch.empty(m2, m2, dtype=torch.float64, device=dev)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()

    def gemm(m, n, k, a, lda, b, ldb, c, ldc, s):
        rc = lib.gpfvm_gemm(m, n, k, 1.0, C.c_void_p(a.data_ptr()), lda, C.c_void_p(b.data_ptr()), ldb, 0.0,
                            C.c_void_p(c.data_ptr()), ldc, C.c_void_p(s.cuda_stream))
        assert rc == 0, lib.gpfvm_last_error()

    gemm(M, N, K, A, K, B, N, Cm, N, sa)
    torch.cuda.synchronize()
    first = Cm.clone()
    ref = (A.cpu().numpy() @ B.cpu().numpy())
    assert np.abs(first.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    bad = 0
    for rep in range(150):
        Cm.zero_()
        torch.cuda.synchronize()
        for q in range(6):
            gemm(m2, m2, k2, A2, k2, B2, m2, C2, m2, sb)
            if q == 2:
                gemm(M, N, K, A, K, B, N, Cm, N, sa)
        torch.cuda.synchronize()
        bad += not torch.equal(Cm, first)
    assert bad == 0, f"{bad} of 150 repetitions differ from the solitary result"
