"""Host logic of the time-sharded multi-GPU path (paper_2406_05020_b200.dist),
world size 2 over gloo on CPU: sharding, all-to-all re-partition, the
K-concatenated time GEMM, allreduce'd CG inner products.  Local arithmetic
uses the CPU test backend (tests/dist_cpu_ops.py); expected values come from
the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gpfvm_inputs as gi
from gpfvm_inputs import Block, Kernel1D, Problem, Term
from oracle.gram import KroneckerGram, dense_gram, factor_matrix

NT, NX = 16, 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _heat_pde_problem(nt=NT, nx=NX, kappa=0.1):
    p = gi.heat_problem(nt, nx, kappa=kappa)
    pde = p.blocks[3]
    return Problem("heat_pde_only", 2, p.kernels, [pde], meta=p.meta)


def _heat_factors(nt=NT, nx=NX):
    p = gi.heat_problem(nt, nx)
    kt, kx = p.kernels[0]
    T, X = p.blocks[3].sites
    f = lambda k, S, m: torch.from_numpy(factor_matrix((k.q, k.lengthscale, k.variance), S, m, S, m))
    return {"T00": f(kt, T, 0), "T11": f(kt, T, 1), "X00": f(kx, X, 0), "X22": f(kx, X, 2)}


def _worker(rank, world, port, out_q, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_cpu_ops import CpuOps
        from paper_2406_05020_b200.dist import ShardedKron, heat_pde_operator, sharded_pcg
        ops = CpuOps()
        if case == "heat":
            fac = _heat_factors()
            A, fd = heat_pde_operator(ops, fac, 0.1, None, rank, world)
            x = torch.from_numpy(gi.random_vectors(NT * NX, 1, 3)[0])
            nt = NT // world
            xl = x.reshape(NT, NX)[rank * nt:(rank + 1) * nt].reshape(-1).clone()
            yl = A.matvec(xl)
            # PCG on G_pp a = b with the sharded FD preconditioner
            b = torch.from_numpy(gi.random_vectors(NT * NX, 1, 5)[0])
            bl = b.reshape(NT, NX)[rank * nt:(rank + 1) * nt].reshape(-1).clone()
            res = sharded_pcg(ops, A, bl, fd, rtol=1e-10, max_iter=20, group=None, world=world)
            out_q.put((rank, yl.numpy().copy(), res.x.numpy().copy(), res.iterations, res.rel_residual))
        else:  # 3D two-term operator
            rng = np.random.default_rng(7)
            shape = (8, 6, 5)
            facs = [[torch.from_numpy(rng.standard_normal((n, n))) for n in shape] for _ in range(2)]
            A = ShardedKron(ops, shape, [0.7, -1.3], facs, None, rank, world)
            x = torch.from_numpy(rng.standard_normal(int(np.prod(shape))))
            nt = shape[0] // world
            xl = x.reshape(shape)[rank * nt:(rank + 1) * nt].reshape(-1).clone()
            out_q.put((rank, A.matvec(xl).numpy().copy(), None, 0, 0.0))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda t: t[0])
    return outs


@pytest.fixture(scope="module", autouse=True)
def _path():
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = os.pathsep.join([here, os.path.dirname(here), os.environ.get("PYTHONPATH", "")])


def test_sharded_heat_matvec_and_pcg_world2():
    outs = _run(2, "heat")
    y = np.concatenate([o[1] for o in outs])
    x = gi.random_vectors(NT * NX, 1, 3)[0]
    p = _heat_pde_problem()
    ref = KroneckerGram(p).matvec(x)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    # PCG: sharded IterGP with the sharded FD preconditioner == dense solve
    b = gi.random_vectors(NT * NX, 1, 5)[0]
    G = dense_gram(p)
    a_ref = np.linalg.solve(G, b)
    a = np.concatenate([o[2] for o in outs])
    assert outs[0][3] <= 4 and outs[0][3] == outs[1][3]
    assert np.linalg.norm(G @ a - b) <= 1e-8 * np.linalg.norm(b)
    assert np.abs(a - a_ref).max() <= 1e-6 * np.abs(a_ref).max()


def test_sharded_matvec_world1_equals_world2():
    y1 = np.concatenate([o[1] for o in _run(1, "heat")])
    y2 = np.concatenate([o[1] for o in _run(2, "heat")])
    assert np.abs(y1 - y2).max() <= 1e-13 * np.abs(y1).max()


def test_sharded_3d_matvec_world2():
    outs = _run(2, "3d")
    y = np.concatenate([o[1] for o in outs])
    rng = np.random.default_rng(7)
    shape = (8, 6, 5)
    facs = [[rng.standard_normal((n, n)) for n in shape] for _ in range(2)]
    x = rng.standard_normal(int(np.prod(shape)))
    ref = sum(c * KroneckerGram.apply_kron(f, x, shape) for c, f in zip([0.7, -1.3], facs))
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
