"""Multi-rank host logic of the time-sharded path on CPU (no GPU needed):

* the library's exchange plan (gpfvm_shard_plan_counts, host-only C++: the
  same code gpfvm_shard_create runs) is consistent across ranks — what rank r
  sends to q is what q expects from r, in both exchanges — and the local slabs
  partition the N observations, for every BASELINE problem shape and 2, 3, 8
  ranks;
* the torch.distributed collectives dist.TorchComm issues (all_to_all_single
  with the plan's uneven split sizes, all_reduce) over gloo, world size 2,
  equal the single-process emulation dist.LocalComm that the GPU tests use to
  check the sharded numerics against the oracle (tests/test_gpu_dist.py)."""
import ctypes as C
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gpfvm_inputs as gi


def _lib():
    from paper_2406_05020_b200 import _lib as L
    try:
        return L.load()
    except RuntimeError:
        pytest.skip("libgpfvm.so not built")


def _plan(gp, rank, world):
    lib = _lib()
    n = C.c_int64()
    arrs = [(C.c_int64 * world)() for _ in range(4)]
    from paper_2406_05020_b200 import _lib as L
    L.check(lib.gpfvm_shard_plan_counts(gp.handle, rank, world, C.byref(n), *arrs))
    return int(n.value), [[int(v) for v in a] for a in arrs]


PROBLEMS = {
    "heat-16x24": lambda: gi.heat_problem(16, 24),
    "wave-8x10x12": lambda: gi.wave_problem(8, 10, 12),
    "shallow-water-6x6x7": lambda: gi.shallow_water_problem(6, 6, 7),
    "config3": gi.config3,
    "config4": gi.config4,
}


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name", list(PROBLEMS))
def test_plan_counts_consistent(name, world):
    from paper_2406_05020_b200 import GpfvmProblem
    from paper_2406_05020_b200._lib import GpfvmError
    p = PROBLEMS[name]()
    gp = GpfvmProblem(p, device=0)
    if world > max(b.shape[0] for b in p.blocks):
        with pytest.raises(GpfvmError):  # more ranks than time sites
            _plan(gp, 0, world)
        return
    plans = [_plan(gp, r, world) for r in range(world)]
    assert sum(n for n, _ in plans) == p.size
    for r in range(world):
        for q in range(world):
            assert plans[r][1][0][q] == plans[q][1][1][r], ("exchange 1", r, q)
            assert plans[r][1][2][q] == plans[q][1][3][r], ("exchange 2", r, q)
    # every rank holds a time slab of the time-extended blocks (IC planes on rank 0)
    assert all(n > 0 for n, _ in plans)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, counts, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_05020_b200.dist import TorchComm
        comm = TorchComm()
        send_counts, recv_counts = counts
        g = torch.Generator().manual_seed(100 + rank)
        send = torch.randn(sum(send_counts[rank]), dtype=torch.float64, generator=g)
        recv = torch.empty(sum(recv_counts[rank]), dtype=torch.float64)
        comm.alltoall([send], [recv], [send_counts[rank]], [recv_counts[rank]])
        red = torch.arange(5, dtype=torch.float64) * (rank + 1)
        comm.allreduce([red])
        q.put((rank, send, recv, red))
    finally:
        dist.destroy_process_group()


def test_torchcomm_gloo_matches_localcomm():
    from paper_2406_05020_b200 import GpfvmProblem
    from paper_2406_05020_b200.dist import LocalComm
    world = 2
    gp = GpfvmProblem(gi.wave_problem(8, 10, 12), device=0)
    plans = [_plan(gp, r, world) for r in range(world)]
    send_counts = [plans[r][1][0] for r in range(world)]
    recv_counts = [plans[r][1][1] for r in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (send_counts, recv_counts), q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict()
    for _ in range(world):
        r, send, recv, red = q.get(timeout=300)
        res[r] = (send, recv, red)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    emu_recv = [torch.empty_like(res[r][1]) for r in range(world)]
    LocalComm(world).alltoall([res[r][0] for r in range(world)], emu_recv, send_counts, recv_counts)
    for r in range(world):
        assert torch.equal(res[r][1], emu_recv[r])
        assert torch.equal(res[r][2], torch.arange(5, dtype=torch.float64) * 3)
