"""Time-mode sharded GP-FVM (north_star multi-GPU row): a thin
orchestrator.  Every arithmetic step — the spatial Kronecker products, the
grouping of terms by time factor (R6 cancellation included), the packing of
the exchange buffers, the K-concatenated time GEMM, the block-Jacobi FD
preconditioner and every IterGP scalar — runs in libgpfvm (gpfvm_shard_*,
gpfvm_iter_*, gpfvm_dot_many).  This module only

  * allocates the exchange buffers the library sizes (gpfvm_shard_counts),
  * moves them with ``all_to_all_single`` (NCCL over NVLink on GPUs), and
  * sums the IterGP partial scalars with ``all_reduce``.

``Comm`` abstracts the two collectives over the ranks held by this process:
``TorchComm`` (one rank per process, torch.distributed) and ``LocalComm``
(W ranks in one process on one GPU, exchanges done as copies: the
single-GPU numerical check of the multi-rank layouts; no kernel ever waits on
another rank).  The sharded objects are lists with one entry per local rank.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from . import _lib as L

SHARD_GRAM, SHARD_PRECOND = 0, 1
ITER_STATE = 8
ST_NY, ST_NR, ST_DONE, ST_COUNT = 0, 1, 5, 6


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else C.c_void_p(0)


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


# ---- collectives -------------------------------------------------------------
class TorchComm:
    """One local rank; all_to_all_single / all_reduce over a process group."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.ranks = [dist.get_rank(group) if dist.is_initialized() else 0]

    def alltoall(self, sends: List[torch.Tensor], recvs: List[torch.Tensor], send_counts, recv_counts):
        if self.world == 1:
            recvs[0].copy_(sends[0])
            return
        dist.all_to_all_single(recvs[0], sends[0], output_split_sizes=list(recv_counts[0]),
                               input_split_sizes=list(send_counts[0]), group=self.group)

    def allreduce(self, ts: List[torch.Tensor]):
        if self.world > 1:
            dist.all_reduce(ts[0], op=dist.ReduceOp.SUM, group=self.group)


class LocalComm:
    """W ranks in this process (one GPU): exchanges are plain device copies."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def alltoall(self, sends, recvs, send_counts, recv_counts):
        W = self.world
        soff = [[0] * (W + 1) for _ in range(W)]
        roff = [[0] * (W + 1) for _ in range(W)]
        for r in range(W):
            for q in range(W):
                soff[r][q + 1] = soff[r][q] + send_counts[r][q]
                roff[r][q + 1] = roff[r][q] + recv_counts[r][q]
        for src in range(W):
            for dst in range(W):
                n = send_counts[src][dst]
                assert n == recv_counts[dst][src], "exchange counts disagree"
                if n:
                    recvs[dst][roff[dst][src]:roff[dst][src] + n].copy_(sends[src][soff[src][dst]:soff[src][dst] + n])

    def allreduce(self, ts):
        total = ts[0].clone()
        for t in ts[1:]:
            total += t
        for t in ts:
            t.copy_(total)


# ---- sharded operators ---------------------------------------------------------
class _ShardOp:
    """One library shard handle per local rank (kind GRAM or PRECOND)."""

    def __init__(self, gps, comm, kind):
        self.lib = L.load()
        self.comm = comm
        self.gps = gps
        self.dev = [torch.device("cuda", gp.device) for gp in gps]
        self.h = []
        for gp, r, dev in zip(gps, comm.ranks, self.dev):
            h = C.c_void_p()
            with torch.cuda.device(dev):
                L.check(self.lib.gpfvm_shard_create(gp.handle, int(r), int(comm.world), int(kind), C.byref(h),
                                                    _stream(dev)))
            self.h.append(h)
        W = comm.world
        self.n = [int(self.lib.gpfvm_shard_local_size(h)) for h in self.h]
        self.phases = 2 if kind == SHARD_PRECOND else 1
        self.counts = []  # per phase: (send1, recv1, send2, recv2), each per local rank a list of W ints
        self.bufs = []
        for ph in range(self.phases):
            cs = [[], [], [], []]
            for h in self.h:
                arr = [(C.c_int64 * W)() for _ in range(4)]
                L.check(self.lib.gpfvm_shard_counts(h, ph, *arr))
                for k in range(4):
                    cs[k].append([int(v) for v in arr[k]])
            self.counts.append(cs)
            self.bufs.append([[torch.empty(max(1, sum(cs[k][i])), dtype=torch.float64, device=self.dev[i])
                               for i in range(len(self.h))] for k in range(4)])

    def layout(self, i=0):
        nb = len(self.gps[i].problem.blocks)
        arrs = [(C.c_int64 * nb)() for _ in range(4)]
        L.check(self.lib.gpfvm_shard_layout(self.h[i], *arrs))
        return [[int(v) for v in a] for a in arrs]

    def apply(self, ph: int, xs: Sequence[torch.Tensor], ys: Sequence[torch.Tensor], x_for_end=True):
        s1, r1, s2, r2 = self.bufs[ph]
        c = self.counts[ph]
        for i, h in enumerate(self.h):
            L.check(self.lib.gpfvm_shard_apply_begin(h, ph, _p(xs[i]), _p(s1[i]), _stream(self.dev[i])))
        self.comm.alltoall(s1, r1, c[0], c[1])
        for i, h in enumerate(self.h):
            L.check(self.lib.gpfvm_shard_apply_mid(h, ph, _p(r1[i]), _p(s2[i]), _stream(self.dev[i])))
        self.comm.alltoall(s2, r2, c[2], c[3])
        for i, h in enumerate(self.h):
            L.check(self.lib.gpfvm_shard_apply_end(h, ph, _p(r2[i]), _p(xs[i]) if x_for_end else C.c_void_p(0),
                                                   _p(ys[i]), _stream(self.dev[i])))

    def close(self):
        for h in self.h:
            if h:
                self.lib.gpfvm_shard_destroy(h)
        self.h = []


@dataclass
class ShardedReport:
    iterations: int
    converged: bool
    breakdown: bool
    rel_residual: float


class ShardedProblem:
    """The GP-FVM Gram, its block-Jacobi FD preconditioner and the IterGP solve,
    sharded along the time mode.  ``gps``: one assembled GpfvmProblem per local
    rank (TorchComm: one; LocalComm(W): W problems on one GPU)."""

    def __init__(self, gps, comm):
        self.lib = L.load()
        self.comm = comm
        self.gps = list(gps)
        self.G = _ShardOp(self.gps, comm, SHARD_GRAM)
        self.P: Optional[_ShardOp] = None
        self.n = self.G.n
        self.dev = self.G.dev

    # -- vectors
    def local(self, full_vectors: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        """Local slabs of full (block-concatenated) device vectors, one per local rank."""
        out = []
        for i, h in enumerate(self.G.h):
            t = torch.empty(max(1, self.n[i]), dtype=torch.float64, device=self.dev[i])[:self.n[i]]
            L.check(self.lib.gpfvm_shard_gather_local(h, _p(full_vectors[i]), _p(t), _stream(self.dev[i])))
            out.append(t)
        return out

    def _empty(self):
        return [torch.empty(max(1, n), dtype=torch.float64, device=d)[:n] for n, d in zip(self.n, self.dev)]

    # -- operators
    def matvec(self, xs):
        ys = self._empty()
        self.G.apply(0, xs, ys)
        return ys

    def precond(self, rs, out=None):
        if self.P is None:
            self.P = _ShardOp(self.gps, self.comm, SHARD_PRECOND)
        tmp = self._empty()
        zs = out if out is not None else self._empty()
        self.P.apply(0, rs, tmp, x_for_end=False)
        for i, h in enumerate(self.P.h):
            L.check(self.lib.gpfvm_shard_precond_scale(h, _p(tmp[i]), _stream(self.dev[i])))
        self.P.apply(1, tmp, zs, x_for_end=False)
        return zs

    # -- IterGP (CG policy, full reorthogonalisation by default) ----------------
    def solve(self, ys, rtol=1e-8, max_iter=200, reorth_window=0, precond=True, check_every=4):
        """alpha = G^{-1} y on the sharded vectors; every scalar stays on the
        device (library kernels), the ranks sum partial scalars with all_reduce."""
        lib, R = self.lib, range(len(self.gps))
        st = [torch.zeros(ITER_STATE, dtype=torch.float64, device=d) for d in self.dev]
        xs = [torch.zeros_like(y) for y in ys]
        rs = [y.clone() for y in ys]
        D = [torch.empty(max_iter + 1, max(1, n), dtype=torch.float64, device=d) for n, d in zip(self.n, self.dev)]
        GD = [torch.empty_like(t) for t in D]
        eta = [torch.zeros(max_iter + 1, dtype=torch.float64, device=d) for d in self.dev]
        cbuf = [torch.zeros(max_iter + 1, dtype=torch.float64, device=d) for d in self.dev]
        p1 = [torch.empty(max(1, max_iter + 1), dtype=torch.float64, device=d) for d in self.dev]
        p2 = [torch.empty(2, dtype=torch.float64, device=d) for d in self.dev]
        s = [_stream(d) for d in self.dev]
        for i in R:
            L.check(lib.gpfvm_dot_many(_p(ys[i]), max(1, self.n[i]), _p(ys[i]), self.n[i], 1, _p(p1[i]), s[i]))
        self.comm.allreduce([t[:1] for t in p1])
        for i in R:
            L.check(lib.gpfvm_iter_init(_p(p1[i]), float(rtol), _p(st[i]), s[i]))
        it = 0
        while it < max_iter:
            if it == 0 or it <= 4 or it % check_every == 0:
                if float(st[0][ST_DONE]) != 0.0:
                    break
            ds = self.precond(rs) if precond else [r.clone() for r in rs]
            gds = self.matvec(ds)
            w = it if reorth_window <= 0 else min(reorth_window, it)
            j0 = it - w
            if w > 0:
                for i in R:
                    L.check(lib.gpfvm_dot_many(_p(D[i][j0]), D[i].stride(0), _p(gds[i]), self.n[i], w, _p(p1[i]), s[i]))
                self.comm.allreduce([t[:w] for t in p1])
                for i in R:
                    L.check(lib.gpfvm_iter_coefs(_p(p1[i]), w, _p(eta[i][j0:]), _p(cbuf[i]), _p(st[i]), s[i]))
            for i in R:
                L.check(lib.gpfvm_iter_update_local(_p(ds[i]), _p(gds[i]), _p(D[i][j0]), _p(GD[i][j0]), D[i].stride(0),
                                                    w, _p(cbuf[i]), _p(rs[i]), _p(D[i][it]), _p(GD[i][it]),
                                                    self.n[i], _p(p2[i]), _p(st[i]), s[i]))
            self.comm.allreduce(p2)
            for i in R:
                L.check(lib.gpfvm_iter_update_final(_p(p2[i]), _p(st[i]), _p(eta[i][it:]), s[i]))
                L.check(lib.gpfvm_iter_step_local(_p(xs[i]), _p(rs[i]), _p(D[i][it]), _p(GD[i][it]), self.n[i],
                                                  _p(p1[i]), _p(st[i]), s[i]))
            self.comm.allreduce([t[:1] for t in p1])
            for i in R:
                L.check(lib.gpfvm_iter_step_final(_p(p1[i]), _p(st[i]), s[i]))
            it += 1
        h = st[0].cpu()
        ny = float(h[ST_NY])
        rep = ShardedReport(int(h[ST_COUNT]), bool(h[ST_DONE] == 1.0 or ny == 0.0), bool(h[ST_DONE] == 2.0),
                            float(h[ST_NR]) / ny if ny > 0 else 0.0)
        return xs, rep

    # -- posterior mean on a grid (Eq. 5): partial sums per rank + all_reduce
    def predict_mean(self, grid, alphas):
        import numpy as np
        d = self.gps[0].problem.ndim
        pts = [np.ascontiguousarray(p, dtype=np.float64) for p in grid.points]
        g = L.Grid()
        for i in range(d):
            g.n[i] = int(pts[i].shape[0])
            g.pts[i] = pts[i].ctypes.data_as(C.POINTER(C.c_double))
        g.output = int(grid.output)
        ng = int(np.prod([p.shape[0] for p in pts]))
        means = [torch.empty(ng, dtype=torch.float64, device=dv) for dv in self.dev]
        for i, h in enumerate(self.G.h):
            L.check(self.lib.gpfvm_shard_predict_mean(h, C.byref(g), _p(alphas[i]), _p(means[i]), _stream(self.dev[i])))
        self.comm.allreduce(means)
        return means

    def close(self):
        self.G.close()
        if self.P is not None:
            self.P.close()
