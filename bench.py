#!/usr/bin/env python
"""GP-FVM hot-path benchmark (BASELINE.json metric: "FVM-Gram matvec GB/s & CG
solve s to 1e-8 resid (N obs)").

One step = one pass of every §8(a) row on BASELINE config 1 (1D heat,
256 x 512 FVM cells + 1,024 IC/BC cells, Matérn-5/2, FP64):
  1. gpfvm_assemble_factors
  2. gpfvm_gram_matvec on a resident block of R = 128 vectors (135 MB > L2)
  3. gpfvm_solve to relative residual 1e-8 (preconditioner built in-step)
  4. gpfvm_predict mean + variance on the 512 x 1024 grid
`value` = Gram-matvec throughput in GB/s: algorithmic bytes R*N*8*2 (read X,
write Y) / matvec device time, summed over ranks / max over ranks.
`cg_solve_s` = device time of row 3.  N > 1: independent replicas per rank
(weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FVM-Gram matvec GB/s & CG solve s to 1e-8 resid (N obs)"
WORKLOAD = "config1_heat1d_256x512"


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML every 10 ms (nvidia-smi every ~0.3 s as a fallback)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self._stop.is_set():
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            self.mx.append(mx)
            bits = int(get_reasons(h))
            for name, bit in self.BITS.items():
                if bits & bit:
                    self.reasons.add(name)
            self._stop.wait(0.01)

    def _run_smi(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    r = [c.strip() for c in line.split(",")]
                    if len(r) > 2 and r[1].replace(".", "").isdigit():
                        self.sm.append(float(r[1]))
                        self.mx.append(float(r[2]))
                    for k, nm in enumerate(names):
                        if len(r) > 4 + k and r[4 + k].lower().startswith("active"):
                            self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
        except Exception:
            return self._run_smi()
        try:
            self._run_nvml(nv)
        except Exception:
            self._run_smi()
        finally:
            try:
                nv.nvmlShutdown()
            except Exception:
                pass

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        import statistics
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_min_mhz": min(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def cpu_baseline(seconds: float = 15.0):
    """The oracle (as it stands) on the host cores: its plain Kronecker matvec
    (oracle.gram.KroneckerGram) on config 1, vectors until ~`seconds` elapse."""
    import numpy as np
    import gpfvm_inputs as gi
    from oracle.gram import KroneckerGram
    p = gi.config1()
    K = KroneckerGram(p)              # factor construction (mpmath) not timed
    x = gi.random_vectors(p.size, 1, 3)[0]
    n = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds or n == 0:
        K.matvec(x)
        n += 1
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    gbs = n * p.size * 8 * 2 / dt / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": int(cores), "kind": "oracle",
            "sample": f"{n} single-vector oracle Kronecker matvecs of config 1 (N={p.size}) in {dt:.1f}s; "
                      f"factor construction excluded"}


def fp64_peak_live(gp):
    """FP64 tensor-core roofline denominator measured in this run
    (gpfvm_probe_fp64_peak: register-only DMMA.8x8x4 probe); MEASURED_PEAKS.json
    has no FP64 entry."""
    import ctypes as C
    import torch
    v = C.c_double(0.0)
    rc = gp.lib.gpfvm_probe_fp64_peak(C.byref(v), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc == 0 and v.value > 1.0:
        return v.value, ("live DMMA.8x8x4 probe in this run (gpfvm_probe_fp64_peak); MEASURED_PEAKS.json has no "
                         "FP64 entry; tools/fp64_peak_bench: DMMA 37.0, cuBLAS DGEMM 35.4 (profiles/fp64_peak.txt)")
    return 37.0, "tools/fp64_peak_bench DMMA.8x8x4 on this pool's B200 (profiles/fp64_peak.txt)"


def _traffic():
    """DRAM bytes (read + write) per matvec from the committed ncu capture
    (profiles/r02_traffic.json, written by tools/ncu_traffic.py from a
    `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` pass over every
    kernel of one matvec)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
    except Exception:
        return {}


def bench_config(builder, R, dev, peak, traffic, world, solve_budget=0, full_reorth=True):
    """Matvec of a BASELINE 3D config (R right-hand sides resident in HBM):
    graph replay timed with CUDA events over 5 launches after 3 warm-ups."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import gpfvm_inputs as gi
    from paper_2406_05020_b200 import GpfvmProblem
    p = builder()
    gp = GpfvmProblem(p, device=dev.index or 0)
    gp.gpfvm_assemble_factors()
    N = gp.N
    X = torch.tensor(gi.random_vectors(N, R, 7), dtype=torch.float64, device=dev)
    Y = torch.empty_like(X)
    for _ in range(3):
        gp.gpfvm_gram_matvec(X, out=Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gp.gpfvm_gram_matvec(X, out=Y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    tt = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    flops = gp.matvec_flops() * R
    out = {"workload": p.name if hasattr(p, "name") else builder.__name__, "n_obs": int(N), "nrhs": R, "matvec_ms": ms,
           "GB_s": world * 16.0 * N * R / (ms * 1e-3) / 1e9, "TFLOP_s": flops / (ms * 1e-3) / 1e12,
           "frac": flops / (ms * 1e-3) / 1e12 / peak, "algorithmic_bytes": 16 * N * R,
           "unsplit_plan_equivalent_tflops": gp.matvec_flops_unsplit() * R / (ms * 1e-3) / 1e12,
           "traffic": traffic.get("dram_bytes"), "traffic_source": traffic.get("source")}
    if solve_budget > 0:
        # the paper's fixed IterGP budget for its 3D problem (P:l.444: 1250
        # iterations), full reorthogonalisation, every action kept (P:l.475)
        y = torch.tensor(p.rhs(), dtype=torch.float64, device=dev)
        alpha = torch.empty_like(y)
        gp.gpfvm_solve(y, rtol=1e-8, max_iter=2, out=alpha)  # preconditioner build, warm-up
        torch.cuda.synchronize()
        e0.record()
        # configs 3/4: 2 x 1250 x N x 8 B of kept actions exceed one GPU's HBM, so
        # their budgeted solve runs the PCG recurrence (reorth_window = 1, actions
        # not kept); the sharded path is where their Krylov store fits
        _, rep = gp.gpfvm_solve(y, rtol=1e-8, max_iter=solve_budget, out=alpha, reorth_window=0 if full_reorth else 1,
                                keep_actions=bool(full_reorth))
        e1.record()
        torch.cuda.synchronize()
        out["solve"] = {"budget": solve_budget, "iterations": rep["iterations"], "converged": bool(rep["converged"]),
                        "rel_residual": rep["rel_residual"], "true_rel_residual": rep["true_rel_residual"],
                        "solve_s": e0.elapsed_time(e1) / 1e3,
                        "reorth": "full" if full_reorth else "window 1 (PCG recurrence)",
                        "actions_kept": rep["iterations"] if full_reorth else 0,
                        "breakdown": bool(rep.get("breakdown", 0)),
                        "precond": "block-Jacobi FD (DESIGN.md 5.4)"}
        rb = p.meta.get("rhs_batch")
        if rb is not None and len(rb) > 1:
            # the 4-RHS batch (BASELINE configs[2]) through gpfvm_solve_many: one
            # IterGP run per RHS sharing the batched preconditioner and matvec;
            # the PCG recurrence (reorth_window=1) over the same budget
            Yb = torch.tensor(np.ascontiguousarray(rb), dtype=torch.float64, device=dev)
            Ab = torch.empty_like(Yb)
            gp.gpfvm_solve(Yb, rtol=1e-8, max_iter=2, out=Ab, reorth_window=1, keep_actions=False)
            torch.cuda.synchronize()
            e0.record()
            _, reps = gp.gpfvm_solve(Yb, rtol=1e-8, max_iter=solve_budget, out=Ab, reorth_window=1,
                                     keep_actions=False)
            e1.record()
            torch.cuda.synchronize()
            out["solve_batch"] = {"nrhs": len(rb), "budget": solve_budget, "reorth": "window 1 (PCG recurrence)",
                                  "solve_s": e0.elapsed_time(e1) / 1e3,
                                  "iterations": [r["iterations"] for r in reps],
                                  "true_rel_residual": [r["true_rel_residual"] for r in reps]}
            del Yb, Ab
        del y, alpha
    del gp, X, Y
    torch.cuda.empty_cache()
    return out


def bench_sharded(builder, dev, world, iters=20):
    """Sharded matvec and IterGP iterations of a full BASELINE 3D problem over
    the ranks of this job (max over ranks of CUDA-event times)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import gpfvm_inputs as gi
    from paper_2406_05020_b200 import GpfvmProblem
    from paper_2406_05020_b200.dist import ShardedProblem, TorchComm
    p = builder()
    gp = GpfvmProblem(p, device=dev.index or 0)
    gp.gpfvm_assemble_factors()
    sp = ShardedProblem([gp], TorchComm())
    x = torch.tensor(gi.random_vectors(p.size, 1, 5)[0], dtype=torch.float64, device=dev)
    xl = sp.local([x])
    for _ in range(3):
        sp.matvec(xl)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        sp.matvec(xl)
    e1.record()
    torch.cuda.synchronize()
    mv = e0.elapsed_time(e1) / 5
    y = torch.tensor(p.rhs(), dtype=torch.float64, device=dev)
    yl = sp.local([y])
    sp.solve(yl, rtol=0.0, max_iter=2, reorth_window=1)  # preconditioner build + warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record()
    _, rep = sp.solve(yl, rtol=0.0, max_iter=iters, reorth_window=1)
    e1.record()
    torch.cuda.synchronize()
    it_ms = e0.elapsed_time(e1) / max(1, iters)
    t = torch.tensor([mv, it_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    mv, it_ms = t.tolist()
    cnt = sp.G.counts[0]
    comm = int(sum(cnt[0][0]) - cnt[0][0][sp.comm.ranks[0]] + sum(cnt[2][0]) - cnt[2][0][sp.comm.ranks[0]]) * 8
    out = {"workload": p.name, "ranks": world, "n_obs": int(p.size), "matvec_ms": mv,
           "GB_s": 16.0 * p.size / (mv * 1e-3) / 1e9, "iteration_ms": it_ms, "iterations_timed": rep.iterations,
           "precond": "sharded block-Jacobi FD", "bytes_sent_per_rank_per_matvec": comm,
           "scaling": "strong (fixed problem split over the ranks)"}
    sp.close()
    del gp
    torch.cuda.empty_cache()
    return out


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    steps_vals = []
    per = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(seconds=per)
        if i >= args.warmup:
            steps_vals.append(cb)
    val = sum(c["value"] for c in steps_vals) / len(steps_vals)
    cb = dict(steps_vals[-1])
    cb["value"] = val
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1000, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_obs": 132096, "note": "oracle Kronecker matvec on host cores"},
            "cpu_baseline": cb, "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nrhs", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sharded", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-budget-solve", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import gpfvm_inputs as gi
    from paper_2406_05020_b200 import GpfvmProblem, launch_count
    from paper_2406_05020_b200.build import build

    rank, world, local = _dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    dev = torch.device(f"cuda:{local}")

    prob = gi.config1(seed=1 + rank)             # weak scaling: one replica per rank
    grid = gi.heat_grid(512, 1024)
    R = args.nrhs
    gp = GpfvmProblem(prob, device=local)
    N = gp.N
    X = torch.tensor(gi.random_vectors(N, R, 11 + rank), dtype=torch.float64, device=dev)
    Y = torch.empty_like(X)
    rhs = torch.tensor(prob.rhs(), dtype=torch.float64, device=dev)
    alpha = torch.empty_like(rhs)
    mean = torch.empty(512 * 1024, dtype=torch.float64, device=dev)
    var = torch.empty_like(mean)

    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(timed: bool):
        e = [ev() for _ in range(5)]
        e[0].record()
        gp.gpfvm_assemble_factors()
        e[1].record()
        gp.gpfvm_gram_matvec(X, out=Y)
        e[2].record()
        _, rep = gp.gpfvm_solve(rhs, rtol=1e-8, out=alpha)
        e[3].record()
        gp.gpfvm_predict(grid, alpha, cov_mode=1, mean=mean, var=var)
        e[4].record()
        return e, rep

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = launch_count()
    times = {"assemble": [], "matvec": [], "solve": [], "predict": [], "step": []}
    reps = []
    with ClockSampler(local) as clk:
        t_all0 = ev()
        t_all1 = ev()
        t_all0.record()
        for _ in range(args.steps):
            e, rep = step(True)
            reps.append(rep)
            torch.cuda.synchronize()
            times["assemble"].append(e[0].elapsed_time(e[1]))
            times["matvec"].append(e[1].elapsed_time(e[2]))
            times["solve"].append(e[2].elapsed_time(e[3]))
            times["predict"].append(e[3].elapsed_time(e[4]))
            times["step"].append(e[0].elapsed_time(e[4]))
        t_all1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = launch_count() - l0
    total_ms = t_all0.elapsed_time(t_all1)
    mv_ms = float(np.mean(times["matvec"]))
    bytes_mv = R * N * 8 * 2
    # max over ranks of the times, sum of the work
    vals = torch.tensor([total_ms, mv_ms, float(np.mean(times["solve"]))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, mv_ms_max, solve_ms_max = vals.tolist()
    value = world * bytes_mv / (mv_ms_max * 1e-3) / 1e9

    # e2e: same metric through the C ABI with pinned HOST buffers (H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        Xh = torch.empty((R, N), dtype=torch.float64, pin_memory=True)
        Xh.copy_(X.cpu())
        Yh = torch.empty((R, N), dtype=torch.float64, pin_memory=True)
        xa, ya = Xh.numpy(), Yh.numpy()
        gp.gpfvm_gram_matvec(xa, out=ya)
        ts = []
        for _ in range(max(2, args.steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gp.gpfvm_gram_matvec(xa, out=ya)
            ts.append(time.perf_counter() - t0)
        e2e_s = float(np.median(ts))
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * bytes_mv / tt.item() / 1e9, "unit": "GB/s", "h2d_bytes_per_step": R * N * 8,
               "d2h_bytes_per_step": R * N * 8}

    flops_mv = gp.matvec_flops() * R
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    fp64_peak, peak_src = fp64_peak_live(gp)
    traffic = _traffic()
    achieved = flops_mv / (mv_ms_max * 1e-3) / 1e12
    roofline = {"bound": "tensor", "kernel": "gpfvm_gram_matvec (DMMA FP64 mode-product GEMMs of the reflection-parity-split plan, whole matvec graph; achieved = executed flops / time)",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "peak_source": peak_src,
                "traffic": traffic.get("config1", {}).get("dram_bytes"),
                "traffic_source": traffic.get("config1", {}).get("source"),
                "algorithmic_bytes": bytes_mv, "flops_per_launch": flops_mv,
                # context: the same matvec through the unsplit plan would execute these flops
                # (the reflection-parity split halves the PDE-PDE pairs)
                "flops_per_launch_unsplit_plan": gp.matvec_flops_unsplit() * R,
                "unsplit_plan_equivalent_tflops": gp.matvec_flops_unsplit() * R / (mv_ms_max * 1e-3) / 1e12}
    configs = None
    if not args.no_configs:
        configs = {}
        for name, builder, nr in (("config2", gi.config2, 4), ("config3", gi.config3, 4), ("config4", gi.config4, 4)):
            try:
                configs[name] = bench_config(builder, nr, dev, fp64_peak, traffic.get(name, {}), world,
                                             solve_budget=0 if args.no_budget_solve else 1250,
                                             full_reorth=(name == "config2"))
            except Exception as e:  # never break the headline line
                configs[name] = {"error": repr(e)[:200]}

    sharded = None
    # The sharded section is the only part of this file that only ever runs on
    # one GPU in development (NCCL all_to_all over several GPUs is the driver's
    # to exercise).  A watchdog keeps the headline: if the section has not
    # finished after GPFVM_BENCH_SHARD_TIMEOUT seconds (default 300), rank 0
    # prints the line without it and every rank exits 0.
    shard_done = threading.Event()
    partial_line = {}

    def _watchdog():
        if shard_done.wait(float(os.environ.get("GPFVM_BENCH_SHARD_TIMEOUT", "300"))):
            return
        if rank == 0 and partial_line:
            line = dict(partial_line)
            line["sharded"] = {"error": "sharded section timed out; headline measured before it"}
            print(json.dumps(line), flush=True)
        os._exit(0)

    if not args.no_sharded:
        if rank == 0:
            rep0 = reps[-1]
            partial_line.update({
                "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOAD, "n_obs": N, "matvec_nrhs": R, "parallelism": f"replicas{world}"},
                "cg_solve_s": solve_ms_max / 1e3, "cg_iters": rep0["iterations"],
                "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": None, "e2e": e2e,
                "clocks": clk.summary(), "configs": configs})
        threading.Thread(target=_watchdog, daemon=True).start()
    if not args.no_sharded:
        # time-sharded full problems (every block: IC planes on rank 0, faces and
        # PDE block split along time; library gpfvm_shard_* + NCCL all_to_all,
        # DESIGN.md §7): strong scaling of the matvec and of IterGP iterations
        sharded = {}
        for name, builder in (("config3", gi.config3), ("config4", gi.config4)):
            try:
                sharded[name] = bench_sharded(builder, dev, world)
            except Exception as e:  # never break the headline line
                sharded[name] = {"error": repr(e)[:200]}
    shard_done.set()
    if rank == 0:
        cb = None
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_baseline(15.0)
        rep = reps[-1]
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_obs": N, "n_pde": 256 * 512, "n_icbc": N - 256 * 512,
                       "matvec_nrhs": R, "predict_grid": [512, 1024], "l2": "matvec block 135 MB > 126 MB L2",
                       "parallelism": f"replicas{world}"},
            "cg_solve_s": solve_ms_max / 1e3, "cg_iters": rep["iterations"],
            "cg_true_rel_residual": rep["true_rel_residual"],
            "ms": {k: float(np.mean(v)) for k, v in times.items()},
            "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
            "clocks": clk.summary(), "hbm_peak_gbs": peaks.get("hbm_gbs"), "sharded": sharded,
            "configs": configs,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
