"""Time the Gram matvec of BASELINE configs (graph replay, CUDA events):
    python tools/time_matvec.py config1:128 config2:4 ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gpfvm_inputs as gi  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem  # noqa: E402

for arg in sys.argv[1:]:
    name, R = arg.split(":")
    R = int(R)
    p = getattr(gi, name)()
    gp = GpfvmProblem(p)
    gp.gpfvm_assemble_factors()
    X = torch.tensor(gi.random_vectors(gp.N, R, 7), dtype=torch.float64, device="cuda:0")
    Y = torch.empty_like(X)
    for _ in range(5):
        gp.gpfvm_gram_matvec(X, out=Y)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record(s)
    for _ in range(n):
        gp.gpfvm_gram_matvec(X, out=Y)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = gp.matvec_flops() * R
    print(f"{name} R={R} N={gp.N} matvec {ms:.3f} ms  {16 * gp.N * R / ms / 1e6:.1f} GB/s  "
          f"{fl / ms / 1e9:.2f} TF/s (executed {fl / R / 1e9:.3f} GFLOP/vector)", flush=True)
    del gp, X, Y
    torch.cuda.empty_cache()
