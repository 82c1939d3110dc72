"""One Gram matvec of a BASELINE config between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures (tools/ncu_traffic.py):
    python tools/matvec_once.py config1 128"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gpfvm_inputs as gi  # noqa: E402
from paper_2406_05020_b200 import GpfvmProblem  # noqa: E402

name, R = sys.argv[1], int(sys.argv[2])
p = getattr(gi, name)()
gp = GpfvmProblem(p)
gp.gpfvm_assemble_factors()
X = torch.tensor(gi.random_vectors(gp.N, R, 7), dtype=torch.float64, device="cuda:0")
Y = torch.empty_like(X)
for _ in range(3):  # direct, capture, replay
    gp.gpfvm_gram_matvec(X, out=Y)
torch.cuda.synchronize()
torch.cuda.profiler.start()
gp.gpfvm_gram_matvec(X, out=Y)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(name, R, "flops", gp.matvec_flops() * R, "N", gp.N)
