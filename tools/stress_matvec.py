"""Repeat the Gram matvec of BASELINE configs and compare every call with the
oracle's Kronecker matvec (cached in /tmp for the session): counts calls with
any element off by more than 1e-12 of max|ref|.
    python tools/stress_matvec.py config4:2:40 config3:2:40 ..."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gpfvm_inputs as gi
from paper_2406_05020_b200 import GpfvmProblem
from oracle.gram import KroneckerGram
for arg in sys.argv[1:]:
    name, R, ncall = arg.split(":"); R = int(R); ncall = int(ncall)
    p = getattr(gi, name)()
    gp = GpfvmProblem(p); gp.gpfvm_assemble_factors()
    X = gi.random_vectors(p.size, R, 9)
    rf = f"/tmp/ref_{name}_{R}.npy"
    if os.path.exists(rf): ref = np.load(rf)
    else:
        ref = KroneckerGram(p).matvec(X[:2]); np.save(rf, ref)
    xt = torch.tensor(X, device="cuda:0"); yt = torch.empty_like(xt)
    bad = 0; worst = 0.0
    for c in range(ncall):
        gp.gpfvm_gram_matvec(xt, out=yt)
        Y = yt[:2].cpu().numpy()
        e = np.abs(Y - ref).max() / np.abs(ref).max()
        worst = max(worst, e); bad += e > 1e-12
    print(f"{name} R={R}: {bad} bad of {ncall} calls, worst {worst:.2e}", flush=True)
    del gp, xt, yt; torch.cuda.empty_cache()
