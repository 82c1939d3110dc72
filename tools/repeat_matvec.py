"""Bitwise repeatability of the Gram matvec: python tools/repeat_matvec.py config4:2:40 ..."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gpfvm_inputs as gi
from paper_2406_05020_b200 import GpfvmProblem
for arg in sys.argv[1:]:
    name, R, ncall = arg.split(":"); R = int(R); ncall = int(ncall)
    p = getattr(gi, name)()
    gp = GpfvmProblem(p); gp.gpfvm_assemble_factors()
    xt = torch.tensor(gi.random_vectors(p.size, R, 13), device="cuda:0")
    first = gp.gpfvm_gram_matvec(xt).clone()
    out = torch.empty_like(xt)
    bad = []
    for c in range(ncall):
        gp.gpfvm_gram_matvec(xt, out=out)
        if not torch.equal(out, first):
            d = (out - first).abs()
            off = 0; blocks = []
            for b in p.blocks:
                m = float(d[:, off:off + b.size].max())
                if m > 0: blocks.append((b.name, m / float(first.abs().max())))
                off += b.size
            bad.append((c, blocks))
    print(name, R, "calls differing from the first:", len(bad), "of", ncall, bad[:6], flush=True)
    del gp, xt, out, first; torch.cuda.empty_cache()
