import sys; sys.path.insert(0, "/root/repo")
import torch, numpy as np
import gpfvm_inputs as gi
from paper_2406_05020_b200 import GpfvmProblem
p = gi.config1(); gp = GpfvmProblem(p); gp.gpfvm_assemble_factors()
y = torch.tensor(p.rhs(), device="cuda:0")
for i in range(3):
    torch.cuda.synchronize()
    a, rep = gp.gpfvm_solve(y, rtol=1e-8)
    torch.cuda.synchronize()
print({k: rep[k] for k in rep if k != "breakdown_detail"})
