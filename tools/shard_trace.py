import sys; sys.path.insert(0, "/root/repo")
import torch
import gpfvm_inputs as gi
from paper_2406_05020_b200 import GpfvmProblem
from paper_2406_05020_b200.dist import ShardedProblem, TorchComm, LocalComm
p = gi.config4(); gp = GpfvmProblem(p); gp.gpfvm_assemble_factors()
sp = ShardedProblem([gp], LocalComm(1))
x = torch.tensor(gi.random_vectors(p.size, 1, 5)[0], dtype=torch.float64, device="cuda:0")
xl = sp.local([x])
sp.matvec(xl); torch.cuda.synchronize()
import os; os.environ["X"]="1"
print("=== traced matvec", flush=True)
sp.matvec(xl); torch.cuda.synchronize()
