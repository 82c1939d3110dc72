"""Per-step times of the bench step (config 1): python tools/step_times.py [steps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import gpfvm_inputs as gi
from paper_2406_05020_b200 import GpfvmProblem
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
prob = gi.config1(); grid = gi.heat_grid(512, 1024)
gp = GpfvmProblem(prob); N = gp.N; dev = torch.device("cuda:0")
X = torch.tensor(gi.random_vectors(N, 128, 11), dtype=torch.float64, device=dev); Y = torch.empty_like(X)
rhs = torch.tensor(prob.rhs(), dtype=torch.float64, device=dev); alpha = torch.empty_like(rhs)
mean = torch.empty(512 * 1024, dtype=torch.float64, device=dev); var = torch.empty_like(mean)
for i in range(steps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    e[0].record(); gp.gpfvm_assemble_factors()
    e[1].record(); gp.gpfvm_gram_matvec(X, out=Y)
    e[2].record(); gp.gpfvm_solve(rhs, rtol=1e-8, out=alpha)
    e[3].record(); gp.gpfvm_predict(grid, alpha, cov_mode=1, mean=mean, var=var)
    e[4].record(); torch.cuda.synchronize()
    free, tot = torch.cuda.mem_get_info()
    print(i, " ".join(f"{e[k].elapsed_time(e[k+1]):7.2f}" for k in range(4)), f"free {free/1e9:.1f} GB", flush=True)
