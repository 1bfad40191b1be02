"""Time the 64-RHS preconditioner apply of config 5 -- dev tool."""
import sys, time
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config5()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
lu = fde.hlu_factor(h, hm, 1e-3)
torch.cuda.synchronize()
r = torch.randn(64, p.n, dtype=torch.float64, device="cuda")
for _ in range(2): z = fde.precond_apply(h, lu, r)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): z = fde.precond_apply(h, lu, r)
torch.cuda.synchronize()
print(f"c5 apply 64 RHS: {1e3*(time.perf_counter()-t0)/5:.2f} ms", flush=True)
