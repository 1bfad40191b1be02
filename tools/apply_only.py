"""A few preconditioner applications on config 4 (for ncu) -- dev tool."""
import sys
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
lu = fde.hlu_factor(h, hm, 1e-3)
r = torch.randn(int(sys.argv[1]) if len(sys.argv) > 1 else 1, p.n, dtype=torch.float64, device="cuda")
for _ in range(4):
    z = fde.precond_apply(h, lu, r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    z = fde.precond_apply(h, lu, r)
e1.record()
torch.cuda.synchronize()
print(f"apply nrhs {r.shape[0]}: {e0.elapsed_time(e1) / 10:.3f} ms")
