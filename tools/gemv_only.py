"""A few dense stiffness matvecs on config 4 (for ncu) -- dev tool."""
import sys
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
x = torch.randn(1, p.n, dtype=torch.float64, device="cuda")
for _ in range(6):
    y = fde.stiffness_matvec(h, op, x, path=fde.PATH_DENSE)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()))
