"""A few 64-RHS dense stiffness contractions (k_gemm_dmma) on config 5 (for ncu) -- dev tool."""
import sys
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config5(nrhs=1)
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
x = torch.randn(64, p.n, dtype=torch.float64, device="cuda")
for _ in range(4):
    y = fde.stiffness_matvec(h, op, x, path=fde.PATH_DENSE)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    y = fde.stiffness_matvec(h, op, x, path=fde.PATH_DENSE)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"c5 64-RHS matvec {ms:.3f} ms, {2.0 * p.n * p.n * 64 / ms / 1e9:.2f} TFLOP/s", float(y.abs().sum()))
