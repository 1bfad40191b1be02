"""A few preconditioner applications (for ncu / A-B) -- dev tool.  usage: apply_only.py [nrhs] [c2|c3|c4|c5]"""
import sys
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
p = {"c2": lambda: fi.config2(1.5), "c3": lambda: fi.config3(16), "c4": fi.config4, "c5": lambda: fi.config5(nrhs=1)}[cfg]()
h = fde.Handle(0)
op = fde.assemble_problem(h, p, flags=fde.OP_TOEPLITZ) if cfg == "c2" else fde.assemble_problem(h, p)
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
print(f"{cfg} apply nrhs {r.shape[0]}: {e0.elapsed_time(e1) / 10:.3f} ms")
