import sys, ctypes
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
for _ in range(3):
    lu = fde.hlu_factor(h, hm, 1e-3); torch.cuda.synchronize(); lu.free()
st = (ctypes.c_ulonglong * 4)()
fde.lib().fde_debug_trunc_stats.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
fde.lib().fde_debug_trunc_stats(st)
print("calls", st[0] / 3, "mean width", st[1] / max(st[0], 1), "mean sweeps", st[2] / max(st[0], 1), "max", st[3])
