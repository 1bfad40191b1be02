"""Per-step phase times of k_apply_pf (FDE_APPLY_TIMELINE=1) -- dev tool.
usage: FDE_APPLY_TIMELINE=1 python tools/apply_timeline.py [c4|c5|c2]"""
import ctypes
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = {"c4": fi.config4(), "c5": fi.config5(nrhs=1), "c2": fi.config2(1.5)}[name]
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
lu = fde.hlu_factor(h, hm, 1e-3)
r = torch.randn(1, p.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    z = fde.precond_apply(h, lu, r)
torch.cuda.synchronize()
L = fde.lib()
L.fde_debug_apply_timeline.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_longlong]
buf = (ctypes.c_ulonglong * (1 << 22))()
n = L.fde_debug_apply_timeline(buf, 1 << 22)
a = np.frombuffer(buf, dtype=np.uint64, count=n).astype(np.int64).reshape(-1, 148, 4)
t0 = a[0, :, 0].min()
print(f"{name}: {a.shape[0]} steps, total {(a[-1, :, 3].max() - t0) / 1e3:.1f} us")
print("step  A(max over CTAs)  barrier1  B(max)  barrier0(next)   [us]")
for s in range(a.shape[0]):
    A = (a[s, :, 1] - a[s, :, 0]).max() / 1e3
    b1 = (a[s, :, 2].min() - a[s, :, 1].max()) / 1e3
    B = (a[s, :, 3] - a[s, :, 2]).max() / 1e3
    nb = (a[s + 1, :, 0].min() - a[s, :, 3].max()) / 1e3 if s + 1 < a.shape[0] else 0
    slowA = int(np.argmax(a[s, :, 1] - a[s, :, 0]))
    print(f"{s:3d}  {A:7.2f} (cta {slowA:3d})  {b1:6.2f}  {B:6.2f}  {nb:6.2f}")
