"""Time one H-LU factorisation of config 4 (host wall vs device) -- dev tool."""
import sys, time
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config5() if (len(sys.argv) > 1 and sys.argv[1] == 'c5') else fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
torch.cuda.synchronize()
for it in range(2):
    t0 = time.perf_counter()
    lu = fde.hlu_factor(h, hm, 1e-3)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"hlu host wall {1e3*(t1-t0):.1f} ms, device {lu.info.factor_ms:.1f} ms, ops {lu.info.nops}, launches {fde.lib().fde_launch_count()}")
    r = torch.randn(1, p.n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): z = fde.precond_apply(h, lu, r)
    torch.cuda.synchronize(); print(f"apply {1e3*(time.perf_counter()-t0)/10:.3f} ms")
    lu.free()
import ctypes
st = (ctypes.c_ulonglong * 4)()
fde.lib().fde_debug_trunc_stats(st)
print("trunc calls", st[0], "avg ke", st[1] / max(st[0], 1), "avg sweeps (2 eigs)", st[2] / max(st[0], 1), "max sweeps (one solve)", st[3])
