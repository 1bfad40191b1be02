"""Truncation statistics and k_bcore phase profile (FDE_TRUNC_STATS=1) -- dev tool.
usage: FDE_TRUNC_STATS=1 python tools/trunc_stats.py [c4|c5]"""
import sys, ctypes
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = fi.config5(nrhs=1) if cfg == "c5" else fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
nf = 3
for _ in range(nf):
    lu = fde.hlu_factor(h, hm, 1e-3); torch.cuda.synchronize(); lu.free()
st = (ctypes.c_ulonglong * 32)()
fde.lib().fde_debug_trunc_profile.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
fde.lib().fde_debug_trunc_profile(st)
calls = max(st[0], 1)
print(cfg, "truncations per factorisation", st[0] / nf, "mean width", st[1] / calls, "mean sweeps", st[2] / calls,
      "max sweeps", st[3])
print("  nonzero width: mean", st[16] / calls, "max", st[17], "| chunks: mean", st[18] / calls, "max", st[19],
      "| max CTA cycles", st[20])
names = ["mask", "gram", "index", "scale", "pivchol", "coreprod", "jacobi", "order", "output"]
tot = sum(st[4 + i] for i in range(9))
print("  phase cycles per CTA (mean):", " | ".join(f"{n} {st[4 + i] / calls:.0f}" for i, n in enumerate(names)),
      f"| total {tot / calls:.0f}")
