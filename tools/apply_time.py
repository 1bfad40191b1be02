"""Median precond_apply time on config 4 (1, 2, 4, 8 RHS) and a hash of z (dev tool:
A/B of apply kernels through FDE_LIB_PATH)."""
import sys, hashlib, statistics
sys.path.insert(0, '.')
import numpy as np
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
lu = fde.hlu_factor(h, hm, 1e-3)
out = []
for nrhs in (1, 2, 4, 8):
    r = torch.tensor(np.random.default_rng(nrhs).standard_normal((nrhs, p.n)), device="cuda")
    ts = []
    for it in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); z = fde.precond_apply(h, lu, r); e1.record(); torch.cuda.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    out.append(f"{nrhs} RHS {statistics.median(ts):.1f} us sha {hashlib.sha256(z.cpu().numpy().tobytes()).hexdigest()[:12]}")
print(" | ".join(out))
