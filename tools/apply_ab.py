"""Preconditioner-application timing and old/new agreement on configs 4 and 5 -- dev tool.
usage: python tools/apply_ab.py out.npz   (run once with FDE_APPLY_OLD=1, once without)"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
h = fde.Handle(0)
res = {}
for name, p in (("c4", fi.config4()), ("c5", fi.config5(nrhs=1)), ("c2", fi.config2(1.5))):
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    for nrhs in ((1, 2, 4, 8, 16, 64) if name != "c2" else (1, 8)):
        r = torch.tensor(np.random.default_rng(nrhs).standard_normal((nrhs, p.n)), device="cuda")
        for _ in range(3):
            z = fde.precond_apply(h, lu, r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            z = fde.precond_apply(h, lu, r)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} apply nrhs {nrhs}: {e0.elapsed_time(e1) / 20 * 1000:.1f} us", flush=True)
        res[f"{name}_{nrhs}"] = z.cpu().numpy()
    for o in (lu, hm, op):
        o.free()
np.savez(sys.argv[1], **res)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    for k in res:
        print(k, "max rel diff vs", sys.argv[2], np.abs(res[k] - ref[k]).max() / np.abs(ref[k]).max())
