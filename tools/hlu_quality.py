"""Preconditioner quality of both H-LU algorithms at Tol_HLU = 1e-3 (dev tool):
GMRES iterations and ||A~ z - r|| / ||r|| for a few configurations."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

cases = [("c3-P12", fi.config3(P=12), 16), ("c3-P16", fi.config3(P=16), 16), ("c3-P8", fi.config3(P=8), 16),
         ("c4", fi.config4(), 64), ("c4-N128", fi.config4(N=128, P=8), 40), ("c2", fi.config2(1.5), 16)]
h = fde.Handle(0)
for name, p, n_min in cases:
    op = fde.assemble_problem(h, p)
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    At = fde.hmatrix_dense_paper(h, hm).cpu().numpy()
    r = np.random.default_rng(6).standard_normal(p.n)
    for mode in (0, 1):
        fde.set_hlu_mode(mode)
        for tol in (1e-3, 1e-5):
            lu = fde.hlu_factor(h, hm, tol)
            z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()[0]
            q = np.linalg.norm(At @ z - r) / np.linalg.norm(r)
            try:
                X, rep = fde.solve(h, op, lu, G, tol=1e-12, maxiter=300)
                its = rep.iterations
            except fde.FdeError as e:
                its = f"fail ({e})"[:40]
            print(f"{name:8s} alg {lu.info.algorithm} tol {tol:.0e}: ||A~z-r||/||r|| {q:.2e}  gmres {its}  "
                  f"hlu {lu.info.factor_ms:.1f} ms max_rank {lu.info.max_rank}", flush=True)
            lu.free()
    fde.set_hlu_mode(0)
    hm.free()
    op.free()
