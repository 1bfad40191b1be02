"""Config-5 preconditioner quality for both H-LU algorithms (1 RHS) -- dev tool."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config5(nrhs=1)
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
G = fde.sem_rhs(h, op, p.forcings)
for n_min in [int(a) for a in sys.argv[1:]] or [64]:
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    for mode in (0, 1):
        fde.set_hlu_mode(mode)
        for tol in (1e-3, 1e-5):
            lu = fde.hlu_factor(h, hm, tol)
            r = torch.tensor(np.random.default_rng(6).standard_normal(p.n), device="cuda").reshape(1, -1)
            z = fde.precond_apply(h, lu, r)
            Az = fde.stiffness_matvec(h, op, z, path=fde.PATH_DENSE)
            X, rep = fde.solve(h, op, lu, G, tol=1e-12, maxiter=500)
            print(f"n_min {n_min} alg {lu.info.algorithm} tol {tol:.0e}: gmres {rep.iterations}  hlu {lu.info.factor_ms:.1f} ms "
                  f"solve {rep.solve_ms:.1f} ms max_rank {lu.info.max_rank} ||A z - r||/||r|| {float((Az - r).norm() / r.norm()):.2e}", flush=True)
            lu.free()
    fde.set_hlu_mode(0)
    hm.free()
