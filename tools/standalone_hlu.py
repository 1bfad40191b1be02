"""NEXT-3: the standalone H-LU solve of
A~ X = G (Tol_HLU 1e-13) against the preconditioned Krylov solve of A X = G
(GMRES 1e-12, = the Galerkin solution) on Example 5.1 -- the H-matrix
approximation error that the standalone solve keeps and the preconditioned
solve removes.  usage: python tools/standalone_hlu.py"""
import json
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

h = fde.Handle(0)
for rho in (0.0, 100.0):
    for N in (100, 300, 1000, 2000):
        for R in (3, 5, 7):
            p = fi.example51(N=N, P=3, R=R, rho=rho)
            op = fde.assemble_problem(h, p)
            G = fde.sem_rhs(h, op, p.forcings)
            hm = fde.hmatrix_build(h, op, R, 1.0, p.n_min)
            try:
                lu_ex = fde.hlu_factor(h, hm, 1e-13)
            except fde.FdeError as e:   # (rank capacity)
                print(json.dumps(dict(rho=rho, N=N, R=R, error=e.name)), flush=True)
                op.free(); hm.free()
                continue
            Xs = fde.precond_apply(h, lu_ex, G)
            lu = fde.hlu_factor(h, hm, 1e-3)
            X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500)
            err = (torch.linalg.norm(Xs - X) / torch.linalg.norm(X)).item()
            res = (torch.linalg.norm(fde.stiffness_matvec(h, op, Xs) - G) / torch.linalg.norm(G)).item()
            print(json.dumps(dict(rho=rho, N=N, R=R, standalone_rel_diff=err, standalone_residual=res,
                                  gmres_its=rep.iterations)), flush=True)
            for o in (lu, lu_ex, hm, op):
                o.free()
