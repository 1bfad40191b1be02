"""Example 5.1 iteration counts (paper Table 1 / Table 2 analogue) on the B200 path."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
h = fde.Handle(0)
Ns = [int(a) for a in sys.argv[1:]] or [100, 400, 800, 1500, 2000]
print("N    R=2     R=3     R=5     R=7   (BiCGSTAB iterations / operator applications; L_inf error)")
for N in Ns:
    row = []
    for R in (2, 3, 5, 7):
        p = fi.example51(N=N, P=3, R=R)
        op = fde.assemble_problem(h, p)
        G = fde.sem_rhs(h, op, p.forcings)
        hm = fde.hmatrix_build(h, op, R, 1.0, p.n_min)
        lu = fde.hlu_factor(h, hm, 1e-3)
        X, rep = fde.solve(h, op, lu, G, method=fde.BICGSTAB, tol=1e-13, maxiter=400)
        row.append(f"{rep.iterations:3d}/{rep.matvecs:3d}")
        for o in (lu, hm, op): o.free()
    print(N, "  ".join(row))
