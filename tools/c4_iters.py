"""GMRES iterations and preconditioner residual of config 4 at Tol_HLU = 1e-3 (dev tool)."""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
G = fde.sem_rhs(h, op, p.forcings)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
At = fde.hmatrix_dense_paper(h, hm)
r = torch.tensor(np.random.default_rng(6).standard_normal(p.n), device="cuda")
lu = fde.hlu_factor(h, hm, 1e-3)
z = fde.precond_apply(h, lu, r)[0]
q = (torch.linalg.norm(At @ z - r) / torch.linalg.norm(r)).item()
X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500)
print(f"||A~z-r||/||r|| {q:.3e} gmres its {rep.iterations} max_rank {lu.info.max_rank} hlu {lu.info.factor_ms:.1f} ms")
