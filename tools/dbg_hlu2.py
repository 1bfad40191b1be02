import numpy as np, torch, sys
sys.path.insert(0, '.')
import fde_inputs as fi, oracle as O
from paper_1808_02937_b200 import fde
h = fde.Handle(0)
for p, n_min, tol in [(fi.config1(), 2, 0.0), (fi.config2(1.5, N=48, P=4), 4, 0.0), (fi.config2(1.5, N=48, P=4), 4, 1e-3), (fi.config3(P=4), 4, 1e-3)]:
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    lu = fde.hlu_factor(h, hm, tol)
    F = fde.hlu_dense_internal(h, lu).cpu().numpy()
    so = O.assemble_system(p)
    At, part = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min)
    perm = fde.internal_to_paper_index(p.N, p.P)
    Ai = At[np.ix_(perm, perm)]
    Lm = np.tril(F, -1) + np.eye(p.n); Um = np.triu(F)
    print(p.name, tol, "||LU-A~||/||A~||", np.linalg.norm(Lm @ Um - Ai) / np.linalg.norm(Ai), "cond(A~)", np.linalg.cond(Ai), "maxrank", lu.info.max_rank)
    r = np.random.default_rng(5).standard_normal(p.n)
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()[0]
    zo = np.linalg.solve(At, r)
    # factor-based solve in internal order
    ri = r[perm]
    zi = np.linalg.solve(Um, np.linalg.solve(Lm, ri))
    zf = np.empty_like(zi); zf[perm] = zi
    print("   apply vs dense:", np.linalg.norm(z - zo) / np.linalg.norm(zo), " F-solve vs dense:", np.linalg.norm(zf - zo) / np.linalg.norm(zo), " apply vs F-solve:", np.linalg.norm(z - zf) / np.linalg.norm(zf))
    lu.free(); hm.free(); op.free()
h.close()
