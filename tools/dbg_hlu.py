import numpy as np, torch, sys
sys.path.insert(0, '.')
import fde_inputs as fi, oracle as O
from paper_1808_02937_b200 import fde
h = fde.Handle(0)
for p, n_min in [(fi.config1(), 2), (fi.config2(1.5, N=48, P=4), 4), (fi.config2(1.5, N=16, P=4), 2)]:
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    lu = fde.hlu_factor(h, hm, 0.0)
    F = fde.hlu_dense_internal(h, lu).cpu().numpy()
    so = O.assemble_system(p)
    At, part = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min)
    perm = fde.internal_to_paper_index(p.N, p.P)
    Ai = At[np.ix_(perm, perm)]
    Lm = np.tril(F, -1) + np.eye(p.n); Um = np.triu(F)
    E = Lm @ Um - Ai
    print(p.name, "n", p.n, "max |LU - A~|", np.abs(E).max(), "scale", np.abs(Ai).max(), "info", lu.info.nops, lu.info.max_rank)
    # exact LU
    def lu_nopiv(A):
        A = A.copy(); n = len(A)
        for k in range(n):
            A[k+1:, k] /= A[k, k]; A[k+1:, k+1:] -= np.outer(A[k+1:, k], A[k, k+1:])
        return A
    Fe = lu_nopiv(Ai)
    D = np.abs(F - Fe)
    bad = np.argwhere(D > 1e-8 * np.abs(Fe).max())
    if len(bad):
        print("  first bad entries (internal r,c):", bad[:10].tolist(), "count", len(bad))
        r, c = bad[0]
        print("  F", F[r, c], "exact", Fe[r, c])
