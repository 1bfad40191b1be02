"""Condition-number diagnostics:
cond_2(A), cond_2(A~) and cond_2(A~^{-1} A) of the assembled SEM system and the
H-LU-preconditioned one, by dense SVD (cuSOLVER via torch.linalg.svdvals, off the
hot path) of matrices formed with the library's own kernels: A from
sem_assemble, A~ from hmatrix_build, A~^{-1} A column by column through
precond_apply (H-LU at Tol_HLU).  usage: python tools/cond_diag.py [names...]"""
import json
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

CASES = {
    "ex51-N100": lambda: fi.example51(N=100, P=3),
    "ex51-N300": lambda: fi.example51(N=300, P=3),
    "ex51-N1000": lambda: fi.example51(N=1000, P=3),
    "ex51-N300-rho100": lambda: fi.example51(N=300, P=3, rho=100.0),
    "c2": lambda: fi.config2(1.5),
    "c4": lambda: fi.config4(),
}


def cond(M):
    s = torch.linalg.svdvals(M)
    return (s[0] / s[-1]).item()


h = fde.Handle(0)
names = sys.argv[1:] or list(CASES)
for name in names:
    p = CASES[name]()
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    A = fde.operator_dense_paper(h, op)
    At = fde.hmatrix_dense_paper(h, hm)
    Z = fde.precond_apply(h, lu, A.T.contiguous())   # rows: A~^{-1} a_j
    MA = Z.T.contiguous()
    out = dict(case=name, n=p.n, R=p.R, hlu_tol=1e-3, cond_A=cond(A), cond_Atilde=cond(At), cond_precond=cond(MA),
               rel_err_Atilde=(torch.linalg.norm(A - At) / torch.linalg.norm(A)).item())
    print(json.dumps(out), flush=True)
    lu.free(); hm.free(); op.free()
