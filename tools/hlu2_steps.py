"""Leaf-ordered H-LU at tol = 0, stopped after s leaf steps, against a dense
right-looking block LU of A~ after s steps (dev tool).
usage: hlu2_steps.py [c2|c4] N P n_min"""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import fde_inputs as fi  # noqa: E402
import oracle.oracle as O  # noqa: E402  (cluster tree only)
from paper_1808_02937_b200 import fde  # noqa: E402

cfg, N, P, n_min = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
p = fi.config2(1.5, N=N, P=P) if cfg == "c2" else fi.config4(N=N, P=P)
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
Ap = fde.hmatrix_dense_paper(h, hm).cpu().numpy()
perm = fde.internal_to_paper_index(p.N, p.P)
A = Ap[np.ix_(perm, perm)]          # internal order
lv = []


def walk(c):
    if c.children:
        for x in c.children:
            walk(x)
    else:
        lv.append((c.e0 * P, min(c.e1 * P, p.n)))


walk(O.cluster_tree(p.N, n_min))
nl = len(lv)
W = A.copy()
d = np.sqrt(np.abs(np.diag(A)))
scale = d[:, None] * d[None, :]
for s in range(nl + 1):
    fde.set_hlu_mode(2 + s)
    lu = fde.hlu_factor(h, hm, 0.0)
    F = fde.hlu_dense_internal(h, lu).cpu().numpy()
    lu.free()
    E = np.abs(F - W) / scale
    bad = [(i, j, E[lv[i][0]:lv[i][1], lv[j][0]:lv[j][1]].max()) for i in range(nl) for j in range(nl)]
    bad = [b for b in bad if b[2] > 1e-10]
    print(f"after {s} steps: max err {E.max():.2e}; bad tiles {[(i, j, f'{e:.1e}') for i, j, e in bad[:12]]}")
    if bad:
        break
    if s == nl:
        break
    # dense reference: step s of the right-looking block LU
    a0, a1 = lv[s]
    D = W[a0:a1, a0:a1]
    for k in range(a1 - a0):
        D[k + 1:, k] /= D[k, k]
        D[k + 1:, k + 1:] -= np.outer(D[k + 1:, k], D[k, k + 1:])
    Lk = np.tril(D, -1) + np.eye(a1 - a0)
    Uk = np.triu(D)
    W[a0:a1, a1:] = np.linalg.solve(Lk, W[a0:a1, a1:])
    W[a1:, a0:a1] = np.linalg.solve(Uk.T, W[a1:, a0:a1].T).T
    W[a1:, a1:] -= W[a1:, a0:a1] @ W[a0:a1, a1:]
fde.set_hlu_mode(0)
