"""Leaf-ordered vs recursive H-LU at tol = 0: per-tile difference map of the
packed factors (dev tool).  usage: hlu2_debug.py [c2|c4] N P n_min"""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

cfg, N, P, n_min = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
p = fi.config2(1.5, N=N, P=P) if cfg == "c2" else fi.config4(N=N, P=P)
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
F = []
for mode in (0, 1):
    fde.set_hlu_mode(mode)
    lu = fde.hlu_factor(h, hm, 0.0)
    print("mode", mode, "algorithm", lu.info.algorithm, "nops", lu.info.nops, "max_rank", lu.info.max_rank)
    F.append(fde.hlu_dense_internal(h, lu).cpu().numpy())
    lu.free()
A = fde.hmatrix_dense_paper(h, hm) if hasattr(fde, "hmatrix_dense_paper") else None
d = np.sqrt(np.abs(np.diag(F[1])))
E = np.abs(F[0] - F[1]) / (d[:, None] * d[None, :])
import oracle.oracle as O   # dev tool: cluster tree only
root = O.cluster_tree(p.N, n_min)
lv = []
def walk(c):
    if c.children:
        for x in c.children:
            walk(x)
    else:
        lv.append((c.e0 * P, min(c.e1 * P, p.n)))
walk(root)
nl = len(lv)
print("leaves", nl, lv[:4], "max err", E.max())
for i in range(nl):
    row = ""
    for j in range(nl):
        e = E[lv[i][0]:lv[i][1], lv[j][0]:lv[j][1]].max()
        row += "." if e < 1e-12 else ("o" if e < 1e-6 else "X")
    print(row)
