"""Host-wall breakdown of one cold solve (config 4 by default) -- dev tool.

Each phase is bracketed by torch.cuda.synchronize() so that host-side gaps
(tree building, schedule building, allocations, frees) show up.
"""
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = {"c4": fi.config4, "c2": lambda: fi.config2(1.5), "c5": lambda: fi.config5(nrhs=64)}[cfg]()
h = fde.Handle(0)


def tick(t):
    torch.cuda.synchronize()
    return time.perf_counter() - t


for it in range(4):
    T = {}
    t0 = time.perf_counter()
    t = time.perf_counter(); op = fde.assemble_problem(h, p); T["assemble"] = tick(t)
    t = time.perf_counter(); G = fde.sem_rhs(h, op, p.forcings); T["rhs"] = tick(t)
    t = time.perf_counter(); hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min); T["hbuild"] = tick(t)
    t = time.perf_counter(); lu = fde.hlu_factor(h, hm, 1e-3); T["hlu"] = tick(t)
    t = time.perf_counter(); X, rep = fde.solve(h, op, lu, G, tol=1e-12); T["solve"] = tick(t)
    t = time.perf_counter(); lu.free(); T["free_lu"] = tick(t)
    t = time.perf_counter(); hm.free(); T["free_hm"] = tick(t)
    t = time.perf_counter(); op.free(); T["free_op"] = tick(t)
    tot = time.perf_counter() - t0
    dev = dict(assemble=op.info.assemble_ms, hbuild=hm.info.build_ms, hlu=lu.info.factor_ms, solve=rep.solve_ms)
    print(f"it {it}: total {1e3*tot:.1f} ms | " + " ".join(f"{k} {1e3*v:.1f}" for k, v in T.items())
          + " | device " + " ".join(f"{k} {v:.1f}" for k, v in dev.items())
          + f" | iters {rep.iterations} hlu ops {lu.info.nops}")
