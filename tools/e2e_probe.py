"""Per-step host timing of cold solves with / without the host copy (dev tool)."""
import sys, time
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
def step(e2e):
    t = [time.perf_counter()]
    op = fde.assemble_problem(h, p); t.append(time.perf_counter())
    G = fde.sem_rhs(h, op, p.forcings); t.append(time.perf_counter())
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min); t.append(time.perf_counter())
    lu = fde.hlu_factor(h, hm, 1e-3); t.append(time.perf_counter())
    X, rep = fde.solve(h, op, lu, G, tol=1e-12); t.append(time.perf_counter())
    if e2e: Xh = X.cpu()
    t.append(time.perf_counter())
    lu.free(); t.append(time.perf_counter()); hm.free(); t.append(time.perf_counter()); op.free(); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [round(1e3 * (t[i + 1] - t[i]), 1) for i in range(len(t) - 1)]
    print("e2e" if e2e else "dev", "asm rhs hb hlu solve copy freeLU freeHM freeOP sync:", d, "total", round(1e3 * (t[-1] - t[0]), 1))
for i in range(10): step(False)
