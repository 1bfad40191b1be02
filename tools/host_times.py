"""Host time of each API call of a config-4 cold solve (the calls are asynchronous:
this is the host work the device may wait for) -- dev tool."""
import sys, time
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
for it in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    op = fde.assemble_problem(h, p); t.append(time.perf_counter())
    G = fde.sem_rhs(h, op, p.forcings); t.append(time.perf_counter())
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min); t.append(time.perf_counter())
    lu = fde.hlu_factor(h, hm, 1e-3); t.append(time.perf_counter())
    X, rep = fde.solve(h, op, lu, G, tol=1e-12, verify=False); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    if it >= 3:
        d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
        print("host ms: assemble %.3f rhs %.3f hbuild %.3f hlu %.3f solve %.3f sync-wait %.3f | total %.3f | plan_ms %.3f" %
              (*d, 1e3 * (t[-1] - t[0]), lu.info.plan_ms))
    for o in (lu, hm, op):
        o.free()
