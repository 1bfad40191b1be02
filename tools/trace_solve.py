"""Kernel timeline of one GMRES solve (after assembly, H-matrix and H-LU) via
torch.profiler -- dev tool.  usage: trace_solve.py c4|c5"""
import collections
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = fi.config5() if cfg == "c5" else fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
G = fde.sem_rhs(h, op, p.forcings)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
lu = fde.hlu_factor(h, hm, 1e-3)
X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500)
    torch.cuda.synchronize()
print("iterations", rep.iterations, "solve_ms", getattr(rep, "solve_ms", None))
tot, cnt = collections.Counter(), collections.Counter()
t0, t1 = None, None
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        n = e.name.split("(")[0].replace("void ", "")
        tot[n] += e.time_range.elapsed_us()
        cnt[n] += 1
        t0 = e.time_range.start if t0 is None else min(t0, e.time_range.start)
        t1 = e.time_range.end if t1 is None else max(t1, e.time_range.end)
print("device span ms", (t1 - t0) / 1e3 if t0 is not None else None)
for n, v in tot.most_common(20):
    print(f"{n[:40]:40s} {cnt[n]:6d} {v/1e3:9.3f} ms")
