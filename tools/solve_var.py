"""Per-kernel device time of several c5 solves (variance hunt) -- dev tool."""
import collections
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

p = fi.config5()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
G = fde.sem_rhs(h, op, p.forcings)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
lu = fde.hlu_factor(h, hm, 1e-3)
for it in range(6):
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500)
        torch.cuda.synchronize()
    tot, cnt = collections.Counter(), collections.Counter()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            n = e.name.split("(")[0].replace("void ", "")
            tot[n] += e.time_range.elapsed_us()
            cnt[n] += 1
    print(f"solve {rep.solve_ms:.1f} ms:", ", ".join(f"{n[:14]} {cnt[n]}x {v/1e3:.1f}" for n, v in tot.most_common(4)), flush=True)
