"""tools/host_phases.py for config 5 (one step) -- dev tool."""
import sys
import time
sys.path.insert(0, '.')
import torch  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

p = fi.config5()
h = fde.Handle(0)
for it in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    op = fde.assemble_problem(h, p); t.append(time.perf_counter())
    G = fde.sem_rhs(h, op, p.forcings); t.append(time.perf_counter())
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min); t.append(time.perf_counter())
    lu = fde.hlu_factor(h, hm, 1e-3); t.append(time.perf_counter())
    X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    names = ["assemble", "rhs", "hbuild", "hlu", "solve", "sync"]
    print("host ms:", " ".join(f"{n} {1e3 * (t[i + 1] - t[i]):.1f}" for i, n in enumerate(names)),
          f"| total {1e3 * (t[-1] - t[0]):.1f} | plan {lu.info.plan_ms:.1f} | device hlu {lu.info.factor_ms:.1f} | "
          f"solve dev {rep.solve_ms:.1f} its {rep.iterations}", flush=True)
    lu.free(); hm.free(); op.free()
