"""Does clock sampling during the timed region slow the cold solve? -- dev tool.

Times 4 cold solves of config 4 with (a) no sampler, (b) the nvidia-smi
subprocess sampler of bench.py, (c) an in-process NVML sampler thread.
"""
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

p = fi.config4()
h = fde.Handle(0)


def step():
    op = fde.assemble_problem(h, p)
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12)
    lu.free(); hm.free(); op.free()


def timed(k=4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t) / k


for _ in range(3):
    step()
print(f"no sampler      {timed():.1f} ms/step")
fde.lib().fde_profile(h.h, 1)
print(f"profiling on    {timed():.1f} ms/step")
fde.lib().fde_profile(h.h, 0)
s = bench.ClockSampler(0)
s.start()
print(f"nvidia-smi      {timed():.1f} ms/step", s.stop())
cls = getattr(bench, "NvmlSampler", None)
if cls:
    s = cls(0)
    s.start()
    print(f"nvml thread     {timed():.1f} ms/step", s.stop())
print(f"no sampler      {timed():.1f} ms/step")
