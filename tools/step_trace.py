"""Device timeline of one config-4 cold solve (bench.py's step) through CUPTI: the idle
gaps between kernels show where the device waits for the host -- dev tool."""
import sys
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
from torch.profiler import profile, ProfilerActivity
p = fi.config4()
h = fde.Handle(0)

def step():
    op = fde.assemble_problem(h, p)
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12, verify=False)
    torch.cuda.synchronize()
    for o in (lu, hm, op):
        o.free()

for _ in range(3):
    step()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
iv = sorted((e.time_range.start - t0, e.time_range.end - t0, e.name) for e in ev)
busy_end = 0.0
gaps = []
for s, e, n in iv:
    if s > busy_end + 5.0:
        gaps.append((busy_end, s, n))
    busy_end = max(busy_end, e)
print("span us", busy_end, "kernels", len(iv))
tot = sum(b - a for a, b, _ in gaps)
print("idle gaps > 5 us:", len(gaps), "total", round(tot, 1), "us")
for a, b, n in sorted(gaps, key=lambda g: -(g[1] - g[0]))[:25]:
    print(f"  {a:9.1f} -> {b:9.1f}  {b - a:7.1f} us  before {n[:60]}")

if len(sys.argv) > 2:
    a, b = float(sys.argv[1]), float(sys.argv[2])
    for s_, e_, n in iv:
        if a <= s_ <= b:
            print(f"{s_:9.1f} {e_:9.1f} {e_ - s_:7.1f} {n[:70]}")
