"""Kernel timeline of one config-4 assembly through CUPTI (torch.profiler) -- dev tool."""
import sys
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
from torch.profiler import profile, ProfilerActivity
p = fi.config4()
h = fde.Handle(0)
for _ in range(3):
    op = fde.assemble_problem(h, p); torch.cuda.synchronize(); op.free()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    op = fde.assemble_problem(h, p)
    torch.cuda.synchronize()
print("assemble_ms", op.info.assemble_ms)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f} {e.name[:60]}")
