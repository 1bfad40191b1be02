"""Kernel timeline of one H-LU factorisation through CUPTI (torch.profiler) -- dev tool.
usage: python tools/kineto_trace.py [c4|c5] out.json"""
import sys, json
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace.json"
p = fi.config5(nrhs=1) if cfg == "c5" else fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
for _ in range(2):
    lu = fde.hlu_factor(h, hm, 1e-3); torch.cuda.synchronize(); lu.free()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    lu = fde.hlu_factor(h, hm, 1e-3)
    torch.cuda.synchronize()
print("factor ms", lu.info.factor_ms)
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        ev.append({"name": e.name, "start": e.time_range.start, "end": e.time_range.end})
prof.export_chrome_trace(out.replace(".json", "_chrome.json"))
json.dump(ev, open(out, "w"))
print(len(ev), "device events")
