"""Kernel timeline of one leaf-ordered H-LU of config 4 via torch.profiler (CUPTI
activity records: every kernel's stream, start and end, concurrent kernels
included) -- dev tool.  usage: trace_hlu.py [n_min] [out.json]"""
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

n_min = int(sys.argv[1]) if len(sys.argv) > 1 else 64
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/hlu_trace.json"
p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, n_min)
for _ in range(2):
    lu = fde.hlu_factor(h, hm, 1e-3)
    torch.cuda.synchronize()
    lu.free()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    lu = fde.hlu_factor(h, hm, 1e-3)
    torch.cuda.synchronize()
print("factor_ms", lu.info.factor_ms)
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() >= 0:
        ev.append({"name": e.name.split("(")[0].replace("void ", ""), "start": e.time_range.start,
                   "end": e.time_range.end, "stream": getattr(e, "device_resource_id", -1)})
ev.sort(key=lambda x: x["start"])
json.dump(ev, open(out, "w"))
print("events", len(ev), "->", out)
