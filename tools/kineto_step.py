"""CUPTI kernel trace of one bench cold solve (c4 by default): device-idle gaps and
per-kernel totals -- dev tool.  usage: python tools/kineto_step.py [c4|c5|c2|c3] out.json"""
import sys, json
sys.path.insert(0, '.')
import torch
import bench
from paper_1808_02937_b200 import fde
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/step_trace.json"
prob = bench.workload(cfg)
flags, path = bench.op_path(cfg, fde)
h = fde.Handle(0, stream=torch.cuda.current_stream().cuda_stream)


def step():
    op = fde.assemble_problem(h, prob, flags)
    G = fde.sem_rhs(h, op, prob.forcings)
    hm = fde.hmatrix_build(h, op, prob.R, prob.lam, prob.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500, path=path, verify=False)
    lu.free(); hm.free(); op.free()
    torch.cuda.synchronize()


for _ in range(3):
    step()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
prof.export_chrome_trace(out)
d = json.load(open(out))
evs = [e for e in d['traceEvents'] if e.get('ph') == 'X' and e.get('cat') in ('kernel', 'gpu_memcpy', 'gpu_memset')]
evs.sort(key=lambda e: e['ts'])
t0 = evs[0]['ts']
t1 = max(e['ts'] + e['dur'] for e in evs)
print(f"{cfg}: {len(evs)} device ops over {t1 - t0:.0f} us")
# device-idle gaps (no op on any stream)
busy_end = t0
gaps = []
for e in evs:
    if e['ts'] > busy_end + 2.0:
        gaps.append((e['ts'] - busy_end, busy_end - t0, e['name'][:50]))
    busy_end = max(busy_end, e['ts'] + e['dur'])
print(f"device idle total {sum(g[0] for g in gaps):.0f} us in {len(gaps)} gaps; largest:")
for g in sorted(gaps, reverse=True)[:15]:
    print(f"  {g[0]:8.1f} us at +{g[1]:8.1f}  before {g[2]}")
tot = {}
for e in evs:
    n = e['name'].split('(')[0].replace('void ', '')[:40]
    tot[n] = tot.get(n, 0) + e['dur']
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"  {v:9.1f} us  {n}")
