"""In-process A/B of H-LU environment switches read per factorisation (dev tool).
usage: python tools/ab_inproc.py c4|c5 "A=1 B=2" "A=0" ...   (each argument one setting;
interleaved over 5 rounds; median factor time and the median cold H-LU + solve time)"""
import os, sys, statistics
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
cfg = sys.argv[1]
sets = sys.argv[2:] or [""]
p = fi.config5(nrhs=1) if cfg == "c5" else fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
G = fde.sem_rhs(h, op, p.forcings)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
keys = set()
for s in sets:
    for kv in s.split():
        keys.add(kv.split("=")[0])
res = {s: [] for s in sets}
its = {s: None for s in sets}
for rnd in range(6):
    for s in sets:
        for k in keys:
            os.environ.pop(k, None)
        for kv in s.split():
            k, v = kv.split("=")
            os.environ[k] = v
        lu = fde.hlu_factor(h, hm, 1e-3)
        X, rep = fde.solve(h, op, lu, G, tol=1e-12)
        torch.cuda.synchronize()
        if rnd > 0:
            res[s].append(lu.info.factor_ms)
        its[s] = rep.iterations
        lu.free()
for s in sets:
    v = res[s]
    print(f"[{s or 'default'}] factor ms median {statistics.median(v):.3f} min {min(v):.3f} max {max(v):.3f} gmres its {its[s]}")
