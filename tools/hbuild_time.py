"""Median hmatrix_build time of config 4 (dev tool: A/B of H-matrix build changes)."""
import sys, statistics
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
ts = []
for _ in range(12):
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    torch.cuda.synchronize()
    ts.append(hm.info.build_ms)
    hm.free()
print("hbuild_ms median", round(statistics.median(ts[2:]), 4), "min", round(min(ts[2:]), 4))
