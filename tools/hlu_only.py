"""Two H-LU factorisations of config 4 (for ncu launch lists) -- dev tool.  usage: hlu_only.py n_min"""
import sys
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
p = fi.config5(nrhs=1) if cfg == "c5" else fi.config4()
n_min = int(sys.argv[1]) if len(sys.argv) > 1 else 16
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, n_min)
for _ in range(2):
    lu = fde.hlu_factor(h, hm, 1e-3)
    torch.cuda.synchronize()
    print("hlu", cfg, lu.info.factor_ms, "ms ops", lu.info.nops, "alg", lu.info.algorithm, "plan ms", lu.info.plan_ms)
    lu.free()
