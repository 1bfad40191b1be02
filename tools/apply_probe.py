"""Time the preconditioner apply (1 and 8 RHS) of config 4/2; save z for
cross-variant comparison -- dev tool.  usage: apply_probe.py tag [c4|c2]"""
import sys, time
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
tag = sys.argv[1]
p = fi.config4() if (len(sys.argv) < 3 or sys.argv[2] == 'c4') else fi.config2()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
lu = fde.hlu_factor(h, hm, 1e-3)
torch.cuda.synchronize()
g = torch.Generator().manual_seed(5)
out = {}
for nrhs in (1, 4, 8):
    r = torch.randn(nrhs, p.n, dtype=torch.float64, generator=g).cuda()
    for _ in range(3): z = fde.precond_apply(h, lu, r)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20): z = fde.precond_apply(h, lu, r)
    torch.cuda.synchronize()
    print(f"{tag} nrhs {nrhs}: apply {1e3*(time.perf_counter()-t0)/20:.3f} ms", flush=True)
    out[nrhs] = z.cpu()
torch.save(out, f"/tmp/apply_{tag}.pt")
