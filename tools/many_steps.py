"""Many cold solves in a row (bench-like), per-step time and pool size -- dev tool."""
import sys, time
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
stream = torch.cuda.current_stream()
h = fde.Handle(0, stream=stream.cuda_stream)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 16):
    torch.cuda.synchronize()
    t = time.perf_counter()
    op = fde.assemble_problem(h, p)
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12)
    Xh = X.cpu()
    lu.free(); hm.free(); op.free()
    torch.cuda.synchronize()
    r, u = fde.pool_bytes(0)
    print(f"it {it}: {1e3*(time.perf_counter()-t):7.1f} ms | asm {op.info.assemble_ms:.1f} hb {hm.info.build_ms:.1f} "
          f"hlu {lu.info.factor_ms:.1f} (plan {lu.info.plan_ms:.1f}) solve {rep.solve_ms:.1f} | pool reserved {r/1e9:.2f} GB used {u/1e9:.2f} GB "
          f"torch reserved {torch.cuda.memory_reserved()/1e9:.2f} GB", flush=True)
