"""Cold-solve phases of config 4 for several leaf sizes n_min (dev tool)."""
import sys, time
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4()
h = fde.Handle(0)
op = fde.assemble_problem(h, p)
G = fde.sem_rhs(h, op, p.forcings)
for n_min in [int(a) for a in sys.argv[1:]] or [16, 32, 64]:
    for it in range(2):
        hm = fde.hmatrix_build(h, op, p.R, p.lam, n_min)
        lu = fde.hlu_factor(h, hm, 1e-3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            z = fde.precond_apply(h, lu, G)
        torch.cuda.synchronize()
        ta = (time.perf_counter() - t0) / 5
        X, rep = fde.solve(h, op, lu, G, tol=1e-12)
        if it == 1:
            print(f"n_min={n_min}: hbuild {hm.info.build_ms:.1f} ms, hlu {lu.info.factor_ms:.1f} ms ({lu.info.nops} ops), "
                  f"apply {1e3*ta:.3f} ms, gmres iters {rep.iterations}, solve {rep.solve_ms:.1f} ms, "
                  f"dense {hm.info.dense_entries*8/1e6:.0f} MB lr {hm.info.lr_entries*8/1e6:.0f} MB")
        lu.free(); hm.free()
