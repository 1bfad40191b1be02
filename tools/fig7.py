"""Fig. fig7 analogue: the preconditioned solve of Example 5.1
on UNIFORM meshes (rho = 0, theta = 1, P = 3, R = 2 and 7, alpha = 1.6 by reading
A16) with the dense O(N_d^2) matvec and with the block-Toeplitz FFT matvec.
Reports per N: cold-solve time (assemble + rhs + H-matrix + H-LU + solve) and the
Krylov time (warm) for both paths, per-matvec times, iterations, and the
difference of the two solutions.  usage: python tools/fig7.py [out.jsonl]"""
import json
import math
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else None
h = fde.Handle(0)


def problem(N, R):
    p = fi.example51(N=N, P=3, R=R)
    p.nodes = fi.uniform_mesh(0.0, 10.0, N)
    p.name = f"ex51-uniform-N{N}-R{R}"
    return p


def ev():
    return torch.cuda.Event(enable_timing=True)


for R in (2, 7):
    for N in (256, 512, 1024, 2048, 4096, 6144, 8192):
        p = problem(N, R)
        rec = {"N": N, "P": 3, "n": p.n, "R": R}
        Xs = {}
        for name, flags, path in (("dense", fde.OP_DENSE, fde.PATH_DENSE), ("fft", fde.OP_TOEPLITZ, fde.PATH_TOEPLITZ)):
            if name == "dense" and N > 8192:
                continue
            try:
                fde.assemble_problem(h, p, flags=flags).free()
            except fde.FdeError as e:   # (the single-CTA shared-memory FFT bounds N)
                rec[name] = str(e)
                continue
            for rep in range(2):   # (second repetition timed)
                torch.cuda.synchronize()
                e0, e1 = ev(), ev()
                e0.record()
                op = fde.assemble_problem(h, p, flags=flags)
                G = fde.sem_rhs(h, op, p.forcings)
                hm = fde.hmatrix_build(h, op, R, 1.0, p.n_min)
                lu = fde.hlu_factor(h, hm, 1e-3)
                X, r = fde.solve(h, op, lu, G, method=fde.BICGSTAB, tol=1e-13, maxiter=400, path=path)
                e1.record()
                torch.cuda.synchronize()
            cold = e0.elapsed_time(e1)
            w0, w1 = ev(), ev()
            w0.record()
            for _ in range(5):
                fde.solve(h, op, lu, G, method=fde.BICGSTAB, tol=1e-13, maxiter=400, path=path)
            w1.record()
            torch.cuda.synchronize()
            m0, m1 = ev(), ev()
            m0.record()
            for _ in range(20):
                fde.stiffness_matvec(h, op, G, path=path)
            m1.record()
            torch.cuda.synchronize()
            rec[name] = {"cold_ms": cold, "krylov_ms": w0.elapsed_time(w1) / 5, "matvec_us": 1e3 * m0.elapsed_time(m1) / 20,
                         "iterations": r.iterations, "matvecs": r.matvecs, "hlu_ms": lu.info.factor_ms}
            Xs[name] = X.clone()
            for o in (lu, hm, op):
                o.free()
        if len(Xs) == 2:
            rec["rel_diff_X"] = (torch.linalg.norm(Xs["fft"] - Xs["dense"]) / torch.linalg.norm(Xs["dense"])).item()
        print(json.dumps(rec), flush=True)
        if out:
            with open(out, "a") as f:
                f.write(json.dumps(rec) + "\n")
