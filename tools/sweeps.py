"""Throughput sweeps (dev tool, BASELINE configs 3 and 4): p-refinement on config 3's
geometric mesh (P = 4..24: cold solves/s, L_inf error against the closed form) and
h-refinement on config 4's graded mesh (N = 128..2048: cold solves/s, GEMV GB/s).
usage: python tools/sweeps.py [p|h|both] > profiles/rNN_sweeps.jsonl"""
import sys, json, time, ctypes
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde

h = fde.Handle(0, stream=torch.cuda.current_stream().cuda_stream)


def cold(p, steps=10, warm=3):
    def step():
        op = fde.assemble_problem(h, p)
        G = fde.sem_rhs(h, op, p.forcings)
        hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
        lu = fde.hlu_factor(h, hm, 1e-3)
        X, rep = fde.solve(h, op, lu, G, tol=1e-12, maxiter=300)
        out = (X, rep.iterations)
        lu.free(); hm.free(); op.free()
        torch.cuda.synchronize()
        return out
    for _ in range(warm):
        step()
    fde.lib().fde_profile(h.h, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        X, its = step()
    e1.record()
    torch.cuda.synchronize()
    prof = (ctypes.c_double * 9)()
    fde.lib().fde_profile_collect(h.h, prof, 1)
    fde.lib().fde_profile(h.h, 0)
    ms = e0.elapsed_time(e1) / steps
    gbs = (prof[2] / prof[0]) / (prof[1] / prof[0] * 1e-3) / 1e9 if prof[0] else None
    return X, its, ms, gbs


mode = sys.argv[1] if len(sys.argv) > 1 else "both"
if mode in ("p", "both"):
    import oracle as O
    from test_gpu_psweep import linf_error
    for P in (4, 8, 12, 16, 20, 24):
        p = fi.config3(P)
        X, its, ms, gbs = cold(p)
        print(json.dumps({"sweep": "p", "config": "c3", "P": P, "n": p.n, "ms_per_solve": ms, "solves_per_s": 1e3 / ms,
                          "iters": its, "linf_err": linf_error(p, X.cpu().numpy()[0]), "gemv_gbs": gbs}), flush=True)
if mode in ("h", "both"):
    for N in (128, 256, 512, 1024, 2048):
        p = fi.config4(N=N)
        X, its, ms, gbs = cold(p, steps=10 if N <= 1024 else 5)
        print(json.dumps({"sweep": "h", "config": "c4", "N": N, "n": p.n, "ms_per_solve": ms, "solves_per_s": 1e3 / ms,
                          "iters": its, "gemv_gbs": gbs}), flush=True)
