import numpy as np, torch, sys, ctypes
sys.path.insert(0, '.')
import fde_inputs as fi, oracle as O
from paper_1808_02937_b200 import fde
L = fde.lib()
L.fde_hlu_solve_debug.argtypes = [ctypes.c_void_p]*3 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
h = fde.Handle(0)
for p, n_min, tol in [(fi.config2(1.5, N=48, P=4), 4, 1e-3), (fi.config2(1.5, N=24, P=4), 4, 1e-3), (fi.config2(1.5, N=16, P=4), 2, 1e-3)]:
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    lu = fde.hlu_factor(h, hm, tol)
    F = fde.hlu_dense_internal(h, lu).cpu().numpy()
    Lm = np.tril(F, -1) + np.eye(p.n); Um = np.triu(F)
    r = np.random.default_rng(5).standard_normal(p.n)
    for which, M in [(0, np.linalg.inv(Lm)), (1, np.linalg.inv(Um)), (2, np.linalg.inv(Um.T))]:
        x = torch.tensor(r, device="cuda")
        rc = L.fde_hlu_solve_debug(h.h, lu.ptr, ctypes.c_void_p(x.data_ptr()), p.n, 1, which)
        xg = x.cpu().numpy(); xe = M @ r
        d = np.abs(xg - xe)
        print(p.name, which, "rel err", np.linalg.norm(d)/np.linalg.norm(xe), "first bad idx", np.argmax(d > 1e-8*np.abs(xe).max()) if (d > 1e-8*np.abs(xe).max()).any() else -1)
    lu.free(); hm.free(); op.free()
