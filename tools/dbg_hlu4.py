import numpy as np, torch, sys, ctypes
sys.path.insert(0, '.')
import fde_inputs as fi, oracle as O
from paper_1808_02937_b200 import fde
L = fde.lib()
L.fde_hlu_solve_debug.argtypes = [ctypes.c_void_p]*3 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
h = fde.Handle(0)
p, n_min, tol = fi.config2(1.5, N=48, P=4), 4, 1e-3
op = fde.assemble_problem(h, p)
hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
lu = fde.hlu_factor(h, hm, tol)
perm = fde.internal_to_paper_index(p.N, p.P)
r = np.random.default_rng(5).standard_normal(p.n)
z_api = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()[0]
x = torch.tensor(r[perm].copy(), device="cuda")
L.fde_hlu_solve_debug(h.h, lu.ptr, ctypes.c_void_p(x.data_ptr()), p.n, 1, 0)
L.fde_hlu_solve_debug(h.h, lu.ptr, ctypes.c_void_p(x.data_ptr()), p.n, 1, 1)
zi = x.cpu().numpy(); z_dbg = np.empty_like(zi); z_dbg[perm] = zi
print("api vs dbg", np.linalg.norm(z_api - z_dbg) / np.linalg.norm(z_dbg))
# api twice
z2 = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()[0]
print("api twice", np.linalg.norm(z_api - z2)/np.linalg.norm(z2))
# api with 2 columns
R2 = np.stack([r, r])
z3 = fde.precond_apply(h, lu, torch.tensor(R2, device="cuda")).cpu().numpy()
print("api 2col", np.linalg.norm(z3[0] - z_dbg)/np.linalg.norm(z_dbg), np.linalg.norm(z3[1] - z_dbg)/np.linalg.norm(z_dbg))
# matvec then apply
y = fde.stiffness_matvec(h, op, torch.tensor(r, device="cuda"))
z4 = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()[0]
print("after matvec", np.linalg.norm(z4 - z_dbg)/np.linalg.norm(z_dbg))
