"""Batched truncation in isolation (fde_debug_truncate) for ncu launch lists -- dev tool.
usage: python tools/trunc_bench.py [k] [m] [nb]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1808_02937_b200 import fde
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 14
h = fde.Handle(0)
rng = np.random.default_rng(0)
U = np.empty((nb, k, m))
V = np.empty((nb, k, m))
for q in range(nb):
    sig = 10.0 ** -np.linspace(0, 5, k)
    X = np.linalg.qr(rng.standard_normal((m, k)))[0]
    Y = np.linalg.qr(rng.standard_normal((m, k)))[0]
    G = rng.standard_normal((k, k)) + 3 * np.eye(k)
    U[q] = (X @ np.diag(sig) @ G).T
    V[q] = (Y @ np.linalg.inv(G).T).T
U = torch.tensor(U, device="cuda")
V = torch.tensor(V, device="cuda")
for _ in range(10):
    Uo, Vo, ov = fde.truncate(h, U, V, 1e-3, 16)
torch.cuda.synchronize()
print("k", k, "m", m, "nb", nb, "kept", int((Uo[0].abs().sum(1) > 0).sum()))
import ctypes
st = (ctypes.c_ulonglong * 32)()
fde.lib().fde_debug_trunc_profile.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
fde.lib().fde_debug_trunc_profile(st)
calls = max(st[0], 1)
names = ["mask", "gram", "index", "scale", "pivchol", "coreprod", "jacobi", "order", "output"]
print("calls", st[0], "mean sweeps", st[2] / calls, "max", st[3], "| max CTA cycles", st[20])
print("  phase cycles per CTA (mean):", " | ".join(f"{n} {st[4 + i] / calls:.0f}" for i, n in enumerate(names)))
