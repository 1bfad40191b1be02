"""Example 5.1 iteration counts on the B200 path: the paper's Table 1 (h-refinement,
P = 3) and Table 2 (p-refinement, N = 300) analogues (SURVEY 8(f)
NEXT-1).  BiCGSTAB on A~^{-1} A X = A~^{-1} G, tol 1e-13, Tol_HLU 1e-3, rho = 0,
theta = 1, alpha = 1.6 (reading A16).  Each cell: iterations / operator
applications (the paper's counts are even: two applications per iteration, A13).
usage: python tools/table1.py [table1|table2|both] [interleaved|paper] [n_min]
(paper: the paper's modal / nodal partition)"""
import sys
sys.path.insert(0, '.')
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

h = fde.Handle(0)
which = sys.argv[1] if len(sys.argv) > 1 else "both"
part = fde.PARTITION_PAPER if (len(sys.argv) > 2 and sys.argv[2] == "paper") else fde.PARTITION_INTERLEAVED
nmin = int(sys.argv[3]) if len(sys.argv) > 3 else None
print(f"# partition: {'paper (modal / nodal trees)' if part else 'interleaved (reading A9)'}, "
      f"n_min {nmin or 'default (16)'}")


def cell(N, P, R):
    p = fi.example51(N=N, P=P, R=R)
    op = fde.assemble_problem(h, p)
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, R, 1.0, nmin or p.n_min, partition=part)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, method=fde.BICGSTAB, tol=1e-13, maxiter=400)
    for o in (lu, hm, op):
        o.free()
    return f"{rep.iterations:3d}/{rep.matvecs:3d}"


if which in ("table1", "both"):
    print("Table 1 analogue (P = 3):  R=2     R=3     R=5     R=7")
    for N in (100, 400, 800, 1500, 2000):
        print(f"  N={N:5d}              ", "  ".join(cell(N, 3, R) for R in (2, 3, 5, 7)), flush=True)
if which in ("table2", "both"):
    print("Table 2 analogue (N = 300): R=2     R=3     R=5     R=7")
    for P in (3, 5, 9, 13, 19):
        print(f"  P={P:3d}                 ", "  ".join(cell(300, P, R) for R in (2, 3, 5, 7)), flush=True)
