"""Development prototype of the formatted H-LU recursion (numpy).

NOT part of the product path and not an oracle: it exists to validate the
block recursion (the same partition as csrc/hmatrix.cu) and to count the
device operations the CUDA implementation will issue.
Usage:  PYTHONPATH=. python tools/hlu_proto.py
"""
import collections
import sys

import numpy as np

COUNT = collections.Counter()


class Blk:
    def __init__(self, t, s, kind):
        self.t, self.s, self.kind = t, s, kind   # kind: D, R, H
        self.ch = None
        self.D = None
        self.U = self.V = None


class Cl:
    def __init__(self, e0, e1, r0, r1, lo, hi):
        self.e0, self.e1, self.r0, self.r1, self.lo, self.hi = e0, e1, r0, r1, lo, hi
        self.ch = None


def cluster(nodes, P, n, e0, e1, n_min):
    N = len(nodes) - 1
    c = Cl(e0, e1, e0 * P, min(e1 * P, n), nodes[e0], nodes[min(e1 + 1, N)])
    if e1 - e0 > n_min:
        m = (e0 + e1) // 2
        c.ch = (cluster(nodes, P, n, e0, m, n_min), cluster(nodes, P, n, m, e1, n_min))
    return c


def admissible(t, s, lam):
    diam = max(t.hi - t.lo, s.hi - s.lo)
    dist = max(s.lo - t.hi, t.lo - s.hi, 0.0)
    return dist > 0 and diam <= lam * dist


def build(t, s, A, lam, R):
    if admissible(t, s, lam):
        b = Blk(t, s, "R")
        M = A[t.r0:t.r1, s.r0:s.r1]
        u, sv, vt = np.linalg.svd(M, full_matrices=False)
        k = min(R, len(sv))
        b.U = u[:, :k] * sv[:k]
        b.V = vt[:k].T.copy()
    elif t.ch is None or s.ch is None:
        b = Blk(t, s, "D")
        b.D = A[t.r0:t.r1, s.r0:s.r1].copy()
    else:
        b = Blk(t, s, "H")
        b.ch = [[build(tc, sc, A, lam, R) for sc in s.ch] for tc in t.ch]
    return b


def rows(b):
    return b.t.r1 - b.t.r0


def cols(b):
    return b.s.r1 - b.s.r0


def to_dense(b):
    if b.kind == "D":
        return b.D
    if b.kind == "R":
        return b.U @ b.V.T
    return np.block([[to_dense(b.ch[0][0]), to_dense(b.ch[0][1])], [to_dense(b.ch[1][0]), to_dense(b.ch[1][1])]])


def split_rows(b, X):
    m0 = rows(b.ch[0][0])
    return X[:m0], X[m0:]


def split_cols_of(b, X):
    """split along b's column clusters"""
    n0 = cols(b.ch[0][0])
    return X[:n0], X[n0:]


# ---------------------------------------------------------------- products
def hmul(A, X, trans=False):
    """op(A) @ X with A an H-block, X dense (rows = op(A) cols)."""
    COUNT["hmul_leaf" if A.kind != "H" else "hmul_rec"] += 1
    if A.kind == "D":
        return (A.D.T if trans else A.D) @ X
    if A.kind == "R":
        return (A.V @ (A.U.T @ X)) if trans else (A.U @ (A.V.T @ X))
    if not trans:
        X0, X1 = split_cols_of(A, X)
        top = hmul(A.ch[0][0], X0) + hmul(A.ch[0][1], X1)
        bot = hmul(A.ch[1][0], X0) + hmul(A.ch[1][1], X1)
        return np.vstack([top, bot])
    X0, X1 = split_rows(A, X)
    left = hmul(A.ch[0][0], X0, True) + hmul(A.ch[1][0], X1, True)
    right = hmul(A.ch[0][1], X0, True) + hmul(A.ch[1][1], X1, True)
    return np.vstack([left, right])


def truncate(U, V, tol, kmax=10 ** 9):
    COUNT["truncate"] += 1
    COUNT[f"trunc_k{min(U.shape[1], 200) // 16 * 16}"] += 1
    if U.shape[1] == 0:
        return U, V
    if tol == 0:
        return U, V
    qu, ru = np.linalg.qr(U)
    qv, rv = np.linalg.qr(V)
    x, s, yt = np.linalg.svd(ru @ rv.T)
    r = int(np.sum(s > tol * s[0])) if s[0] > 0 else 0
    r = min(r, kmax)
    return qu @ (x[:, :r] * s[:r]), qv @ yt[:r].T


def product_lr(A, B, tol):
    """A @ B as low rank (U, V)."""
    if A.kind == "R":
        return A.U, hmul(B, A.V, trans=True)
    if B.kind == "R":
        return hmul(A, B.U), B.V
    if A.kind == "H" and B.kind == "H":
        COUNT["hh_to_lr"] += 1
        m0, m1 = rows(A.ch[0][0]), rows(A.ch[1][0])
        n0, n1 = cols(B.ch[0][0]), cols(B.ch[0][1])
        Us, Vs = [], []
        for i in range(2):
            for j in range(2):
                u_parts, v_parts = [], []
                for k in range(2):
                    u, v = product_lr(A.ch[i][k], B.ch[k][j], tol)
                    u_parts.append(u)
                    v_parts.append(v)
                u, v = truncate(np.hstack(u_parts), np.hstack(v_parts), tol)
                U = np.zeros((m0 + m1, u.shape[1]))
                V = np.zeros((n0 + n1, u.shape[1]))
                U[(0 if i == 0 else m0):(m0 if i == 0 else m0 + m1)] = u
                V[(0 if j == 0 else n0):(n0 if j == 0 else n0 + n1)] = v
                Us.append(U)
                Vs.append(V)
        return truncate(np.hstack(Us), np.hstack(Vs), tol)
    # dense x H or H x dense or dense x dense
    COUNT["dense_to_lr"] += 1
    if A.kind == "D":
        P = hmul(B, A.D.T, trans=True).T
    else:
        P = hmul(A, B.D)
    if P.shape[0] <= P.shape[1]:
        return truncate(np.eye(P.shape[0]), P.T.copy(), tol)
    return truncate(P.copy(), np.eye(P.shape[1]), tol)


def add_lr(C, U, V, tol):
    """C += U V^T (formatted)."""
    if U.shape[1] == 0:
        return
    if C.kind == "D":
        COUNT["dense_update"] += 1
        C.D += U @ V.T
    elif C.kind == "R":
        C.U, C.V = truncate(np.hstack([C.U, U]), np.hstack([C.V, V]), tol)
    else:
        m0 = rows(C.ch[0][0])
        n0 = cols(C.ch[0][0])
        Us = (U[:m0], U[m0:])
        Vs = (V[:n0], V[n0:])
        for i in range(2):
            for j in range(2):
                add_lr(C.ch[i][j], Us[i], Vs[j], tol)


def gemm_sub(C, A, B, tol):
    """C -= A B."""
    COUNT["gemm_sub"] += 1
    if A.kind == "H" and B.kind == "H" and C.kind == "H":
        for i in range(2):
            for j in range(2):
                for k in range(2):
                    gemm_sub(C.ch[i][j], A.ch[i][k], B.ch[k][j], tol)
        return
    if C.kind == "D" and A.kind != "R" and B.kind != "R":
        COUNT["dense_gemm"] += 1
        if A.kind == "D" and B.kind == "D":
            C.D -= A.D @ B.D
        elif A.kind == "D":
            C.D -= hmul(B, A.D.T, trans=True).T
        else:
            C.D -= hmul(A, B.D)
        return
    U, V = product_lr(A, B, tol)
    add_lr(C, -U, V, tol)


# ------------------------------------------------------------- triangular
def solve_L(L, X):
    """X <- L^{-1} X (L unit lower, H format)."""
    if L.kind == "D":
        COUNT["leaf_trsm"] += 1
        Lm = np.tril(L.D, -1) + np.eye(L.D.shape[0])
        return np.linalg.solve(Lm, X)
    X0, X1 = split_rows(L, X)
    Y0 = solve_L(L.ch[0][0], X0)
    X1 = X1 - hmul(L.ch[1][0], Y0)
    return np.vstack([Y0, solve_L(L.ch[1][1], X1)])


def solve_U(U, X):
    """X <- U^{-1} X."""
    if U.kind == "D":
        COUNT["leaf_trsm"] += 1
        return np.linalg.solve(np.triu(U.D), X)
    X0, X1 = split_rows(U, X)
    Y1 = solve_U(U.ch[1][1], X1)
    X0 = X0 - hmul(U.ch[0][1], Y1)
    return np.vstack([solve_U(U.ch[0][0], X0), Y1])


def solve_UT(U, X):
    """X <- U^{-T} X."""
    if U.kind == "D":
        COUNT["leaf_trsm"] += 1
        return np.linalg.solve(np.triu(U.D).T, X)
    X0, X1 = split_rows(U, X)
    Y0 = solve_UT(U.ch[0][0], X0)
    X1 = X1 - hmul(U.ch[0][1], Y0, trans=True)
    return np.vstack([Y0, solve_UT(U.ch[1][1], X1)])


def trsm_L(L, B, tol):
    """B <- L^{-1} B (formatted)."""
    if B.kind == "R":
        B.U = solve_L(L, B.U)
    elif B.kind == "D":
        B.D = solve_L(L, B.D)
    else:
        for j in range(2):
            trsm_L(L.ch[0][0], B.ch[0][j], tol)
            gemm_sub(B.ch[1][j], L.ch[1][0], B.ch[0][j], tol)
            trsm_L(L.ch[1][1], B.ch[1][j], tol)


def trsm_U(U, B, tol):
    """B <- B U^{-1} (formatted)."""
    if B.kind == "R":
        B.V = solve_UT(U, B.V)
    elif B.kind == "D":
        B.D = solve_UT(U, B.D.T).T
    else:
        for i in range(2):
            trsm_U(U.ch[0][0], B.ch[i][0], tol)
            gemm_sub(B.ch[i][1], B.ch[i][0], U.ch[0][1], tol)
            trsm_U(U.ch[1][1], B.ch[i][1], tol)


def hlu(A, tol):
    if A.kind == "D":
        COUNT["leaf_lu"] += 1
        D = A.D
        m = D.shape[0]
        for k in range(m):
            D[k + 1:, k] /= D[k, k]
            D[k + 1:, k + 1:] -= np.outer(D[k + 1:, k], D[k, k + 1:])
        return
    hlu(A.ch[0][0], tol)
    trsm_L(A.ch[0][0], A.ch[0][1], tol)
    trsm_U(A.ch[0][0], A.ch[1][0], tol)
    gemm_sub(A.ch[1][1], A.ch[1][0], A.ch[0][1], tol)
    hlu(A.ch[1][1], tol)


def apply_inverse(F, r):
    return solve_U(F, solve_L(F, r))


def main():
    sys.path.insert(0, ".")
    import fde_inputs as fi
    import oracle as O
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2small"
    if cfg == "c1":
        p = fi.config1()
    elif cfg == "c4":
        p = fi.config4(N=256, P=8)
        p.n_min = 16
    else:
        p = fi.config2(1.5, N=64, P=4)
        p.n_min = 4
    tol = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    so = O.assemble_system(p)
    At, _ = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=p.n_min)
    N, P, n = p.N, p.P, p.n
    perm = np.array([e * (P - 1) + q if q < P - 1 else N * (P - 1) + e
                     for r in range(n) for e, q in [divmod(r, P)]])
    Ai = At[np.ix_(perm, perm)]
    root = cluster(p.nodes, P, n, 0, N, p.n_min)
    H = build(root, root, Ai, 1.0, p.R + 4)
    print("max |H - A~| =", np.abs(to_dense(H) - Ai).max())
    hlu(H, tol)
    rng = np.random.default_rng(0)
    r = rng.standard_normal(n)
    z = apply_inverse(H, r.reshape(-1, 1)).ravel()
    zd = np.linalg.solve(Ai, r)
    print(f"tol={tol}: rel err vs dense solve {np.linalg.norm(z - zd) / np.linalg.norm(zd):.3e}")
    for k, v in sorted(COUNT.items()):
        print(f"  {k:16s} {v}")


if __name__ == "__main__":
    main()
