"""Plain CPU fp64/long-double oracle for the SEM system of arXiv 1808.02937.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
passage of /root/reference/PAPER.md (or the DESIGN.md reading) it follows.

Index conventions (oracle side, independent of the CUDA path):
  * paper order: X = [u^1_1..u^{P-1}_1; ...; u^1_N..u^{P-1}_N; u~_1..u~_{N-1}]
  * extended order = paper order + [hat of node 0, hat of node N] (for lifting).

Parity: every function here is pinned in tests/test_oracle_pins.py and
tests/test_oracle_branch_pins.py (the latter also runs each pin against a
deliberately broken copy of the branch it pins, which must fail): theta != 1/2
orientation, t-expansion and upper (1-theta) W Q^T blocks, Legendre-series and
singular power loads, boundary-hat lifting.  Not pinned:
  * `hlu`-related behaviour at Tol_HLU = 1e-3, which has no plain definition
    (DESIGN.md "parity unpinned" list).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fde_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile oracle/fde_oracle.c (plain gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


def load_library(path: str):
    """ctypes handle of a compiled oracle library with its signatures declared
    (the mutation pins load deliberately broken copies through this)."""
    L = ctypes.CDLL(path)
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    L.orc_pair_offdiag.restype = ctypes.c_long
    L.orc_pair_offdiag.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, dp]
    L.orc_pair_self.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, dp]
    L.orc_assemble_Sl.argtypes = [ctypes.c_int, dp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                  ctypes.c_int, dp, ctypes.c_int]
    L.orc_assemble_mass.argtypes = [ctypes.c_int, dp, ctypes.c_int, dp]
    L.orc_load.argtypes = [ctypes.c_int, dp, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                           ctypes.c_int, dp, ctypes.c_int, ip, dp, dp, dp]
    L.orc_eval_solution.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, dp, dp]
    L.orc_gl_table.argtypes = [ctypes.c_int, dp, dp]
    L.orc_gj_table.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, dp, dp]
    L.orc_local_deriv.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, dp]
    L.orc_local_value.argtypes = [ctypes.c_int, ctypes.c_double, dp]
    L.orc_frac_integral_monomial.restype = ctypes.c_double
    L.orc_frac_integral_monomial.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int]
    return L


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = load_library(_SO)
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ------------------------------------------------------------------ tables
def gl_table(n: int) -> Tuple[np.ndarray, np.ndarray]:
    x, w = np.zeros(n), np.zeros(n)
    assert lib().orc_gl_table(n, _p(x), _p(w)) == 0
    return x, w


def gj_table(n: int, a: float, b: float) -> Tuple[np.ndarray, np.ndarray]:
    """Gauss-Jacobi nodes/weights for the weight (1-x)^a (1+x)^b on [-1,1]."""
    x, w = np.zeros(n), np.zeros(n)
    assert lib().orc_gj_table(n, a, b, _p(x), _p(w)) == 0
    return x, w


def local_deriv(P: int, h: float, xi: float) -> np.ndarray:
    """Physical derivatives of [left hat, psi_1..psi_{P-1}, right hat]."""
    o = np.zeros(P + 1)
    lib().orc_local_deriv(P, h, xi, _p(o))
    return o


def local_value(P: int, xi: float) -> np.ndarray:
    o = np.zeros(P + 1)
    lib().orc_local_value(P, xi, _p(o))
    return o


def frac_integral_monomial(x: float, beta: float, gam: float, q: int = 24) -> float:
    """0I^beta s^gam at x by the oracle's singular rule (PAPER.md:43 definition)."""
    return lib().orc_frac_integral_monomial(x, beta, gam, q)


# --------------------------------------------------------------- pair / assembly
def pair_integral(P: int, alpha: float, nodes: np.ndarray, i: int, j: int) -> np.ndarray:
    """gamma0 int_{e_i} int_{e_j, s<t} phi_a'(t)(t-s)^{1-alpha} phi_b'(s) for local fns a,b.

    (P+1)x(P+1), zero if j > i (S_l vanishes when the trial element lies right of
    the test element)."""
    out = np.zeros((P + 1) * (P + 1))
    if j > i:
        return out.reshape(P + 1, P + 1)
    hi = nodes[i + 1] - nodes[i]
    if i == j:
        assert lib().orc_pair_self(P, alpha, hi, _p(out)) == 0
    else:
        hj = nodes[j + 1] - nodes[j]
        d = nodes[i] - nodes[j + 1]
        assert lib().orc_pair_offdiag(P, alpha, d, hi, hj, _p(out)) >= 0
    return out.reshape(P + 1, P + 1)


def sizes(N: int, P: int) -> Tuple[int, int]:
    """(n, n_modal): n = NP-1 unknowns (reading A3 of PAPER.md:190)."""
    return N * P - 1, N * (P - 1)


def assemble_Sl_ext(nodes: np.ndarray, P: int, alpha: float, e0: int = 0, e1: Optional[int] = None,
                    threads: Optional[int] = None) -> np.ndarray:
    """Rows of S_l (extended order) contributed by test elements e0..e1-1 (Eq. (lsys))."""
    N = len(nodes) - 1
    e1 = N if e1 is None else e1
    next_ = N * P + 1
    S = np.zeros((next_, next_))
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    th = threads if threads is not None else (os.cpu_count() or 1)
    assert lib().orc_assemble_Sl(N, _p(nodes), P, alpha, e0, e1, _p(S), th) == 0
    return S


def mass_ext(nodes: np.ndarray, P: int) -> np.ndarray:
    """M_IJ = (phi_J, phi_I), extended order."""
    N = len(nodes) - 1
    next_ = N * P + 1
    Mm = np.zeros((next_, next_))
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    lib().orc_assemble_mass(N, _p(nodes), P, _p(Mm))
    return Mm


def load_ext(nodes: np.ndarray, P: int, a: float, b: float, forcing) -> np.ndarray:
    """g_I = (f, phi_I), extended order."""
    N = len(nodes) - 1
    G = np.zeros(N * P + 1)
    leg = np.ascontiguousarray(forcing.leg, dtype=np.float64)
    side = np.array([0 if s == "L" else 1 for s, _, _ in forcing.terms], dtype=np.int32)
    pw = np.array([p for _, p, _ in forcing.terms], dtype=np.float64)
    cf = np.array([c for _, _, c in forcing.terms], dtype=np.float64)
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    lib().orc_load(N, _p(nodes), P, a, b, len(leg), _p(leg) if len(leg) else None, len(cf),
                   side.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) if len(cf) else None,
                   _p(pw) if len(cf) else None, _p(cf) if len(cf) else None, _p(G))
    return G


@dataclass
class System:
    A: np.ndarray          # n x n, paper order
    Abnd: np.ndarray       # n x 2, columns of the boundary hats (node 0, node N)
    Sl_ext: np.ndarray
    M_ext: np.ndarray


def assemble_system(prob, threads: Optional[int] = None) -> System:
    """A = rho M + theta S_l + (1-theta) S_l^T (Eq. (lsys); reading A1)."""
    S = assemble_Sl_ext(prob.nodes, prob.P, prob.alpha, threads=threads)
    Mm = mass_ext(prob.nodes, prob.P)
    Afull = prob.rho * Mm + prob.theta * S + (1 - prob.theta) * S.T
    n = prob.n
    return System(A=Afull[:n, :n].copy(), Abnd=Afull[:n, n:n + 2].copy(), Sl_ext=S, M_ext=Mm)


def rhs(prob, sysm: System, forcing) -> np.ndarray:
    """G with boundary-hat lifting (reading A15): G_int - A[int,{0,N}] [c1,c2]."""
    Gext = load_ext(prob.nodes, prob.P, prob.a, prob.b, forcing)
    n = prob.n
    return Gext[:n] - sysm.Abnd @ np.array([prob.c1, prob.c2])


def solve_dense(A: np.ndarray, G: np.ndarray, refine: int = 3) -> np.ndarray:
    """Direct solve: Jacobi equilibration, LAPACK LU with partial pivoting, iterative
    refinement with long-double residuals (SURVEY.md §8(c) oracle step 6)."""
    G2 = G.reshape(G.shape[0], -1)
    d = 1.0 / np.sqrt(np.abs(np.diag(A)))
    As = A * d[:, None] * d[None, :]
    import scipy.linalg as sla
    lu = sla.lu_factor(As)
    Y = sla.lu_solve(lu, G2 * d[:, None])
    X = Y * d[:, None]
    Al = A.astype(np.longdouble)
    for _ in range(refine):
        R = (G2.astype(np.longdouble) - Al @ X.astype(np.longdouble)).astype(np.float64)
        X = X + sla.lu_solve(lu, R * d[:, None]) * d[:, None]
    return X.reshape(G.shape)


def eval_solution(prob, X: np.ndarray, xis: np.ndarray) -> np.ndarray:
    """u_h at reference points xis of every element; returns (N, len(xis))."""
    n = prob.n
    Xext = np.concatenate([X, [prob.c1, prob.c2]])
    out = np.zeros(prob.N * len(xis))
    xis = np.ascontiguousarray(xis, dtype=np.float64)
    lib().orc_eval_solution(prob.N, prob.P, _p(Xext), len(xis), _p(xis), _p(out))
    return out.reshape(prob.N, len(xis))


# -------------------------------------------------------------- index maps
def paper_index_of_element_dofs(N: int, P: int, e0: int, e1: int) -> np.ndarray:
    """Paper-order indices of the dofs of element cluster [e0,e1): modal dofs of
    the elements and the hats of their right nodes (node e+1, if interior).
    (Cluster dof groups, reading A9 of DESIGN.md.)"""
    n, nm = sizes(N, P)
    idx = []
    for e in range(e0, e1):
        idx.extend(e * (P - 1) + p for p in range(P - 1))
        if e + 1 <= N - 1:
            idx.append(nm + e)
    return np.array(idx, dtype=np.int64)


# ---------------------------------------------------------------- H-matrix
@dataclass
class Cluster:
    e0: int
    e1: int
    children: Tuple["Cluster", ...] = ()


def cluster_tree(N: int, n_min: int, e0: int = 0, e1: Optional[int] = None) -> Cluster:
    """Binary cluster tree over element index ranges, median split (reading A9)."""
    e1 = N if e1 is None else e1
    c = Cluster(e0, e1)
    if e1 - e0 > n_min:
        m = (e0 + e1) // 2
        c.children = (cluster_tree(N, n_min, e0, m), cluster_tree(N, n_min, m, e1))
    return c


def cluster_support(nodes: np.ndarray, c: Cluster) -> Tuple[float, float]:
    """Union of the supports of the cluster's dofs: modal dofs
    cover [x_e0, x_e1]; the hat of node e1 reaches x_{e1+1}."""
    N = len(nodes) - 1
    return nodes[c.e0], nodes[min(c.e1 + 1, N)]


# The paper's own partition (Fig. fig200): the modal functions
# and the nodal hats are clustered separately; S_l = [B F; E C]
# is the first block level.  Dofs in the paper order.
@dataclass
class PCluster:
    kind: str            # "modal" (elements [a, b)), "nodal" (interior nodes [a, b)), "root"
    a: int
    b: int
    children: Tuple["PCluster", ...] = ()


def paper_cluster_tree(N: int, P: int, n_min: int) -> PCluster:
    """Median bisection of the element range (modal tree) and of the interior node
    range 1..N-1 (nodal tree) down to n_min elements / nodes, under a virtual root."""
    def rec(kind, a, b):
        c = PCluster(kind, a, b)
        if b - a > n_min:
            m = (a + b) // 2
            c.children = (rec(kind, a, m), rec(kind, m, b))
        return c
    parts = []
    if P > 1:
        parts.append(rec("modal", 0, N))
    if N > 1:
        parts.append(rec("nodal", 1, N))
    return parts[0] if len(parts) == 1 else PCluster("root", 0, N, tuple(parts))


def pcluster_support(nodes: np.ndarray, c: PCluster) -> Tuple[float, float]:
    """Union of the supports: element e is [x_e, x_{e+1}], the hat of node j is
    [x_{j-1}, x_{j+1}]."""
    if c.kind == "modal":
        return nodes[c.a], nodes[c.b]
    if c.kind == "nodal":
        return nodes[c.a - 1], nodes[c.b]
    return nodes[0], nodes[-1]


def pcluster_dofs(N: int, P: int, c: PCluster) -> np.ndarray:
    """Paper-order indices of the cluster's dofs."""
    nm = N * (P - 1)
    if c.kind == "modal":
        return np.array([e * (P - 1) + p - 1 for e in range(c.a, c.b) for p in range(1, P)], dtype=np.int64)
    if c.kind == "nodal":
        return np.array([nm + j - 1 for j in range(c.a, c.b)], dtype=np.int64)
    return np.arange(N * P - 1, dtype=np.int64)


def support_of(nodes, c):
    return cluster_support(nodes, c) if isinstance(c, Cluster) else pcluster_support(nodes, c)


def dofs_of(N, P, c):
    return paper_index_of_element_dofs(N, P, c.e0, c.e1) if isinstance(c, Cluster) else pcluster_dofs(N, P, c)


def admissible(tau: Tuple[float, float], sig: Tuple[float, float], lam: float) -> bool:
    """max(diam tau, diam sigma) <= lambda dist(tau, sigma)  (Eq. (admis))."""
    diam = max(tau[1] - tau[0], sig[1] - sig[0])
    dist = max(sig[0] - tau[1], tau[0] - sig[1], 0.0)
    return dist > 0 and diam <= lam * dist


def block_partition(nodes, root, lam: float):
    """Leaves of the block tree: list of (tau, sigma, 'lr'|'dense'); root is a
    Cluster (interleaved tree) or a PCluster (the paper's partition)."""
    out = []

    def rec(t, s):
        if admissible(support_of(nodes, t), support_of(nodes, s), lam):
            out.append((t, s, "lr"))
        elif not t.children or not s.children:
            out.append((t, s, "dense"))
        else:
            for tc in t.children:
                for sc in s.children:
                    rec(tc, sc)

    rec(root, root)
    return out


def _rising(x: float, k: int) -> float:
    r = 1.0
    for l in range(k):
        r *= x + l
    return r


def _elem_dof_derivs(nodes, P, e, xs_ref):
    """Physical derivatives of the element's local functions at reference points."""
    h = nodes[e + 1] - nodes[e]
    return np.array([local_deriv(P, h, xr) for xr in xs_ref])  # (q, P+1)


def taylor_factors(prob, test, trial, R: int, q: int = 48):
    """Low-rank factors of S_l on an admissible block with `test` right of `trial`.

    s-expansion about s0 = mid(trial support) unless diam(trial) > diam(test),
    then t-expansion about t0 = mid(test support) (Lemma 3.2 Eq. (eqn:Lexpan),
    PAPER.md:229-235; Remark PAPER.md:285-298; reading A10).  Returns (Q, W) with
    rows in the order of the clusters' dofs (paper_index_of_element_dofs for the
    interleaved tree, pcluster_dofs for the paper's partition) and
        S_l[test, trial] ~= Q @ W.T,   Q = gamma0 int h_nu phi_I',  W = int g_nu phi_J'
    (PAPER.md:365-370, 383-388)."""
    nodes, P, alpha = prob.nodes, prob.P, prob.alpha
    N = len(nodes) - 1
    g0 = 1.0 / math.gamma(2 - alpha)
    ts = support_of(nodes, test)
    ss = support_of(nodes, trial)
    c = np.array([_rising(alpha - 1, nu) / math.factorial(nu) for nu in range(R)])  # (alpha-1)_nu/nu!
    gx, gw = gl_table(q)
    s_expand = (ss[1] - ss[0]) <= (ts[1] - ts[0])

    def factor(cl, fn):
        """int fn(x) phi_I'(x) dx for the cluster's dofs (rows in cluster dof order)."""
        per_elem = {}

        def elem(e):   # (P+1, R): the element's local functions against fn
            if e not in per_elem:
                h = nodes[e + 1] - nodes[e]
                xs = nodes[e] + 0.5 * h * (gx + 1)
                D = _elem_dof_derivs(nodes, P, e, gx)            # (q, P+1)
                F = fn(xs, e)                                       # (q, R)
                per_elem[e] = (0.5 * h * gw[:, None] * D).T @ F     # (P+1, R)
            return per_elem[e]

        def hat(j):    # hat of interior node j: rising half on element j-1, falling half on j
            return elem(j - 1)[P] + elem(j)[0]

        rows = []
        if isinstance(cl, Cluster):
            for e in range(cl.e0, cl.e1):
                for p in range(1, P):
                    rows.append(elem(e)[p])
                if e + 1 <= N - 1:
                    rows.append(hat(e + 1))
        elif cl.kind == "modal":
            for e in range(cl.a, cl.b):
                for p in range(1, P):
                    rows.append(elem(e)[p])
        else:
            for j in range(cl.a, cl.b):
                rows.append(hat(j))
        return np.array(rows).reshape(-1, R)

    nus = np.arange(R)
    if s_expand:
        s0 = 0.5 * (ss[0] + ss[1])
        Q = g0 * factor(test, lambda x, e: c[None, :] * (x[:, None] - s0) ** (1 - alpha - nus[None, :]))
        W = factor(trial, lambda x, e: (x[:, None] - s0) ** nus[None, :])
    else:
        t0 = 0.5 * (ts[0] + ts[1])
        Q = g0 * factor(test, lambda x, e: (x[:, None] - t0) ** nus[None, :])
        W = factor(trial, lambda x, e: ((-1.0) ** nus * c)[None, :] * (t0 - x[:, None]) ** (1 - alpha - nus[None, :]))
    return Q, W


def hmatrix_dense(prob, sysm: System, R: int, lam: float = 1.0, n_min: int = 16, partition: str = "interleaved"):
    """Dense A~ = rho M + theta H + (1-theta) H^T (Eq. (approxsys) PAPER.md:594,
    reading A2): exact entries on inadmissible leaves, Taylor
    low-rank factors on admissible leaves.  Paper order.  partition:
    "interleaved" (reading A9) or "paper" (separate modal / nodal trees,
    PAPER.md:327-338).  Returns (A~, partition)."""
    N, P = prob.N, prob.P
    root = cluster_tree(N, n_min) if partition == "interleaved" else paper_cluster_tree(N, P, n_min)
    part = block_partition(prob.nodes, root, lam)
    At = sysm.A.copy()
    for t, s, kind in part:
        if kind != "lr":
            continue
        rows = dofs_of(N, P, t)
        cols = dofs_of(N, P, s)
        if len(rows) == 0 or len(cols) == 0:
            continue
        if support_of(prob.nodes, t)[0] >= support_of(prob.nodes, s)[1]:   # test cluster right of trial: lower part
            Q, W = taylor_factors(prob, t, s, R)
            At[np.ix_(rows, cols)] = prob.theta * (Q @ W.T)
        else:                                           # upper part: (1-theta) (S_l[s,t])^T
            Q, W = taylor_factors(prob, s, t, R)
            At[np.ix_(rows, cols)] = (1 - prob.theta) * (W @ Q.T)
    return At, part


# ------------------------------------------------------------ full problem
def reference_solve(prob, threads: Optional[int] = None):
    """The oracle's answer for a Problem: (A, G (n x nrhs), X (n x nrhs), System)."""
    sysm = assemble_system(prob, threads=threads)
    G = np.stack([rhs(prob, sysm, f) for f in prob.forcings], axis=1)
    X = solve_dense(sysm.A, G)
    return sysm, G, X
