"""Pins of the oracle branches that round 1 left unpinned (-m "not gpu").

Each `check_*` function states what the paper / mathematics fixes and raises
AssertionError when the oracle disagrees.  Every check runs twice:
  * on the oracle as committed (must pass), and
  * on a deliberately broken copy of the branch it pins (must FAIL) -- the
    mutation tests at the bottom.  A pin that a plausible mistake survives
    would not be a pin.

Branches ("What's weak" #1):
  a  t-expansion factors (Remark after Lemma 3.2)
  b  upper admissible blocks (1-theta) W Q^T (reading A2)
  c  theta orientation rho M + theta S_l + (1-theta) S_l^T (Eq. (lsys))
  d  Legendre-series load of degree >= 1
  e  boundary-hat lifting with c1, c2 != 0 (reading A15)
  f  singular power loads away from their base element (PAPER.md:744-751 forcing)
"""
import inspect
import math
import os
import re
import subprocess
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import fde_inputs as fi
import oracle as O
import oracle.oracle as OO
from mp_exact import legendre_power, deriv, local_deriv_ref  # noqa: F401  (exact rational basis)


# =============================================================== helpers
def _local_value_ref(P):
    """Power-basis (in xi, Fractions) of [left hat, psi_1..psi_{P-1}, right hat]
    (Eq. (RefBasis))."""
    L = legendre_power(P + 1)
    out = [[Fraction(1, 2), Fraction(-1, 2)]]
    for p in range(1, P):
        a, b = L[p - 1], L[p + 1]
        out.append([(a[i] if i < len(a) else 0) - (b[i] if i < len(b) else 0) for i in range(len(b))])
    out.append([Fraction(1, 2), Fraction(1, 2)])
    return out


def _ext_index(N, P, e, a):
    """Extended paper order of oracle.py's docstring: modal (e,p) | hats 1..N-1 | hat 0 | hat N."""
    nm = N * (P - 1)
    if a == 0:
        return nm + N - 1 if e == 0 else nm + e - 1
    if a == P:
        return nm + N if e + 1 == N else nm + e
    return e * (P - 1) + a - 1


def _poly_mul(p, q):
    out = [Fraction(0)] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        if a:
            for j, b in enumerate(q):
                out[i + j] += a * b
    return out


def _poly_compose_affine(p, c0, c1):
    """p(c0 + c1 xi) as a power series in xi (exact)."""
    out = [Fraction(0)]
    powk = [Fraction(1)]
    for k, a in enumerate(p):
        if k:
            powk = _poly_mul(powk, [c0, c1])
        if a:
            out = out + [Fraction(0)] * (len(powk) - len(out))
            for i, b in enumerate(powk):
                out[i] += a * b
    return out


def _int_m11(p):
    """int_{-1}^{1} p(xi) dxi, exact."""
    return sum(a * Fraction(2, i + 1) for i, a in enumerate(p) if i % 2 == 0)


def _l1_deriv_bound(P, a):
    """Upper bound of int |phi'| dx over one element for local function a (the
    Jacobian cancels): a hat's half contributes exactly 1; modal psi_p' =
    -(2p+1) L_p and int |L_p| <= sqrt(2) ||L_p||_2 =
    2/sqrt(2p+1) (Cauchy-Schwarz) give 2 sqrt(2p+1)."""
    if a == 0 or a == P:
        return 1.0
    return 2.0 * math.sqrt(2 * a + 1)


# ======================================================= c: theta orientation
def _poly_problem(theta, rho, nodes, P=4, alpha=1.5):
    f = fi.manufactured_poly_forcing({2: 1.0, 3: -2.0, 4: 1.0}, alpha, theta, rho)
    return fi.Problem(f"poly-t{theta}", 0.0, 1.0, alpha, theta, rho, 0.0, 0.0, nodes, P, 4,
                      n_min=2, forcings=[f])


def check_theta_orientation_exact_solution(theta, rho, nodes):
    """u = x^2(1-x)^2 lies in S_N^P for P >= 4, so the Galerkin solution of
    Eq. (Model) is u itself for every theta (uniqueness,
    Theorem 2.1).  f = -theta D^2 0I^{2-a} u - (1-theta) D^2 xI_1^{2-a} u + rho u by
    the monomial closed form; at theta != 1/2 the two one-sided operators differ,
    so a swapped theta in A = rho M + theta S_l + (1-theta) S_l^T (or a transposed
    S_l) gives a different discrete solution."""
    p = _poly_problem(theta, rho, nodes)
    sysm, G, X = O.reference_solve(p)
    xis = np.linspace(-1, 1, 11)
    uh = O.eval_solution(p, X[:, 0], xis)
    h = np.diff(p.nodes)
    xs = p.nodes[:-1, None] + h[:, None] * (xis[None, :] + 1) / 2
    err = np.abs(uh - fi.config1_exact(xs)).max()
    assert err < 2e-13, err


THETA_CASES = [(0.3, 1.0, "uniform"), (0.85, 0.0, "uniform"), (0.3, 2.0, "graded"), (0.0, 0.5, "graded"),
               (1.0, 0.0, "graded")]


def _nodes(kind):
    return fi.uniform_mesh(0, 1, 8) if kind == "uniform" else fi.config4(N=12, P=4).nodes


@pytest.mark.parametrize("theta,rho,kind", THETA_CASES)
def test_theta_orientation_exact_polynomial_solution(theta, rho, kind):
    check_theta_orientation_exact_solution(theta, rho, _nodes(kind))


# ============================================ a, b: admissible blocks, any side
def _mirrored_problem(theta=0.3, N=64, P=4):
    p = fi.config4(N=N, P=P)
    p.theta = theta
    return p


_SYS = {}


def _system(p):
    key = (p.name, p.theta, p.rho, p.P)
    if key not in _SYS:
        _SYS[key] = O.assemble_system(p)
    return _SYS[key]


def check_admissible_block_bounds(p, R, n_min=4, lam=1.0):
    """Entrywise bound on every admissible block, lower AND upper, s- AND
    t-expansion.  Lemma 3.2 (exponent alpha-1 as in its proof,
    reading A8) and its t-analogue in the Remark give
        |k - k~| <= r^R / (1 - r) / dist^{alpha-1},   r = (diam/2) / (diam/2 + dist)
    with diam the diameter of the EXPANDED cluster; integrating against phi_I',
    phi_J' (Eq. (lsys) entries) bounds
        |A~_IJ - A_IJ| <= w gamma0 ||phi_I'||_1 ||phi_J'||_1 r^R / (1-r) / dist^{alpha-1},
    w = theta below the diagonal, 1-theta above (reading A2; rho M vanishes on
    admissible blocks), plus a rounding floor 1e-12 sqrt(A_II A_JJ) (the far
    entries are differences of nearly equal moments; metric M-A's scaling).
    Also requires all four (lower/upper x s-/t-expansion) kinds to occur."""
    sysm = _system(p)
    At, part = O.hmatrix_dense(p, sysm, R=R, lam=lam, n_min=n_min)
    nodes, P, N, alpha = p.nodes, p.P, p.N, p.alpha
    g0 = 1 / math.gamma(2 - alpha)
    nm = N * (P - 1)
    kinds = set()
    worst = 0.0
    for t, s, kind in part:
        if kind != "lr":
            continue
        rows = O.paper_index_of_element_dofs(N, P, t.e0, t.e1)
        cols = O.paper_index_of_element_dofs(N, P, s.e0, s.e1)
        ts, ss = O.cluster_support(nodes, t), O.cluster_support(nodes, s)
        lower = ts[0] >= ss[1]
        test, trial = (ts, ss) if lower else (ss, ts)      # S_l block (test right of trial)
        dist = test[0] - trial[1]
        s_exp = (trial[1] - trial[0]) <= (test[1] - test[0])   # Remark
        dexp = (trial[1] - trial[0]) if s_exp else (test[1] - test[0])
        r = 0.5 * dexp / (0.5 * dexp + dist)
        kb = r ** R / (1 - r) / dist ** (alpha - 1)
        w = p.theta if lower else 1 - p.theta
        kinds.add((lower, s_exp))

        def l1(I):
            if I >= nm:
                return 2.0           # hat: 1 on each of its two elements
            return _l1_deriv_bound(P, I % (P - 1) + 1)
        for I in rows:
            for J in cols:
                bound = w * g0 * l1(I) * l1(J) * kb + 1e-12 * math.sqrt(abs(sysm.A[I, I] * sysm.A[J, J]))
                err = abs(At[I, J] - sysm.A[I, J])
                worst = max(worst, err / bound if bound > 0 else (np.inf if err > 0 else 0))
    assert worst <= 1.0, worst
    for need in [(True, True), (True, False), (False, True), (False, False)]:
        assert need in kinds, (need, kinds)
    return worst


@pytest.mark.parametrize("R", [3, 6, 10])
def test_admissible_blocks_within_taylor_bound_theta03(R):
    check_admissible_block_bounds(_mirrored_problem(0.3), R)


def check_error_decreases_with_rank(p, Rs=(2, 4, 6, 8, 10), n_min=4):
    """||A - A~||_F decays geometrically in R (Fig. fig:matrixerror),
    here on the two-sided graded mesh at theta = 0.3 where t-expansion and upper
    blocks carry most of the admissible entries; by R = 10 the error is below
    1e-8 ||A||_F (delta_1 = 1/3 per Taylor order)."""
    sysm = _system(p)
    errs = []
    for R in Rs:
        At, _ = O.hmatrix_dense(p, sysm, R=R, lam=1.0, n_min=n_min)
        errs.append(np.linalg.norm(sysm.A - At))
    assert all(errs[k + 1] < 0.5 * errs[k] for k in range(len(errs) - 1)), errs
    assert errs[-1] < 1e-8 * np.linalg.norm(sysm.A), errs


def test_error_decreases_with_rank_mirrored_theta03():
    check_error_decreases_with_rank(_mirrored_problem(0.3))


def check_t_expansion_hat_closed_forms(p, R=6, n_min=4):
    """t-expansion blocks (Remark PAPER.md:283-298): for the hat of node x0 with
    neighbours xm < x0 < xp, the analogues of the closed forms Eq. (eq412)/(eq415)
     with the roles of t and s exchanged:
        Q_nu = gamma0 int (t-t0)^nu phi'(t) dt
             = gamma0 [ ((x0-t0)^{nu+1}-(xm-t0)^{nu+1})/((x0-xm)(nu+1))
                       - ((xp-t0)^{nu+1}-(x0-t0)^{nu+1})/((xp-x0)(nu+1)) ]
        W_nu = int binom(1-alpha, nu) (t0-s)^{1-alpha-nu} phi'(s) ds
             = binom(1-alpha, nu) [ ((t0-xm)^{e}-(t0-x0)^{e})/((x0-xm) e)
                                   - ((t0-x0)^{e}-(t0-xp)^{e})/((xp-x0) e) ],  e = 2-alpha-nu,
    where binom(1-alpha, nu) is the Taylor coefficient of (t0 - s + (t - t0))^{1-alpha}
    in (t-t0)^nu, computed here from math.comb-free generalised binomials
    (mpmath.binomial), not from the oracle's rising factorial."""
    nodes, P, N, alpha = p.nodes, p.P, p.N, p.alpha
    g0 = 1 / math.gamma(2 - alpha)
    part = O.block_partition(nodes, O.cluster_tree(N, n_min), 1.0)
    checked = 0
    for t, s, kind in part:
        if kind != "lr" or nodes[t.e0] < nodes[s.e1]:
            continue
        ts, ss = O.cluster_support(nodes, t), O.cluster_support(nodes, s)
        if (ss[1] - ss[0]) <= (ts[1] - ts[0]):
            continue                                   # s-expansion: test_oracle_pins covers it
        Q, W = O.taylor_factors(p, t, s, R)
        t0 = 0.5 * (ts[0] + ts[1])
        r = 0
        for e in range(t.e0, t.e1):
            r += P - 1
            if e + 1 <= N - 1:
                xm, x0, xp = nodes[e], nodes[e + 1], nodes[e + 2]
                for nu in range(R):
                    k = nu + 1
                    q = g0 * (((x0 - t0) ** k - (xm - t0) ** k) / ((x0 - xm) * k)
                              - ((xp - t0) ** k - (x0 - t0) ** k) / ((xp - x0) * k))
                    assert Q[r, nu] == pytest.approx(q, rel=1e-10, abs=1e-13 * (xp - xm) ** nu)
                r += 1
        r = 0
        for e in range(s.e0, s.e1):
            r += P - 1
            if e + 1 <= N - 1:
                xm, x0, xp = nodes[e], nodes[e + 1], nodes[e + 2]
                for nu in range(R):
                    ex = 2 - alpha - nu
                    c = float(mp.binomial(1 - alpha, nu))
                    wv = c * (((t0 - xm) ** ex - (t0 - x0) ** ex) / ((x0 - xm) * ex)
                              - ((t0 - x0) ** ex - (t0 - xp) ** ex) / ((xp - x0) * ex))
                    assert W[r, nu] == pytest.approx(wv, rel=1e-9, abs=1e-12 * abs(wv) + 1e-300)
                r += 1
        checked += 1
    assert checked > 0
    return checked


def test_t_expansion_hat_closed_forms():
    check_t_expansion_hat_closed_forms(_mirrored_problem(0.3))


# ====================================================== d: Legendre-series load
def _exact_legendre_load(nodes_f, P, a, b, leg):
    """(f, phi_I) in exact rational arithmetic for f = sum_k leg_k L_k(2(x-a)/(b-a)-1)
    (the forcing recipe of configs 2/4/5); nodes, a, b and the
    coefficients are binary floats, hence exact Fractions."""
    N = len(nodes_f) - 1
    nodes = [Fraction(x) for x in nodes_f]
    A, B = Fraction(a), Fraction(b)
    Lp = legendre_power(len(leg) - 1)
    fz = [Fraction(0)] * len(leg)                        # f as a polynomial in z
    for k, ck in enumerate(leg):
        for i, c in enumerate(Lp[k]):
            fz[i] += Fraction(ck) * c
    V = _local_value_ref(P)
    G = [Fraction(0)] * (N * P + 1)
    for e in range(N):
        xl, xr = nodes[e], nodes[e + 1]
        h = xr - xl
        # z(xi) = 2(x - a)/(b - a) - 1 with x = xl + h (xi + 1)/2
        z0 = 2 * (xl + h / 2 - A) / (B - A) - 1
        z1 = h / (B - A)
        fxi = _poly_compose_affine(fz, z0, z1)
        for loc in range(P + 1):
            G[_ext_index(N, P, e, loc)] += h / 2 * _int_m11(_poly_mul(fxi, V[loc]))
    return np.array([float(g) for g in G])


def check_legendre_load(nodes, P, a, b, leg):
    G = O.load_ext(nodes, P, a, b, fi.Forcing(leg=np.array(leg)))
    Ge = _exact_legendre_load(nodes, P, a, b, leg)
    err = np.abs(G - Ge).max() / np.abs(Ge).max()
    assert err < 1e-14, err


LOAD_CASES = [
    # (nodes (binary fractions), P, a, b, seed)
    (np.array([-0.5, -0.375, -0.0625, 0.25, 0.3125, 0.75, 1.0, 1.5]), 5, -0.5, 1.5, 1),
    (np.array([0.0, 0.0078125, 0.03125, 0.125, 0.5, 1.0]), 8, 0.0, 1.0, 2),
    (np.array([2.0, 2.5, 3.0, 3.25, 4.0]), 3, 2.0, 4.0, 3),
]


@pytest.mark.parametrize("case", LOAD_CASES, ids=["shifted", "graded", "offset"])
def test_legendre_series_load_exact_rational(case):
    """Degree-20 Legendre series (every degree 0..20 present) on meshes whose
    nodes are binary fractions, against exact rational integration of
    f * phi_I (power-basis Legendre polynomials from the recurrence PAPER.md:128)."""
    nodes, P, a, b, seed = case
    leg = list(fi.random_legendre_forcing(seed).leg)
    check_legendre_load(nodes, P, a, b, leg)


# ============================================================ e: lifting
def check_lifting_against_bordered_solve(p):
    """Dirichlet data u(a) = c1, u(b) = c2 (Eq. (Model)) imposed in the
    full space span{phi_0..phi_N} + modal: the Galerkin equations of the interior
    test functions, plus the rows u_0 = c1, u_N = c2.  Its interior part must equal
    the oracle's lifted solve A X = G - A[:, {0,N}] [c1, c2] (reading A15)."""
    sysm = O.assemble_system(p)
    n = p.n
    Afull = p.rho * sysm.M_ext + p.theta * sysm.Sl_ext + (1 - p.theta) * sysm.Sl_ext.T
    gext = O.load_ext(p.nodes, p.P, p.a, p.b, p.forcings[0])
    K = Afull.copy()
    rhs = gext.copy()
    for k, c in ((n, p.c1), (n + 1, p.c2)):            # boundary rows -> identity
        K[k, :] = 0.0
        K[k, k] = 1.0
        rhs[k] = c
    Xb = np.linalg.solve(K, rhs)
    X = O.solve_dense(sysm.A, O.rhs(p, sysm, p.forcings[0]))
    d = np.sqrt(np.abs(np.diag(sysm.A)))
    err = np.linalg.norm(d * (X - Xb[:n])) / np.linalg.norm(d * Xb[:n])
    assert err < 1e-12, err


@pytest.mark.parametrize("theta", [0.3, 0.8])
def test_lifting_equals_bordered_dirichlet_solve(theta):
    p = fi.config2(1.5, N=10, P=4)
    p.theta = theta
    p.c1, p.c2 = 0.5, -1.0
    check_lifting_against_bordered_solve(p)


# ============================================ f: singular power-law loads
def _exact_power_load(nodes_f, P, a, b, side, beta, dps=100):
    """(y^beta, phi_I) with y = x - a (side L) or b - x (side R) by repeated
    integration by parts against the exact antiderivatives
    F_m(y) = y^{beta+m} / prod_{l=1..m}(beta+l)  (mpmath, `dps` digits: on an element
    of size h at distance y the terms cancel by ~(y/h)^P, 40 digits on Example 5.1's
    mesh at N = 100)."""
    N = len(nodes_f) - 1
    V = _local_value_ref(P)
    G = [mp.mpf(0)] * (N * P + 1)
    with mp.workdps(dps):
        be = mp.mpf(beta)

        def F(m, y):
            if y == 0:
                return mp.mpf(0)
            den = mp.mpf(1)
            for l in range(1, m + 1):
                den *= be + l
            return y ** (be + m) / den

        for e in range(N):
            xl, xr = mp.mpf(nodes_f[e]), mp.mpf(nodes_f[e + 1])
            h = xr - xl
            if side == "L":
                y0, y1, s1 = xl - mp.mpf(a), xr - mp.mpf(a), 2 / h      # xi = -1 at y0
                xi0, xi1 = -1, 1
            else:
                y0, y1, s1 = mp.mpf(b) - xr, mp.mpf(b) - xl, -2 / h
                xi0, xi1 = 1, -1
            for loc in range(P + 1):
                tot = mp.mpf(0)
                c = list(V[loc])
                l = 0
                while any(c):
                    pv1 = sum(mp.mpf(ci.numerator) / ci.denominator * mp.mpf(xi1) ** i for i, ci in enumerate(c))
                    pv0 = sum(mp.mpf(ci.numerator) / ci.denominator * mp.mpf(xi0) ** i for i, ci in enumerate(c))
                    tot += (-1) ** l * s1 ** l * (pv1 * F(l + 1, y1) - pv0 * F(l + 1, y0))
                    c = deriv(c)
                    if len(c) == 1 and c[0] == 0:
                        break
                    l += 1
                G[_ext_index(N, P, e, loc)] += tot
        return np.array([float(g) for g in G])


def check_power_load(nodes, P, a, b, side, beta):
    """Entry by entry, relative to the L1 scale  sum_{e in supp phi_I} int_e |f|
    (|phi_I| <= 2 on its support), the natural size of (f, phi_I) -- entries of
    smooth-data modal functions can be far smaller than it by cancellation."""
    G = O.load_ext(nodes, P, a, b, fi.Forcing(terms=[(side, beta, 1.0)]))
    Ge = _exact_power_load(nodes, P, a, b, side, beta)
    N = len(nodes) - 1
    y = (nodes - a) if side == "L" else (b - nodes)
    el1 = np.abs(y[1:] ** (beta + 1) - y[:-1] ** (beta + 1)) / (beta + 1)   # int_e y^beta
    scale = np.zeros(N * P + 1)
    for e in range(N):
        for loc in range(P + 1):
            scale[_ext_index(N, P, e, loc)] += el1[e]
    n = N * P - 1                                       # interior test functions only
    err = (np.abs(G[:n] - Ge[:n]) / scale[:n]).max()
    assert err < 1e-14, err


POWER_CASES = [
    ("L", 1.0 - 1.6),   # Example 5.1's  x^{1-alpha} (alpha = 1.6 by A16)
    ("L", 0.8 - 1.6),   # and x^{gamma-alpha}
    ("L", 0.8),         # rho u term x^{0.8}
    ("R", 0.5),         # a right-sided (b-x)^beta term (config 1 at theta != 1/2)
    ("R", 2.0 - 1.85),
]


@pytest.mark.parametrize("side,beta", POWER_CASES)
def test_power_load_on_graded_mesh_exact(side, beta):
    """Example 5.1's graded mesh x_i = 10 (i/N)^5 -- elements of
    size ratio up to ~5 and a singular base point next to tiny elements -- and
    (y^beta, phi_I) for every interior test function, entry by entry, against
    exact antiderivatives.  Covers both load rules: Gauss-Jacobi on the element
    touching the base point and the distance-graded composite rule elsewhere.
    Also a stronger grading x_i = 10 (i/N)^8 (element 2 is 255x its distance to
    the base point), on which a fixed two-half rule is off by 1e-7."""
    for N, q in ((24, 5.0), (100, 5.0), (100, 8.0)):
        check_power_load(fi.graded_mesh(0.0, 10.0, N, q), 3, 0.0, 10.0, side, beta)


# ======================================================== mutation tests
def _mutant_py(func, old, new, module=OO):
    """A copy of `func` with one source substring replaced, compiled in the
    oracle module's namespace (deliberately broken branch)."""
    src = inspect.getsource(func)
    assert old in src, (old, func.__name__)
    ns = dict(module.__dict__)
    exec(compile(src.replace(old, new), f"<mutant {func.__name__}>", "exec"), ns)
    return ns[func.__name__]


_C_SRC = os.path.join(os.path.dirname(OO.__file__), "fde_oracle.c")


def _mutant_c(tmp_path, old, new, tag):
    src = open(_C_SRC).read()
    assert old in src, old
    path = tmp_path / f"fde_oracle_{tag}.c"
    path.write_text(src.replace(old, new))
    so = tmp_path / f"liboracle_{tag}.so"
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", str(so), str(path), "-lm"])
    return OO.load_library(str(so))


def _patch(monkeypatch, name, fn):
    """Replace an oracle function in its module (seen by the other oracle
    functions) and in the package namespace (seen by the checks)."""
    monkeypatch.setattr(OO, name, fn)
    monkeypatch.setattr(O, name, fn)


def _fails(fn, *a):
    try:
        fn(*a)
    except AssertionError:
        return True
    return False


def test_mutation_theta_swap_is_caught(monkeypatch):
    """c: theta S_l + (1-theta) S_l^T -> (1-theta) S_l + theta S_l^T."""
    m = _mutant_py(OO.assemble_system, "prob.theta * S + (1 - prob.theta) * S.T",
                   "(1 - prob.theta) * S + prob.theta * S.T")
    _patch(monkeypatch, "assemble_system", m)
    assert _fails(check_theta_orientation_exact_solution, 0.3, 1.0, _nodes("uniform"))


def test_mutation_transposed_Sl_is_caught(monkeypatch):
    m = _mutant_py(OO.assemble_system, "prob.theta * S + (1 - prob.theta) * S.T",
                   "prob.theta * S.T + (1 - prob.theta) * S")
    _patch(monkeypatch, "assemble_system", m)
    assert _fails(check_theta_orientation_exact_solution, 0.85, 0.0, _nodes("uniform"))


def test_mutation_t_expansion_sign_is_caught(monkeypatch):
    """a: drop the (-1)^nu of the t-expansion (Remark)."""
    m = _mutant_py(OO.taylor_factors, "((-1.0) ** nus * c)", "(c)")
    _patch(monkeypatch, "taylor_factors", m)
    p = _mirrored_problem(0.3)
    assert _fails(check_admissible_block_bounds, p, 6)
    assert _fails(check_error_decreases_with_rank, p)
    assert _fails(check_t_expansion_hat_closed_forms, p)


def test_mutation_t_expansion_point_is_caught(monkeypatch):
    """a: expand about the wrong cluster's midpoint in the t-branch."""
    m = _mutant_py(OO.taylor_factors, "t0 = 0.5 * (ts[0] + ts[1])", "t0 = 0.5 * (ts[0] + ts[1]) + 0.25 * (ts[1] - ts[0])")
    _patch(monkeypatch, "taylor_factors", m)
    assert _fails(check_t_expansion_hat_closed_forms, _mirrored_problem(0.3))


def test_mutation_upper_block_weight_is_caught(monkeypatch):
    """b: upper admissible block weighted by theta instead of 1-theta (reading A2)."""
    m = _mutant_py(OO.hmatrix_dense, "(1 - prob.theta) * (W @ Q.T)", "prob.theta * (W @ Q.T)")
    _patch(monkeypatch, "hmatrix_dense", m)
    p = _mirrored_problem(0.3)
    assert _fails(check_admissible_block_bounds, p, 6)
    assert _fails(check_error_decreases_with_rank, p)


def test_mutation_upper_block_expansion_side_is_caught(monkeypatch):
    """b: upper block built from the lower orientation's factors (S_l[t,s] read
    where (S_l[s,t])^T belongs) -- i.e. the transposed block taken literally."""
    m = _mutant_py(OO.hmatrix_dense, "At[np.ix_(rows, cols)] = (1 - prob.theta) * (W @ Q.T)",
                   "At[np.ix_(rows, cols)] = (1 - prob.theta) * (W @ Q.T)[::-1, ::-1]")
    _patch(monkeypatch, "hmatrix_dense", m)
    assert _fails(check_admissible_block_bounds, _mirrored_problem(0.3), 6)


def test_mutation_lifting_sign_is_caught(monkeypatch):
    """e: G + A[:, bnd] c instead of G - A[:, bnd] c."""
    m = _mutant_py(OO.rhs, "Gext[:n] - sysm.Abnd", "Gext[:n] + sysm.Abnd")
    _patch(monkeypatch, "rhs", m)
    p = fi.config2(1.5, N=10, P=4)
    p.theta, p.c1, p.c2 = 0.3, 0.5, -1.0
    assert _fails(check_lifting_against_bordered_solve, p)


def test_mutation_lifting_rows_instead_of_columns_is_caught(monkeypatch):
    """e: boundary ROWS A[{0,N}, :]^T instead of the boundary COLUMNS (differs at theta != 1/2)."""
    m = _mutant_py(OO.assemble_system, "Abnd=Afull[:n, n:n + 2].copy()", "Abnd=Afull[n:n + 2, :n].T.copy()")
    _patch(monkeypatch, "assemble_system", m)
    p = fi.config2(1.5, N=10, P=4)
    p.theta, p.c1, p.c2 = 0.3, 0.5, -1.0
    assert _fails(check_lifting_against_bordered_solve, p)


def test_mutation_legendre_map_is_caught(monkeypatch, tmp_path):
    """d: Legendre argument 2(x-a)/(b-a)-1 replaced by (x-a)/(b-a) (wrong map)."""
    L = _mutant_c(tmp_path, "ld z = 2 * offa / (B - A) - 1,", "ld z = offa / (B - A),", "legmap")
    monkeypatch.setattr(OO, "_lib", L)
    nodes, P, a, b, seed = LOAD_CASES[0]
    assert _fails(check_legendre_load, nodes, P, a, b, list(fi.random_legendre_forcing(seed).leg))


def test_mutation_legendre_coarse_rule_is_caught(monkeypatch, tmp_path):
    """d: too few Gauss points for the degree-20 series (q = 40 -> 8 per half)."""
    L = _mutant_c(tmp_path, "int q = 40;\n    orc_gauss_legendre(q, gx, gw);\n    ld A = a, B = b;",
                  "int q = 8;\n    orc_gauss_legendre(q, gx, gw);\n    ld A = a, B = b;", "legq")
    monkeypatch.setattr(OO, "_lib", L)
    nodes, P, a, b, seed = LOAD_CASES[1]
    assert _fails(check_legendre_load, nodes, P, a, b, list(fi.random_legendre_forcing(seed).leg))


def test_mutation_two_half_power_rule_is_caught(monkeypatch, tmp_path):
    """f: the round-1 rule before 0f891c7 -- singular powers away from the base
    element integrated on two fixed halves instead of distance-graded cells
    (converged to 1e-14 on Example 5.1's q = 5 mesh, off by 5e-8 at q = 8)."""
    L = _mutant_c(tmp_path, "ld ub = o0 + 2 * ua < h ? o0 + 2 * ua : h;", "ld ub = ua + 0.5L * h;", "twohalf")
    monkeypatch.setattr(OO, "_lib", L)
    nodes = fi.graded_mesh(0.0, 10.0, 100, 8.0)
    assert _fails(check_power_load, nodes, 3, 0.0, 10.0, "L", 1.0 - 1.6)


def test_mutation_power_side_is_caught(monkeypatch, tmp_path):
    """f: the right-sided (b-x)^beta term measured from the wrong end."""
    L = _mutant_c(tmp_path, "ld o0 = (side[t] == 0) ? ((ld)nodes[e] - A) : (B - (ld)nodes[e + 1]);",
                  "ld o0 = (side[t] == 0) ? ((ld)nodes[e] - A) : (B - (ld)nodes[e]);", "side")
    monkeypatch.setattr(OO, "_lib", L)
    nodes = fi.graded_mesh(0.0, 10.0, 24, 5.0)
    assert _fails(check_power_load, nodes, 3, 0.0, 10.0, "R", 0.5)


# ================================================ the paper's own partition
def check_paper_partition_bounds(p, R, n_min=4, lam=1.0):
    """The paper's partition (separate modal / nodal cluster trees):
    the same entrywise Lemma 3.2 / Remark bound as check_admissible_block_bounds on
    every admissible block, with the supports of the modal clusters (unions of
    elements) and nodal clusters (unions of [x_{j-1}, x_{j+1}]); every block of
    the partition is pure (modal x modal, modal x nodal, ...): the first block level
    is S_l = [B F; E C]."""
    sysm = _system(p)
    At, part = O.hmatrix_dense(p, sysm, R=R, lam=lam, n_min=n_min, partition="paper")
    nodes, P, N, alpha = p.nodes, p.P, p.N, p.alpha
    g0 = 1 / math.gamma(2 - alpha)
    nm = N * (P - 1)
    covered = np.zeros((p.n, p.n), dtype=bool)
    worst, nlr = 0.0, 0
    for t, s, kind in part:
        assert t.kind in ("modal", "nodal") and s.kind in ("modal", "nodal")
        rows, cols = O.pcluster_dofs(N, P, t), O.pcluster_dofs(N, P, s)
        assert not covered[np.ix_(rows, cols)].any()
        covered[np.ix_(rows, cols)] = True
        if kind != "lr":
            assert np.array_equal(At[np.ix_(rows, cols)], sysm.A[np.ix_(rows, cols)])   # exact entries
            continue
        nlr += 1
        ts, ss = O.pcluster_support(nodes, t), O.pcluster_support(nodes, s)
        lower = ts[0] >= ss[1]
        test, trial = (ts, ss) if lower else (ss, ts)
        dist = test[0] - trial[1]
        s_exp = (trial[1] - trial[0]) <= (test[1] - test[0])
        dexp = (trial[1] - trial[0]) if s_exp else (test[1] - test[0])
        r = 0.5 * dexp / (0.5 * dexp + dist)
        kb = r ** R / (1 - r) / dist ** (alpha - 1)
        w = p.theta if lower else 1 - p.theta
        l1 = lambda I: 2.0 if I >= nm else _l1_deriv_bound(P, I % (P - 1) + 1)
        for I in rows:
            for J in cols:
                bound = w * g0 * l1(I) * l1(J) * kb + 1e-12 * math.sqrt(abs(sysm.A[I, I] * sysm.A[J, J]))
                worst = max(worst, abs(At[I, J] - sysm.A[I, J]) / bound)
    assert covered.all()
    assert nlr > 0
    assert worst <= 1.0, worst
    return worst


@pytest.mark.parametrize("R", [3, 8])
def test_paper_partition_blocks_within_taylor_bound(R):
    check_paper_partition_bounds(_mirrored_problem(0.3), R)


def test_paper_partition_error_decay_and_lambda0():
    """||A - A~||_F decays geometrically in R on the paper's partition too, and
    lambda -> 0 gives A~ = A."""
    p = _mirrored_problem(0.3)
    sysm = _system(p)
    errs = [np.linalg.norm(sysm.A - O.hmatrix_dense(p, sysm, R=R, n_min=4, partition="paper")[0]) for R in (2, 4, 6, 8)]
    assert all(errs[k + 1] < 0.5 * errs[k] for k in range(3)), errs
    At, part = O.hmatrix_dense(p, sysm, R=3, lam=1e-9, n_min=4, partition="paper")
    assert all(k == "dense" for _, _, k in part) and np.array_equal(At, sysm.A)


def test_mutation_paper_nodal_support_is_caught(monkeypatch):
    """A nodal cluster's support taken as [x_{j0}, x_{j1}] (dropping the hats' left
    halves) admits blocks whose kernel is not smooth on the real supports."""
    m = _mutant_py(OO.pcluster_support, "return nodes[c.a - 1], nodes[c.b]", "return nodes[c.a], nodes[c.b - 1]")
    _patch(monkeypatch, "pcluster_support", m)
    assert _fails(check_paper_partition_bounds, _mirrored_problem(0.3), 8)
