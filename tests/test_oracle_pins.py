"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of them re-types the oracle's own
formula: they use closed forms, an independent exact method (tests/mp_exact.py,
iterated antiderivatives at 60 digits), invariants, special cases with a known
exact solution and the paper's own error bounds.
"""
import math

import numpy as np
import pytest

import fde_inputs as fi
import oracle as O
from mp_exact import pair_exact


# ----------------------------------------------------------------- tables
@pytest.mark.parametrize("n", [1, 4, 9, 17, 30])
def test_gauss_legendre_exact_on_monomials(n):
    x, w = O.gl_table(n)
    for k in range(2 * n):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 1e-14 * (1 + abs(exact))


@pytest.mark.parametrize("n,a,b", [(3, 0.0, 0.5), (8, 0.0, -0.7), (12, 0.3, 0.0), (20, 0.0, 0.2), (10, 0.4, -0.6)])
def test_gauss_jacobi_exact_on_moments(n, a, b):
    """int (1-x)^a (1+x)^{b+k} dx = 2^{a+b+k+1} B(a+1, b+k+1), k <= 2n-1."""
    x, w = O.gj_table(n, a, b)
    for k in range(2 * n):
        exact = 2.0 ** (a + b + k + 1) * math.gamma(a + 1) * math.gamma(b + k + 1) / math.gamma(a + b + k + 2)
        assert abs(np.dot(w, (1 + x) ** k) - exact) < 2e-14 * exact


# ------------------------------------------------------------------ basis
@pytest.mark.parametrize("P", [2, 5, 11])
def test_modal_basis_facts(P):
    """psi_p(+-1) = 0; psi_p' = -(2p+1) L_p; hats are the linear
    nodal functions."""
    for xi in [-1.0, 1.0]:
        v = O.local_value(P, xi)
        assert np.all(np.abs(v[1:P]) < 1e-14)
        assert v[0] == pytest.approx((1 - xi) / 2) and v[P] == pytest.approx((1 + xi) / 2)
    h = 0.37
    for xi in np.linspace(-1, 1, 7):
        d = O.local_deriv(P, h, xi)
        for p in range(1, P):
            Lp = np.polynomial.legendre.legval(xi, [0] * p + [1])
            assert d[p] == pytest.approx((2 / h) * (-(2 * p + 1)) * Lp, abs=1e-12)
        assert d[0] == pytest.approx(-1 / h) and d[P] == pytest.approx(1 / h)


# --------------------------------------------- fractional integral closed form
@pytest.mark.parametrize("beta", [0.2, 0.5, 0.8])
@pytest.mark.parametrize("gam", [0, 1, 3, 6])
def test_fractional_integral_of_monomial(beta, gam):
    """aI^beta (x-a)^gam = Gamma(gam+1)/Gamma(gam+1+beta) (x-a)^{gam+beta}
    (definition; closed form named in BASELINE north_star)."""
    for x in [0.3, 1.0, 7.5]:
        got = O.frac_integral_monomial(x, beta, gam)
        exact = math.gamma(gam + 1) / math.gamma(gam + 1 + beta) * x ** (gam + beta)
        assert abs(got - exact) <= 1e-14 * exact


def test_right_sided_fractional_integral_by_reflection():
    """xI_b^beta (b-x)^gam = Gamma(gam+1)/Gamma(gam+1+beta) (b-x)^{gam+beta}: the
    reflection s -> a+b-s maps it onto the left-sided closed form."""
    b, beta, gam = 2.0, 0.6, 2
    for x in [0.1, 1.3]:
        got = O.frac_integral_monomial(b - x, beta, gam)
        exact = math.gamma(gam + 1) / math.gamma(gam + 1 + beta) * (b - x) ** (gam + beta)
        assert abs(got - exact) <= 1e-14 * exact


# ----------------------------------------------- pair integrals (S_l entries)
CASES = [  # (d, h_test, h_trial, self)
    (0.0, 1.0, 1.0, True),
    (0.0, 1.0, 1.0, False),
    (0.0, 1.0, 0.15, False),
    (0.0, 0.15, 1.0, False),
    (0.15, 1.0, 0.0225, False),
    (1.0, 1.0, 1.0, False),
    (3.0, 0.5, 2.0, False),
    (1e-3, 1.0, 0.3, False),
]


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.85])
@pytest.mark.parametrize("case", CASES)
def test_pair_integral_vs_exact_antiderivatives(alpha, case):
    """S_l element-pair blocks (reading A1) against the exact
    corner formula (independent method, 60 digits)."""
    d, hi, hj, selfp = case
    P = 4
    ex = np.array(pair_exact(P, alpha, d, hi, hj, selfp))
    if selfp:
        got = O.pair_integral(P, alpha, np.array([0.0, hi]), 0, 0)
    else:
        nodes = np.array([0.0, hj, hj + d, hj + d + hi])
        if d == 0.0:
            nodes = np.array([0.0, hj, hj + hi])
            got = O.pair_integral(P, alpha, nodes, 1, 0)
        else:
            got = O.pair_integral(P, alpha, nodes, 2, 0)
    assert np.abs(got - ex).max() <= 2e-15 * np.abs(ex).max()


def test_hat_hat_entries_uniform_closed_form():
    """Uniform mesh, h=2: S_l hat-hat entries = 1/4 [2K(k) - K(k-1) - K(k+1)] with
    the lag moment K(k) = gamma0 2^{3-a} ((k+1)^{3-a} - 2k^{3-a} + (k-1)^{3-a})/((2-a)(3-a)),
    K(0) = gamma0 2^{3-a}/((2-a)(3-a)) (direct integration of (xi-eta+2k)^{1-a}; cf.
    the Toeplitz symbols of PAPER.md:697-702 and SURVEY.md A5)."""
    for alpha in [1.3, 1.5, 1.9]:
        N, P = 10, 2
        nodes = np.arange(N + 1) * 2.0
        S = O.assemble_Sl_ext(nodes, P, alpha)
        n, nm = O.sizes(N, P)
        H = S[nm:nm + N - 1, nm:nm + N - 1]
        g0 = 1 / math.gamma(2 - alpha)
        a = alpha

        def K(k):
            if k == 0:
                return g0 * 2 ** (3 - a) / ((2 - a) * (3 - a))
            return g0 * 2 ** (3 - a) * ((k + 1) ** (3 - a) - 2 * k ** (3 - a) + (k - 1) ** (3 - a)) / ((2 - a) * (3 - a))

        I = 4
        assert H[I, I] == pytest.approx(0.25 * (2 * K(0) - K(1)), rel=1e-14)
        assert H[I, I + 1] == pytest.approx(-0.25 * K(0), rel=1e-14)
        assert H[I, I + 2] == 0.0
        for k in range(1, 4):
            assert abs(H[I, I - k] - 0.25 * (2 * K(k) - K(k - 1) - K(k + 1))) < 1e-15 * K(0)


def test_hat_values_alpha15_printed():
    """The alpha=1.5 numbers recorded in SURVEY.md §8(c) pin table."""
    N, P, alpha = 8, 2, 1.5
    S = O.assemble_Sl_ext(np.arange(N + 1) * 2.0, P, alpha)
    n, nm = O.sizes(N, P)
    H = S[nm:nm + N - 1, nm:nm + N - 1]
    assert H[4, 4] == pytest.approx(0.6231866060136242, abs=1e-15)
    assert H[4, 3] == pytest.approx(0.0625307855272551, abs=1e-15)
    assert H[4, 5] == pytest.approx(-0.5319230405352436, abs=1e-15)


# ------------------------------------------------------------------- mass
def test_mass_closed_forms():
    """int psi_p^2 = 2/(2p-1) + 2/(2p+3) on [-1,1] (orthogonality PAPER.md:131);
    hat diagonal (h_j + h_{j+1})/3."""
    nodes = np.array([0.0, 0.3, 1.0, 1.2])
    P = 5
    Mm = O.mass_ext(nodes, P)
    N = 3
    n, nm = O.sizes(N, P)
    h = np.diff(nodes)
    for e in range(N):
        for p in range(1, P):
            I = e * (P - 1) + p - 1
            assert Mm[I, I] == pytest.approx(0.5 * h[e] * (2 / (2 * p - 1) + 2 / (2 * p + 3)), rel=1e-14)
    for j in range(1, N):
        assert Mm[nm + j - 1, nm + j - 1] == pytest.approx((h[j - 1] + h[j]) / 3, rel=1e-14)


# ------------------------------------------------------------- invariants
def test_theta_half_symmetric_and_toeplitz_uniform():
    """theta=1/2 => A symmetric; uniform mesh => K_{i,i-k} independent of i
    (Toeplitz structure)."""
    p = fi.config1()
    sysm = O.assemble_system(p)
    assert np.abs(sysm.A - sysm.A.T).max() < 1e-14 * np.abs(sysm.A).max()
    nodes = fi.uniform_mesh(0, 1, 9)
    P, alpha = 3, 1.6
    ref = [O.pair_integral(P, alpha, nodes, 5, 5 - k) for k in range(4)]
    for i in range(4, 9):
        for k in range(4):
            assert np.abs(O.pair_integral(P, alpha, nodes, i, i - k) - ref[k]).max() <= 1e-13 * np.abs(ref[k]).max()


def test_geometric_mesh_pair_scaling_law():
    """Single-ratio geometric mesh: the nodes are o + c q^e, so
    t_i - s_j = q^j (t_{i-j} - s_0) and every pair integral is the first-column one
    scaled by w_j = (h_j/h_0)^{1-alpha} (the reading the geometric Toeplitz matvec
    uses); pinned against the oracle's per-pair quadrature."""
    for q, alpha in [(1.25, 1.6), (0.8, 1.3)]:
        nodes = fi.geometric_mesh(0, 1, 9, q)
        P = 3
        h = np.diff(nodes)
        for i in range(2, 9):
            for j in range(1, i + 1):
                ref = O.pair_integral(P, alpha, nodes, i - j, 0)
                got = O.pair_integral(P, alpha, nodes, i, j)
                w = (h[j] / h[0]) ** (1 - alpha)
                assert np.abs(got - w * ref).max() <= 1e-12 * np.abs(w * ref).max()


def test_coercivity_symmetric_part_positive_definite():
    """Theorem 2.1: the symmetric part of A is positive definite."""
    p = fi.config2(1.8, N=12, P=4)
    sysm = O.assemble_system(p)
    ev = np.linalg.eigvalsh(0.5 * (sysm.A + sysm.A.T))
    assert ev.min() > 0


# ----------------------------------------------------------- whole chain
def test_config1_reproduces_exact_polynomial_solution():
    """u = x^2(1-x)^2 lies in S_N^P for P>=4, so the Galerkin solution is exact
    (uniqueness, Theorem 2.1); f from the monomial closed form."""
    p = fi.config1()
    sysm, G, X = O.reference_solve(p)
    xis = np.linspace(-1, 1, 13)
    uh = O.eval_solution(p, X[:, 0], xis)
    h = np.diff(p.nodes)
    xs = p.nodes[:-1, None] + h[:, None] * (xis[None, :] + 1) / 2
    assert np.abs(uh - fi.config1_exact(xs)).max() < 1e-14
    # nodal coefficients are the nodal values
    n, nm = O.sizes(p.N, p.P)
    assert np.abs(X[nm:, 0] - fi.config1_exact(p.nodes[1:-1])).max() < 1e-14


@pytest.mark.slow
def test_config3_p_refinement_converges_to_closed_form_solution():
    """theta=1/2, rho=0, u=(x(1-x))^{alpha/2} => f = -cos(pi alpha/2) Gamma(alpha+1)
    (fractional-Laplacian identity); L_inf error must fall under p-refinement on
    the geometric mesh (BASELINE config 3)."""
    errs = []
    xis = np.linspace(-1, 1, 50)
    for P in (4, 8, 12):
        p = fi.config3(P)
        sysm, G, X = O.reference_solve(p)
        uh = O.eval_solution(p, X[:, 0], xis)
        h = np.diff(p.nodes)
        xl = p.nodes[:-1, None] + h[:, None] * (xis[None, :] + 1) / 2
        xr = (p.nodes[-1] - p.nodes[1:])[:, None] + h[:, None] * (1 - xis[None, :]) / 2
        errs.append(np.abs(uh - fi.config3_exact(xl, xr)).max())
    assert errs[0] < 3e-5 and errs[1] < errs[0] / 30 and errs[2] < errs[1] / 30


# --------------------------------------------------------------- H-matrix
def _graded_problem(N=48, P=3, alpha=1.6):
    nodes = fi.graded_mesh(0.0, 10.0, N, 5.0)
    return fi.Problem("g", 0.0, 10.0, alpha, 1.0, 0.0, 0.0, 0.0, nodes, P, 5)


def test_hmatrix_lambda_to_zero_is_exact():
    """lambda -> 0: no block is admissible, so A~ = A."""
    p = _graded_problem(N=24)
    sysm = O.assemble_system(p)
    At, part = O.hmatrix_dense(p, sysm, R=3, lam=1e-9, n_min=4)
    assert all(k == "dense" for _, _, k in part)
    assert np.array_equal(At, sysm.A)


def test_hmatrix_error_decreases_with_rank():
    """||A - A~||_F decays (exponentially) in R (Fig. fig:matrixerror)."""
    p = _graded_problem()
    sysm = O.assemble_system(p)
    errs = []
    for R in (2, 4, 6, 8, 10):
        At, _ = O.hmatrix_dense(p, sysm, R=R, lam=1.0, n_min=4)
        errs.append(np.linalg.norm(sysm.A - At))
    assert all(errs[k + 1] < 0.5 * errs[k] for k in range(len(errs) - 1))


def test_taylor_factor_structure_and_closed_forms():
    """W_{j0} = 0 and W^q_{j nu} = 0 for q > nu (int phi' = 0, orthogonality);
    hat factors match the closed forms of Eq. (eq412) and Eq. (eq415)
    (PAPER.md:492-504, 531-546)."""
    p = _graded_problem(N=32, P=4)
    nodes, P, alpha = p.nodes, p.P, p.alpha
    root = O.cluster_tree(p.N, 4)
    part = O.block_partition(nodes, root, 1.0)
    g0 = 1 / math.gamma(2 - alpha)
    checked = 0
    for t, s, kind in part:
        if kind != "lr" or nodes[t.e0] < nodes[s.e1]:
            continue
        ss, ts = O.cluster_support(nodes, s), O.cluster_support(nodes, t)
        if (ss[1] - ss[0]) > (ts[1] - ts[0]):
            continue                     # s-expansion blocks only (the theorem's setting)
        R = 6
        Q, W = O.taylor_factors(p, t, s, R)
        s0 = 0.5 * (ss[0] + ss[1])
        # rows in cluster order: for each element, P-1 modal then the right-node hat
        r = 0
        for e in range(s.e0, s.e1):
            for q in range(1, P):
                assert abs(W[r, 0]) < 1e-13
                for nu in range(min(q, R)):
                    assert abs(W[r, nu]) < 1e-12 * max(1.0, np.abs(W[r]).max())
                r += 1
            if e + 1 <= p.N - 1:
                j = e + 1                # hat of node j
                xm, x0, xp = nodes[j - 1], nodes[j], nodes[min(j + 1, p.N)]
                for nu in range(R):
                    wbar = ((x0 - s0) ** (nu + 1) - (xm - s0) ** (nu + 1)) / ((x0 - xm) * (nu + 1)) \
                        - ((xp - s0) ** (nu + 1) - (x0 - s0) ** (nu + 1)) / ((xp - x0) * (nu + 1))
                    assert W[r, nu] == pytest.approx(wbar, rel=1e-11, abs=1e-13 * abs(xp - xm) ** nu)
                r += 1
        r = 0
        for e in range(t.e0, t.e1):
            r += P - 1
            if e + 1 <= p.N - 1:
                i = e + 1
                xm, x0, xp = nodes[i - 1], nodes[i], nodes[min(i + 1, p.N)]
                for nu in range(R):
                    pr = 1.0
                    for l in range(1, nu + 1):
                        pr *= alpha + l - 2
                    ex = 2 - alpha - nu
                    qbar = g0 / math.factorial(nu) * pr * (
                        ((x0 - s0) ** ex - (xm - s0) ** ex) / ((x0 - xm) * ex)
                        - ((xp - s0) ** ex - (x0 - s0) ** ex) / ((xp - x0) * ex))
                    assert Q[r, nu] == pytest.approx(qbar, rel=1e-10, abs=1e-14)
                r += 1
        checked += 1
    assert checked > 0


def test_theorem33_entrywise_bounds():
    """|B - B~| <= 8 h_i c0/Gamma(2-a) delta^R on s-expansion admissible blocks
    (Theorem 3.3, Eq. (eq408))."""
    p = _graded_problem(N=32, P=3)
    sysm = O.assemble_system(p)
    nodes, P, alpha, lam, R = p.nodes, p.P, p.alpha, 1.0, 4
    root = O.cluster_tree(p.N, 4)
    n, nm = O.sizes(p.N, p.P)
    part = O.block_partition(nodes, root, lam)
    g0 = 1 / math.gamma(2 - alpha)
    delta = lam / (2 + lam)
    nchk = 0
    for t, s, kind in part:
        if kind != "lr" or nodes[t.e0] < nodes[s.e1]:
            continue
        ss, ts = O.cluster_support(nodes, s), O.cluster_support(nodes, t)
        if (ss[1] - ss[0]) > (ts[1] - ts[0]):
            continue
        Q, W = O.taylor_factors(p, t, s, R)
        rows = O.paper_index_of_element_dofs(p.N, P, t.e0, t.e1)
        cols = O.paper_index_of_element_dofs(p.N, P, s.e0, s.e1)
        exact = sysm.Sl_ext[np.ix_(rows, cols)]
        approx = Q @ W.T
        a_, d_ = ts[0], ss[1]
        s0 = 0.5 * (ss[0] + ss[1])
        c0 = (1 / (abs(a_ - d_) + abs(d_ - s0)) ** alpha) * (1 + lam / 2) * (R + 1 + lam / 2)
        for ri, I in enumerate(rows):
            for ci, J in enumerate(cols):
                if I < nm and J < nm:               # B block: modal x modal
                    e = I // (P - 1)
                    h_i = nodes[e + 1] - nodes[e]
                    bound = 8 * h_i * c0 * g0 * delta ** R
                    assert abs(exact[ri, ci] - approx[ri, ci]) <= bound
                    nchk += 1
    assert nchk > 0


def test_lemma32_kernel_bound():
    """Lemma 3.2 with the proof's exponent (alpha-1) (reading A8)."""
    alpha, lam = 1.6, 1.0
    c_, d_ = 0.0, 1.0                 # sigma
    a_, b_ = 2.0, 3.0                 # tau: max diam 1 <= lam * dist 1
    s0 = 0.5 * (c_ + d_)
    for R in (2, 4, 8):
        bound = (1 / (a_ - d_) ** (alpha - 1)) * (1 + lam / 2) * (lam / (2 + lam)) ** R
        worst = 0.0
        for t in np.linspace(a_, b_, 21):
            for s in np.linspace(c_, d_, 21):
                kt = 0.0
                for nu in range(R):
                    cnu = 1.0
                    for l in range(nu):
                        cnu *= (alpha - 1 + l)
                    cnu /= math.factorial(nu)
                    kt += cnu * (t - s0) ** (1 - alpha - nu) * (s - s0) ** nu
                worst = max(worst, abs((t - s) ** (1 - alpha) - kt))
        assert worst <= bound


def test_geometric_mesh_recipe_single_ratio():
    """The seeded-input recipe for geometric meshes (fde_inputs.geometric_mesh,
    PAPER.md:634): every node from its own power, so h_{e+1}/h_e equals q to far
    below the 1e-10 the library's single-ratio test (and Toeplitz path) requires,
    even on long meshes; endpoints exact, nodes strictly increasing."""
    for q, N in [(1.001, 4096), (1.01, 256), (0.97, 100), (1.2, 24), (0.8, 9)]:
        x = fi.geometric_mesh(0.0, 1.0, N, q)
        h = np.diff(x)
        assert x[0] == 0.0 and x[-1] == 1.0 and (h > 0).all()
        assert np.abs(h[1:] / h[:-1] / q - 1).max() < 1e-11
