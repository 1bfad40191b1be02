"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Metrics:
  M-A  max |dA_IJ| / sqrt(A_II A_JJ)            <= 1e-10 (assembly, A~)
  M-B  max |dy_I| / (|A| |x|)_I                 <= 1e-10 (matvec)
  M-D  ||X - X_ora||_D / ||X_ora||_D, D=diag(A) <= 1e-10 (solve)
"""
import numpy as np
import pytest

import fde_inputs as fi
import oracle as O
from parity_util import md_check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def fde():
    from paper_1808_02937_b200 import fde as F
    return F


@pytest.fixture(scope="module")
def h(fde):
    return fde.Handle(0)


def metric_A(Ag, Ao):
    d = np.sqrt(np.abs(np.diag(Ao)))
    return np.max(np.abs(Ag - Ao) / (d[:, None] * d[None, :]))


def graded_mirrored(N):
    p = fi.config4(N=N, P=8)
    return p


def problems_small():
    out = [fi.config1()]
    for a in (1.2, 1.5, 1.8):
        out.append(fi.config2(a, N=24, P=8))
    out.append(fi.config3(P=4))
    out.append(fi.config3(P=9))
    out.append(fi.config4(N=40, P=6))
    rng = np.random.default_rng(7)
    x = np.sort(rng.uniform(0.0, 3.0, 17))
    nodes = np.concatenate([[0.0], x, [3.0]])
    out.append(fi.Problem("random", 0.0, 3.0, 1.65, 0.25, 0.5, 0.3, -0.7, nodes, 5, 6, n_min=3,
                          forcings=[fi.random_legendre_forcing(3)]))
    out.append(fi.Problem("P1", 0.0, 1.0, 1.3, 0.6, 1.0, 0.0, 0.0, fi.uniform_mesh(0, 1, 12), 1, 4, n_min=2,
                          forcings=[fi.random_legendre_forcing(4)]))
    return out


_ORA = {}


def oracle_system(p):
    key = (p.name, p.N, p.P, p.alpha, p.theta, p.rho, float(p.nodes.sum()))
    if key not in _ORA:
        _ORA[key] = O.assemble_system(p)
    return _ORA[key]


@pytest.mark.parametrize("p", problems_small(), ids=lambda p: p.name)
def test_assembly_matches_oracle(fde, h, p):
    op = fde.assemble_problem(h, p)
    Ag = fde.operator_dense_paper(h, op).cpu().numpy()
    so = oracle_system(p)
    assert metric_A(Ag, so.A) <= TOL
    B = fde.operator_boundary_columns(h, op).cpu().numpy()
    d = np.sqrt(np.abs(np.diag(so.A)))
    for k in range(2):
        Ab = so.Abnd[:, k]
        # scale by sqrt(A_II * A_bb); boundary hat diagonal from the extended matrix
        nb = p.n + k
        Abb = p.rho * so.M_ext[nb, nb] + so.Sl_ext[nb, nb]
        assert np.max(np.abs(B[k] - Ab) / (d * np.sqrt(abs(Abb)))) <= TOL
    op.free()


@pytest.mark.parametrize("p", problems_small(), ids=lambda p: p.name)
def test_rhs_matches_oracle(fde, h, p):
    if not p.forcings:
        pytest.skip("no forcing")
    op = fde.assemble_problem(h, p)
    Gg = fde.sem_rhs(h, op, p.forcings).cpu().numpy()[0]
    so = oracle_system(p)
    Go = O.rhs(p, so, p.forcings[0])
    scale = np.abs(Go).max() + 1e-300
    assert np.max(np.abs(Gg - Go)) <= 1e-12 * scale + 1e-13
    op.free()


@pytest.mark.parametrize("p", problems_small(), ids=lambda p: p.name)
def test_dense_matvec_matches_oracle(fde, h, p):
    op = fde.assemble_problem(h, p)
    so = oracle_system(p)
    rng = np.random.default_rng(1)
    X = rng.standard_normal((3, p.n))
    Y = fde.stiffness_matvec(h, op, torch.tensor(X, device="cuda"), path=fde.PATH_DENSE).cpu().numpy()
    Yo = (so.A.astype(np.longdouble) @ X.T.astype(np.longdouble)).T.astype(np.float64)
    den = (np.abs(so.A) @ np.abs(X.T)).T
    assert np.max(np.abs(Y - Yo) / den) <= TOL
    op.free()


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.8])
@pytest.mark.parametrize("N", [24, 100])
def test_toeplitz_fft_matvec_matches_oracle(fde, h, alpha, N):
    p = fi.config2(alpha, N=N, P=8)
    op = fde.assemble_problem(h, p, flags=fde.OP_DENSE | fde.OP_TOEPLITZ)
    rng = np.random.default_rng(2)
    X = torch.tensor(rng.standard_normal((2, p.n)), device="cuda")
    Yf = fde.stiffness_matvec(h, op, X, path=fde.PATH_TOEPLITZ).cpu().numpy()
    Yd = fde.stiffness_matvec(h, op, X, path=fde.PATH_DENSE).cpu().numpy()
    Ag = fde.operator_dense_paper(h, op).cpu().numpy()
    den = (np.abs(Ag) @ np.abs(X.cpu().numpy().T)).T
    assert np.max(np.abs(Yf - Yd) / den) <= TOL
    if N == 24:
        so = oracle_system(p)
        Yo = (so.A @ X.cpu().numpy().T).T
        assert np.max(np.abs(Yf - Yo) / den) <= TOL
    op.free()


@pytest.mark.parametrize("qhat,N,P,alpha", [(1.05, 24, 8, 1.5), (0.9, 24, 4, 1.3), (1.2, 24, 6, 1.8),
                                           (1.02, 100, 8, 1.6), (0.97, 100, 5, 1.4)])
def test_toeplitz_fft_matvec_geometric_mesh(fde, h, qhat, N, P, alpha):
    """Geometric meshes: K_ij = w_j K_{i-j,0}, Toeplitz after a
    diagonal scaling; the FFT matvec equals the dense one and (N = 24) the oracle's A x."""
    p = fi.geometric_problem(qhat, N=N, P=P, alpha=alpha)
    op = fde.assemble_problem(h, p, flags=fde.OP_DENSE | fde.OP_TOEPLITZ)
    rng = np.random.default_rng(3)
    X = torch.tensor(rng.standard_normal((3, p.n)), device="cuda")
    Yf = fde.stiffness_matvec(h, op, X, path=fde.PATH_TOEPLITZ).cpu().numpy()
    Yd = fde.stiffness_matvec(h, op, X, path=fde.PATH_DENSE).cpu().numpy()
    Ag = fde.operator_dense_paper(h, op).cpu().numpy()
    den = (np.abs(Ag) @ np.abs(X.cpu().numpy().T)).T
    assert np.max(np.abs(Yf - Yd) / den) <= TOL
    if N == 24:
        so = oracle_system(p)
        Yo = (so.A @ X.cpu().numpy().T).T
        assert np.max(np.abs(Yf - Yo) / den) <= TOL
    op.free()


def test_toeplitz_rejects_graded_mesh_but_not_geometric(fde, h):
    p = fi.config4(N=16, P=4)   # x_j = (2j/N)^2 / 2: ratios vary
    with pytest.raises(fde.FdeError) as e:
        fde.assemble_problem(h, p, flags=fde.OP_TOEPLITZ)
    assert e.value.name == "FDE_EUNSUPPORTED_MESH"
    op = fde.assemble_problem(h, fi.geometric_problem(1.1, N=16, P=4), flags=fde.OP_TOEPLITZ)
    op.free()


def test_toeplitz_rejects_nonuniform(fde, h):
    p = fi.config4(N=16, P=4)
    with pytest.raises(fde.FdeError) as e:
        fde.assemble_problem(h, p, flags=fde.OP_TOEPLITZ)
    assert e.value.name == "FDE_EUNSUPPORTED_MESH"


@pytest.mark.parametrize("p", [fi.config1(), fi.config2(1.5, N=24, P=8), fi.config3(P=6)], ids=lambda p: p.name)
def test_unpreconditioned_gmres_matches_oracle(fde, h, p):
    op = fde.assemble_problem(h, p)
    G = fde.sem_rhs(h, op, p.forcings)
    X, rep = fde.solve(h, op, None, G, tol=1e-13, maxiter=4000, restart=200)
    so = oracle_system(p)
    Go = O.rhs(p, so, p.forcings[0])
    md_check(p, X.cpu().numpy()[0], so, Go)      # M-D: D-norm, u_h pointwise, backward error
    op.free()


@pytest.mark.parametrize("p", [fi.config1(), fi.config2(1.5, N=48, P=4), fi.config4(N=64, P=4)],
                         ids=lambda p: p.name)
@pytest.mark.parametrize("R", [3, 6])
def test_hmatrix_matches_oracle(fde, h, p, R):
    n_min = 2 if p.N <= 8 else 4
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, R, 1.0, n_min)
    Ag = fde.hmatrix_dense_paper(h, hm).cpu().numpy()
    so = oracle_system(p)
    At, part = O.hmatrix_dense(p, so, R=R, lam=1.0, n_min=n_min)
    assert hm.info.nblocks_lr == sum(1 for _, _, k in part if k == "lr")
    assert hm.info.nblocks_dense == sum(1 for _, _, k in part if k == "dense")
    assert metric_A(Ag, At) <= TOL
    hm.free()
    op.free()


def test_invalid_inputs_raise(fde, h):
    p = fi.config1()
    with pytest.raises(fde.FdeError) as e:
        fde.sem_assemble(h, 0.0, 1.0, 2.5, 0.5, 1.0, 0, 0, p.nodes, 4)
    assert e.value.name == "FDE_EINVAL_PARAM"
    with pytest.raises(fde.FdeError) as e:
        fde.sem_assemble(h, 1.0, 0.0, 1.5, 0.5, 1.0, 0, 0, p.nodes, 4)
    assert e.value.name == "FDE_EINVAL_DOMAIN"
    bad = p.nodes.copy()
    bad[3] = bad[2]
    with pytest.raises(fde.FdeError) as e:
        fde.sem_assemble(h, 0.0, 1.0, 1.5, 0.5, 1.0, 0, 0, bad, 4)
    assert e.value.name == "FDE_EINVAL_MESH"
    with pytest.raises(fde.FdeError) as e:
        fde.sem_assemble(h, 0.0, 1.0, 1.5, 0.5, 1.0, 0, 0, p.nodes, 0)
    assert e.value.name == "FDE_EDEGREE"
    nan, inf = float("nan"), float("inf")
    for args, code in [((0.0, 1.0, nan, 0.5, 1.0, 0, 0), "FDE_EINVAL_PARAM"),      # non-finite parameters
                       ((0.0, 1.0, 1.5, nan, 1.0, 0, 0), "FDE_EINVAL_PARAM"),
                       ((0.0, 1.0, 1.5, 0.5, nan, 0, 0), "FDE_EINVAL_PARAM"),
                       ((0.0, 1.0, 1.5, 0.5, inf, 0, 0), "FDE_EINVAL_PARAM"),
                       ((0.0, 1.0, 1.5, 0.5, 1.0, nan, 0), "FDE_EINVAL_PARAM"),
                       ((0.0, 1.0, 1.5, 0.5, 1.0, 0, inf), "FDE_EINVAL_PARAM")]:
        with pytest.raises(fde.FdeError) as e:
            fde.sem_assemble(h, *args, p.nodes, 4)
        assert e.value.name == code, args
    for nodes, a, b in [(np.concatenate([[-inf], p.nodes[1:]]), -inf, 1.0), (np.where(np.arange(p.nodes.size) == 3, nan, p.nodes), 0.0, 1.0)]:
        with pytest.raises(fde.FdeError) as e:
            fde.sem_assemble(h, a, b, 1.5, 0.5, 1.0, 0, 0, nodes, 4)
        assert e.value.name in ("FDE_EINVAL_DOMAIN", "FDE_EINVAL_MESH")


# ------------------------------------------------------------------ H-LU
HLU_CASES = [
    (fi.config1(), 2),
    (fi.config2(1.5, N=48, P=4), 4),
    (fi.config4(N=64, P=4), 4),
    (fi.config3(P=4), 4),
]


HLU2_CASES = HLU_CASES + [
    (fi.config4(N=96, P=8), 4),          # 24 leaves of 32 dofs: several low-rank levels
    (fi.config2(1.3, N=64, P=8), 16),    # leaves of exactly 128 dofs (kernel limit)
    (fi.config4(N=44, P=6), 5),          # leaves at two depths (dense blocks spanning two leaves)
    (fi.config4(N=128, P=8), 40),        # 256-dof leaves: two sweep tiles per leaf
    (fi.config3(P=12), 16),              # geometric layers, 192-dof leaves (two tiles of 96)
]


@pytest.fixture(params=[0, 1], ids=["leaf-ordered", "recursive"])
def hlu_mode(fde, request):
    fde.set_hlu_mode(request.param)
    yield request.param
    fde.set_hlu_mode(0)


@pytest.mark.parametrize("case", HLU2_CASES, ids=lambda c: f"{c[0].name}-nmin{c[1]}")
def test_hlu_exact_mode_equals_dense_solve_of_Atilde(fde, h, case, hlu_mode):
    """tol = 0: the formatted H-LU is the exact LU of A~ (up to rounding), so
    precond_apply must equal a dense solve with the oracle's A~ (metric M-C).
    Both algorithms (leaf-ordered batched, recursive) are checked."""
    p, n_min = case
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    lu = fde.hlu_factor(h, hm, 0.0)
    assert lu.info.algorithm == (1 if hlu_mode == 0 else 0)
    so = oracle_system(p)
    At, _ = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min)
    rng = np.random.default_rng(5)
    r = rng.standard_normal((2, p.n))
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()
    zo = np.linalg.solve(At, r.T).T
    err = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert err <= TOL, err
    for o in (lu, hm, op):
        o.free()


@pytest.mark.parametrize("case", HLU2_CASES[-5:], ids=lambda c: f"{c[0].name}-nmin{c[1]}")
def test_hlu_deferred_updates_exact_mode(fde, h, case, monkeypatch):
    """The deferred dense updates (default for >= 128 sweep tiles, forced here with
    FDE_H2_DEFER=1; small flush threshold and scratch ring so that every flush path
    runs) give the exact LU of A~ at tol = 0 like the step-by-step updates."""
    monkeypatch.setenv("FDE_H2_DEFER", "1")
    monkeypatch.setenv("FDE_H2_KFLUSH", "32")
    monkeypatch.setenv("FDE_H2_RING", "3")
    p, n_min = case
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    lu = fde.hlu_factor(h, hm, 0.0)
    so = oracle_system(p)
    At, _ = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min)
    r = np.random.default_rng(7).standard_normal((2, p.n))
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()
    zo = np.linalg.solve(At, r.T).T
    err = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert err <= TOL, err
    for o in (lu, hm, op):
        o.free()


@pytest.mark.parametrize("tol", [0.0, 1e-3])
def test_hlu_planner_threads_bitwise(fde, h, tol, monkeypatch):
    """The deferred dense-update terms are built by planner threads (tiles split by
    row, each tile's terms in the serial order): 1 and 4 threads give the same
    factorisation bit for bit (precond_apply compared with torch.equal)."""
    monkeypatch.setenv("FDE_H2_DEFER", "1")
    monkeypatch.setenv("FDE_H2_KFLUSH", "32")
    p = fi.config4(N=256, P=8)
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, 16)
    r = torch.tensor(np.random.default_rng(5).standard_normal((3, p.n)), device="cuda")
    z = {}
    for nt in ("1", "4"):
        monkeypatch.setenv("FDE_H2_PLAN_THREADS", nt)
        lu = fde.hlu_factor(h, hm, tol)
        z[nt] = fde.precond_apply(h, lu, r)
        lu.free()
    assert torch.equal(z["1"], z["4"])
    hm.free()
    op.free()


@pytest.mark.parametrize("gemm_path", [False, True], ids=["tiles", "gemm-tasks"])
@pytest.mark.parametrize("nrhs", [9, 19, 64])
def test_hlu_apply_many_rhs_equals_dense_solve_of_Atilde(fde, h, nrhs, gemm_path, monkeypatch):
    """precond_apply with more right-hand sides than the register chunk (nrhs > 8:
    8 x 8 output tiles of rows x RHS, ragged at 9 and 19) against the dense solve
    with the oracle's A~ in exact mode (tol = 0), like the two-RHS test above."""
    p, n_min = fi.config4(N=96, P=8), 4   # 24 leaves, several low-rank levels
    if gemm_path:   # the opt-in multi-term GEMM-task substitutions (nrhs >= 16)
        monkeypatch.setenv("FDE_APPLY_GEMM_MIN", "16")
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    lu = fde.hlu_factor(h, hm, 0.0)
    so = oracle_system(p)
    At, _ = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min)
    r = np.random.default_rng(nrhs).standard_normal((nrhs, p.n))
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()
    zo = np.linalg.solve(At, r.T).T
    err = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert err <= TOL, err
    for o in (lu, hm, op):
        o.free()


@pytest.mark.parametrize("case", HLU2_CASES, ids=lambda c: f"{c[0].name}-nmin{c[1]}")
def test_hlu_preconditioned_gmres_matches_oracle(fde, h, case, hlu_mode):
    """tol = 1e-3: A~^{-1} is only approximate (parity unpinned
    for the factor itself), but the preconditioned solve must reach the oracle's
    X (metric M-D) and need fewer iterations than the unpreconditioned one."""
    p, n_min = case
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    G = fde.sem_rhs(h, op, p.forcings)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12)   # BASELINE: GMRES tol 1e-12
    try:
        X0, rep0 = fde.solve(h, op, None, G, tol=1e-12, maxiter=3000, restart=200)
        its0 = rep0.iterations
    except fde.FdeError as e:   # ill-conditioned cases (c3: kappa ~ 1e11) need the preconditioner
        assert e.name == "FDE_EMAXITER"
        its0 = 10 ** 9
    so = oracle_system(p)
    md_check(p, X.cpu().numpy()[0], so, O.rhs(p, so, p.forcings[0]))   # M-D, all three parts
    assert rep.iterations < its0
    # the factor approximates A~: ||A~ z - r|| small relative to ||r||
    At, _ = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min)
    r = np.random.default_rng(6).standard_normal(p.n)
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()[0]
    assert np.linalg.norm(At @ z - r) / np.linalg.norm(r) < 5e-2
    for o in (lu, hm, op):
        o.free()


@pytest.mark.parametrize("tma", ["1", "0"], ids=["tma", "cpasync"])
@pytest.mark.parametrize("splitk", [None, "3"], ids=["auto", "splitK3"])
@pytest.mark.parametrize("nrhs", [8, 37, 64])
def test_multi_rhs_dmma_matvec_matches_oracle(fde, h, nrhs, splitk, tma, monkeypatch):
    """nrhs >= 8 routes the dense matvec to the FP64 tensor-core GEMM (DMMA): the TMA
    kernel (64 x 16 swizzled tiles, mbarrier ring, zero-filled ragged edges) or the
    cp.async one (FDE_GEMM_TMA=0); with FDE_GEMM_SPLITK=3 the K dimension is cut
    into three slices whose partial products k_sum_splits adds (c5 uses 4)."""
    monkeypatch.setenv("FDE_GEMM_TMA", tma)
    if splitk:
        monkeypatch.setenv("FDE_GEMM_SPLITK", splitk)
    p = fi.config4(N=40, P=6)
    op = fde.assemble_problem(h, p)
    so = oracle_system(p)
    X = np.random.default_rng(nrhs).standard_normal((nrhs, p.n))
    Y = fde.stiffness_matvec(h, op, torch.tensor(X, device="cuda"), path=fde.PATH_DENSE).cpu().numpy()
    Yo = (so.A.astype(np.longdouble) @ X.T.astype(np.longdouble)).T.astype(np.float64)
    den = (np.abs(so.A) @ np.abs(X.T)).T
    assert np.max(np.abs(Y - Yo) / den) <= TOL
    op.free()


def test_multi_rhs_solve_matches_single(fde, h):
    """64 RHS in lockstep (config-5 style) give the same X as one-by-one solves."""
    p = fi.config2(1.6, N=32, P=8)
    p.forcings = [fi.random_legendre_forcing(s) for s in range(12)]
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, 8, 1.0, 4)
    lu = fde.hlu_factor(h, hm, 1e-3)
    G = fde.sem_rhs(h, op, p.forcings)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12)
    for c in (0, 5, 11):
        Xc, _ = fde.solve(h, op, lu, G[c:c + 1].clone(), tol=1e-12)
        assert np.max(np.abs(X[c].cpu().numpy() - Xc[0].cpu().numpy())) <= 1e-9 * np.abs(Xc.cpu().numpy()).max()
    for o in (lu, hm, op):
        o.free()


def test_example51_bicgstab_iterations_pattern(fde, h):
    """Example 5.1 (Table 1 setting PAPER.md:794-815): preconditioned
    BiCGSTAB at tol 1e-13 converges in a handful of iterations, non-increasing in R
    (the table's pattern), and the solution approximates the exact u."""
    its = []
    for R in (2, 3, 5, 7):
        p = fi.example51(N=100, P=3, R=R)
        op = fde.assemble_problem(h, p)
        G = fde.sem_rhs(h, op, p.forcings)
        hm = fde.hmatrix_build(h, op, R, 1.0, p.n_min)
        lu = fde.hlu_factor(h, hm, 1e-3)
        X, rep = fde.solve(h, op, lu, G, method=fde.BICGSTAB, tol=1e-13, maxiter=400)
        its.append(rep.iterations)
        if R == 7:
            so = oracle_system(p)
            x = X.cpu().numpy()[0]
            md_check(p, x, so, O.rhs(p, so, p.forcings[0]))
            xis = np.linspace(-1, 1, 9)
            uh = O.eval_solution(p, x, xis)
            hh = np.diff(p.nodes)
            xs = p.nodes[:-1, None] + hh[:, None] * (xis[None, :] + 1) / 2
            assert np.abs(uh - fi.example51_exact(xs)).max() < 1e-3
        for o in (lu, hm, op):
            o.free()
    assert its[-1] <= 10
    assert all(its[k + 1] <= its[k] + 1 for k in range(3)), its


def test_hlu_leaf_ordered_matches_recursive_factors(fde, h):
    """At tol = 0 both algorithms compute the unique LU of A~ (no pivoting): the
    packed factors agree entry by entry up to rounding (scaled like M-A)."""
    p = fi.config4(N=96, P=8)
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, 4)
    F = []
    for mode in (0, 1):
        fde.set_hlu_mode(mode)
        lu = fde.hlu_factor(h, hm, 0.0)
        F.append(fde.hlu_dense_internal(h, lu).cpu().numpy())
        lu.free()
    fde.set_hlu_mode(0)
    d = np.sqrt(np.abs(np.diag(F[1])))
    assert np.max(np.abs(F[0] - F[1]) / (d[:, None] * d[None, :])) <= 1e-9
    hm.free()
    op.free()


def test_condition_numbers_example51(fde, h):
    """NEXT-4: on Example 5.1's graded mesh cond_2(A)
    grows past 1e9 already at N = 300 (6.8e11 at N = 1000, profiles/r1f_cond_diag.jsonl)
    while the H-LU-preconditioned operator A~^{-1} A (Tol_HLU = 1e-3) has
    cond_2 < 10; A~^{-1} A formed column by column through precond_apply."""
    p = fi.example51(N=300, P=3)
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    A = fde.operator_dense_paper(h, op)
    s = torch.linalg.svdvals(A)
    MA = fde.precond_apply(h, lu, A.T.contiguous()).T
    sp = torch.linalg.svdvals(MA)
    assert (s[0] / s[-1]).item() > 1e9
    assert (sp[0] / sp[-1]).item() < 10.0
    lu.free(); hm.free(); op.free()


@pytest.mark.parametrize("NP", [(1, 2), (2, 1), (1, 4), (3, 1), (2, 2), (1, 9)], ids=lambda t: f"N{t[0]}P{t[1]}")
def test_tiny_problems_full_path(fde, h, NP):
    """The degenerate sizes of the method: one or two elements, P = 1 (n = N P - 1 =
    1 .. 8 unknowns), through every call of the path (assembly, load, H-matrix with
    a single leaf, H-LU, preconditioned GMRES) against the oracle's system and
    Galerkin solution."""
    N, P = NP
    p = fi.Problem(f"tiny-N{N}-P{P}", 0.0, 1.0, 1.55, 0.4, 0.5, 0.25, -0.5, fi.uniform_mesh(0, 1, N), P, 3,
                   n_min=1, forcings=[fi.random_legendre_forcing(11)])
    op = fde.assemble_problem(h, p)
    so = oracle_system(p)
    Ag = fde.operator_dense_paper(h, op).cpu().numpy()
    assert Ag.shape == (p.n, p.n)
    assert metric_A(Ag, so.A) <= TOL
    G = fde.sem_rhs(h, op, p.forcings)
    Go = O.rhs(p, so, p.forcings[0])
    assert np.max(np.abs(G.cpu().numpy()[0] - Go)) <= TOL * np.max(np.abs(Go))
    hm = fde.hmatrix_build(h, op, p.R, 1.0, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12)
    Xo = np.linalg.solve(so.A, Go)
    assert np.linalg.norm(X.cpu().numpy()[0] - Xo) <= 1e-10 * np.linalg.norm(Xo)
    for o in (lu, hm, op):
        o.free()


def test_non_finite_inputs_fail_loudly(fde, h):
    """Non-finite data never hangs or passes silently: a NaN in the load vector makes
    GMRES and BiCGSTAB stop with FDE_EBREAKDOWN (before round 2's fix a NaN norm
    read as a zero right-hand side: X = 0 returned as converged), precond_apply
    propagates NaN, the binding rejects float32 and host tensors (they would be
    read as garbage through the C-ABI), and the handle stays usable."""
    p = fi.config4(N=32, P=4)
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, 4)
    lu = fde.hlu_factor(h, hm, 1e-3)
    G = fde.sem_rhs(h, op, p.forcings)
    Gn = G.clone()
    Gn[0, 5] = float("nan")
    for method in (fde.GMRES, fde.BICGSTAB):
        with pytest.raises(fde.FdeError) as e:
            fde.solve(h, op, lu, Gn, tol=1e-12, method=method)
        assert e.value.name == "FDE_EBREAKDOWN"
    z = fde.precond_apply(h, lu, torch.full((1, p.n), float("nan"), device="cuda", dtype=torch.float64))
    assert torch.isnan(z).all()                                                        # NaN in, NaN out
    with pytest.raises(TypeError):                                                     # float32 is rejected
        fde.precond_apply(h, lu, torch.zeros((1, p.n), device="cuda"))
    with pytest.raises(ValueError):                                                    # so is host memory
        fde.precond_apply(h, lu, torch.zeros((1, p.n), dtype=torch.float64))
    X, rep = fde.solve(h, op, lu, G, tol=1e-12)                                        # still usable
    assert torch.isfinite(X).all() and rep.iterations >= 1
    for o in (lu, hm, op):
        o.free()


def _edge_problems():
    out = []
    rng = np.random.default_rng(21)
    for alpha in (1.02, 1.98):        # near both ends of (1, 2): the kernel |x-s|^{1-alpha} almost flat / almost 1/|x-s|
        out.append(fi.Problem(f"alpha{alpha}", 0.0, 1.0, alpha, 0.35, 0.5, 0.2, -0.1, fi.graded_mesh(0.0, 1.0, 20, 2.0),
                              5, 6, n_min=2, forcings=[fi.random_legendre_forcing(5)]))
    for theta in (0.0, 1.0):          # one-sided operators (right- / left-sided only)
        out.append(fi.Problem(f"theta{theta}", -1.0, 2.0, 1.45, theta, 0.0, 0.0, 0.0, fi.uniform_mesh(-1.0, 2.0, 16),
                              6, 6, n_min=2, forcings=[fi.random_legendre_forcing(6)]))
    out.append(fi.Problem("Pmax", 0.0, 1.0, 1.6, 0.5, 1.0, 0.0, 0.0, fi.uniform_mesh(0.0, 1.0, 3), 32, 4, n_min=1,
                          forcings=[fi.random_legendre_forcing(7)]))                 # P = FDE_MAX_P
    nodes = np.concatenate([[0.0], np.sort(rng.uniform(0.0, 1.0, 9)) ** 4, [1.0]])   # clustered random mesh
    out.append(fi.Problem("clustered", 0.0, 1.0, 1.7, 0.8, 3.0, 1.0, 2.0, nodes, 7, 6, n_min=2,
                          forcings=[fi.random_legendre_forcing(8)]))
    return out


@pytest.mark.parametrize("p", _edge_problems(), ids=lambda p: p.name)
def test_edge_parameters_full_path(fde, h, p):
    """alpha near 1 and 2, theta = 0 and 1, P = FDE_MAX_P = 32, a clustered random
    mesh with rho = 3 and nonzero boundary values: assembly (M-A), load, and the
    preconditioned solve (M-D) against the oracle."""
    op = fde.assemble_problem(h, p)
    so = oracle_system(p)
    assert metric_A(fde.operator_dense_paper(h, op).cpu().numpy(), so.A) <= TOL
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-13, maxiter=300)
    md_check(p, X.cpu().numpy()[0], so, O.rhs(p, so, p.forcings[0]))
    for o in (lu, hm, op):
        o.free()


@pytest.mark.parametrize("tol", [0.0, 1e-3])
def test_rank_limit_R32(fde, h, tol):
    """R = 32 (the largest Taylor rank): A~ against the oracle's A~ (M-A), and the
    H-LU (exact at tol = 0, truncated to capacity 32 at 1e-3) preconditioning a
    GMRES solve that reaches the oracle's Galerkin solution."""
    p = fi.config4(N=48, P=4)
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, 32, 1.0, 2)
    so = oracle_system(p)
    At, _ = O.hmatrix_dense(p, so, R=32, lam=1.0, n_min=2)
    assert metric_A(fde.hmatrix_dense_paper(h, hm).cpu().numpy(), At) <= TOL
    lu = fde.hlu_factor(h, hm, tol)
    G = fde.sem_rhs(h, op, p.forcings)
    X, rep = fde.solve(h, op, lu, G, tol=1e-13)
    md_check(p, X.cpu().numpy()[0], so, O.rhs(p, so, p.forcings[0]))
    for o in (lu, hm, op):
        o.free()


def test_toeplitz_edge_sizes(fde, h):
    """The FFT path at its edges: one element (n = P - 1), P = 32, and P = 1 (hats
    only), against the dense operator of the same mesh."""
    for N, P in [(1, 4), (2, 1), (4, 32), (3, 7)]:
        p = fi.Problem(f"u{N}-{P}", 0.0, 2.0, 1.35, 0.3, 1.0, 0.0, 0.0, fi.uniform_mesh(0.0, 2.0, N), P, 3, n_min=1,
                       forcings=[fi.random_legendre_forcing(2)])
        if p.n < 1:
            continue
        opd = fde.assemble_problem(h, p)
        opt = fde.assemble_problem(h, p, flags=fde.OP_TOEPLITZ)
        x = torch.tensor(np.random.default_rng(N * 100 + P).standard_normal((2, p.n)), device="cuda")
        yd = fde.stiffness_matvec(h, opd, x, path=fde.PATH_DENSE).cpu().numpy()
        yt = fde.stiffness_matvec(h, opt, x, path=fde.PATH_TOEPLITZ).cpu().numpy()
        so = oracle_system(p)
        den = (np.abs(so.A) @ np.abs(x.cpu().numpy().T)).T
        assert np.max(np.abs(yt - yd) / den) <= TOL, (N, P)
        opd.free()
        opt.free()


def test_hundred_rhs_solve(fde, h):
    """100 right-hand sides (two 64-wide DMMA column tiles, the many-RHS apply) give
    the one-by-one solutions."""
    p = fi.config4(N=64, P=4)
    p.forcings = [fi.random_legendre_forcing(s) for s in range(100)]
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, 4)
    lu = fde.hlu_factor(h, hm, 1e-3)
    G = fde.sem_rhs(h, op, p.forcings)
    X, rep = fde.solve(h, op, lu, G, tol=1e-13)
    for c in (0, 63, 64, 99):
        x1, _ = fde.solve(h, op, lu, G[c:c + 1].contiguous(), tol=1e-13)
        assert np.linalg.norm(X[c].cpu().numpy() - x1[0].cpu().numpy()) <= 1e-10 * np.linalg.norm(x1[0].cpu().numpy())
    for o in (lu, hm, op):
        o.free()


def test_many_handles_lifecycle(fde):
    """Handles and objects created and released many times (streams, pools,
    communicator-free contexts): no failure, and the pool's used bytes do not grow
    with the number of lifecycles (measured against the state after the first one,
    so buffers other tests' live handles hold do not count)."""
    import ctypes
    p = fi.config1()
    fde.lib().fde_debug_pool_bytes.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong),
                                               ctypes.POINTER(ctypes.c_ulonglong)]

    def used():
        torch.cuda.synchronize()
        r, u = ctypes.c_ulonglong(0), ctypes.c_ulonglong(0)
        fde.lib().fde_debug_pool_bytes(0, ctypes.byref(r), ctypes.byref(u))
        return u.value

    u0 = None
    for it in range(40):
        hh = fde.Handle(0)
        op = fde.assemble_problem(hh, p)
        hm = fde.hmatrix_build(hh, op, p.R, p.lam, p.n_min)
        lu = fde.hlu_factor(hh, hm, 1e-3)
        G = fde.sem_rhs(hh, op, p.forcings)
        fde.solve(hh, op, lu, G, tol=1e-12)
        for o in (lu, hm, op):
            o.free()
        hh.close()
        if it == 0:
            u0 = used()
    u1 = used()
    assert u1 - u0 < (4 << 20), (u0, u1)


@pytest.mark.parametrize("lam,n_min", [(0.3, 2), (3.0, 2), (1.0, 64)], ids=["lam0.3", "lam3", "one-leaf"])
def test_admissibility_and_leaf_extremes(fde, h, lam, n_min):
    """The admissibility parameter lambda (Def. 3.1) far below and
    above 1 (few / many admissible blocks) and a leaf size covering the whole mesh
    (A~ = A: the H-LU is the dense LU): A~ against the oracle's A~, block counts,
    exact-mode H-LU against the dense solve with A~."""
    p = fi.config4(N=40, P=5)
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, 6, lam, n_min)
    so = oracle_system(p)
    At, part = O.hmatrix_dense(p, so, R=6, lam=lam, n_min=n_min)
    assert hm.info.nblocks_lr == sum(1 for _, _, k in part if k == "lr")
    assert metric_A(fde.hmatrix_dense_paper(h, hm).cpu().numpy(), At) <= TOL
    lu = fde.hlu_factor(h, hm, 0.0)
    r = np.random.default_rng(1).standard_normal((2, p.n))
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()
    zo = np.linalg.solve(At, r.T).T
    assert np.linalg.norm(z - zo) <= TOL * np.linalg.norm(zo)
    for o in (lu, hm, op):
        o.free()
