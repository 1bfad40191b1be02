"""Parity at the BASELINE sizes, in the launch configuration bench.py times.

* config 2 (N=256, P=8, alpha=1.5): the full dense operator against the oracle
  (metric M-A) and the Toeplitz FFT matvec against the oracle's A x (M-B).
* config 3 (geometric layers, P=16): full operator (M-A) and the solve (M-D with
  its kappa-dependent bar, reported).
* config 4 (N=1024, P=8, n=8191 -- the bench workload):
  - FULL oracle rows of sampled elements (pair integrals against every other
    element): the GPU's rows (M-A) and the GEMV's y on those rows (M-B);
  - the GEMV kernels that bench.py times (k_gemv_bulk, 1 and 4 right-hand
    sides, every ring stage and phase flip) on ALL rows against a long-double
    product of the same operator;
  - the cold solve of bench.py (assemble + rhs + hmatrix + H-LU + GMRES) to
    backward error at rounding level;
  - bitwise determinism of repeated cold solves.
* H-LU exact mode in the production leaf shape (P=8, n_min=64: 512-dof leaves
  of four 128-dof sweep tiles, R=12) against the oracle's A~ (M-C).
* config 5 (N=4096, 64 RHS): sampled oracle rows; the FFT matvec against the
  DMMA GEMM on all 64 right-hand sides.
"""
import json
import os

import numpy as np
import pytest

import fde_inputs as fi
import oracle as O
from parity_util import metric_A, md_check, oracle_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fde():
    from paper_1808_02937_b200 import fde as F
    return F


@pytest.fixture(scope="module")
def h(fde):
    return fde.Handle(0)


def _record(name, **kw):
    """Measured parity values land in gpurun_out/parity_values.jsonl (evidence)."""
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "parity_values.jsonl"), "a") as f:
        f.write(json.dumps({"test": name, **{k: (float(v) if v is not None else None) for k, v in kw.items()}}) + "\n")


def test_config2_full_operator_and_fft(fde, h):
    p = fi.config2(1.5)
    op = fde.assemble_problem(h, p, flags=fde.OP_DENSE | fde.OP_TOEPLITZ)
    Ag = fde.operator_dense_paper(h, op).cpu().numpy()
    so = O.assemble_system(p)
    mA = metric_A(Ag, so.A)
    assert mA <= 1e-10
    X = np.random.default_rng(11).standard_normal((2, p.n))
    Yf = fde.stiffness_matvec(h, op, torch.tensor(X, device="cuda"), path=fde.PATH_TOEPLITZ).cpu().numpy()
    Yo = (so.A.astype(np.longdouble) @ X.T.astype(np.longdouble)).T.astype(np.float64)
    den = (np.abs(so.A) @ np.abs(X.T)).T
    mB = np.max(np.abs(Yf - Yo) / den)
    assert mB <= 1e-10
    G = fde.sem_rhs(h, op, p.forcings)
    Go = O.rhs(p, so, p.forcings[0])
    assert np.max(np.abs(G.cpu().numpy()[0] - Go)) <= 1e-12 * np.abs(Go).max()
    _record("c2_full", MA=mA, MB_fft=mB)
    op.free()


def test_config3_full_P16_operator_and_solve(fde, h):
    p = fi.config3(16)
    op = fde.assemble_problem(h, p)
    Ag = fde.operator_dense_paper(h, op).cpu().numpy()
    so = O.assemble_system(p)
    mA = metric_A(Ag, so.A)
    assert mA <= 1e-10
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, 4)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-13)
    Go = O.rhs(p, so, p.forcings[0])
    # h_min = 1.5e-14 next to x = 0 and 1: the equilibrated kappa decides the bar
    r = md_check(p, X.cpu().numpy()[0], so, Go)
    _record("c3_P16_solve", MA=mA, **r)
    for o in (lu, hm, op):
        o.free()


C4_ELEMS = [0, 1, 2, 100, 511, 512, 700, 1021, 1022, 1023]


@pytest.fixture(scope="module")
def c4(fde, h):
    p = fi.config4()
    op = fde.assemble_problem(h, p)                       # as in bench.py
    Ag = fde.operator_dense_paper(h, op)
    idx, rows = oracle_rows(p, C4_ELEMS)
    yield p, op, Ag, idx, rows
    op.free()


def test_config4_oracle_rows_and_gemv(fde, h, c4):
    """Full rows (every column) of 10 sampled elements -- both ends, the middle,
    the mesh's smallest and largest elements -- against the oracle (M-A), and
    y = A x of the bench's GEMV on those rows against the oracle's rows (M-B)."""
    p, op, Ag, idx, rows = c4
    A = Ag[torch.tensor(idx, device="cuda")].cpu().numpy()
    d_g = np.sqrt(np.abs(np.diag(Ag.cpu().numpy())))     # (diagonal of the GPU operator: pinned by the rows)
    assert np.max(np.abs(np.diag(A[:, idx]) - np.diag(rows[:, idx])) / np.abs(np.diag(rows[:, idx]))) <= 1e-12
    mA = np.max(np.abs(A - rows) / (d_g[idx][:, None] * d_g[None, :]))
    assert mA <= 1e-10
    X = np.random.default_rng(21).standard_normal((4, p.n))
    mB = 0.0
    for nrhs in (1, 4):
        Y = fde.stiffness_matvec(h, op, torch.tensor(X[:nrhs], device="cuda"), path=fde.PATH_DENSE).cpu().numpy()
        Yo = (rows.astype(np.longdouble) @ X[:nrhs].T.astype(np.longdouble)).T.astype(np.float64)
        den = (np.abs(rows) @ np.abs(X[:nrhs].T)).T
        mB = max(mB, np.max(np.abs(Y[:, idx] - Yo) / den))
    assert mB <= 1e-10
    _record("c4_oracle_rows", MA=mA, MB=mB, rows=len(idx))


@pytest.mark.parametrize("nrhs", [1, 2, 3, 4, 5])
def test_config4_gemv_all_rows_long_double(fde, h, c4, nrhs):
    """The bulk-copy GEMV (NR = 1: 1024-column slabs; NR = 2..4: 512-column
    slabs; nrhs = 5 = a 4-pass plus a 1-pass) on all 8191 rows -- 71 CTAs' worth
    of row blocks per SM slot, every stage of the 3-stage ring and its phase
    flips -- against the long-double product of the same operator (M-B)."""
    p, op, Ag, idx, rows = c4
    A = Ag.cpu().numpy()
    X = np.random.default_rng(100 + nrhs).standard_normal((nrhs, p.n))
    Y = fde.stiffness_matvec(h, op, torch.tensor(X, device="cuda"), path=fde.PATH_DENSE).cpu().numpy()
    Yo = (A.astype(np.longdouble) @ X.T.astype(np.longdouble)).T.astype(np.float64)
    den = (np.abs(A) @ np.abs(X.T)).T
    mB = np.max(np.abs(Y - Yo) / den)
    assert mB <= 1e-10
    _record(f"c4_gemv_all_rows_nrhs{nrhs}", MB=mB)


def test_config4_cold_solve_backward_error(fde, h, c4):
    p, op, Ag, idx, rows = c4
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12, restart=50, maxiter=500)
    AX = fde.stiffness_matvec(h, op, X).cpu().numpy()[0]
    g, x = G.cpu().numpy()[0], X.cpu().numpy()[0]
    A = Ag.cpu().numpy()
    r = (g.astype(np.longdouble) - A.astype(np.longdouble) @ x.astype(np.longdouble)).astype(np.float64)
    berr = np.abs(r).max() / (np.abs(A).sum(axis=1).max() * np.abs(x).max() + np.abs(g).max())
    assert berr <= 1e-14, berr
    assert rep.iterations <= 4, rep.iterations
    # preconditioner quality: ||A~ z - r|| / ||r|| with z = (L_H U_H)^{-1} r
    At = fde.hmatrix_dense_paper(h, hm)
    rr = torch.tensor(np.random.default_rng(6).standard_normal(p.n), device="cuda")
    z = fde.precond_apply(h, lu, rr)[0]
    q = (torch.linalg.norm(At @ z - rr) / torch.linalg.norm(rr)).item()
    assert q <= 1e-5, q
    _record("c4_cold_solve", berr=berr, iters=rep.iterations, precond_resid=q)
    del At
    for o in (lu, hm):
        o.free()


@pytest.mark.parametrize("hold", [None, "200"], ids=["free-running", "host-held"])
def test_config4_cold_solves_bitwise_deterministic(fde, h, hold, monkeypatch):
    """Ten cold solves of the bench workload give the same X bit for bit, with
    the host running ahead of the device and with the device held until the
    whole H-LU is enqueued (FDE_H2_HOLD_US): the seven-stream H-LU, the deferred
    updates and the plan/flatten overlap must not change the arithmetic (the
    row-sharded job relies on identical replicas)."""
    if hold:
        monkeypatch.setenv("FDE_H2_HOLD_US", hold)
    p = fi.config4()
    ref = None
    for k in range(10):
        op = fde.assemble_problem(h, p)
        G = fde.sem_rhs(h, op, p.forcings)
        hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
        lu = fde.hlu_factor(h, hm, 1e-3)
        X, rep = fde.solve(h, op, lu, G, tol=1e-12)
        if ref is None:
            ref = X.clone()
        else:
            assert torch.equal(X, ref), f"solve {k} differs"
        for o in (lu, hm, op):
            o.free()


def test_hlu_exact_mode_production_leaf_shape(fde, h):
    """tol = 0 with the bench's partition parameters (P = 8, n_min = 64 -> 512-dof
    leaves, each four 128-dof sweep tiles; R = 12) on the mirrored graded mesh
    at N = 256: precond_apply equals the dense solve with the oracle's A~ (M-C)."""
    p = fi.config4(N=256, P=8)
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 0.0)
    so = O.assemble_system(p)
    At, part = O.hmatrix_dense(p, so, R=p.R, lam=p.lam, n_min=p.n_min)
    assert any(k == "lr" for _, _, k in part)
    mA = metric_A(fde.hmatrix_dense_paper(h, hm).cpu().numpy(), At)
    assert mA <= 1e-10
    r = np.random.default_rng(5).standard_normal((3, p.n))
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()
    zo = np.linalg.solve(At, r.T).T
    err = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert err <= 1e-10, err
    _record("hlu_exact_production_shape", MA=mA, MC=err)
    for o in (lu, hm, op):
        o.free()


def test_config5_sampled_rows_and_fft_vs_dmma(fde, h):
    """Config 5 (uniform N = 4096, P = 8, n = 32767, 64 RHS): full oracle rows of
    three sampled elements (M-A, M-B of the 64-RHS DMMA GEMM on them); the FFT
    matvec against the DMMA GEMM on all rows and all 64 right-hand sides (M-B
    against |A||x|, both paths of the same operator)."""
    p = fi.config5()
    op = fde.assemble_problem(h, p, flags=fde.OP_DENSE | fde.OP_TOEPLITZ)
    X = torch.tensor(np.random.default_rng(64).standard_normal((64, p.n)), device="cuda")
    Yd = fde.stiffness_matvec(h, op, X, path=fde.PATH_DENSE)
    Yf = fde.stiffness_matvec(h, op, X, path=fde.PATH_TOEPLITZ)
    Ag = fde.operator_dense_paper(h, op)
    den = torch.abs(Ag) @ torch.abs(X.T)
    mB_cross = (torch.abs(Yf - Yd).T / den).max().item()
    assert mB_cross <= 1e-10
    elems = [0, 2047, 4095]
    idx, rows = oracle_rows(p, elems)
    A = Ag[torch.tensor(idx, device="cuda")].cpu().numpy()
    d = np.sqrt(np.abs(torch.diagonal(Ag).cpu().numpy()))
    mA = np.max(np.abs(A - rows) / (d[idx][:, None] * d[None, :]))
    assert mA <= 1e-10
    Xn = X.cpu().numpy()
    Yo = (rows.astype(np.longdouble) @ Xn.T.astype(np.longdouble)).astype(np.float64)   # (rows, 64)
    denr = np.abs(rows) @ np.abs(Xn.T)
    mB = np.max(np.abs(Yd.cpu().numpy()[:, idx].T - Yo) / denr)
    assert mB <= 1e-10
    _record("c5_rows_fft_dmma", MA=mA, MB_dmma=mB, MB_fft_vs_dmma=mB_cross)
    del Ag, den
    op.free()


def test_hlu_launch_variants(fde, h, monkeypatch):
    """The H-LU sweep's launch-level options: programmatic dependent
    launches and the operand snapshots on their own stream change only WHEN kernels
    run, so the preconditioner is bitwise the default one with them off; the fused
    16 x 16 cores (formed in-CTA by the product tiles, a different summation order)
    give another tol = 1e-3 preconditioner, and every variant's solve reaches the
    oracle's X (M-D).  Mirrored graded mesh N = 256, P = 8: 16 sweep tiles, so the
    fused cores are on by default."""
    p = fi.config4(N=256, P=8)
    op = fde.assemble_problem(h, p)
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    so = O.assemble_system(p)
    Go = O.rhs(p, so, p.forcings[0])
    Xo = O.solve_dense(so.A, Go).reshape(-1)
    r = torch.tensor(np.random.default_rng(11).standard_normal((2, p.n)), device="cuda")
    zs = {}
    for name, env in [("default", {}), ("no-pdl", {"FDE_H2_PDL": "0"}), ("late-snap", {"FDE_H2_SNAP_EARLY": "0"}),
                      ("no-fuse", {"FDE_H2_FUSECORE": "0"})]:
        for k in ("FDE_H2_PDL", "FDE_H2_SNAP_EARLY", "FDE_H2_FUSECORE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        lu = fde.hlu_factor(h, hm, 1e-3)
        zs[name] = fde.precond_apply(h, lu, r).clone()
        X, rep = fde.solve(h, op, lu, G, tol=1e-12)
        md_check(p, X.cpu().numpy()[0], so, Go, Xo=Xo)
        lu.free()
    assert torch.equal(zs["no-pdl"], zs["default"])
    assert torch.equal(zs["late-snap"], zs["default"])
    q = (torch.linalg.norm(zs["no-fuse"] - zs["default"]) / torch.linalg.norm(zs["default"])).item()
    assert q <= 1e-3, q
    for o in (hm, op):
        o.free()
