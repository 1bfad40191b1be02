"""The paper's own H-matrix partition (Fig. fig200): separate
cluster trees for the modal functions and the nodal hats, the first block level
being S_l = [B F; E C] -- `hmatrix_build_partition(...,
FDE_PARTITION_PAPER)` against the oracle's `hmatrix_dense(partition="paper")`:
A~ entry by entry (M-A), the exact-mode leaf-ordered H-LU (M-C), the
preconditioned solve (M-D), and the Table 1 iteration pattern.
"""
import json
import os

import numpy as np
import pytest

import fde_inputs as fi
import oracle as O
from parity_util import md_check, metric_A

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


_SYS = {}


def system(p):
    key = (p.name, p.theta, p.rho, p.N)
    if key not in _SYS:
        _SYS[key] = O.assemble_system(p)
    return _SYS[key]


CASES = [(fi.config1(), 2), (fi.config4(N=64, P=4), 4), (fi.config2(1.5, N=48, P=4), 4),
         (fi.example51(N=300, P=3, R=5), 16), (fi.config4(N=96, P=8), 4)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0].name}-nmin{c[1]}")
def test_paper_partition_Atilde_matches_oracle(fde, h, case):
    p, n_min = case
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min, partition=fde.PARTITION_PAPER)
    Ag = fde.hmatrix_dense_paper(h, hm).cpu().numpy()
    so = system(p)
    At, part = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min, partition="paper")
    assert hm.info.nblocks_lr == sum(1 for _, _, k in part if k == "lr")
    assert hm.info.nblocks_dense == sum(1 for _, _, k in part if k == "dense")
    assert metric_A(Ag, At) <= 1e-10
    hm.free()
    op.free()


@pytest.mark.parametrize("case", CASES[1:], ids=lambda c: f"{c[0].name}-nmin{c[1]}")
def test_paper_partition_hlu_exact_mode(fde, h, case):
    """tol = 0: the (leaf-ordered) H-LU on the paper's partition is the exact LU of
    its A~, so precond_apply equals np.linalg.solve with the oracle's A~ (M-C).
    The recursive fallback refuses the paper partition (FDE_EINVAL_PARAM)."""
    p, n_min = case
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min, partition=fde.PARTITION_PAPER)
    lu = fde.hlu_factor(h, hm, 0.0)
    so = system(p)
    At, _ = O.hmatrix_dense(p, so, R=p.R, lam=1.0, n_min=n_min, partition="paper")
    r = np.random.default_rng(17).standard_normal((3, p.n))
    z = fde.precond_apply(h, lu, torch.tensor(r, device="cuda")).cpu().numpy()
    zo = np.linalg.solve(At, r.T).T
    err = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert err <= 1e-10, err
    fde.set_hlu_mode(1)
    try:
        with pytest.raises(fde.FdeError) as e:
            fde.hlu_factor(h, hm, 0.0)
        assert e.value.name == "FDE_EINVAL_PARAM"
    finally:
        fde.set_hlu_mode(0)
    for o in (lu, hm, op):
        o.free()


@pytest.mark.parametrize("case", CASES[1:], ids=lambda c: f"{c[0].name}-nmin{c[1]}")
def test_paper_partition_preconditioned_solve(fde, h, case):
    p, n_min = case
    op = fde.assemble_problem(h, p)
    hm = fde.hmatrix_build(h, op, p.R, 1.0, n_min, partition=fde.PARTITION_PAPER)
    lu = fde.hlu_factor(h, hm, 1e-3)
    G = fde.sem_rhs(h, op, p.forcings)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12)
    so = system(p)
    md_check(p, X.cpu().numpy()[0], so, O.rhs(p, so, p.forcings[0]))
    assert rep.iterations <= 8
    for o in (lu, hm, op):
        o.free()


def test_paper_partition_rejects_sharded_or_fft_operator(fde, h):
    p = fi.config2(1.5, N=32, P=4)
    op = fde.assemble_problem(h, p, flags=fde.OP_TOEPLITZ)
    with pytest.raises(fde.FdeError) as e:
        fde.hmatrix_build(h, op, p.R, 1.0, 4, partition=fde.PARTITION_PAPER)
    assert e.value.name == "FDE_EINVAL_PARAM"
    op.free()


def test_table1_pattern_paper_partition(fde, h):
    """Table 1 on the paper's partition, Example 5.1 at N = 400,
    P = 3, n_min = 16: BiCGSTAB operator applications non-increasing in R, fewer
    at R = 7 than at R = 2 (paper: 10, 8, 4, 4), every solve at the oracle's X."""
    apps = {}
    p0 = fi.example51(N=400, P=3, R=2)
    so = system(p0)
    Go = O.rhs(p0, so, p0.forcings[0])
    for R in (2, 3, 5, 7):
        p = fi.example51(N=400, P=3, R=R)
        op = fde.assemble_problem(h, p)
        G = fde.sem_rhs(h, op, p.forcings)
        hm = fde.hmatrix_build(h, op, R, 1.0, p.n_min, partition=fde.PARTITION_PAPER)
        lu = fde.hlu_factor(h, hm, 1e-3)
        X, rep = fde.solve(h, op, lu, G, method=fde.BICGSTAB, tol=1e-13, maxiter=400)
        apps[R] = rep.matvecs
        md_check(p, X.cpu().numpy()[0], so, Go, berr_tol=1e-13)
        for o in (lu, hm, op):
            o.free()
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "parity_values.jsonl"), "a") as f:
        f.write(json.dumps({"test": "table1_paper_partition_N400", "applications": apps}) + "\n")
    Rs = sorted(apps)
    assert all(apps[Rs[k + 1]] <= apps[Rs[k]] for k in range(len(Rs) - 1)), apps
    assert apps[7] < apps[2], apps
