"""The preconditioned solve on the block-Toeplitz FFT matvec alone (config 2,
PAPER.md:632-735, 914-919): the operator is assembled with FDE_OP_TOEPLITZ only
(no dense matrix anywhere), so hmatrix_build recomputes the inadmissible
leaves from pair moments and every Krylov matvec is the O(P N log N + P^2 N)
FFT product.  The solve must reach the oracle's direct solution (metric M-D,
1e-10) for all three alphas of config 2, at full size.
"""
import numpy as np
import pytest

import fde_inputs as fi
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def md_error(x, Xo, A):
    D = np.abs(np.diag(A))
    return np.sqrt(np.sum(D * (x - Xo) ** 2) / np.sum(D * Xo ** 2))


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.8])
def test_config2_toeplitz_only_preconditioned_solve(fde, h, alpha):
    p = fi.config2(alpha)                                    # N = 256, P = 8, n = 2047
    op = fde.assemble_problem(h, p, flags=fde.OP_TOEPLITZ)   # no dense operator
    assert op.info.flags == fde.OP_TOEPLITZ
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)       # near field: recompute path
    lu = fde.hlu_factor(h, hm, 1e-3)
    X, rep = fde.solve(h, op, lu, G, tol=1e-12, path=fde.PATH_TOEPLITZ)
    with pytest.raises(fde.FdeError):                         # no dense form to fall back on
        fde.stiffness_matvec(h, op, G, path=fde.PATH_DENSE)
    so = O.assemble_system(p)
    Go = O.rhs(p, so, p.forcings[0])
    assert np.max(np.abs(G.cpu().numpy()[0] - Go)) <= 1e-12 * np.abs(Go).max()
    Xo = O.solve_dense(so.A, Go)
    x = X.cpu().numpy()[0]
    err = md_error(x, Xo, so.A)
    assert err <= 1e-10, (err, rep.iterations)
    assert rep.iterations <= 6, rep.iterations
    # the recomputed near field equals the dense-path (copied) one
    opd = fde.assemble_problem(h, p, flags=fde.OP_DENSE)
    hmd = fde.hmatrix_build(h, opd, p.R, p.lam, p.n_min)
    At = fde.hmatrix_dense_paper(h, hm).cpu().numpy()
    Atd = fde.hmatrix_dense_paper(h, hmd).cpu().numpy()
    assert metric_A(At, Atd) <= 1e-14
    # and the oracle's A~
    Ato, _ = O.hmatrix_dense(p, so, R=p.R, lam=p.lam, n_min=p.n_min)
    assert metric_A(At, Ato) <= 1e-10
    for o in (hmd, opd, lu, hm, op):
        o.free()


def test_toeplitz_and_dense_solves_agree_on_uniform_c5_mesh(fde, h):
    """Fig. fig7's comparison on the config-5 mesh (uniform,
    N = 4096, P = 8, n = 32767) with 4 of its right-hand sides: the FFT-matvec
    solve and the dense-matvec solve (DMMA/GEMV) reach the same X (both are
    solves of the same A to 1e-12; D-norm difference <= 1e-10)."""
    p = fi.config5(nrhs=4)
    op = fde.assemble_problem(h, p, flags=fde.OP_DENSE | fde.OP_TOEPLITZ)
    G = fde.sem_rhs(h, op, p.forcings)
    hm = fde.hmatrix_build(h, op, p.R, p.lam, p.n_min)
    lu = fde.hlu_factor(h, hm, 1e-3)
    Xf, rf = fde.solve(h, op, lu, G, tol=1e-12, path=fde.PATH_TOEPLITZ)
    Xd, rd = fde.solve(h, op, lu, G, tol=1e-12, path=fde.PATH_DENSE)
    A = fde.operator_dense_paper(h, op)
    D = torch.abs(torch.diagonal(A))
    for c in range(4):
        e = torch.sqrt(torch.sum(D * (Xf[c] - Xd[c]) ** 2) / torch.sum(D * Xd[c] ** 2)).item()
        assert e <= 1e-10, (c, e)
    # backward error of the FFT solve against the dense operator
    R = G - (A @ Xf.T).T
    berr = (torch.abs(R).max() / (torch.abs(A).sum(1).max() * torch.abs(Xf).max() + torch.abs(G).max())).item()
    assert berr <= 1e-14, berr
    del A
    for o in (lu, hm, op):
        o.free()
