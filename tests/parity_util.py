"""Parity metrics shared by the GPU tests:

  M-A  max |dA_IJ| / sqrt(A_II A_JJ)                         <= 1e-10
  M-B  max |dy_I| / (|A| |x|)_I                               <= 1e-10
  M-D  ||X - X_ora||_D / ||X_ora||_D (D = diag A)             <= max(1e-10, 10 kappa eps)
       max |u_h - u_h^ora| / max |u_h^ora| on 50 points/elem  <= the same bar
       backward error ||G - A X|| / (||A|| ||X|| + ||G||)      <= 1e-14 (oracle's A, long double)

and the oracle's rows of A for sampled elements at full size (pair integrals of
the sampled element against every other element, in parallel threads; ctypes
releases the GIL inside the oracle's C code).  Test infrastructure only.
"""
from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np

import oracle as O

EPS = np.finfo(np.float64).eps


def metric_A(Ag, Ao):
    d = np.sqrt(np.abs(np.diag(Ao)))
    return np.max(np.abs(Ag - Ao) / (d[:, None] * d[None, :]))


def ext_index(N, P, e, a):
    """Paper order extended by [hat 0, hat N] (oracle.py convention)."""
    nm = N * (P - 1)
    if a == 0:
        return nm + N - 1 if e == 0 else nm + e - 1
    if a == P:
        return nm + N if e + 1 == N else nm + e
    return e * (P - 1) + a - 1


def oracle_rows(p, elems, threads=None):
    """Full rows of A = rho M + theta S_l + (1-theta) S_l^T (Eq. (lsys))
    for the modal dofs of the elements `elems`, paper order, (len, n), computed by
    the oracle's pair integrals: S_l[I, :] from the pairs (e, j <= e), S_l[:, I]
    from the pairs (j >= e, e), M from the oracle's mass of the one-element mesh."""
    N, P, n = p.N, p.P, p.n
    threads = threads or (os.cpu_count() or 1)
    rows, idx = [], []
    for e in elems:
        jobs = [("r", j) for j in range(0, e + 1)] + [("c", j) for j in range(e + 1, N)]

        def run(job):
            kind, j = job
            if kind == "r":
                return job, O.pair_integral(P, p.alpha, p.nodes, e, j)
            return job, O.pair_integral(P, p.alpha, p.nodes, j, e)

        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(run, jobs))
        Sr = np.zeros((P + 1, n + 2))       # S_l[I, :], local test fn a of element e
        Sc = np.zeros((P + 1, n + 2))       # S_l[:, I] as a row
        for (kind, j), blk in res:
            for b in range(P + 1):
                J = ext_index(N, P, j, b)
                if kind == "r":
                    Sr[:, J] += blk[:, b]
                    if j == e:
                        Sc[:, J] += blk[b, :]   # the self pair also feeds S_l[J, I] with J in e
                else:
                    Sc[:, J] += blk[b, :]
        Mloc = O.mass_ext(np.array([p.nodes[e], p.nodes[e + 1]]), P)   # 1-element mesh, ext order
        loc_of = lambda a: P - 1 if a == 0 else (P if a == P else a - 1)
        Mr = np.zeros((P + 1, n + 2))
        for a in range(P + 1):
            for b in range(P + 1):
                Mr[a, ext_index(N, P, e, b)] += Mloc[loc_of(a), loc_of(b)]
        Ar = p.rho * Mr + p.theta * Sr + (1 - p.theta) * Sc
        for a in range(1, P):
            rows.append(Ar[a, :n])
            idx.append(ext_index(N, P, e, a))
    return np.array(idx), np.array(rows)


def kappa_equilibrated(A):
    d = 1.0 / np.sqrt(np.abs(np.diag(A)))
    return np.linalg.cond(A * d[:, None] * d[None, :])


def md_check(p, x, so, Go, Xo=None, xis=50, berr_tol=1e-14, kappa=None):
    """Metric M-D for one right-hand side.  Returns a dict of the measured values;
    raises AssertionError if any part exceeds its bar."""
    A = so.A
    if Xo is None:
        Xo = O.solve_dense(A, Go)
    D = np.abs(np.diag(A))
    err = np.sqrt(np.sum(D * (x - Xo) ** 2) / np.sum(D * Xo ** 2))
    if kappa is None:
        kappa = kappa_equilibrated(A) if p.n <= 4096 else None
    bar = max(1e-10, 10 * kappa * EPS) if kappa is not None else 1e-10
    pts = np.linspace(-1, 1, xis)
    uh = O.eval_solution(p, x, pts)
    uo = O.eval_solution(p, Xo, pts)
    uerr = np.abs(uh - uo).max() / np.abs(uo).max()
    Al = A.astype(np.longdouble)
    r = (Go.astype(np.longdouble) - Al @ x.astype(np.longdouble)).astype(np.float64)
    berr = np.abs(r).max() / (np.abs(A).sum(axis=1).max() * np.abs(x).max() + np.abs(Go).max())
    out = dict(md=err, uh=uerr, berr=berr, kappa=kappa, bar=bar)
    assert err <= bar, out
    assert uerr <= bar, out
    assert berr <= berr_tol, out
    return out
