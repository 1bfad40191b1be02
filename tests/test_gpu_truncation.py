"""The H-LU's formatted truncation (H-LU "with a prescribed
tolerance Tol_HLU", Boerm's truncation of a low-rank sum U V^T to the singular
values sigma_i > tol * sigma_1) through `fde_debug_truncate`, which runs the
batched path of the factorisation (k_bgram -> k_bcore -> k_bapply).

Pinned to the mathematics, not to an oracle routine (the oracle has no tol > 0
H-LU): with sigma = svd(U V^T) (numpy, fp64) and r = #{sigma_i > tol sigma_1},
  * the kept rank is r (spectra keep a clear gap around the threshold), capped
    at kc with the overflow flag raised;
  * Uo Vo^T is the best rank-r approximation (Eckart-Young: ||U V^T - Uo Vo^T||_2
    equals sigma_{r+1}, and Uo Vo^T equals the truncated SVD, up to the Gram
    method's accuracy ~1e-8 sigma_1);
  * columns >= r of Uo, Vo are exactly zero.
Widths 1..16 take the one-warp core (nonzero width <= 16), 17..64 the CTA core;
unused capacity (zero columns), dependent columns (the pivoted Cholesky stops
early), equal singular values (Jacobi ties), all-zero sums and ragged row
chunks (m, n not multiples of 64) are covered.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fde():
    from paper_1808_02937_b200 import fde as F
    return F


@pytest.fixture(scope="module")
def h(fde):
    return fde.Handle(0)


def make_sum(rng, m, n, k, sig, zero_cols=0, dup_cols=0):
    """U (m x k), V (n x k) with U V^T = X diag(sig) Y^T, mixed by a random G (so U
    and V are not orthogonal), plus zero columns (unused capacity) and duplicated
    U columns (a dependent Gram)."""
    r0 = len(sig)
    X = np.linalg.qr(rng.standard_normal((m, max(r0, 1))))[0][:, :r0]
    Y = np.linalg.qr(rng.standard_normal((n, max(r0, 1))))[0][:, :r0]
    G = rng.standard_normal((r0, r0)) + 3 * np.eye(r0)
    U = X @ np.diag(sig) @ G
    V = Y @ np.linalg.inv(G).T
    cols_u = [U[:, i] for i in range(r0)]
    cols_v = [V[:, i] for i in range(r0)]
    for d in range(dup_cols):                    # u_d = u_0 again, with its own v
        cols_u.append(cols_u[0] * (1.0 + d))
        cols_v.append(rng.standard_normal(n) * sig[0] * 1e-2)
    for _ in range(zero_cols):
        cols_u.append(np.zeros(m))
        cols_v.append(np.zeros(n))
    order = rng.permutation(len(cols_u))
    Uk = np.stack([cols_u[i] for i in order], axis=1)
    Vk = np.stack([cols_v[i] for i in order], axis=1)
    assert Uk.shape[1] == k, (Uk.shape, k)
    return Uk, Vk


def check(fde, h, sums, tol, kc):
    U = torch.tensor(np.stack([u.T for u, _ in sums]), device="cuda")
    V = torch.tensor(np.stack([v.T for _, v in sums]), device="cuda")
    Uo, Vo, ov = fde.truncate(h, U, V, tol, kc)
    Uo = Uo.cpu().numpy()
    Vo = Vo.cpu().numpy()
    any_over = False
    for q, (u, v) in enumerate(sums):
        P = u @ v.T
        s = np.linalg.svd(P, compute_uv=False)
        s1 = s[0] if s.size else 0.0
        r = int(np.sum(s > tol * s1)) if s1 > 0 else 0
        over = r > kc
        any_over |= over
        r = min(r, kc)
        nz = [c for c in range(kc) if np.any(Uo[q, c]) or np.any(Vo[q, c])]
        assert nz == list(range(r)), (q, nz, r, s[:r + 2] / max(s1, 1e-300))
        Q = Uo[q].T @ Vo[q]
        if s1 == 0.0:
            assert not np.any(Q)
            continue
        err = np.linalg.norm(P - Q, 2)
        nxt = s[r] if r < s.size else 0.0
        assert abs(err - nxt) <= 1e-6 * s1, (q, err, nxt, s1)
        Xs, ss, Yst = np.linalg.svd(P)
        best = (Xs[:, :r] * ss[:r]) @ Yst[:r]
        assert np.linalg.norm(Q - best, 2) <= 1e-6 * s1, (q, np.linalg.norm(Q - best, 2) / s1)
    assert ov == any_over


def spectrum(rng, nsig, decades):
    """nsig singular values spanning `decades` decades below 1, none within 10^0.3
    of the tol = 1e-3 threshold (the rank decision is then unambiguous)."""
    sig = 10.0 ** -np.sort(rng.uniform(0, decades, nsig))
    sig = sig[np.abs(np.log10(sig / sig.max()) + 3) > 0.3]
    return sig if sig.size else np.array([1.0])


@pytest.mark.parametrize("k", [1, 2, 5, 8, 9, 12, 16])
def test_truncation_warp_core(fde, h, k):
    """One batch per (m, n) shape, three sums each (batched entries)."""
    rng = np.random.default_rng(100 + k)
    for (m, n) in [(200, 77), (64, 64), (20, 130), (513, 65)]:
        sums = []
        for _ in range(3):
            zero = k // 3
            sig = spectrum(rng, max(1, k - zero - (1 if k >= 4 else 0)), 6)
            dup = k - sig.size - zero
            sums.append(make_sum(rng, m, n, k, sig * rng.uniform(0.5, 20), zero, dup))
        check(fde, h, sums, 1e-3, 16)


@pytest.mark.parametrize("k", [17, 24, 40, 64])
def test_truncation_cta_core(fde, h, k):
    rng = np.random.default_rng(200 + k)
    for (m, n) in [(300, 257), (128, 96)]:
        sums = []
        for _ in range(2):
            sig = spectrum(rng, k - 4, 8)
            sums.append(make_sum(rng, m, n, k, sig, k - sig.size, 0))
        check(fde, h, sums, 1e-3, 64)


def test_truncation_ties_zero_overflow(fde, h):
    rng = np.random.default_rng(7)
    # equal sigmas (Jacobi ties) beside an all-zero sum
    check(fde, h, [make_sum(rng, 150, 90, 8, np.array([1.0, 1.0, 1.0, 0.5, 0.5]), 3, 0),
                   (np.zeros((150, 8)), np.zeros((90, 8)))], 1e-3, 10)
    # more than kc = 10 kept: overflow flag, the best rank-10 approximation
    check(fde, h, [make_sum(rng, 90, 90, 12, np.linspace(2.0, 1.0, 12), 0, 0)], 1e-3, 10)
    check(fde, h, [make_sum(rng, 65, 129, 16, 10.0 ** -np.linspace(0, 2, 16), 0, 0)], 1e-3, 10)


@pytest.mark.parametrize("tol", [1e-6, 1e-2])
def test_truncation_other_tolerances(fde, h, tol):
    rng = np.random.default_rng(int(-np.log10(tol)))
    for k in (4, 10, 15):
        sig = np.array([1.0, 0.3, 3e-2, 3e-3, 3e-4, 3e-5, 3e-7, 1e-7])[:max(1, k - 3)]
        check(fde, h, [make_sum(rng, 180, 100, k, sig, k - sig.size, 0) for _ in range(2)], tol, 16)
