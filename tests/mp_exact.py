"""Exact (multi-precision) pair integrals for pinning the oracle.

A method independent of any quadrature: for polynomial test/trial derivatives
p(t), q(s) the double integral
    I = gamma0 int_{t0}^{t1} p(t) int_{s0}^{s1} q(s) (t-s)_+^{1-alpha} ds dt
is a finite sum of corner terms of the iterated antiderivatives
    F_m(z) = z_+^{1-alpha+m} / prod_{l=1..m} (1-alpha+l),   F_m' = F_{m-1},
by repeated integration by parts in s and then in t:
    I = gamma0 sum_{k,l} (-1)^l { q^(k)(s0) [p^(l) F_{k+l+2}(t-s0)]_{t0}^{t1}
                                 - q^(k)(s1) [p^(l) F_{k+l+2}(t-s1)]_{t0}^{t1} }.
Evaluated with mpmath at `dps` digits the corner cancellation is harmless for
the small meshes used in the pins.  The basis polynomials are built from the
Legendre recurrence with exact rational arithmetic.
"""
from fractions import Fraction

import mpmath as mp


def legendre_power(n):
    """Power-basis coefficients (Fractions) of L_0..L_n."""
    L = [[Fraction(1)], [Fraction(0), Fraction(1)]]
    for k in range(1, n):
        a = [Fraction(0)] + [c * Fraction(2 * k + 1, k + 1) for c in L[k]]
        b = [c * Fraction(k, k + 1) for c in L[k - 1]] + [Fraction(0)] * 2
        L.append([a[i] - b[i] for i in range(k + 2)])
    return L[: n + 1]


def deriv(c):
    return [c[i] * i for i in range(1, len(c))] or [Fraction(0)]


def local_deriv_ref(P):
    """d/dxi of the local functions [left hat, psi_1..psi_{P-1}, right hat] (power basis in xi)."""
    L = legendre_power(P + 1)
    out = [[Fraction(-1, 2)]]
    for p in range(1, P):
        a, b = L[p - 1], L[p + 1]
        psi = [(a[i] if i < len(a) else 0) - (b[i] if i < len(b) else 0) for i in range(len(b))]
        out.append(deriv(psi))
    out.append([Fraction(1, 2)])
    return out


def polyval(c, x):
    s = mp.mpf(0)
    for ci in reversed(c):
        s = s * x + mp.mpf(ci.numerator) / ci.denominator
    return s


def pair_exact(P, alpha, d, hi, hj, self_pair=False, dps=60):
    """(P+1)x(P+1) pair integral; geometry as in oracle.pair_integral.

    Off-diagonal (trial element j left of test element i): d = x_i - x_{j+1} >= 0.
    Self pair: test = trial element of size hi."""
    with mp.workdps(dps):
        a = mp.mpf(alpha)
        g0 = 1 / mp.gamma(2 - a)
        hi_, hj_ = mp.mpf(hi), mp.mpf(hj)
        d_ = mp.mpf(d)
        if self_pair:
            t0, t1, s0, s1 = mp.mpf(0), hi_, mp.mpf(0), hi_
        else:
            # coordinates relative to x_{j+1}: s in [-hj, 0], t in [d, d+hi]
            t0, t1, s0, s1 = d_, d_ + hi_, -hj_, mp.mpf(0)
        hs = hi_ if self_pair else hj_

        def F(m, z):
            if z <= 0:
                return mp.mpf(0)
            den = mp.mpf(1)
            for l in range(1, m + 1):
                den *= (1 - a + l)
            return z ** (1 - a + m) / den

        D = local_deriv_ref(P)
        maxdeg = P + 1
        # derivative tables: physical d^l/dt^l of (2/h) * (d/dxi local fn)
        def derivs(c, h):
            out, cur = [], list(c)
            for l in range(maxdeg + 1):
                out.append((cur, (2 / h) ** (l + 1)))
                cur = deriv(cur)
            return out

        M = P + 1
        res = [[mp.mpf(0)] * M for _ in range(M)]
        for ia in range(M):
            pd = derivs(D[ia], hi_)
            for ib in range(M):
                qd = derivs(D[ib], hs)
                tot = mp.mpf(0)
                for k, (qc, qs) in enumerate(qd):
                    q_s0 = qs * polyval(qc, -1)
                    q_s1 = qs * polyval(qc, 1)
                    if q_s0 == 0 and q_s1 == 0:
                        continue
                    for l, (pc, ps) in enumerate(pd):
                        p_t0 = ps * polyval(pc, -1)
                        p_t1 = ps * polyval(pc, 1)
                        if p_t0 == 0 and p_t1 == 0:
                            continue
                        m = k + l + 2
                        term = q_s0 * (p_t1 * F(m, t1 - s0) - p_t0 * F(m, t0 - s0)) \
                            - q_s1 * (p_t1 * F(m, t1 - s1) - p_t0 * F(m, t0 - s1))
                        tot += (-1) ** l * term
                res[ia][ib] = g0 * tot
        return [[float(v) for v in row] for row in res]
