/*
 * fde_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this code.  It shares nothing with the CUDA path (paper_1808_02937_b200/):
 * its own quadrature-table generators, its own basis code, its own integration
 * rules.  Plain and slow on purpose.
 *
 * What it computes (Eq. (lsys), reading A1 of DESIGN.md):
 *   S_l[I,J] = gamma0 * int int_{s<t} phi_I'(t) (t-s)^{1-alpha} phi_J'(s) ds dt,
 *   gamma0 = 1/Gamma(2-alpha),
 * for the nodal hats phi_j and the modal functions
 * phi_i^p = psi_p(xi_i(x)), psi_p = L_{p-1} - L_{p+1} (Eq. (RefBasis)/(LocalBasis),
 * PAPER.md:133-143), plus the mass matrix M_IJ = (phi_J, phi_I) and the load
 * vector (f, phi_I).
 *
 * Integration (per element pair, in physical offsets so that no kernel
 * argument suffers cancellation -- SURVEY.md §7 hard part 2):
 *   - same element:   t-s = (t-x_i) - (s-x_i); nested Gauss-Jacobi in long double
 *                     (inner weight y^{1-alpha}, outer weight u^{2-alpha}); exact
 *                     for the polynomial basis.
 *   - element j < i:  t-s = d + u + v with d = x_i - x_{j+1} >= 0, u = t - x_i,
 *                     v = x_{j+1} - s.  Adaptive 2-D subdivision: a cell is
 *                     integrated by a tensor Gauss-Legendre rule (checked against
 *                     a second, larger rule) once its distance to the singular
 *                     point (u,v)=(-d,-d..) exceeds its size; the corner cell of a
 *                     touching pair (d=0) is dropped once its a-priori bound is
 *                     below 1e-19 of the pair scale.
 * Every table (Gauss-Legendre by Newton on the recurrence, Gauss-Jacobi by
 * sign-change bracketing + bisection + Newton on P_n^{(a,b)}) is computed here in long double.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

typedef long double ld;

#define MAXQ 64
#define MAXP 40

/* ---------------------------------------------------------------- Legendre */
/* L_n(x) and L_n'(x) from the three-term recurrence of PAPER.md:128 and its
 * term-by-term derivative  L'_{k+1} = ((2k+1)(L_k + x L'_k) - k L'_{k-1})/(k+1). */
static void legendre_ld(int n, ld x, ld *val, ld *der)
{
    ld p0 = 1.0L, p1 = x, d0 = 0.0L, d1 = 1.0L;
    if (n == 0) { *val = 1.0L; *der = 0.0L; return; }
    for (int k = 1; k < n; ++k) {
        ld p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
        ld d2 = ((2 * k + 1) * (p1 + x * d1) - k * d0) / (k + 1);
        p0 = p1; p1 = p2; d0 = d1; d1 = d2;
    }
    *val = p1; *der = d1;
}

/* all L_0..L_n and derivatives at x */
static void legendre_all(int n, ld x, ld *L, ld *dL)
{
    L[0] = 1.0L; dL[0] = 0.0L;
    if (n >= 1) { L[1] = x; dL[1] = 1.0L; }
    for (int k = 1; k < n; ++k) {
        L[k + 1] = ((2 * k + 1) * x * L[k] - k * L[k - 1]) / (k + 1);
        dL[k + 1] = ((2 * k + 1) * (L[k] + x * dL[k]) - k * dL[k - 1]) / (k + 1);
    }
}

/* ------------------------------------------------------ Gauss-Legendre rule */
int orc_gauss_legendre(int n, ld *x, ld *w)
{
    if (n < 1 || n > MAXQ) return -1;
    const ld pi = 3.141592653589793238462643383279502884L;
    for (int i = 0; i < n; ++i) {
        ld z = cosl(pi * (i + 0.75L) / (n + 0.5L)), v, d;
        for (int it = 0; it < 100; ++it) {
            legendre_ld(n, z, &v, &d);
            ld dz = v / d;
            z -= dz;
            if (fabsl(dz) < 1e-21L) break;
        }
        legendre_ld(n, z, &v, &d);
        x[n - 1 - i] = z;
        w[n - 1 - i] = 2.0L / ((1.0L - z * z) * d * d);
    }
    return 0;
}

/* ---------------------------------------- Gauss-Jacobi (1-x)^a (1+x)^b rule */
/* Jacobi polynomial P_n^{(a,b)} and derivative (standard three-term recurrence). */
static void jacobi_ld(int n, ld a, ld b, ld x, ld *val, ld *der)
{
    ld p0 = 1.0L, p1 = 0.5L * (a - b + (a + b + 2) * x);
    if (n == 0) { *val = 1.0L; *der = 0.0L; return; }
    for (int k = 2; k <= n; ++k) {
        ld c = 2 * k + a + b;
        ld a1 = 2 * k * (k + a + b) * (c - 2);
        ld a2 = (c - 1) * (a * a - b * b);
        ld a3 = (c - 2) * (c - 1) * c;
        ld a4 = 2 * (k + a - 1) * (k + b - 1) * c;
        ld p2 = ((a2 + a3 * x) * p1 - a4 * p0) / a1;
        p0 = p1; p1 = p2;
    }
    /* derivative: d/dx P_n^{(a,b)} = (n+a+b+1)/2 P_{n-1}^{(a+1,b+1)} */
    if (n >= 1) {
        ld q0 = 1.0L, q1 = 0.5L * ((a + 1) - (b + 1) + ((a + 1) + (b + 1) + 2) * x), qa = a + 1, qb = b + 1;
        ld q = (n - 1 == 0) ? q0 : q1;
        for (int k = 2; k <= n - 1; ++k) {
            ld c = 2 * k + qa + qb;
            ld a1 = 2 * k * (k + qa + qb) * (c - 2);
            ld a2 = (c - 1) * (qa * qa - qb * qb);
            ld a3 = (c - 2) * (c - 1) * c;
            ld a4 = 2 * (k + qa - 1) * (k + qb - 1) * c;
            ld q2 = ((a2 + a3 * x) * q1 - a4 * q0) / a1;
            q0 = q1; q1 = q2; q = q2;
        }
        *der = 0.5L * (n + a + b + 1) * q;
    } else *der = 0.0L;
    *val = p1;
}

/* Gauss-Jacobi rule from the polynomial itself: the nodes are the n simple zeros
 * of P_n^{(a,b)} in (-1,1).  They are bracketed by sign changes of P_n on a
 * Chebyshev-spaced grid of 256 n + 1 points (dense near +-1, where the zeros
 * crowd like O(1/n^2)), each bracket is narrowed by bisection and polished by
 * Newton steps.  Weights from the closed form (Szego, Orthogonal Polynomials,
 * Thm. 15.3.1 / Abramowitz-Stegun 25.4.33, second form):
 *   w_i = 2^{a+b+1} Gamma(n+a+1) Gamma(n+b+1) / (Gamma(n+a+b+1) n!)
 *         / ((1 - x_i^2) P_n'(x_i)^2).
 * Pinned by tests/test_oracle_pins.py::test_gauss_jacobi_exact_on_moments
 * (exactness on (1+x)^k, k <= 2n-1). */
int orc_gauss_jacobi(int n, ld a, ld b, ld *x, ld *w)
{
    if (n < 1 || n > MAXQ) return -1;
    const ld pi = 3.141592653589793238462643383279502884L;
    const int M = 256 * n;
    int found = 0;
    ld xl = -1.0L, vl, dv;
    jacobi_ld(n, a, b, xl, &vl, &dv);
    for (int k = M - 1; k >= 0 && found < n; --k) {
        ld xr = cosl(pi * k / M), vr;           /* ascending from -1 to +1 */
        jacobi_ld(n, a, b, xr, &vr, &dv);
        if (vl == 0.0L) { x[found++] = xl; }
        else if ((vl < 0) != (vr < 0) && vr != 0.0L) {
            ld lo = xl, hi = xr, flo = vl;
            for (int it = 0; it < 200 && hi - lo > 1e-12L * (1 + fabsl(lo)); ++it) {
                ld mid = 0.5L * (lo + hi), fm;
                jacobi_ld(n, a, b, mid, &fm, &dv);
                if ((fm < 0) == (flo < 0)) { lo = mid; flo = fm; } else hi = mid;
            }
            ld z = 0.5L * (lo + hi);
            for (int it = 0; it < 6; ++it) {
                ld v, d;
                jacobi_ld(n, a, b, z, &v, &d);
                if (d == 0) break;
                ld zn = z - v / d;
                if (zn <= lo || zn >= hi) break;      /* stay inside the bracket */
                z = zn;
            }
            x[found++] = z;
        }
        xl = xr; vl = vr;
    }
    if (found != n) return -2;
    ld lc = (a + b + 1) * logl(2.0L) + lgammal(n + a + 1) + lgammal(n + b + 1)
          - lgammal(n + a + b + 1) - lgammal(n + 1.0L);
    ld c = expl(lc);
    for (int i = 0; i < n; ++i) {
        ld v, d;
        jacobi_ld(n, a, b, x[i], &v, &d);
        w[i] = c / ((1 - x[i] * x[i]) * d * d);
    }
    return 0;
}

/* ------------------------------------------------------------ local basis */
/* Physical derivative of the P+1 local functions on an element of size h at
 * reference point xi: index 0 = hat of the left node (phi = (1-xi)/2),
 * index P = hat of the right node (phi = (1+xi)/2), 1..P-1 = modal psi_p. */
static void local_deriv(int P, ld h, ld xi, ld *out)
{
    ld L[MAXP + 2], dL[MAXP + 2];
    legendre_all(P, xi, L, dL);
    out[0] = -1.0L / h;
    out[P] = 1.0L / h;
    for (int p = 1; p < P; ++p) out[p] = (2.0L / h) * (dL[p - 1] - dL[p + 1]);
}

static void local_value(int P, ld xi, ld *out)
{
    ld L[MAXP + 2], dL[MAXP + 2];
    legendre_all(P, xi, L, dL);
    out[0] = 0.5L * (1 - xi);
    out[P] = 0.5L * (1 + xi);
    for (int p = 1; p < P; ++p) out[p] = L[p - 1] - L[p + 1];
}

/* ------------------------------------------------------ pair integrals */
typedef struct {
    int P;
    ld alpha, d, hi, hj;
    ld gx1[MAXQ], gw1[MAXQ], gx2[MAXQ], gw2[MAXQ];
    int q1, q2;
    ld scale, drop;
    long ncells;
} pairctx;

static void cell_rule(pairctx *c, ld u0, ld u1, ld v0, ld v1, const ld *gx, const ld *gw, int q, ld *acc)
{
    const int P = c->P, M = P + 1;
    ld fu[MAXQ][MAXP + 1], gv[MAXQ][MAXP + 1];
    ld wu[MAXQ], wv[MAXQ], uu[MAXQ], vv[MAXQ];
    for (int k = 0; k < q; ++k) {
        uu[k] = u0 + 0.5L * (u1 - u0) * (gx[k] + 1);
        wu[k] = 0.5L * (u1 - u0) * gw[k];
        vv[k] = v0 + 0.5L * (v1 - v0) * (gx[k] + 1);
        wv[k] = 0.5L * (v1 - v0) * gw[k];
        /* test element: t = x_i + u  ->  xi = 2u/h_i - 1 */
        local_deriv(P, c->hi, 2 * uu[k] / c->hi - 1, fu[k]);
        /* trial element: s = x_{j+1} - v  ->  eta = 1 - 2v/h_j */
        local_deriv(P, c->hj, 1 - 2 * vv[k] / c->hj, gv[k]);
    }
    for (int a = 0; a < M * M; ++a) acc[a] = 0;
    for (int k = 0; k < q; ++k) {
        ld tmp[MAXP + 1];
        for (int b = 0; b < M; ++b) tmp[b] = 0;
        for (int l = 0; l < q; ++l) {
            ld ker = wv[l] * powl(c->d + uu[k] + vv[l], 1 - c->alpha);
            for (int b = 0; b < M; ++b) tmp[b] += ker * gv[l][b];
        }
        for (int a = 0; a < M; ++a)
            for (int b = 0; b < M; ++b) acc[a * M + b] += wu[k] * fu[k][a] * tmp[b];
    }
}

static void integrate_cell(pairctx *c, ld u0, ld u1, ld v0, ld v1, ld *out, int depth)
{
    const int M = c->P + 1;
    ld du = u1 - u0, dv = v1 - v0;
    ld dist = c->d + u0 + v0;
    ld size = du > dv ? du : dv;
    if (dist >= size && depth < 200) {
        ld r1[(MAXP + 1) * (MAXP + 1)], r2[(MAXP + 1) * (MAXP + 1)];
        cell_rule(c, u0, u1, v0, v1, c->gx1, c->gw1, c->q1, r1);
        cell_rule(c, u0, u1, v0, v1, c->gx2, c->gw2, c->q2, r2);
        ld err = 0;
        for (int a = 0; a < M * M; ++a) { ld e = fabsl(r1[a] - r2[a]); if (e > err) err = e; }
        if (err <= 1e-19L * c->scale || depth > 150) {
            for (int a = 0; a < M * M; ++a) out[a] += r2[a];
            c->ncells++;
            return;
        }
    } else if (dist == 0 && size <= c->drop) {
        return; /* corner cell of a touching pair: a-priori bound below 1e-19 * scale */
    }
    /* subdivide: the long side only if the aspect ratio exceeds 2 */
    if (du > 2 * dv) {
        ld um = 0.5L * (u0 + u1);
        integrate_cell(c, u0, um, v0, v1, out, depth + 1);
        integrate_cell(c, um, u1, v0, v1, out, depth + 1);
    } else if (dv > 2 * du) {
        ld vm = 0.5L * (v0 + v1);
        integrate_cell(c, u0, u1, v0, vm, out, depth + 1);
        integrate_cell(c, u0, u1, vm, v1, out, depth + 1);
    } else {
        ld um = 0.5L * (u0 + u1), vm = 0.5L * (v0 + v1);
        integrate_cell(c, u0, um, v0, vm, out, depth + 1);
        integrate_cell(c, um, u1, v0, vm, out, depth + 1);
        integrate_cell(c, u0, um, vm, v1, out, depth + 1);
        integrate_cell(c, um, u1, vm, v1, out, depth + 1);
    }
}

/* Pair integral for test element i and trial element j < i.
 * out[(P+1)*(P+1)] (row = local test fn a, col = local trial fn b):
 *   gamma0 * int_{e_i} int_{e_j} phi_a'(t) (t-s)^{1-alpha} phi_b'(s) ds dt.
 * d = x_i - x_{j+1} >= 0 (gap), hi, hj element sizes.  Returns #cells. */
long orc_pair_offdiag(int P, double alpha, double d, double hi, double hj, double *out)
{
    if (P < 1 || P > MAXP) return -1;
    pairctx c;
    memset(&c, 0, sizeof(c));
    c.P = P; c.alpha = alpha; c.d = d; c.hi = hi; c.hj = hj;
    c.q1 = 14 + P / 2; c.q2 = c.q1 + 6;
    orc_gauss_legendre(c.q1, c.gx1, c.gw1);
    orc_gauss_legendre(c.q2, c.gx2, c.gw2);
    ld a = alpha;
    /* scale ~ size of the pair integral for unit-sized derivatives */
    ld Mi = (2.0L / hi) * (2 * P + 1), Mj = (2.0L / hj) * (2 * P + 1);
    c.scale = Mi * Mj * hi * hj * powl(d + hi + hj, 1 - a);
    /* corner bound: int_0^delta int_0^delta (u+v)^{1-a} = (2^{3-a}-2) delta^{3-a}/((2-a)(3-a)) */
    ld cb = Mi * Mj * (powl(2.0L, 3 - a) - 2) / ((2 - a) * (3 - a));
    c.drop = powl(1e-19L * c.scale / cb, 1.0L / (3 - a));
    const int M = P + 1;
    ld acc[(MAXP + 1) * (MAXP + 1)];
    for (int k = 0; k < M * M; ++k) acc[k] = 0;
    integrate_cell(&c, 0.0L, (ld)hi, 0.0L, (ld)hj, acc, 0);
    ld g0 = 1.0L / tgammal(2 - a);
    for (int k = 0; k < M * M; ++k) out[k] = (double)(g0 * acc[k]);
    return c.ncells;
}

/* Same element: gamma0 int_{e} phi_a'(t) int_{x_i}^{t} (t-s)^{1-alpha} phi_b'(s) ds dt.
 * u = t - x_i in [0,h], s = t - u*y: t-s = u y, ds = u dy  =>
 * int_0^h u^{2-alpha} phi_a'(u) int_0^1 y^{1-alpha} phi_b'(u(1-y)) dy du, both
 * Gauss-Jacobi (exact: the basis derivatives are polynomials). */
int orc_pair_self(int P, double alpha, double h, double *out)
{
    if (P < 1 || P > MAXP) return -1;
    const int M = P + 1;
    int q = P + 4;
    ld yx[MAXQ], yw[MAXQ], ux[MAXQ], uw[MAXQ];
    ld a = alpha;
    /* weight (1+x)^{1-a} on [-1,1], y = (1+x)/2 : y^{1-a} dy = 2^{a-2} (1+x)^{1-a} dx */
    if (orc_gauss_jacobi(q, 0.0L, 1 - a, yx, yw)) return -2;
    if (orc_gauss_jacobi(q, 0.0L, 2 - a, ux, uw)) return -2;
    ld acc[(MAXP + 1) * (MAXP + 1)];
    for (int k = 0; k < M * M; ++k) acc[k] = 0;
    ld H = h;
    for (int k = 0; k < q; ++k) {
        ld u = 0.5L * H * (ux[k] + 1);                      /* u in [0,h] */
        ld wu = uw[k] * powl(0.5L * H, 3 - a);              /* u^{2-a} du = (h/2)^{3-a} (1+x)^{2-a} dx */
        ld fa[MAXP + 1];
        local_deriv(P, H, 2 * u / H - 1, fa);
        ld tmp[MAXP + 1];
        for (int b = 0; b < M; ++b) tmp[b] = 0;
        for (int l = 0; l < q; ++l) {
            ld y = 0.5L * (yx[l] + 1);
            ld wy = yw[l] * powl(0.5L, 2 - a);
            ld s_off = u * (1 - y);                          /* s - x_i */
            ld gb[MAXP + 1];
            local_deriv(P, H, 2 * s_off / H - 1, gb);
            for (int b = 0; b < M; ++b) tmp[b] += wy * gb[b];
        }
        for (int a2 = 0; a2 < M; ++a2)
            for (int b = 0; b < M; ++b) acc[a2 * M + b] += wu * fa[a2] * tmp[b];
    }
    ld g0 = 1.0L / tgammal(2 - a);
    for (int k = 0; k < M * M; ++k) out[k] = (double)(g0 * acc[k]);
    return 0;
}

/* --------------------------------------------------------- global assembly */
/* Extended paper ordering: [modal (e,p) e=0..N-1, p=1..P-1 | hats node 1..N-1 |
 * hat node 0 | hat node N].  n = NP-1 interior unknowns (A3). */
static long gidx_local(int N, int P, int e, int a)
{
    long nmod = (long)N * (P - 1);
    if (a == 0) {            /* left node of element e = node e */
        if (e == 0) return nmod + (N - 1);          /* boundary node 0 */
        return nmod + (e - 1);
    }
    if (a == P) {            /* right node = node e+1 */
        if (e + 1 == N) return nmod + (N - 1) + 1;  /* boundary node N */
        return nmod + e;
    }
    return (long)e * (P - 1) + (a - 1);
}

/* Assemble rows of S_l (extended ordering, (n+2) x (n+2) row-major) for test
 * elements in [e0, e1).  Only pairs (i, j<=i) contribute (S_l vanishes for s > t). */
int orc_assemble_Sl(int N, const double *nodes, int P, double alpha, int e0, int e1, double *Sl, int nthreads)
{
    const int M = P + 1;
    const long next = (long)N * P + 1;
    int err = 0;
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int i = e0; i < e1; ++i) {
        double loc[(MAXP + 1) * (MAXP + 1)];
        double hi = nodes[i + 1] - nodes[i];
        for (int j = 0; j <= i; ++j) {
            if (j == i) {
                if (orc_pair_self(P, alpha, hi, loc)) { err = -1; continue; }
            } else {
                double hj = nodes[j + 1] - nodes[j];
                double d = nodes[i] - nodes[j + 1];
                if (orc_pair_offdiag(P, alpha, d, hi, hj, loc) < 0) { err = -1; continue; }
            }
            for (int a = 0; a < M; ++a) {
                long I = gidx_local(N, P, i, a);
                for (int b = 0; b < M; ++b) {
                    long J = gidx_local(N, P, j, b);
                    /* rows of element i are touched only by iteration i, except the
                     * hat rows shared with element i-1/i+1: protect with atomic. */
#pragma omp atomic
                    Sl[I * next + J] += loc[a * M + b];
                }
            }
        }
    }
    return err;
}

/* Mass matrix (extended ordering), exact Gauss-Legendre with P+2 points. */
int orc_assemble_mass(int N, const double *nodes, int P, double *Mm)
{
    const int M = P + 1;
    const long next = (long)N * P + 1;
    ld gx[MAXQ], gw[MAXQ];
    int q = P + 2;
    orc_gauss_legendre(q, gx, gw);
    for (int e = 0; e < N; ++e) {
        ld h = (ld)nodes[e + 1] - (ld)nodes[e];
        ld loc[(MAXP + 1) * (MAXP + 1)];
        for (int k = 0; k < M * M; ++k) loc[k] = 0;
        for (int k = 0; k < q; ++k) {
            ld v[MAXP + 1];
            local_value(P, gx[k], v);
            for (int a = 0; a < M; ++a)
                for (int b = 0; b < M; ++b) loc[a * M + b] += 0.5L * h * gw[k] * v[a] * v[b];
        }
        for (int a = 0; a < M; ++a)
            for (int b = 0; b < M; ++b)
                Mm[gidx_local(N, P, e, a) * next + gidx_local(N, P, e, b)] += (double)loc[a * M + b];
    }
    return 0;
}

/* Load vector (extended ordering) for
 *   f(x) = sum_k leg[k] L_k(2(x-a)/(b-a)-1) + sum_t coef_t (x-a)^pw_t [side 0]
 *                                          + sum_t coef_t (b-x)^pw_t [side 1].
 * Smooth parts: Gauss-Legendre with 40 points per element.  Power terms on the
 * element touching their base point: Gauss-Jacobi with the endpoint weight
 * (exact for the polynomial test functions); elsewhere composite GL (2 halves,
 * 40 points), which is converged to rounding because the base point is at least
 * one element away. */
int orc_load(int N, const double *nodes, int P, double a, double b,
             int nleg, const double *leg, int nterm, const int *side, const double *pw,
             const double *coef, double *G)
{
    const int M = P + 1;
    ld gx[MAXQ], gw[MAXQ];
    int q = 40;
    orc_gauss_legendre(q, gx, gw);
    ld A = a, B = b;
    for (int e = 0; e < N; ++e) {
        ld xl = nodes[e], xr = nodes[e + 1], h = xr - xl;
        ld loc[MAXP + 1];
        for (int k = 0; k < M; ++k) loc[k] = 0;
        /* Legendre part (and integer powers): Gauss-Legendre on two halves */
        for (int half = 0; half < 2; ++half) {
            for (int k = 0; k < q; ++k) {
                ld xi = -1 + half + 0.5L * (gx[k] + 1);          /* reference point in the half */
                ld w = 0.5L * gw[k] * 0.5L * h;
                ld v[MAXP + 1];
                local_value(P, xi, v);
                ld offa = ((ld)nodes[e] - A) + 0.5L * h * (xi + 1);
                ld offb = (B - (ld)nodes[e + 1]) + 0.5L * h * (1 - xi);
                ld fx = 0;
                if (nleg > 0) {
                    ld z = 2 * offa / (B - A) - 1, Lk[64], dLk[64];
                    legendre_all(nleg - 1, z, Lk, dLk);
                    for (int kk = 0; kk < nleg; ++kk) fx += leg[kk] * Lk[kk];
                }
                for (int t = 0; t < nterm; ++t) {
                    int integer_pw = (pw[t] == floor(pw[t]) && pw[t] >= 0);
                    if (!integer_pw) continue;
                    fx += coef[t] * powl(side[t] == 0 ? offa : offb, pw[t]);
                }
                for (int k2 = 0; k2 < M; ++k2) loc[k2] += w * fx * v[k2];
            }
        }
        /* non-integer powers away from their base element: composite Gauss-Legendre on
         * cells [o, 2o] of the distance o to the base point (cell size = distance).
         * Points are placed by their offset u = o - o0 in [0, h] from the element's
         * near end, so the reference coordinate xi is formed without cancellation
         * (o0 can exceed h by many orders of magnitude on graded meshes). */
        for (int t = 0; t < nterm; ++t) {
            int touches = (side[t] == 0) ? (e == 0) : (e == N - 1);
            int integer_pw = (pw[t] == floor(pw[t]) && pw[t] >= 0);
            if (touches || integer_pw) continue;
            ld o0 = (side[t] == 0) ? ((ld)nodes[e] - A) : (B - (ld)nodes[e + 1]);
            ld ua = 0;
            while (ua < h) {
                ld ub = o0 + 2 * ua < h ? o0 + 2 * ua : h;     /* o_b = 2 o_a, capped */
                for (int k = 0; k < q; ++k) {
                    ld u = ua + 0.5L * (ub - ua) * (gx[k] + 1);
                    ld w = 0.5L * (ub - ua) * gw[k] * coef[t] * powl(o0 + u, (ld)pw[t]);
                    ld xi = (side[t] == 0) ? (2 * u / h - 1) : (1 - 2 * u / h);
                    ld v[MAXP + 1];
                    local_value(P, xi, v);
                    for (int k2 = 0; k2 < M; ++k2) loc[k2] += w * v[k2];
                }
                ua = ub;
            }
        }
        /* singular power terms on the touching element: Gauss-Jacobi */
        for (int t = 0; t < nterm; ++t) {
            int touches = (side[t] == 0) ? (e == 0) : (e == N - 1);
            int integer_pw = (pw[t] == floor(pw[t]) && pw[t] >= 0);
            if (!touches || integer_pw) continue;
            ld jx[MAXQ], jw[MAXQ];
            int qq = P + 4;
            if (side[t] == 0) {       /* (x-a)^p, x-a = h(1+xi)/2 -> weight (1+xi)^p */
                orc_gauss_jacobi(qq, 0.0L, (ld)pw[t], jx, jw);
                for (int k = 0; k < qq; ++k) {
                    ld v[MAXP + 1];
                    local_value(P, jx[k], v);
                    ld w = jw[k] * powl(0.5L * h, (ld)pw[t]) * 0.5L * h;
                    for (int k2 = 0; k2 < M; ++k2) loc[k2] += w * coef[t] * v[k2];
                }
            } else {                  /* (b-x)^p, b-x = h(1-xi)/2 -> weight (1-xi)^p */
                orc_gauss_jacobi(qq, (ld)pw[t], 0.0L, jx, jw);
                for (int k = 0; k < qq; ++k) {
                    ld v[MAXP + 1];
                    local_value(P, jx[k], v);
                    ld w = jw[k] * powl(0.5L * h, (ld)pw[t]) * 0.5L * h;
                    for (int k2 = 0; k2 < M; ++k2) loc[k2] += w * coef[t] * v[k2];
                }
            }
        }
        for (int k = 0; k < M; ++k) G[gidx_local(N, P, e, k)] += (double)loc[k];
    }
    return 0;
}

/* Evaluate u_h at reference points of every element from extended-order
 * coefficients (boundary hats included). out[e*m + k]. */
int orc_eval_solution(int N, int P, const double *Xext, int m, const double *xis, double *out)
{
    const int M = P + 1;
    for (int e = 0; e < N; ++e)
        for (int k = 0; k < m; ++k) {
            ld v[MAXP + 1], s = 0;
            local_value(P, xis[k], v);
            for (int a = 0; a < M; ++a) s += v[a] * Xext[gidx_local(N, P, e, a)];
            out[(long)e * m + k] = (double)s;
        }
    return 0;
}

/* exported table generators (for the pins) in double precision */
int orc_gl_table(int n, double *x, double *w)
{
    ld xx[MAXQ], ww[MAXQ];
    int r = orc_gauss_legendre(n, xx, ww);
    for (int i = 0; i < n; ++i) { x[i] = (double)xx[i]; w[i] = (double)ww[i]; }
    return r;
}

int orc_gj_table(int n, double a, double b, double *x, double *w)
{
    ld xx[MAXQ], ww[MAXQ];
    int r = orc_gauss_jacobi(n, a, b, xx, ww);
    for (int i = 0; i < n; ++i) { x[i] = (double)xx[i]; w[i] = (double)ww[i]; }
    return r;
}

/* local derivative / value exports for pins */
int orc_local_deriv(int P, double h, double xi, double *out)
{
    ld o[MAXP + 1];
    local_deriv(P, h, xi, o);
    for (int a = 0; a <= P; ++a) out[a] = (double)o[a];
    return 0;
}

int orc_local_value(int P, double xi, double *out)
{
    ld o[MAXP + 1];
    local_value(P, xi, o);
    for (int a = 0; a <= P; ++a) out[a] = (double)o[a];
    return 0;
}

/* Inner singular integral used by the self-pair rule, exported for the
 * monomial pin:  (1/Gamma(beta)) int_0^x (x-s)^{beta-1} s^gamma ds  computed
 * with the same substitution (s = x(1-y), Gauss-Jacobi weight y^{beta-1}). */
double orc_frac_integral_monomial(double x, double beta, double gam, int q)
{
    ld yx[MAXQ], yw[MAXQ];
    if (orc_gauss_jacobi(q, 0.0L, (ld)beta - 1, yx, yw)) return NAN;
    ld acc = 0;
    for (int l = 0; l < q; ++l) {
        ld y = 0.5L * (yx[l] + 1);
        ld wy = yw[l] * powl(0.5L, (ld)beta);
        acc += wy * powl((ld)x * (1 - y), (ld)gam);
    }
    return (double)(acc * powl((ld)x, (ld)beta) / tgammal((ld)beta));
}
