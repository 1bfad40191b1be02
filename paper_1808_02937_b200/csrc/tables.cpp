// Quadrature tables for the device kernels (host, long double).
//
// Gauss rules are the eigenvalues of the Jacobi matrix of the weight (here
// (1-x)^a (1+x)^b on [-1,1]); we locate them by bisection on the Sturm sequence
// of the tridiagonal matrix and take the weights from the Christoffel numbers
// w_i = mu0 / sum_k p~_k(x_i)^2 of the orthonormal recurrence.  These tables
// are the constants behind the Gauss-Legendre / Gauss-Jacobi rules the
// assembly kernels use for the singular kernel |t-s|^{1-alpha}.
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "fde_internal.h"

namespace fdeq {

typedef long double ld;

static void jacobi_matrix(int n, ld a, ld b, std::vector<ld>& diag, std::vector<ld>& off, ld& mu0)
{
    diag.assign(n, 0);
    off.assign(n, 0);  // off[k] couples k-1 and k  (off[0] unused)
    for (int k = 0; k < n; ++k) {
        ld c = 2 * k + a + b;
        if (k == 0)
            diag[k] = (b - a) / (a + b + 2);
        else
            diag[k] = (b * b - a * a) / (c * (c + 2));
        if (k >= 1) {
            ld num = 4 * (ld)k * (k + a) * (k + b) * (k + a + b);
            ld den = c * c * (c + 1) * (c - 1);
            off[k] = sqrtl(num / den);
        }
    }
    mu0 = powl(2.0L, a + b + 1) * tgammal(a + 1) * tgammal(b + 1) / tgammal(a + b + 2);
}

// number of eigenvalues of the tridiagonal matrix strictly below x
static int sturm_count(int n, const std::vector<ld>& d, const std::vector<ld>& e, ld x)
{
    int cnt = 0;
    ld q = d[0] - x;
    if (q < 0) cnt++;
    for (int k = 1; k < n; ++k) {
        if (q == 0) q = 1e-300L;
        q = d[k] - x - e[k] * e[k] / q;
        if (q < 0) cnt++;
    }
    return cnt;
}

static void gauss_from_jacobi(int n, ld a, ld b, std::vector<double>& xo, std::vector<double>& wo)
{
    std::vector<ld> d, e;
    ld mu0;
    jacobi_matrix(n, a, b, d, e, mu0);
    xo.assign(n, 0);
    wo.assign(n, 0);
    for (int i = 0; i < n; ++i) {
        // i-th smallest eigenvalue in (-1, 1)
        ld lo = -1.0L, hi = 1.0L;
        for (int it = 0; it < 200; ++it) {
            ld mid = 0.5L * (lo + hi);
            if (mid == lo || mid == hi) break;
            if (sturm_count(n, d, e, mid) > i)
                hi = mid;
            else
                lo = mid;
        }
        ld x = 0.5L * (lo + hi);
        // Christoffel number with the orthonormal recurrence
        ld p0 = 1.0L, s = 1.0L, pm = 0.0L;
        for (int k = 0; k < n - 1; ++k) {
            ld p1 = ((x - d[k]) * p0 - (k > 0 ? e[k] * pm : 0.0L)) / e[k + 1];
            s += p1 * p1;
            pm = p0;
            p0 = p1;
        }
        xo[i] = (double)x;
        wo[i] = (double)(mu0 / s);
    }
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w)
{
    gauss_from_jacobi(n, 0.0L, 0.0L, x, w);
}

void gauss_jacobi(int n, double a, double b, std::vector<double>& x, std::vector<double>& w)
{
    // memoised per (n, a, b): a rule is a pure function of them, and the Sturm
    // bisection of the Jacobi matrix in long double took ~40 us of host time per rule
    // at the start of every assembly (the device waited for it)
    typedef std::tuple<int, unsigned long long, unsigned long long> Key;
    static std::mutex mu;
    static std::map<Key, std::pair<std::vector<double>, std::vector<double>>> memo;
    unsigned long long ua, ub;
    std::memcpy(&ua, &a, sizeof ua);
    std::memcpy(&ub, &b, sizeof ub);
    const Key key(n, ua, ub);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = memo.find(key);
        if (it != memo.end()) {
            x = it->second.first;
            w = it->second.second;
            return;
        }
    }
    gauss_from_jacobi(n, (ld)a, (ld)b, x, w);
    std::lock_guard<std::mutex> lk(mu);
    if (memo.size() < 4096) memo.emplace(key, std::make_pair(x, w));
}

}  // namespace fdeq
