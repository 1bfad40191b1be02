"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path.

This module holds NO arithmetic of the method (no quadrature, no assembly, no
solver). It only produces the *inputs* of the problem statement, Eq. (Model),
PAPER.md:33-40: the interval (a, b), alpha, theta, rho, the boundary values
c1, c2, the forcing f (as a description, see `Forcing`), the partition
x_0 < ... < x_N (Eq. (Partition)), the polynomial degree P
and the H-matrix parameters (R, lambda, n_min).

Mesh recipes:
  * uniform           x_i = a + i (b-a)/N                          (q^=1)
  * graded            x_i = a + (i/N)^q (b-a)
  * two-sided graded  (PAPER.md:941 / BASELINE config 4 "mirrored")
  * geometric layers  (BASELINE config 3, SURVEY.md §8(d) reading A17)

Forcing f is described as
    f(x) = sum_k leg[k] * L_k(2 (x-a)/(b-a) - 1)
         + sum_t coef_t * (x-a)^{pow_t}        (side 'L')
         + sum_t coef_t * (b-x)^{pow_t}        (side 'R')
which covers the Legendre-series forcings of configs 2, 4, 5, the constant
forcing of config 3 and the manufactured monomial forcing of config 1.
The manufactured f of config 1 is the *input* derived from the closed form
aI^beta (x-a)^gamma = Gamma(gamma+1)/Gamma(gamma+1+beta) (x-a)^{gamma+beta}
(PAPER.md:43-44 definition; BASELINE.json north_star), i.e. part of the
problem statement, not of the method.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np


# --------------------------------------------------------------------------
# meshes
# --------------------------------------------------------------------------
def uniform_mesh(a: float, b: float, N: int) -> np.ndarray:
    x = a + (b - a) * np.arange(N + 1, dtype=np.float64) / N
    x[0], x[-1] = a, b
    return x


def graded_mesh(a: float, b: float, N: int, q: float) -> np.ndarray:
    i = np.arange(N + 1, dtype=np.float64)
    x = a + (i / N) ** q * (b - a)
    x[0], x[-1] = a, b
    return x


def two_sided_graded_mesh(a: float, b: float, N: int, qL: float, qR: float) -> np.ndarray:
    """x_i = m + (m-a)*((2i/N)^qL - 1) for i <= N/2, mirrored with qR."""
    assert N % 2 == 0
    m = 0.5 * (a + b)
    x = np.empty(N + 1)
    for i in range(N + 1):
        if i <= N // 2:
            x[i] = a + (m - a) * (2.0 * i / N) ** qL
        else:
            x[i] = b - (b - m) * ((2.0 * (N - i)) / N) ** qR
    x[0], x[N // 2], x[-1] = a, m, b
    return x


def geometric_layer_mesh(sigma: float = 0.15, layers: int = 16, interior: int = 32) -> np.ndarray:
    """BASELINE config 3 on (0,1), reading A17:
    x_0=0, x_k = x_g sigma^(layers-k) (k=1..layers), `interior` uniform elements
    on [x_g, 1-x_g], right side mirrored; x_g chosen so the largest layer
    element equals the interior width."""
    xg = 1.0 / (2.0 + interior * (1.0 - sigma))
    left = [0.0] + [xg * sigma ** (layers - k) for k in range(1, layers + 1)]
    mid = [xg + k * (1.0 - 2.0 * xg) / interior for k in range(1, interior)]
    right = [1.0 - xg * sigma ** (layers - k) for k in range(layers, 0, -1)] + [1.0]
    x = np.array(left + mid + right, dtype=np.float64)
    assert len(x) == 2 * layers + interior + 1
    assert np.all(np.diff(x) > 0)
    return x


def geometric_mesh(a: float, b: float, N: int, qhat: float) -> np.ndarray:
    """h_{i+1} = qhat h_i."""
    if qhat == 1.0:
        return uniform_mesh(a, b, N)
    # every node from its own power (not a running sum): relative spacing errors
    # stay at rounding level for long meshes
    k = np.arange(N + 1, dtype=np.float64)
    x = a + (b - a) * np.expm1(k * np.log(qhat)) / np.expm1(N * np.log(qhat))
    x[0], x[-1] = a, b
    return x


# --------------------------------------------------------------------------
# forcing
# --------------------------------------------------------------------------
@dataclass
class Forcing:
    leg: np.ndarray = field(default_factory=lambda: np.zeros(0))       # Legendre coeffs on (a,b)
    terms: List[Tuple[str, float, float]] = field(default_factory=list)  # (side 'L'|'R', power, coef)

    def evaluate(self, x: np.ndarray, a: float, b: float) -> np.ndarray:
        """Pointwise f(x) (used only to *describe* inputs / plots)."""
        x = np.asarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        if len(self.leg):
            y += np.polynomial.legendre.legval(2 * (x - a) / (b - a) - 1, self.leg)
        for side, pw, c in self.terms:
            base = (x - a) if side == "L" else (b - x)
            y += c * np.power(np.maximum(base, 0.0), pw)
        return y


def random_legendre_forcing(seed: int, degree: int = 20) -> Forcing:
    """BASELINE config 2: coeffs z_k/(k+1)^2, z = default_rng(seed).standard_normal(deg+1)."""
    z = np.random.default_rng(seed).standard_normal(degree + 1)
    k = np.arange(degree + 1)
    return Forcing(leg=z / (k + 1.0) ** 2)


def manufactured_poly_forcing(coeffs: dict, alpha: float, theta: float, rho: float,
                              symmetric_about_mid: bool = True) -> Forcing:
    """f for u(x) = sum_k c_k x^k on (0,1) with u(x)=u(1-x) (config 1).

    -D^2 aI^{2-alpha} x^k = -Gamma(k+1)/Gamma(k+1-alpha) x^{k-alpha} (monomial closed
    form of the fractional integral), mirrored for the right-sided operator because
    u(1-x) = u(x); plus rho*u.
    """
    assert symmetric_about_mid
    terms = []
    for k, c in coeffs.items():
        g = math.gamma(k + 1) / math.gamma(k + 1 - alpha)
        terms.append(("L", k - alpha, -theta * c * g))
        terms.append(("R", k - alpha, -(1 - theta) * c * g))
        if rho != 0.0:
            terms.append(("L", float(k), rho * c))
    return Forcing(terms=terms)


# --------------------------------------------------------------------------
# configs (BASELINE.json "configs"; concrete readings SURVEY.md §8(d))
# --------------------------------------------------------------------------
@dataclass
class Problem:
    name: str
    a: float
    b: float
    alpha: float
    theta: float
    rho: float
    c1: float
    c2: float
    nodes: np.ndarray
    P: int
    R: int
    lam: float = 1.0
    n_min: int = 16
    forcings: List[Forcing] = field(default_factory=list)   # one per RHS
    mesh_kind: str = "custom"                               # uniform|graded|geometric|custom

    @property
    def N(self) -> int:
        return len(self.nodes) - 1

    @property
    def n(self) -> int:
        return self.N * self.P - 1


def config1() -> Problem:
    alpha, theta, rho = 1.5, 0.5, 1.0
    f = manufactured_poly_forcing({2: 1.0, 3: -2.0, 4: 1.0}, alpha, theta, rho)
    return Problem("c1", 0.0, 1.0, alpha, theta, rho, 0.0, 0.0, uniform_mesh(0, 1, 8), 4, 4,
                   n_min=2, forcings=[f], mesh_kind="uniform")


def config1_exact(x: np.ndarray) -> np.ndarray:
    return x ** 2 * (1 - x) ** 2


def config2(alpha: float = 1.5, seed: Optional[int] = None, N: int = 256, P: int = 8) -> Problem:
    if seed is None:
        seed = {1.2: 0, 1.5: 1, 1.8: 2}.get(alpha, 0)
    return Problem(f"c2-a{alpha}-N{N}-P{P}", 0.0, 1.0, alpha, 0.3, 1.0, 0.5, -1.0, uniform_mesh(0, 1, N), P, 8,
                   forcings=[random_legendre_forcing(seed)], mesh_kind="uniform")


def geometric_problem(qhat: float, N: int = 64, P: int = 8, alpha: float = 1.5, theta: float = 0.3,
                      rho: float = 1.0, seed: int = 0) -> Problem:
    """Single-ratio geometric mesh on (0, 1) (h_{i+1} = qhat h_i): the
    paper's second structured case for the Toeplitz matvec."""
    return Problem(f"geo-q{qhat}-N{N}-P{P}-a{alpha}", 0.0, 1.0, alpha, theta, rho, 0.0, 0.0,
                   geometric_mesh(0, 1, N, qhat), P, 8, forcings=[random_legendre_forcing(seed)],
                   mesh_kind="geometric")


def config3(P: int = 16) -> Problem:
    alpha = 1.7
    fconst = -math.cos(math.pi * alpha / 2) * math.gamma(alpha + 1)
    return Problem(f"c3-P{P}", 0.0, 1.0, alpha, 0.5, 0.0, 0.0, 0.0, geometric_layer_mesh(), P, 10,
                   forcings=[Forcing(leg=np.array([fconst]))], mesh_kind="custom")


def config3_exact(x_left_dist: np.ndarray, x_right_dist: np.ndarray, alpha: float = 1.7) -> np.ndarray:
    """u = (x(1-x))^{alpha/2}, with x and 1-x passed separately (cancellation near 1)."""
    return (x_left_dist * x_right_dist) ** (alpha / 2)


def config4(N: int = 1024, P: int = 8) -> Problem:
    x = np.empty(N + 1)
    for j in range(N + 1):
        if j <= N // 2:
            x[j] = 0.5 * (2.0 * j / N) ** 2
        else:
            x[j] = 1.0 - 0.5 * (2.0 * (N - j) / N) ** 2
    return Problem(f"c4-N{N}-P{P}", 0.0, 1.0, 1.4, 0.7, 2.0, 0.0, 0.0, x, P, 12, n_min=64,
                   forcings=[random_legendre_forcing(0)], mesh_kind="graded")


def config5(N: int = 4096, P: int = 8, nrhs: int = 64) -> Problem:
    return Problem(f"c5-N{N}-P{P}", 0.0, 1.0, 1.6, 0.4, 1.0, 0.0, 0.0, uniform_mesh(0, 1, N), P, 16, n_min=64,
                   forcings=[random_legendre_forcing(s) for s in range(nrhs)], mesh_kind="uniform")


def example51(N: int = 100, P: int = 3, alpha: float = 1.6, rho: float = 0.0, R: int = 5,
              n_min: int = 16) -> Problem:
    """Example 5.1: theta=1, u = (x-a) - (b-a)^{1-g}(x-a)^g, a=0, b=10,
    g=0.8, graded mesh x_i = (i/N)^5 (b-a); alpha = 1.6 (reading A16).
    f = -D^2 aI^{2-alpha} u + rho u from the monomial closed form
    -D^2 aI^{2-alpha} x^k = -Gamma(k+1)/Gamma(k+1-alpha) x^{k-alpha}."""
    a, b, g = 0.0, 10.0, 0.8
    c = (b - a) ** (1 - g)
    terms = [("L", 1.0 - alpha, -math.gamma(2.0) / math.gamma(2.0 - alpha)),
             ("L", g - alpha, c * math.gamma(g + 1) / math.gamma(g + 1 - alpha))]
    if rho != 0.0:
        terms += [("L", 1.0, rho), ("L", g, -rho * c)]
    return Problem(f"ex51-N{N}-P{P}-R{R}", a, b, alpha, 1.0, rho, 0.0, 0.0, graded_mesh(a, b, N, 5.0), P, R,
                   n_min=n_min, forcings=[Forcing(terms=terms)], mesh_kind="graded")


def example51_exact(x: np.ndarray) -> np.ndarray:
    return x - 10.0 ** 0.2 * np.power(x, 0.8)


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}
