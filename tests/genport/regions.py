"""Region partition [0, inf) = A u B u C of the table-free scheme: x0 (Eq. 20),
x1 (Eq. 12, safeguarded Newton) and the downward-recursion weights rho_A,k
(Eq. 18).  Restates `regions.hpp`/`regions.cpp`."""
from dataclasses import dataclass

import mpmath
from mpmath import mpf

from . import hp


@dataclass
class RegionPartition:
    x0: float = 0.0
    x1: float = 0.0
    k_max: int = 0
    eps_tol: float = 0.0


def compute_x0(k_max):
    """x0 = max{1, (prod_{k<kmax} (k+1/2))^(1/kmax)} (regions.cpp:10-17)."""
    if k_max < 1:
        raise ValueError("compute_x0: k_max must be >= 1")
    with hp.precision():
        prod = hp.gamma_half(k_max) / hp.sqrt_pi()
        x0 = mpmath.power(prod, mpf(1) / k_max)
        return +max(x0, mpf(1))


def _asymptotic_error(k_max, x):
    return hp.upper_gamma_half(k_max, x) / (2 * mpmath.power(x, mpf(k_max) + mpf("0.5")))


def compute_x1(k_max, eps_tol):
    """Root of Gamma(kmax+1/2, x)/(2 x^(kmax+1/2)) = eps_tol by bracketing from
    kmax+35 and safeguarded Newton, residual <= eps_tol*1e-21 (regions.cpp:28-72)."""
    if k_max < 0:
        raise ValueError("compute_x1: k_max must be non-negative")
    with hp.precision():
        eps = mpf(eps_tol)
        if not (0 < eps < 1):
            raise ValueError("compute_x1: eps_tol must lie in (0, 1)")
        s = mpf(k_max) + mpf("0.5")
        hi = mpf(k_max) + 35
        lo = hi
        if _asymptotic_error(k_max, hi) > eps:
            while _asymptotic_error(k_max, hi) > eps:
                lo = hi
                hi *= 2
                if hi > k_max + 100000:
                    raise RuntimeError("compute_x1: failed to bracket root (right)")
        else:
            while _asymptotic_error(k_max, lo) <= eps:
                hi = lo
                lo *= mpf("0.5")
                if lo < mpf(1) / 1048576:
                    raise RuntimeError("compute_x1: failed to bracket root (left)")
        x = (lo + hi) / 2
        tol = eps * mpf(10) ** -21
        trace = []
        for it in range(500):
            err = _asymptotic_error(k_max, x)
            h = err - eps
            trace.append("iter %d x=%s h/eps=%s" % (it, mpmath.nstr(x, 20), mpmath.nstr(h / eps, 5)))
            if abs(h) <= tol:
                return x
            if h > 0:
                lo = x
            else:
                hi = x
            hprime = -hp.exp(-x) / (2 * x) - s * err / x
            nxt = x - h / hprime
            if not (lo < nxt < hi):
                nxt = (lo + hi) / 2
            x = nxt
        raise RuntimeError("compute_x1: Newton did not converge; trace:\n" + "\n".join(trace))


def weight_rho_A(k, x):
    """rho_A,k(x) = max_{l=0..k} prod_{n=l}^{k-1} x/(n+1/2) (regions.cpp:74-85)."""
    if k < 0:
        raise ValueError("weight_rho_A: k must be non-negative")
    x = mpf(x)
    if x < 0:
        raise ValueError("weight_rho_A: x must be non-negative")
    prod = mpf(1)
    best = mpf(1)
    for l in range(k - 1, -1, -1):
        prod *= x
        prod /= (l + mpf("0.5"))
        if prod > best:
            best = prod
    return best


def make_partition(k_max, eps_tol):
    return RegionPartition(x0=float(compute_x0(k_max)), x1=float(compute_x1(k_max, eps_tol)),
                           k_max=k_max, eps_tol=eps_tol)
