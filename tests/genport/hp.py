"""Extended-precision substrate of the coefficient generator (mpmath).

Restates `highprec.hpp`/`highprec.cpp` and `reference.hpp`/`reference.cpp` of
the reference (/root/reference/proj/core): working precision 50 decimal digits
plus 12 guard digits (`highprec.hpp:18-19`), erf by its Taylor series below
x = 2 and Gamma(1/2, x^2) by a modified-Lentz continued fraction above
(`highprec.cpp:75-131`), Gamma(k+1/2, x) built upward from Gamma(1/2, x)
(`highprec.cpp:133-151`), and the equal-sign Boys series oracle
(`reference.cpp:10-23`).

The reference keeps the precision in a process-global MPFR default; here every
public entry point of the generator runs inside `precision()`, a context that
sets mpmath's working precision and restores it on exit.
"""
import contextlib
import math

import mpmath
from mpmath import mp, mpf

DEFAULT_DIGITS = 50  # highprec.hpp:18
GUARD_DIGITS = 12    # highprec.hpp:19
_digits = DEFAULT_DIGITS


def set_working_digits(digits10):
    """highprec.cpp:36-41."""
    global _digits
    if digits10 < 16:
        raise ValueError("working precision must be at least 16 digits")
    _digits = int(digits10)


def working_digits():
    return _digits


@contextlib.contextmanager
def precision():
    """Working digits + guard digits for the duration of a generator call."""
    with mp.workdps(_digits + GUARD_DIGITS):
        yield


def series_eps():
    """Termination tolerance of series / continued fractions (highprec.cpp:28-32)."""
    return mpf(10) ** (-(_digits + GUARD_DIGITS - 2))


def sqrt_pi():
    return mpmath.sqrt(mp.pi)


def exp(x):
    x = mpf(x)
    if not mpmath.isfinite(x):
        raise ValueError("hp::exp: non-finite argument")
    return mpmath.exp(x)


def gamma_half(k):
    """Gamma(k + 1/2) by Gamma(s+1) = s Gamma(s) from sqrt(pi) (highprec.cpp:62-68)."""
    if k < 0:
        raise ValueError("hp::gamma_half: k must be non-negative")
    v = sqrt_pi()
    for i in range(1, k + 1):
        v *= mpf(i) - mpf("0.5")
    return v


def _erf_series(x):
    eps = series_eps()
    xx = x * x
    u = mpf(x)
    s = mpf(x)
    for n in range(1, 100000):
        u *= -xx
        u /= n
        term = u / (2 * n + 1)
        s += term
        if abs(term) <= abs(s) * eps:
            break
    return 2 * s / sqrt_pi()


def _upper_gamma_cf(a, z):
    """Modified Lentz continued fraction for Gamma(a, z) (highprec.cpp:95-117)."""
    eps = series_eps()
    fpmin = mpf(10) ** (-(_digits + GUARD_DIGITS) * 8)
    b = z + 1 - a
    c = 1 / fpmin
    d = 1 / b
    h = d
    for i in range(1, 100000):
        an = -i * (i - a)
        b += 2
        d = an * d + b
        if abs(d) < fpmin:
            d = fpmin
        c = b + an / c
        if abs(c) < fpmin:
            c = fpmin
        d = 1 / d
        dl = d * c
        h *= dl
        if abs(dl - 1) <= eps:
            break
    return exp(-z + a * mpmath.log(z)) * h


def erf(x):
    x = mpf(x)
    if x < 0:
        raise ValueError("hp::erf: negative argument unsupported")
    return _erf_series(x) if x < 2 else 1 - erfc(x)


def erfc(x):
    x = mpf(x)
    if x < 0:
        raise ValueError("hp::erfc: negative argument unsupported")
    if x < 2:
        return 1 - _erf_series(x)
    return _upper_gamma_cf(mpf("0.5"), x * x) / sqrt_pi()


def upper_gamma_half(k, x):
    """Gamma(k + 1/2, x), x >= 0 (highprec.cpp:133-151)."""
    x = mpf(x)
    if k < 0:
        raise ValueError("hp::upper_gamma_half: k must be non-negative")
    if x < 0:
        raise ValueError("hp::upper_gamma_half: x must be non-negative")
    if x == 0:
        return gamma_half(k)
    g = sqrt_pi() * erfc(mpmath.sqrt(x))
    if k == 0:
        return g
    e = exp(-x)
    xpow = mpmath.sqrt(x)
    for j in range(k):
        g = (j + mpf("0.5")) * g + xpow * e
        xpow *= x
    return g


def reference_terms_for(k, x, rel_target=1e-30):
    """Series length L (multiple of 25, >= 150) whose Eq. (22) bound meets
    rel_target (reference.cpp:46-54)."""
    if x <= 0:
        return 150
    lt = math.log(rel_target)
    for L in range(150, 20001, 25):
        s = k + L + 1.5
        if s * math.log(x) - math.lgamma(s) <= lt:
            return L
    raise RuntimeError("reference_terms_for: no L below cap reaches target")


def boys_reference(k, x, L=150):
    """F_k(x) = e^{-x}/2 sum_{l=0..L} x^l / prod_{j=0..l} (k+j+1/2) (reference.cpp:10-23)."""
    x = mpf(x)
    if k < 0:
        raise ValueError("boys_reference: k must be non-negative")
    if x < 0:
        raise ValueError("boys_reference: x must be non-negative")
    if L < 1:
        raise ValueError("boys_reference: truncation_terms must be >= 1")
    term = 1 / (k + mpf("0.5"))
    s = term
    for l in range(1, L + 1):
        term *= x
        term /= (k + l + mpf("0.5"))
        s += term
    return exp(-x) / 2 * s


def boys_reference_batch(kmax, x, L=150):
    """F_0..F_kmax: the series at kmax, then the downward recurrence (reference.cpp:25-35)."""
    x = mpf(x)
    v = [mpf(0)] * (kmax + 1)
    v[kmax] = boys_reference(kmax, x, L)
    if kmax == 0:
        return v
    e = exp(-x)
    for l in range(kmax - 1, -1, -1):
        v[l] = (2 * x * v[l + 1] + e) / (2 * l + 1)
    return v


def truncation_bound(k, x, L):
    """x^(k+L+3/2) / Gamma(k+L+3/2) (reference.cpp:37-44)."""
    x = mpf(x)
    if k < 0 or L < 0:
        raise ValueError("truncation_bound: k, L must be non-negative")
    if x < 0:
        raise ValueError("truncation_bound: x must be non-negative")
    if x == 0:
        return mpf(0)
    return mpmath.power(x, mpf(k) + L + mpf("1.5")) / gamma_half(k + L + 1)


def boys_target(k):
    """The generator's target F_k in working precision, with the series long
    enough that its Eq. (22) bound is below 10^-(digits+2) over the generation
    domain (x <= x1 < 60 for every supported table set)."""
    def f(x):
        x = mpf(x)
        xf = float(x)
        L = reference_terms_for(k, xf, 10.0 ** -(_digits + 2)) if xf > 0 else 150
        return boys_reference(k, x, L)
    return f
