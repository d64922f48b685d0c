"""Monomial-basis polynomials in working precision: Horner evaluation,
trimming, Sturm root counting, Newton interpolation and Leja ordering.
Restates `polynomial.hpp`/`polynomial.cpp`; coefficients ascend in degree."""
import mpmath
from mpmath import mpf

from . import hp


def poly_eval(p, x):
    """polynomial.cpp:9-14."""
    if not p:
        return mpf(0)
    acc = p[-1]
    for c in reversed(p[:-1]):
        acc = acc * x + c
    return acc


def poly_derivative(p):
    if len(p) <= 1:
        return [mpf(0)]
    return [i * p[i] for i in range(1, len(p))]


def poly_trim(p, rel_tol):
    """Drop leading coefficients below rel_tol * max|c| (polynomial.cpp:23-32)."""
    maxc = max((abs(c) for c in p), default=mpf(0))
    if maxc == 0:
        return [mpf(0)]
    cut = maxc * rel_tol
    n = len(p)
    while n > 1 and abs(p[n - 1]) <= cut:
        n -= 1
    return list(p[:n])


def poly_degree(p):
    for i in range(len(p) - 1, -1, -1):
        if p[i] != 0:
            return i
    return 0


def _poly_rem(u, v):
    u = list(u)
    dv = len(v) - 1
    while len(u) - 1 >= dv and not (len(u) == 1 and u[0] == 0):
        du = len(u) - 1
        q = u[-1] / v[-1]
        for i in range(dv + 1):
            u[du - dv + i] -= q * v[i]
        u.pop()
        while len(u) > 1 and u[-1] == 0:
            u.pop()
        if max(abs(c) for c in u) == 0:
            return [mpf(0)]
    return u


def _normalize_scale(p):
    maxc = max(abs(c) for c in p)
    return p if maxc == 0 else [c / maxc for c in p]


def _sign(v, tiny):
    return 1 if v > tiny else (-1 if v < -tiny else 0)


def _sign_variations(chain, x, tiny):
    count, prev = 0, 0
    for q in chain:
        s = _sign(poly_eval(q, x), tiny)
        if s == 0:
            continue
        if prev != 0 and s != prev:
            count += 1
        prev = s
    return count


def sturm_root_count(p, a, b):
    """Distinct real roots of p in (a, b] (polynomial.cpp:88-115)."""
    if a > b:
        raise ValueError("sturm_root_count: a > b")
    d = hp.working_digits() + hp.GUARD_DIGITS
    trim_tol = mpf(10) ** (-(d - 6))
    p0 = poly_trim(p, trim_tol)
    if len(p0) == 1 and p0[0] == 0:
        raise ValueError("sturm_root_count: zero polynomial")
    if len(p0) == 1:
        return 0
    chain = [_normalize_scale(p0), _normalize_scale(poly_derivative(_normalize_scale(p0)))]
    while len(chain[-1]) > 1:
        r = poly_trim(_poly_rem(chain[-2], chain[-1]), trim_tol)
        if len(r) == 1 and r[0] == 0:
            break
        chain.append(_normalize_scale([-c for c in r]))
    tiny = mpf(10) ** (-(d - 8))
    return _sign_variations(chain, mpf(a), tiny) - _sign_variations(chain, mpf(b), tiny)


def newton_interpolate(xs, ys):
    """Divided differences expanded to the monomial basis (polynomial.cpp:117-141)."""
    n = len(xs)
    if n == 0 or len(ys) != n:
        raise ValueError("newton_interpolate: size mismatch")
    c = list(ys)
    for j in range(1, n):
        for i in range(n - 1, j - 1, -1):
            c[i] = (c[i] - c[i - 1]) / (xs[i] - xs[i - j])
    result = [c[0]]
    basis = [mpf(1)]
    for i in range(1, n):
        nxt = [mpf(0)] * (len(basis) + 1)
        for j, bj in enumerate(basis):
            nxt[j + 1] += bj
            nxt[j] -= bj * xs[i - 1]
        basis = nxt
        if len(result) < len(basis):
            result += [mpf(0)] * (len(basis) - len(result))
        for j, bj in enumerate(basis):
            result[j] += c[i] * bj
    return result


def leja_order(xs):
    """Greedy maximal-separation ordering (polynomial.cpp:143-164)."""
    n = len(xs)
    first = max(range(n), key=lambda i: (abs(xs[i]), -i))
    order, used = [first], [False] * n
    used[first] = True
    logdist = [mpf(0)] * n
    for _ in range(1, n):
        best = -1
        for i in range(n):
            if used[i]:
                continue
            logdist[i] += mpmath.log(abs(xs[i] - xs[order[-1]]))
            if best < 0 or logdist[i] > logdist[best]:
                best = i
        order.append(best)
        used[best] = True
    return order
