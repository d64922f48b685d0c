"""Cyclic Jacobi eigensolver for real symmetric matrices in working precision
(restates `linalg.cpp:9-71`).  Returns (values, vectors) with vectors[j] the
eigenvector of values[j]."""
import mpmath
from mpmath import mpf

from . import hp


def jacobi_eigensolve(a, max_sweeps=100):
    d = len(a)
    if any(len(row) != d for row in a):
        raise ValueError("jacobi_eigensolve: matrix not square")
    a = [list(map(mpf, row)) for row in a]
    v = [[mpf(1) if i == j else mpf(0) for j in range(d)] for i in range(d)]
    norm = mpmath.sqrt(sum(a[i][j] ** 2 for i in range(d) for j in range(d)))
    stop = norm * mpf(10) ** (-(hp.working_digits() + hp.GUARD_DIGITS - 4))
    for _ in range(max_sweeps):
        off = sum(a[p][q] ** 2 for p in range(d) for q in range(p + 1, d))
        if mpmath.sqrt(2 * off) <= stop:
            break
        for p in range(d):
            for q in range(p + 1, d):
                if abs(a[p][q]) <= stop / (d * d):
                    continue
                theta = (a[q][q] - a[p][p]) / (2 * a[p][q])
                t = 1 / (abs(theta) + mpmath.sqrt(theta * theta + 1))
                if theta < 0:
                    t = -t
                c = 1 / mpmath.sqrt(t * t + 1)
                s = t * c
                tau = s / (1 + c)
                apq = a[p][q]
                a[p][p] -= t * apq
                a[q][q] += t * apq
                a[p][q] = a[q][p] = mpf(0)
                for i in range(d):
                    if i != p and i != q:
                        aip, aiq = a[i][p], a[i][q]
                        a[i][p] = a[p][i] = aip - s * (aiq + tau * aip)
                        a[i][q] = a[q][i] = aiq + s * (aip - tau * aiq)
                    vip, viq = v[i][p], v[i][q]
                    v[i][p] = vip - s * (viq + tau * vip)
                    v[i][q] = viq + s * (vip - tau * viq)
    values = [a[j][j] for j in range(d)]
    vectors = [[v[i][j] for i in range(d)] for j in range(d)]
    return values, vectors
