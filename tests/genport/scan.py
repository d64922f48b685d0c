"""B200 backend of the Remez extremum search (replaces remez.cpp:33-108's grid
scan + golden-section refinement in working precision).

The weighted error e(x) = rho(x) (F_k(x) - p(x)/q(x)) is evaluated in
double-double on the device (`boysfn_gen_error_scan`, csrc/gen_scan.cu) on a
uniform grid of `grid` points over [a, b]; every grid local maximum of |e| is
then refined on a zoomed grid of `zoom` points spanning its two neighbouring
cells, all zooms in one launch.  The located extremum sits within
(b-a)*2/(grid*zoom) (about 1e-9 of the interval) of the true one, where the
error curve is flat to second order: the sup error is underestimated by a
relative ~1e-17, far below the exchange's convergence threshold (eps_tol/100).

Node positions are doubles; the fixed-node solves, f at the nodes and the
approximant stay in working precision (remez.py).  No silent fallback: with no
GPU or no library the calls raise.
"""
import ctypes

import numpy as np
from mpmath import mpf

from paper_2512_10059_b200 import _capi
from . import hp

WEIGHTS = {"one": 0, "rho_A": 1}


def _dd(coeffs):
    hi = np.array([float(c) for c in coeffs], dtype=np.float64)
    lo = np.array([float(mpf(c) - mpf(h)) for c, h in zip(coeffs, hi)], dtype=np.float64)
    return hi, lo


def error_scan(k, weight, numer, denom, xs):
    """e(x) = rho (F_k - p/q) at xs (float64 array) on the device."""
    L = _capi.lib()
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    nh, nl = _dd(numer)
    dh, dl = _dd(denom)
    err = np.empty_like(xs)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = L.boysfn_gen_error_scan(int(k), ptr(nh), ptr(nl), len(numer) - 1, ptr(dh), ptr(dl), len(denom) - 1,
                                 WEIGHTS[weight], ptr(xs), ctypes.c_size_t(xs.size), ptr(err))
    if st:
        raise RuntimeError("boysfn_gen_error_scan: " + _capi.last_error())
    return err


def boys_dd(k, xs):
    """F_k(xs) in double-double on the device: (hi, lo) arrays."""
    L = _capi.lib()
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    hi, lo = np.empty_like(xs), np.empty_like(xs)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = L.boysfn_gen_boys_dd(int(k), ptr(xs), ctypes.c_size_t(xs.size), ptr(hi), ptr(lo))
    if st:
        raise RuntimeError("boysfn_gen_boys_dd: " + _capi.last_error())
    return hi, lo


class GpuScan:
    """Extremum search for the Remez problem rho (F_k - r) on [a, b]:
    weight "one" (r_B) or "rho_A" (r_A[k])."""

    def __init__(self, k, weight="one", grid=1 << 16, zoom=2048):
        if weight not in WEIGHTS:
            raise ValueError("weight must be 'one' or 'rho_A'")
        self.k, self.weight, self.grid, self.zoom = int(k), weight, int(grid), int(zoom)
        self.a = self.b = None
        self.max_extrema = 1 << 12

    def bind(self, problem):
        c = GpuScan(self.k, self.weight, self.grid, self.zoom)
        c.a, c.b = float(problem.a), float(problem.b)
        c.width = mpf(problem.b) - mpf(problem.a)
        c.max_extrema = 64 * (problem.n + problem.m + 2)  # the reference's grid size bounds its count
        return c

    def errors(self, r, xs):
        return error_scan(self.k, self.weight, r.numer, r.denom, xs)

    def error_at(self, r, x):
        return mpf(float(self.errors(r, np.array([float(x)]))[0]))

    def refined_extrema(self, r):
        xs = np.linspace(self.a, self.b, self.grid)
        e = np.abs(self.errors(r, xs))
        K = xs.size
        left = np.concatenate(([-1.0], e[:-1]))
        right = np.concatenate((e[1:], [-1.0]))
        idx = np.nonzero((e >= left) & (e >= right))[0]
        if idx.size == 0:
            return []
        if idx.size > self.max_extrema:  # flat/noise-level curves: keep the largest
            idx = np.sort(idx[np.argsort(e[idx])[-self.max_extrema:]])
        lo = xs[np.maximum(idx - 1, 0)]
        hi = xs[np.minimum(idx + 1, K - 1)]
        t = np.linspace(0.0, 1.0, self.zoom)
        zx = (lo[:, None] + (hi - lo)[:, None] * t[None, :]).ravel()
        ze = self.errors(r, zx).reshape(idx.size, self.zoom)
        best = np.argmax(np.abs(ze), axis=1)
        out = []
        ev = self.errors(r, xs[idx])
        for j, i in enumerate(idx):
            xb, eb = zx[j * self.zoom + best[j]], ze[j, best[j]]
            if abs(eb) < abs(ev[j]):
                xb, eb = xs[i], ev[j]
            out.append((mpf(float(xb)), mpf(float(eb))))
        from .remez import _merge
        return _merge(out, self.width)
