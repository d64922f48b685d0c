"""Weighted rational Remez exchange (Steps 1-6 of the paper's Fig. 1) and the
Walsh-table degree search.  Restates `remez.hpp`/`remez.cpp`:

  guess_nodes         uniform order statistics from std::mt19937_64 (remez.cpp:175-191)
  solve_fixed_nodes   Lagrange weights, node-orthonormal Stieltjes basis, symmetric
                      (m+1)x(m+1) eigenproblem for the denominator, Newton-Leja
                      interpolation for the numerator (remez.cpp:193-315)
  select_pole_free    Sturm count of the denominator on [a, b] (remez.cpp:317-337)
  golden_section_max  (remez.cpp:339-370)
  ErrorCurve          grid of 64*(n+m+2) points, local maxima refined by golden
                      section, merged (remez.cpp:33-108)
  select_alternating  N alternating extrema including the global maximum (remez.cpp:114-171)
  remez_solve         exchange loop with de la Vallee-Poussin check and the Step-6
                      early abort (remez.cpp:407-511)
  walsh_search        anti-diagonals n+m = 0, 1, ... (remez.cpp:513-581)

The extremum search has two interchangeable backends.  "mp" is the reference's
algorithm in working precision.  "gpu" (gen/scan.py) evaluates the weighted
error on a dense grid on the B200 in double-double and refines each local
maximum on a zoomed grid; the fixed-node solves stay in working precision.
"""
import dataclasses
import enum
from typing import Callable, List, Optional

import mpmath
from mpmath import mpf

from . import hp
from .linalg import jacobi_eigensolve
from .poly import leja_order, newton_interpolate, poly_eval, poly_trim, sturm_root_count


class MT19937_64:
    """std::mt19937_64 (the C++ standard's 64-bit Mersenne Twister)."""
    N, M = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    MASK = (1 << 64) - 1

    def __init__(self, seed=5489):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.mti = self.N

    def __call__(self):
        if self.mti >= self.N:
            mt, N, M = self.mt, self.N, self.M
            for i in range(N):
                x = (mt[i] & self.UM) | (mt[(i + 1) % N] & self.LM)
                xa = x >> 1
                if x & 1:
                    xa ^= self.MATRIX_A
                mt[i] = mt[(i + M) % N] ^ xa
            self.mti = 0
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & self.MASK


class RemezStatus(enum.IntEnum):
    Converged = 0
    Infeasible = 1
    IterationLimit = 2
    ReguessLimit = 3


@dataclasses.dataclass
class RationalHP:
    numer: List
    denom: List

    def eval(self, x):
        return poly_eval(self.numer, x) / poly_eval(self.denom, x)


@dataclasses.dataclass
class RemezProblem:
    f: Callable
    rho: Optional[Callable] = None  # None => 1
    a: object = 0
    b: object = 1
    n: int = 0
    m: int = 0
    eps_conv: object = 0
    abort_error_tol: object = 0  # <= 0 disables the Step-6 abort
    grid_points: int = 0         # 0 => 64*(n+m+2)
    rng_seed: int = 1
    max_iterations: int = 200
    max_reguesses: int = 100
    trace: object = None         # a list collecting trace lines
    scan: object = None          # None: "mp" backend; else a gen.scan.GpuScan for (f, rho)


@dataclasses.dataclass
class RemezIterationRecord:
    levelled_error_abs: object
    sup_error: object


@dataclasses.dataclass
class RemezResult:
    status: RemezStatus = RemezStatus.IterationLimit
    approximant: Optional[RationalHP] = None
    nodes: list = dataclasses.field(default_factory=list)
    sup_error: object = 0
    levelled_error: object = 0
    lower_bound: object = 0
    iterations: int = 0
    reguesses: int = 0
    alternation_count: int = 0
    node_error_spread: object = 0
    monotonicity_warnings: int = 0
    history: list = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class FixedNodeCandidate:
    numer: list
    denom: list
    denom_node_values: list
    levelled_error: object
    residual: object


@dataclasses.dataclass
class NodeUpdate:
    ok: bool = False
    nodes: list = dataclasses.field(default_factory=list)
    sup_error: object = 0
    min_node_error: object = 0


def _validate(p):
    if p.f is None:
        raise ValueError("remez: target function not set")
    if not (mpf(p.a) < mpf(p.b)):
        raise ValueError("remez: need a < b")
    if p.n < 0 or p.m < 0:
        raise ValueError("remez: degrees must be non-negative")
    N = p.n + p.m + 2
    if p.grid_points != 0 and p.grid_points < 4 * N:
        raise ValueError("remez: grid_points must be at least 4*(n+m+2)")
    if mpf(p.eps_conv) < 0:
        raise ValueError("remez: eps_conv must be >= 0")


def _rho(p, x):
    return p.rho(x) if p.rho is not None else mpf(1)


def _sign(v):
    return 1 if v > 0 else (-1 if v < 0 else 0)


def golden_section_max(g, a, b, tol):
    """Argmax of a unimodal g on [a, b] to within tol (remez.cpp:339-370)."""
    tol = mpf(tol)
    if not tol > 0:
        raise ValueError("golden_section_max: tol must be positive")
    sqrt5 = mpmath.sqrt(5)
    invphi = (sqrt5 - 1) / 2
    invphi2 = (3 - sqrt5) / 2
    lo, hi = mpf(a), mpf(b)
    h = hi - lo
    if h <= tol:
        return (lo + hi) / 2
    c = lo + invphi2 * h
    d = lo + invphi * h
    yc, yd = g(c), g(d)
    while h > tol:
        if yc >= yd:
            hi, d, yd = d, c, yc
            h = hi - lo
            c = lo + invphi2 * h
            yc = g(c)
        else:
            lo, c, yc = c, d, yd
            h = hi - lo
            d = lo + invphi * h
            yd = g(d)
    return (lo + hi) / 2


class ErrorCurve:
    """Grid scan plus golden-section refinement of rho (f - r) (remez.cpp:33-108)."""

    def __init__(self, p):
        self.p = p
        N = p.n + p.m + 2
        K = p.grid_points or 64 * N
        a, b = mpf(p.a), mpf(p.b)
        self.xs = [a + (b - a) * i / (K - 1) for i in range(K)]
        self.fv = [p.f(x) for x in self.xs]
        self.rv = [_rho(p, x) for x in self.xs]
        self.golden_tol = (b - a) * mpf(10) ** (-(hp.working_digits() * 2 // 5))

    def error_at(self, r, x):
        return _rho(self.p, x) * (self.p.f(x) - r.eval(x))

    def refined_extrema(self, r):
        p = self.p
        K = len(self.xs)
        e = [self.rv[i] * (self.fv[i] - r.eval(self.xs[i])) for i in range(K)]
        out = []
        for i in range(K):
            ai = abs(e[i])
            if i > 0 and ai < abs(e[i - 1]):
                continue
            if i + 1 < K and ai < abs(e[i + 1]):
                continue
            lo = mpf(p.a) if i == 0 else self.xs[i - 1]
            hi = mpf(p.b) if i + 1 == K else self.xs[i + 1]
            xs = golden_section_max(lambda x: abs(self.error_at(r, x)), lo, hi, self.golden_tol)
            es = self.error_at(r, xs)
            if abs(es) < ai:
                xs, es = self.xs[i], e[i]
            out.append((xs, es))
        return _merge(out, mpf(p.b) - mpf(p.a))


def _merge(out, width):
    out.sort(key=lambda t: t[0])
    close = width * mpf(10) ** (-(hp.working_digits() // 3))
    merged = []
    for ex in out:
        if merged and ex[0] - merged[-1][0] < close:
            if abs(ex[1]) > abs(merged[-1][1]):
                merged[-1] = ex
        else:
            merged.append(ex)
    return merged


def select_alternating(extrema, N, levelled_error_abs):
    """N alternating-sign extrema incl. the global maximum (remez.cpp:114-171)."""
    upd = NodeUpdate(sup_error=mpf(0))
    for _, v in extrema:
        if abs(v) > upd.sup_error:
            upd.sup_error = abs(v)
    floor_level = levelled_error_abs * (1 - mpf(10) ** -10)
    alt = []
    for ex in extrema:
        s = _sign(ex[1])
        if s == 0 or abs(ex[1]) < floor_level:
            continue
        if alt and _sign(alt[-1][1]) == s:
            if abs(ex[1]) > abs(alt[-1][1]):
                alt[-1] = ex
        else:
            alt.append(ex)
    if len(alt) < N:
        return upd

    def global_index():
        g = 0
        for i in range(1, len(alt)):
            if abs(alt[i][1]) > abs(alt[g][1]):
                g = i
        return g

    while len(alt) > N:
        g = global_index()
        if len(alt) == N + 1:
            if abs(alt[0][1]) <= abs(alt[-1][1]):
                alt.pop(0)
            else:
                alt.pop()
            continue
        best, best_score = None, mpf(0)
        for i in range(len(alt) - 1):
            if i == g or i + 1 == g:
                continue
            score = max(abs(alt[i][1]), abs(alt[i + 1][1]))
            if best is None or score < best_score:
                best, best_score = i, score
        if best is None:
            return upd
        del alt[best:best + 2]
    upd.ok = True
    upd.nodes = [x for x, _ in alt]
    upd.min_node_error = min(abs(v) for _, v in alt)
    return upd


def guess_nodes(problem, rng):
    """N = n+m+2 sorted distinct uniform draws on [a, b] (remez.cpp:175-191)."""
    N = problem.n + problem.m + 2
    a, b = mpf(problem.a), mpf(problem.b)
    width = b - a
    for _ in range(1000):
        nodes = sorted(a + width * mpf((rng() >> 11) * 2.0 ** -53) for _ in range(N))
        if all(nodes[i] - nodes[i - 1] >= width * mpf("1e-12") for i in range(1, N)):
            return nodes
    raise RuntimeError("guess_nodes: could not draw distinct nodes")


def solve_fixed_nodes(nodes, fvals, rhovals, n, m):
    """All pole-free-or-not candidates of rho (f - p/q)(x_i) = (-1)^i E
    (remez.cpp:193-315)."""
    N = n + m + 2
    if len(nodes) != N or len(fvals) != N or len(rhovals) != N:
        raise ValueError("solve_fixed_nodes: need n+m+2 nodes and matching values")
    omega = []
    for i in range(N):
        prod = mpf(1)
        for j in range(N):
            if j != i:
                prod *= nodes[i] - nodes[j]
        if prod == 0:
            return []
        omega.append(1 / prod)
    mu = []
    for i in range(N):
        if not rhovals[i] > 0:
            raise ValueError("solve_fixed_nodes: weight must be positive")
        mu.append(abs(omega[i]) / rhovals[i])

    def dot(u, v):
        return mpmath.fsum(mu[i] * u[i] * v[i] for i in range(N))

    phi = [[mpf(0)] * N for _ in range(m + 1)]
    phi_mono = [None] * (m + 1)
    norm0 = mpmath.sqrt(mpmath.fsum(mu))
    phi[0] = [1 / norm0] * N
    phi_mono[0] = [1 / norm0]
    prev, bprev, prev_mono = None, mpf(0), None
    for j in range(m):
        w = [nodes[i] * phi[j][i] for i in range(N)]
        aj = dot(w, phi[j])
        for i in range(N):
            w[i] -= aj * phi[j][i]
            if j > 0:
                w[i] -= bprev * prev[i]
        bj = mpmath.sqrt(dot(w, w))
        if bj == 0:
            return []
        w = [wi / bj for wi in w]
        wm = [mpf(0)] * (len(phi_mono[j]) + 1)
        for c, pc in enumerate(phi_mono[j]):
            wm[c + 1] += pc
            wm[c] -= aj * pc
        if j > 0:
            for c, pc in enumerate(prev_mono):
                wm[c] -= bprev * pc
        wm = [c / bj for c in wm]
        prev, prev_mono, bprev = phi[j], phi_mono[j], bj
        phi[j + 1], phi_mono[j + 1] = w, wm

    A = [[mpf(0)] * (m + 1) for _ in range(m + 1)]
    for s in range(m + 1):
        for t in range(s, m + 1):
            A[s][t] = A[t][s] = mpmath.fsum(omega[i] * fvals[i] * phi[s][i] * phi[t][i] for i in range(N))
    values, vectors = jacobi_eigensolve(A)
    e_sign = 1 if (N - 1) % 2 == 0 else -1
    scale = max(abs(rhovals[i] * fvals[i]) for i in range(N))
    d = hp.working_digits()
    residual_tol = mpf(10) ** (-(d - 8))
    order = leja_order(nodes)
    out = []
    for j in range(m + 1):
        E = e_sign * values[j]
        qv = [mpmath.fsum(vectors[j][s] * phi[s][i] for s in range(m + 1)) for i in range(N)]
        qmono = [mpf(0)] * (m + 1)
        for s in range(m + 1):
            for c, pc in enumerate(phi_mono[s]):
                qmono[c] += vectors[j][s] * pc
        qmax = max(abs(v) for v in qv)
        if not qmax > 0:
            continue
        qtiny = qmax * mpf(10) ** (-(d + hp.GUARD_DIGITS - 6))
        if any(abs(v) <= qtiny for v in qv):
            continue
        pxs, pys = [], []
        for t in range(n + 1):
            i = order[t]
            sigma = 1 if i % 2 == 0 else -1
            pxs.append(nodes[i])
            pys.append((fvals[i] - sigma * E / rhovals[i]) * qv[i])
        numer = newton_interpolate(pxs, pys)
        res = mpf(0)
        for i in range(N):
            sigma = 1 if i % 2 == 0 else -1
            v = rhovals[i] * (fvals[i] - poly_eval(numer, nodes[i]) / qv[i]) - sigma * E
            res = max(res, abs(v))
        denom_scale = max(abs(E), scale) or mpf(1)
        cand = FixedNodeCandidate(numer, qmono, qv, E, res / denom_scale)
        if cand.residual <= residual_tol:
            out.append(cand)
    return out


def select_pole_free(candidates, a, b):
    """The candidate whose denominator has no root in [a, b] (remez.cpp:317-337)."""
    best = None
    trim_tol = mpf(10) ** (-(hp.working_digits() + hp.GUARD_DIGITS - 8))
    a, b = mpf(a), mpf(b)
    for cand in candidates:
        q = poly_trim(cand.denom, trim_tol)
        if len(q) == 1:
            if q[0] == 0:
                continue
        else:
            maxc = max(abs(c) for c in q)
            if abs(poly_eval(q, a)) <= maxc * trim_tol:
                continue
            if sturm_root_count(q, a, b) != 0:
                continue
        if best is None or cand.residual < best.residual:
            best = cand
    return best


def update_nodes(problem, r, levelled_error_abs):
    """Step 5 for the current approximant (remez.cpp:372-378)."""
    _validate(problem)
    with hp.precision():
        curve = problem.scan.bind(problem) if problem.scan is not None else ErrorCurve(problem)
        return select_alternating(curve.refined_extrema(r), problem.n + problem.m + 2, levelled_error_abs)


def _finalize_monic(cand):
    trim_tol = mpf(10) ** (-(hp.working_digits() - 4))
    denom = poly_trim(cand.denom, trim_tol)
    lead = denom[-1]
    denom = [c / lead for c in denom]
    denom[-1] = mpf(1)
    numer = [c / lead for c in cand.numer]
    return RationalHP(numer, denom)


def _trace(p, line):
    if p.trace is not None:
        p.trace.append(line)


def remez_solve(problem):
    """The exchange loop of Fig. 1 (remez.cpp:407-511)."""
    _validate(problem)
    with hp.precision():
        return _remez_solve(problem)


def _remez_solve(problem):
    res = RemezResult()
    N = problem.n + problem.m + 2
    rng = MT19937_64(problem.rng_seed)
    curve = problem.scan.bind(problem) if problem.scan is not None else ErrorCurve(problem)
    a, b = mpf(problem.a), mpf(problem.b)
    nodes = guess_nodes(problem, rng)
    prev_absE = mpf(-1)
    while True:
        fvals = [problem.f(x) for x in nodes]
        rhovals = [_rho(problem, x) for x in nodes]

        def reguess():
            nonlocal nodes, prev_absE
            if res.reguesses >= problem.max_reguesses:
                return False
            res.reguesses += 1
            nodes = guess_nodes(problem, rng)
            prev_absE = mpf(-1)
            return True

        sel = select_pole_free(solve_fixed_nodes(nodes, fvals, rhovals, problem.n, problem.m), a, b)
        if sel is None:
            if reguess():
                continue
            res.status = RemezStatus.ReguessLimit
            return res
        res.iterations += 1
        r = RationalHP(sel.numer, sel.denom)
        absE = abs(sel.levelled_error)
        upd = select_alternating(curve.refined_extrema(r), N, absE)
        sup = upd.sup_error
        if absE > sup * (1 + mpf(10) ** -10):
            raise ArithmeticError("remez_solve: de la Vallee-Poussin inequality violated")
        if prev_absE >= 0 and absE < prev_absE * (1 - mpf(10) ** -20):
            res.monotonicity_warnings += 1
            _trace(problem, "remez warning: |E| decreased")
        prev_absE = absE
        res.history.append(RemezIterationRecord(absE, sup))
        _trace(problem, "remez n=%d m=%d iter=%d E=%s sup=%s" % (
            problem.n, problem.m, res.iterations, mpmath.nstr(absE, 6), mpmath.nstr(sup, 6)))
        if sup - absE <= mpf(problem.eps_conv):
            res.status = RemezStatus.Converged
            res.approximant = _finalize_monic(sel)
            res.sup_error = sup
            res.levelled_error = sel.levelled_error
            if upd.ok:
                res.nodes = upd.nodes
                res.alternation_count = len(upd.nodes)
                errs = [abs(curve.error_at(r, x)) for x in upd.nodes]
                res.node_error_spread = max(errs) - min(errs)
            else:
                res.nodes = nodes
                res.alternation_count = 0
                res.node_error_spread = mpf(0)
            return res
        if not upd.ok:
            if reguess():
                continue
            res.status = RemezStatus.ReguessLimit
            return res
        if mpf(problem.abort_error_tol) > 0 and upd.min_node_error > mpf(problem.abort_error_tol):
            res.status = RemezStatus.Infeasible
            res.lower_bound = upd.min_node_error
            res.sup_error = sup
            res.levelled_error = sel.levelled_error
            return res
        if res.iterations >= problem.max_iterations:
            res.status = RemezStatus.IterationLimit
            res.sup_error = sup
            res.levelled_error = sel.levelled_error
            return res
        nodes = upd.nodes


@dataclasses.dataclass
class WalshCell:
    n: int
    m: int
    status: RemezStatus
    sup_error: object = 0
    lower_bound: object = 0


@dataclasses.dataclass
class WalshResult:
    met_tolerance: bool = False
    approximant: Optional[RationalHP] = None
    n: int = 0
    m: int = 0
    sup_error: object = 0
    cells: list = dataclasses.field(default_factory=list)
    # every cell of the winning anti-diagonal that met the tolerance, best
    # first, as (n, m, sup_error, approximant): the runners-up of the selection
    alternatives: list = dataclasses.field(default_factory=list)


def walsh_search(f, rho, a, b, eps_tol, max_total_degree, rng_seed=1, require_numer_le_denom=False,
                 eps_conv=0, trace=None, scan=None):
    """Minimal n+m meeting eps_tol, ties on the winning anti-diagonal broken by
    the smallest error; cells pruned by the Step-6 abort (remez.cpp:513-581)."""
    eps = mpf(eps_tol)
    if not eps > 0:
        raise ValueError("walsh_search: eps_tol must be positive")
    result = WalshResult()
    have_best = False
    with hp.precision():
        for d in range(max_total_degree + 1):
            hit, best = False, WalshResult()
            for n in range(d + 1):
                m = d - n
                if require_numer_le_denom and n > m:
                    continue
                seed = (rng_seed + 0x9E3779B97F4A7C15 * (n * 64 + m + 1)) & ((1 << 64) - 1)
                prob = RemezProblem(f=f, rho=rho, a=a, b=b, n=n, m=m,
                                    eps_conv=mpf(eps_conv) if mpf(eps_conv) > 0 else eps / 100,
                                    abort_error_tol=eps, rng_seed=seed, trace=trace, scan=scan)
                cell = _remez_solve(prob)
                result.cells.append(WalshCell(n, m, cell.status, cell.sup_error, cell.lower_bound))
                if trace is not None:
                    trace.append("walsh cell (%d,%d) status=%d sup=%s lb=%s" % (
                        n, m, int(cell.status), mpmath.nstr(cell.sup_error, 6), mpmath.nstr(cell.lower_bound, 6)))
                if cell.status == RemezStatus.Converged:
                    if not have_best or cell.sup_error < result.sup_error:
                        have_best = True
                        result.approximant, result.n, result.m = cell.approximant, n, m
                        result.sup_error = cell.sup_error
                    if cell.sup_error <= eps:
                        best.alternatives.append((n, m, cell.sup_error, cell.approximant))
                        if not hit or cell.sup_error < best.sup_error:
                            hit = True
                            best.approximant, best.n, best.m, best.sup_error = cell.approximant, n, m, cell.sup_error
            if hit:
                best.met_tolerance = True
                best.cells = result.cells
                best.alternatives.sort(key=lambda t: t[2])
                return best
    result.met_tolerance = False
    return result
