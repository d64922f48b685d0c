"""The generator pipeline of SPEC.md:475 (cmd_gen; section II.C-II.D):
x0 (Eq. 20), x1 (Eq. 12), then a Walsh-table search per table -- r_B for F_0
on [x0, x1] with rho = 1, r_A,k for F_k on [0, x0] with rho_A,k -- rounded once
to double and emitted in the reference's text format (tables.cpp:79-160).

The reference ships no driver for this pipeline (its CLI and tools/ are
absent); this module is the restatement of the specified pipeline on top of the
restated pieces (regions.py, remez.py) with the B200 extremum scan (scan.py).
"""
import dataclasses
import time
from typing import List, Optional

from mpmath import mpf

from paper_2512_10059_b200 import tables as T
from . import hp
from .regions import compute_x0, compute_x1, weight_rho_A
from .remez import WalshResult, walsh_search
from .scan import GpuScan


@dataclasses.dataclass
class TableReport:
    name: str
    k: int
    n: int
    m: int
    sup_error: float
    met_tolerance: bool
    cells: int
    seconds: float


@dataclasses.dataclass
class GenerateResult:
    tables: "T.CoefficientTableSet"
    reports: List[TableReport]
    x0: object
    x1: object
    alternatives: dict = dataclasses.field(default_factory=dict)  # k -> runner-up r_A cells


def _rational_to_double(res: WalshResult):
    num = [float(c) for c in res.approximant.numer]
    den = [float(c) for c in res.approximant.denom]
    den[-1] = 1.0  # monic, exact
    return T.RationalApproximant(numer=num, denom=den)


def search_table(k, region, a, b, eps_tol, max_total_degree=24, backend="gpu", rng_seed=1, trace=None):
    """One Walsh search: region "B" (F_0, rho = 1) or "A" (F_k, rho_A,k)."""
    f = hp.boys_target(k)
    rho = None if region == "B" else (lambda x, k=k: weight_rho_A(k, x))
    scan = None
    if backend == "gpu":
        scan = GpuScan(k, "one" if region == "B" else "rho_A")
    elif backend != "mp":
        raise ValueError("backend must be 'gpu' or 'mp'")
    t0 = time.time()
    res = walsh_search(f, rho, a, b, eps_tol, max_total_degree, rng_seed=rng_seed, trace=trace, scan=scan)
    rep = TableReport("B" if region == "B" else "A[%d]" % k, k, res.n, res.m, float(res.sup_error),
                      res.met_tolerance, len(res.cells), time.time() - t0)
    return res, rep


def _alternatives(res):
    return [(n, m, float(sup), _rational_to_double(WalshResult(approximant=r))) for n, m, sup, r in res.alternatives]


def _search_A_task(args):
    """Process-pool task: one r_A,k search, returned as plain floats."""
    k, x0, eps_tol, max_total_degree, backend, rng_seed = args
    with hp.precision():
        res, rep = search_table(k, "A", mpf(0), mpf(x0), eps_tol, max_total_degree, backend, rng_seed)
    rat = _rational_to_double(res) if res.approximant is not None else None
    return k, rat, rep, _alternatives(res)


def certify(tables, alternatives, samples=10000, xmax=200.0, seed=1, log=None):
    """verify_tables on the GPU (SPEC.md: gen output passes verify before gen
    reports success).  For an order whose region-A error exceeds eps_tol the
    next-best cell of its winning anti-diagonal is tried (same total degree,
    so the same cost; the selection rule of remez.cpp:571-576 ranks by the sup
    error of the exact rational, which does not see the rounding of the
    coefficients to double or the double-precision recurrence).  Returns
    (passed, report)."""
    from paper_2512_10059_b200.eval import verify_tables
    rep = verify_tables(tables, samples, xmax, seed)
    tried = {k: 0 for k in range(tables.k_max + 1)}
    while rep.max_err > tables.eps_tol:
        bad = [e.k for e in rep.per_k if e.max_err_a > tables.eps_tol]
        swapped = False
        for k in bad:
            alts = alternatives.get(k, [])
            if tried[k] + 1 < len(alts):
                tried[k] += 1
                n, m, sup, rat = alts[tried[k]]
                tables.r_A[k] = rat
                swapped = True
                if log is not None:
                    log.append("certify: r_A[%d] -> (%d,%d) sup %.3e" % (k, n, m, sup))
        if not swapped:
            return False, rep
        rep = verify_tables(tables, samples, xmax, seed)
    return True, rep


def generate_tables(k_max, eps_tol, max_total_degree=24, backend="gpu", orders: Optional[List[int]] = None,
                    rng_seed=1, trace=None, workers=1):
    """Build a CoefficientTableSet for (k_max, eps_tol).  `orders` restricts the
    r_A searches (the others are left empty, for partial runs and tests).
    `workers` > 1 runs the r_A searches in that many processes (the tables are
    independent, SPEC.md: "gen may run per-k Remez jobs concurrently"); each
    process drives the device scan through its own CUDA context."""
    with hp.precision():
        x0 = compute_x0(k_max)
        x1 = compute_x1(k_max, eps_tol)
    reports = []
    resB, rep = search_table(0, "B", x0, x1, eps_tol, max_total_degree, backend, rng_seed, trace)
    reports.append(rep)
    ks = [k for k in range(k_max + 1) if orders is None or k in orders]
    r_A = [None] * (k_max + 1)
    alternatives = {}
    if workers > 1 and len(ks) > 1:
        import concurrent.futures as cf
        import multiprocessing as mpc
        tasks = [(k, str(x0), eps_tol, max_total_degree, backend, rng_seed) for k in ks]
        with cf.ProcessPoolExecutor(max_workers=workers, mp_context=mpc.get_context("spawn")) as ex:
            # largest orders first: their searches are the longest
            for k, rat, rep, alts in ex.map(_search_A_task, sorted(tasks, key=lambda t: -t[0])):
                r_A[k] = rat
                alternatives[k] = alts
                reports.append(rep)
        reports[1:] = sorted(reports[1:], key=lambda r: r.k)
    else:
        for k in ks:
            resA, rep = search_table(k, "A", mpf(0), x0, eps_tol, max_total_degree, backend, rng_seed, trace)
            reports.append(rep)
            r_A[k] = _rational_to_double(resA) if resA.approximant is not None else None
            alternatives[k] = _alternatives(resA)
    tset = T.CoefficientTableSet(x0=float(x0), x1=float(x1), k_max=k_max, eps_tol=float(eps_tol),
                                 r_B=_rational_to_double(resB), r_A=r_A)
    return GenerateResult(tset, reports, x0, x1, alternatives)
