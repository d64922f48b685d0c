"""python -m paper_2512_10059_b200.gen regions --kmax 32 --eps 5e-14
   python -m paper_2512_10059_b200.gen gen --kmax 32 --eps 5e-14 --out tables.txt [--orders 0,1,2]
                                          [--backend gpu|mp] [--workers 16]

The `regions` and `gen` subcommands of SPEC.md:464-480 (the reference's CLI is
absent from /root/reference).  Exit codes as specified there: 0 success,
1 input error, 2 verification failure, 3 internal non-convergence.  `gen`
verifies the generated set on the GPU before writing it (SPEC.md: gen output
always passes verify), trying the runner-up cells of an order's winning
anti-diagonal when the rounded-to-double table misses eps_tol."""
import argparse
import sys

from .. import tables as T
from .generate import certify, generate_tables
from .regions import compute_x0, compute_x1


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2512_10059_b200.gen")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("regions")
    r.add_argument("--kmax", type=int, required=True)
    r.add_argument("--eps", type=float, required=True)
    g = sub.add_parser("gen")
    g.add_argument("--kmax", type=int, required=True)
    g.add_argument("--eps", type=float, required=True)
    g.add_argument("--out", required=True)
    g.add_argument("--orders", default=None, help="comma-separated subset of r_A orders (partial run)")
    g.add_argument("--max-degree", type=int, default=24)
    g.add_argument("--backend", default="gpu", choices=["gpu", "mp"])
    g.add_argument("--workers", type=int, default=1, help="processes for the r_A searches")
    g.add_argument("--verify-samples", type=int, default=10000, help="verify_tables samples per region")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "regions":
            print("x0=%.17g x1=%.17g" % (float(compute_x0(a.kmax)), float(compute_x1(a.kmax, a.eps))))
            return 0
        orders = [int(v) for v in a.orders.split(",")] if a.orders else None
        res = generate_tables(a.kmax, a.eps, a.max_degree, a.backend, orders, workers=a.workers)
    except ValueError as e:
        print("error: %s" % e, file=sys.stderr)
        return 1
    for rep in res.reports:
        print("%-6s n=%2d m=%2d sup=%.3e met=%s cells=%d %.1fs" % (rep.name, rep.n, rep.m, rep.sup_error,
                                                                rep.met_tolerance, rep.cells, rep.seconds))
    if not all(rep.met_tolerance for rep in res.reports):
        return 3
    if orders is None:
        log = []
        ok, vrep = certify(res.tables, res.alternatives, a.verify_samples, log=log)
        for line in log:
            print(line)
        print("verify_tables: max_err %.4e at k=%d region %s -> %s" % (
            vrep.max_err, vrep.worst_k, vrep.worst_region, "PASS" if ok else "FAIL"))
        if not ok:
            return 2
        with open(a.out, "w") as f:
            f.write(T.emit_tables(res.tables))
    return 0


if __name__ == "__main__":
    sys.exit(main())
