"""Throughput of the run-time-k (generic) kernel for orders above 32
(development aid).  The table set is the embedded one with r_A[32] repeated
up to k_max = 64: numerically meaningless above 32, but the kernel does the
same work as for a real k_max = 64 set.   python tools/probe_generic.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402
from paper_2512_10059_b200 import tables as T  # noqa: E402


def main():
    e = pkg.embedded_default()
    if len(sys.argv) > 1:  # a table file (e.g. a generated set)
        t = T.parse_tables(open(sys.argv[1]).read())
    else:
        t = T.CoefficientTableSet(x0=e.x0, x1=e.x1, k_max=64, eps_tol=e.eps_tol, r_B=e.r_B,
                                  r_A=list(e.r_A) + [e.r_A[32]] * 32)
    n = 50_000_000
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0)
    out = torch.empty(n * 65, dtype=torch.float64, device="cuda")
    for k in tuple(int(v) for v in os.environ.get("PG_KS", "32,33,48,64").split(",")):
        for lay in ("soa", "aos"):
            o = out[: n * (k + 1)]
            pkg.eval_device(x, k, o, tables=t, layout=lay)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                pkg.eval_device(x, k, o, tables=t, layout=lay)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            print("k=%2d %s  %.3f ms  %.0f GB/s" % (k, lay, ms, n * (16 + 8 * k) / ms / 1e6), flush=True)


if __name__ == "__main__":
    main()
