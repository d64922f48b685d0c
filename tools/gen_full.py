"""Full table generation for (kmax, eps) on the B200 box, compared with the
embedded Appendix-C set and self-verified on the GPU (development aid).

    python tools/gen_full.py 32 5e-14 16 out.txt
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_10059_b200 as pkg  # noqa: E402
from paper_2512_10059_b200 import tables as T  # noqa: E402
from genport.generate import generate_tables  # noqa: E402


def rat(r, x):
    return np.polyval(r.numer[::-1], x) / np.polyval(r.denom[::-1], x)


def main():
    kmax, eps, workers, out = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    t = time.time()
    res = generate_tables(kmax, eps, workers=workers)
    from genport.generate import certify
    log = []
    ok, _ = certify(res.tables, res.alternatives, 10000, log=log)
    print("\n".join(log), "certified" if ok else "NOT certified", flush=True)
    print("generated in %.1f s" % (time.time() - t), flush=True)
    with open(out, "w") as f:
        f.write(T.emit_tables(res.tables))
    emb = pkg.embedded_default()
    same_deg = 0
    for rep in res.reports:
        e = emb.r_B if rep.name == "B" else (emb.r_A[rep.k] if kmax == emb.k_max else None)
        tag = ""
        if e is not None:
            tag = "embedded (%d,%d)" % (e.degree_n(), e.degree_m())
            same_deg += (e.degree_n(), e.degree_m()) == (rep.n, rep.m)
        print("%-6s n=%2d m=%2d sup=%.4e met=%s cells=%3d %7.1fs  %s" % (
            rep.name, rep.n, rep.m, rep.sup_error, rep.met_tolerance, rep.cells, rep.seconds, tag), flush=True)
    print("degree profile identical to the embedded set for %d of %d tables" % (same_deg, len(res.reports)))
    rep = pkg.verify_tables(res.tables, 10000, 200.0, 7)
    print("verify_tables(generated, 1e4/region): max_err %.4e at k=%d region %s (eps %.1e) -> %s" % (
        rep.max_err, rep.worst_k, rep.worst_region, eps, "PASS" if rep.max_err <= eps else "FAIL"))


if __name__ == "__main__":
    main()
