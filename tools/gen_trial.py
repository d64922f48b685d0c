"""Generator trial on the B200 (development aid): the device error scan
against working precision, r_B by remez_solve (5,6) and by walsh_search, and
one r_A table, with timings.   python tools/gen_trial.py [k_A]"""
import os
import sys
import time

import numpy as np
from mpmath import mpf

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_10059_b200 as pkg  # noqa: E402
import genport as gen  # noqa: E402
from genport import hp, scan  # noqa: E402
from genport.generate import search_table  # noqa: E402


def main():
    kA = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    emb = pkg.embedded_default()
    with hp.precision():
        x0, x1 = gen.compute_x0(32), gen.compute_x1(32, 5e-14)
        # 1. device scan vs working precision
        rng = np.random.default_rng(1)
        for k, w, r, a, b in ((0, "one", emb.r_B, float(x0), float(x1)), (kA, "rho_A", emb.r_A[kA], 0.0, float(x0))):
            xs = rng.uniform(a, b, 64)
            e = scan.error_scan(k, w, [mpf(c) for c in r.numer], [mpf(c) for c in r.denom], xs)
            f = hp.boys_target(k)
            dmax = 0
            for x, ev in zip(xs, e):
                rho = gen.weight_rho_A(k, x) if w == "rho_A" else 1
                num = gen.poly_eval([mpf(c) for c in r.numer], mpf(x))
                den = gen.poly_eval([mpf(c) for c in r.denom], mpf(x))
                ref = rho * (f(mpf(x)) - num / den)
                dmax = max(dmax, abs(float(ref) - ev))
            print("scan k=%d %s: max |device - mp| = %.3e (errors ~%.1e)" % (k, w, dmax, np.abs(e).max()), flush=True)
        # 2. remez (5,6) for r_B
        t = time.time()
        res = gen.remez_solve(gen.RemezProblem(f=hp.boys_target(0), a=x0, b=x1, n=5, m=6, eps_conv=mpf("5e-16"),
                                               scan=scan.GpuScan(0, "one")))
        xs = np.linspace(float(x0), float(x1), 1000)
        rel = 0
        for x in xs:
            mine = res.approximant.eval(mpf(x))
            ref = gen.poly_eval([mpf(c) for c in emb.r_B.numer], mpf(x)) / gen.poly_eval(
                [mpf(c) for c in emb.r_B.denom], mpf(x))
            rel = max(rel, abs(float((mine - ref) / ref)))
        print("remez r_B (5,6): status %s, %d iterations, %d reguesses, alternation %d, sup %.4e, %.1f s; "
              "max rel |r - embedded r_B| on 1000 points %.2e" % (res.status.name, res.iterations, res.reguesses,
                                                                  res.alternation_count, float(res.sup_error),
                                                                  time.time() - t, rel), flush=True)
    # 3. walsh r_B
    resB, rep = search_table(0, "B", x0, x1, 5e-14, 14)
    print("walsh r_B:", rep, flush=True)
    # 4. one r_A table
    resA, rep = search_table(kA, "A", mpf(0), x0, 5e-14, 24)
    print("walsh r_A[%d]:" % kA, rep, "embedded (n,m) = (%d,%d)" % (emb.r_A[kA].degree_n(), emb.r_A[kA].degree_m()),
          flush=True)


if __name__ == "__main__":
    main()
