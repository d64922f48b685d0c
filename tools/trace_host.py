import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg
n, k = 5_000_000, 32
xs = np.random.default_rng(1).uniform(0, 100, n)
out = np.empty(n * (k + 1))
s = pkg.embedded_default()
pkg.boys_batch_many(xs, k, s, out, layout=sys.argv[1])
os.environ["BOYSFN_TRACE"] = "1"
t = time.time(); pkg.boys_batch_many(xs, k, s, out, layout=sys.argv[1]); print("total %.3f s  %.1f GB/s" % (time.time() - t, out.nbytes / (time.time() - t) / 1e9), flush=True)
