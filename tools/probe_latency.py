"""Host-API latency for small batches (development aid): boys_batch_many with
pageable NumPy buffers at n = 1 .. 1e6, k = 8 and 32, median of 50 calls,
against the compiled reference (oracle/_ref) on one host thread."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2512_10059_b200 as pkg  # noqa: E402
import pyoracle  # noqa: E402


def med(fn, reps):
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts)


def main():
    s = pkg.embedded_default()
    ref = pyoracle.Ref()
    rng = np.random.default_rng(1)
    for k in (8, 32):
        for n in (1, 100, 10_000, 1_000_000):
            xs = rng.uniform(0, 50, n)
            out = np.empty(n * (k + 1))
            pkg.boys_batch_many(xs, k, s, out)
            reps = 50 if n <= 10_000 else 10
            tg = med(lambda: pkg.boys_batch_many(xs, k, s, out), reps)
            ro = np.empty(n * (k + 1))
            tr = med(lambda: ref.boys_batch_many(xs, k, out=ro), max(3, reps // 5))
            print("k=%2d n=%8d  B200 host API %9.1f us  reference 1 thread %10.1f us  ratio %.1f" % (
                k, n, tg * 1e6, tr * 1e6, tr / tg), flush=True)


if __name__ == "__main__":
    main()
