"""Host-API call time vs n for the small-batch (host-mapped) path and the
staged pipeline (development aid).   BOYSFN_SMALL_VALUES / BOYSFN_NO_SMALL_PATH select."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def main():
    s = pkg.embedded_default()
    rng = np.random.default_rng(1)
    for k in (8, 32):
        for n in (1000, 3000, 10000, 30000):
            xs = rng.uniform(0, 50, n)
            out = np.empty(n * (k + 1))
            row = []
            for mode in ("small", "pipeline"):
                if mode == "small":
                    os.environ["BOYSFN_SMALL_VALUES"] = str(1 << 20)
                    os.environ.pop("BOYSFN_NO_SMALL_PATH", None)
                else:
                    os.environ["BOYSFN_NO_SMALL_PATH"] = "1"
                pkg.boys_batch_many(xs, k, s, out)
                ts = []
                for _ in range(30):
                    t = time.perf_counter()
                    pkg.boys_batch_many(xs, k, s, out)
                    ts.append(time.perf_counter() - t)
                row.append(statistics.median(ts) * 1e6)
            print("k=%2d n=%6d values=%7d  small %8.1f us  pipeline %8.1f us" % (k, n, n * (k + 1), row[0], row[1]),
                  flush=True)


if __name__ == "__main__":
    main()
