"""Pageable-buffer host API, copy-pool vs per-call threads, interleaved
(development aid).   python tools/probe_pageable.py [n] [k] [rounds]"""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    xs = np.random.default_rng(1).uniform(0, 100, n)
    out = np.empty(n * (k + 1))
    s = pkg.embedded_default()
    pkg.boys_batch_many(xs, k, s, out)
    res = {"pool": []} if os.environ.get("PP_POOL_ONLY") else {"pool": [], "spawn": []}
    for _ in range(rounds):
        for mode in res:
            if mode == "spawn":
                os.environ["BOYSFN_COPY_SPAWN"] = "1"
            else:
                os.environ.pop("BOYSFN_COPY_SPAWN", None)
            for lay in ("aos",):
                t = time.perf_counter()
                pkg.boys_batch_many(xs, k, s, out, layout=lay)
                res[mode].append(out.nbytes / (time.perf_counter() - t) / 1e9)
    for mode, v in res.items():
        print("%-5s pageable aos k=%d n=%d: median %.1f GB/s  [%s]" % (
            mode, k, n, statistics.median(v), " ".join("%.1f" % a for a in v)))


if __name__ == "__main__":
    main()
