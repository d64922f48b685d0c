"""Host-API throughput at configs[1]'s shape with pinned buffers (development
aid): boys_batch_many over n x at order k, both layouts, median of 3.

    python tools/probe_e2e.py [n] [k]
"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0)
    hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hx.copy_(x)
    hout = torch.empty(n * (k + 1), dtype=torch.float64, pin_memory=True)
    xs, out = hx.numpy(), hout.numpy()
    s = pkg.embedded_default()
    for lay in ("soa", "aos"):
        pkg.boys_batch_many(xs, k, s, out, layout=lay)
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            pkg.boys_batch_many(xs, k, s, out, layout=lay)
            ts.append(time.perf_counter() - t)
        el = statistics.median(ts)
        print("%s %s pinned k=%d n=%d: %.4f s  %.3e values/s  D2H %.1f GB/s" % (
            os.environ.get("TAG", ""), lay, k, n, el, n * (k + 1) / el, n * (k + 1) * 8 / el / 1e9), flush=True)


if __name__ == "__main__":
    main()
