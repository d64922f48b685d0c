"""Kernel timing sweep for A/B decisions (development aid; bench.py is the contract).

    python tools/quick_perf.py N k1,k2,.. layout[:path],.. [rounds]

Variants are interleaved round by round and the median per (variant, k) is
reported, so clock or neighbour drift does not favour whichever ran first.
Paths: soa:warp soa:block soa:binned soa:blocktma aos:xpose aos:binned aos:blocktma.
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402

HBM = 6541.5


def set_path(spec):
    lay, _, path = spec.partition(":")
    os.environ.pop("BOYSFN_SOA_PATH", None)
    os.environ.pop("BOYSFN_AOS_PATH", None)
    if path:
        os.environ["BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH"] = path
    return lay


def time_one(x, k, o, lay, reps=10):
    for _ in range(2):
        pkg.eval_device(x, k, o, layout=lay)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        pkg.eval_device(x, k, o, layout=lay)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    ks = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [32, 16, 8, 4, 0]
    specs = sys.argv[3].split(",") if len(sys.argv) > 3 else ["soa", "aos"]
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    if os.environ.get("QP_DIST") == "logu":
        pkg.generate_loguniform(x, 4, -12.0, 4.0)
    elif os.environ.get("QP_DIST") == "boundary":
        pkg.generate_boundary(x, 3)
    else:
        pkg.generate_uniform(x, 2, 0.0, 100.0)
    out = torch.empty(n * (max(ks) + 1), dtype=torch.float64, device="cuda")
    res = {}
    for _ in range(rounds):
        for k in ks:
            for spec in specs:
                lay = set_path(spec)
                res.setdefault((spec, k), []).append(time_one(x, k, out[: n * (k + 1)], lay))
    for k in ks:
        for spec in specs:
            ms = statistics.median(res[(spec, k)])
            gbs = n * (16 + 8 * k) / (ms * 1e-3) / 1e9
            print("%-10s k=%2d n=%d  %.3f ms (min %.3f max %.3f)  %.3e values/s  %5.0f GB/s  %5.1f%% of HBM"
                  % (spec, k, n, ms, min(res[(spec, k)]), max(res[(spec, k)]), n * (k + 1) / (ms * 1e-3), gbs,
                     100 * gbs / HBM), flush=True)


if __name__ == "__main__":
    main()
