"""Ad-hoc kernel timing sweep (development aid; bench.py is the contract).

    python tools/quick_perf.py [N] [k,k,...] [layouts]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402

HBM = 6541.5


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    ks = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [32, 16, 8, 4, 0]
    layouts = sys.argv[3].split(",") if len(sys.argv) > 3 else ["soa", "aos"]
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0)
    out = torch.empty(n * 33, dtype=torch.float64, device="cuda")
    for lay in layouts:
        for k in ks:
            o = out[: n * (k + 1)]
            for _ in range(3):
                pkg.eval_device(x, k, o, layout=lay)
            torch.cuda.synchronize()
            reps = 10
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(reps):
                pkg.eval_device(x, k, o, layout=lay)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1]) / reps
            gbs = n * (16 + 8 * k) / (ms * 1e-3) / 1e9
            print("layout=%s k=%2d n=%d  %.3f ms  %.3e values/s  %.0f GB/s  %.1f%% of HBM"
                  % (lay, k, n, ms, n * (k + 1) / (ms * 1e-3), gbs, 100 * gbs / HBM), flush=True)


if __name__ == "__main__":
    main()
