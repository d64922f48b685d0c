"""Low-k launch times right after a sustained high-k burst vs after an idle
gap (development aid): is the configs[2] sweep's slower k <= 2 the board's
power cap?   python tools/probe_powercap.py [N]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def times(x, k, out, m):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(m + 1)]
    ev[0].record()
    for j in range(m):
        pkg.eval_device(x, k, out[: x.numel() * (k + 1)], layout="soa")
        ev[j + 1].record()
    return ev


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_boundary(x, 3)
    out = torch.empty(n * 33, dtype=torch.float64, device="cuda")
    for k in (0, 1, 32):
        pkg.eval_device(x, k, out[: n * (k + 1)], layout="soa")
    torch.cuda.synchronize()
    for label, burst in (("after 1 s idle", 0), ("after 40 x k=32 (165 ms)", 40), ("after 200 x k=32 (0.8 s)", 200)):
        time.sleep(1.0)
        if burst:
            times(x, 32, out, burst)
        ev0 = times(x, 0, out, 12)
        ev1 = times(x, 1, out, 6)
        torch.cuda.synchronize()
        t0 = [ev0[j].elapsed_time(ev0[j + 1]) for j in range(12)]
        t1 = [ev1[j].elapsed_time(ev1[j + 1]) for j in range(6)]
        print("%-26s k=0: %s | k=1: %s" % (label, " ".join("%.3f" % v for v in t0), " ".join("%.3f" % v for v in t1)),
              flush=True)


if __name__ == "__main__":
    main()
