"""Short-train kernel timing for A/B decisions (development aid).

    python tools/ab_time.py N spec[,spec..] [rounds]     spec = layout:path:k (path '' = default)

Each measurement is a train of 8 back-to-back launches after 0.2 s idle,
CUDA-event timed per launch (median of the last 6): long trains at full HBM
write rate hit the board power cap and then measure the cap, not the kernel.
Specs are interleaved round by round; the median over rounds is printed.
"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def set_path(lay, path):
    os.environ.pop("BOYSFN_SOA_PATH", None)
    os.environ.pop("BOYSFN_AOS_PATH", None)
    if path:
        os.environ["BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH"] = path


def train(x, k, o, lay, m=8):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(m + 1)]
    ev[0].record()
    for j in range(m):
        pkg.eval_device(x, k, o, layout=lay)
        ev[j + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[j].elapsed_time(ev[j + 1]) for j in range(2, m))


def main():
    n = int(float(sys.argv[1]))
    specs = [s.split(":") for s in sys.argv[2].split(",")]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    kmax = max(int(s[2]) for s in specs)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    if os.environ.get("AB_DIST") == "logu":
        pkg.generate_loguniform(x, 4, -12.0, 4.0)
    elif os.environ.get("AB_DIST") == "boundary":
        pkg.generate_boundary(x, 3)
    else:
        pkg.generate_uniform(x, 2, 0.0, 100.0)
    out = torch.empty(n * (kmax + 1), dtype=torch.float64, device="cuda")
    res = {}
    for s in specs:  # warm every kernel once
        set_path(s[0], s[1])
        pkg.eval_device(x, int(s[2]), out[: n * (int(s[2]) + 1)], layout=s[0])
    for _ in range(rounds):
        for s in specs:
            lay, path, k = s[0], s[1], int(s[2])
            set_path(lay, path)
            time.sleep(0.2)
            res.setdefault(tuple(s), []).append(train(x, k, out[: n * (k + 1)], lay))
    for s in specs:
        k = int(s[2])
        ms = statistics.median(res[tuple(s)])
        gbs = n * (16 + 8 * k) / (ms * 1e-3) / 1e9
        print("%-4s %-12s k=%2d  %.4f ms  [%s]  %6.0f GB/s" % (
            s[0], s[1] or "default", k, ms, " ".join("%.3f" % v for v in res[tuple(s)]), gbs), flush=True)


if __name__ == "__main__":
    main()
