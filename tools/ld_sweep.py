"""SoA kernel time against the row stride ld (development aid): the 33 row
streams of an SoA tile land on DRAM channels according to ld, so the same
kernel runs at different rates for different ld.

    python tools/ld_sweep.py [N] [k] [path]
"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2512_10059_b200 as pkg  # noqa: E402
from tma_edge_time import train  # noqa: E402


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    path = sys.argv[3] if len(sys.argv) > 3 else ""
    if path:
        os.environ["BOYSFN_SOA_PATH"] = path
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0)
    pads = [0, 1, 2, 3, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 4096, 65536 - n % 65536]
    if os.environ.get("LD_PADS"):
        pads = [int(v) for v in os.environ["LD_PADS"].split(",")]
    buf = torch.empty((k + 1) * (n + max(pads)), dtype=torch.float64, device="cuda")
    res = {}
    for _ in range(3):
        for p in pads:
            ld = n + p
            o = buf[: (k + 1) * ld]
            pkg.eval_device(x, k, o, layout="soa", ld=ld)
            torch.cuda.synchronize()
            time.sleep(0.1)
            res.setdefault(p, []).append(train(x, k, o, ld))
    for p in pads:
        ms = statistics.median(res[p])
        print("k=%d path=%s ld=n+%-6d (ld*8 mod 1024 = %4d)  %.4f ms  %6.0f GB/s" % (
            k, path or "default", p, (n + p) * 8 % 1024, ms, n * (16 + 8 * k) / (ms * 1e-3) / 1e9), flush=True)


if __name__ == "__main__":
    main()
