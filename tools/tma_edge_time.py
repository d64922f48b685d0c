"""Kernel time of the SoA TMA store at its edges against the aligned case
(development aid): odd ld (odd n with ld = n), an 8-B-aligned output, and the
LSU block fallback for reference.  Short trains (tools/ab_time.py's method).

    python tools/tma_edge_time.py [N] [k]
"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def train(x, k, out, ld, m=8):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(m + 1)]
    ev[0].record()
    for j in range(m):
        pkg.eval_device(x, k, out, layout="soa", ld=ld)
        ev[j + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[j].elapsed_time(ev[j + 1]) for j in range(2, m))


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    x = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0)
    buf = torch.empty((k + 1) * (n + 16) + 2, dtype=torch.float64, device="cuda")
    cases = [("aligned, ld=n even (default)", x[:n], buf[: (k + 1) * n], n, None),
             ("aligned, tensor store", x[:n], buf[: (k + 1) * n], n, "blocktma"),
             ("aligned, per-row bulk copies", x[:n], buf[: (k + 1) * n], n, "blockbulk"),
             ("odd ld = n+1 (default)", x[: n + 1], buf[: (k + 1) * (n + 1)], n + 1, None),
             ("out 8 B off 16-B alignment", x[:n], buf[1: 1 + (k + 1) * n], n, None),
             ("LSU block (round-1 fallback)", x[:n], buf[: (k + 1) * n], n, "block"),
             ("odd ld = n+1, LSU block", x[: n + 1], buf[: (k + 1) * (n + 1)], n + 1, "block"),
             ("ld = n+2 (16 B, not 128 B rows)", x[:n], buf[: (k + 1) * (n + 2)], n + 2, None),
             ("ld = n+2, bulk", x[:n], buf[: (k + 1) * (n + 2)], n + 2, "blockbulk"),
             ("ld = n+16 (128 B rows)", x[:n], buf[: (k + 1) * (n + 16)], n + 16, None)]
    res = {}
    for _ in range(3):
        for name, xx, o, ld, path in cases:
            if path:
                os.environ["BOYSFN_SOA_PATH"] = path
            else:
                os.environ.pop("BOYSFN_SOA_PATH", None)
            pkg.eval_device(xx, k, o, layout="soa", ld=ld)
            torch.cuda.synchronize()
            time.sleep(0.2)
            res.setdefault(name, []).append(train(xx, k, o, ld))
    base = statistics.median(res[cases[0][0]])
    for name, xx, o, ld, path in cases:
        ms = statistics.median(res[name])
        nn = min(xx.numel(), ld)
        gbs = nn * (16 + 8 * k) / (ms * 1e-3) / 1e9
        print("k=%d %-32s %.4f ms  %6.0f GB/s  %.3f of aligned" % (k, name, ms, gbs, base / ms), flush=True)


if __name__ == "__main__":
    main()
