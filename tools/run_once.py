"""One evaluation per (layout[:path], k) on configs[1]'s input (1e8 U[0,100]),
for ncu captures (development aid).

    python tools/run_once.py soa:blocktma:8 aos:binned:8 ...
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def main():
    n = int(float(os.environ.get("RO_N", "1e8")))
    specs = [s.split(":") for s in sys.argv[1:]]
    kmax = max(int(s[-1]) for s in specs)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    if os.environ.get("RO_DIST") == "boundary":
        pkg.generate_boundary(x, 3)
    else:
        pkg.generate_uniform(x, 2, 0.0, 100.0)
    out = torch.empty(n * (kmax + 1), dtype=torch.float64, device="cuda")
    for s in specs:
        lay, k = s[0], int(s[-1])
        os.environ.pop("BOYSFN_SOA_PATH", None)
        os.environ.pop("BOYSFN_AOS_PATH", None)
        if len(s) == 3:
            os.environ["BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH"] = s[1]
        pkg.eval_device(x, k, out[: n * (k + 1)], layout=lay)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
