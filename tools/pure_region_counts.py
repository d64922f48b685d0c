"""Instructions per x of a kernel path on single-region inputs (development
aid; run under ncu --metrics smsp__inst_executed.sum): separates a low-k
kernel's fixed overhead and per-region arithmetic from its mixed-tile waste.

    python tools/pure_region_counts.py soa:sorted soa:binned ...   (k = 0, 1, 2)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402

N = 1 << 24


def main():
    t = pkg.embedded_default()
    bounds = {"A": (0.0, t.x0), "B": (t.x0, t.x1), "C": (t.x1, 100.0), "U": (0.0, 100.0)}
    xs = {}
    for r, (lo, hi) in bounds.items():
        x = torch.empty(N, dtype=torch.float64, device="cuda")
        pkg.generate_uniform(x, 11, lo, hi)
        if r != "U":
            x[x >= hi] = lo
        xs[r] = x
    out = torch.empty(N * 3, dtype=torch.float64, device="cuda")
    for spec in sys.argv[1:]:
        lay, path = spec.split(":")
        os.environ["BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH"] = path
        ks = [int(v) for v in os.environ.get("PR_K", "0,1,2").split(",")]
        regs = os.environ.get("PR_R", "ABCU")
        for k in ks:
            for r in regs:
                print(spec, k, r, flush=True)
                pkg.eval_device(xs[r], k, out[: N * (k + 1)], layout=lay)
        os.environ.pop("BOYSFN_SOA_PATH", None)
        os.environ.pop("BOYSFN_AOS_PATH", None)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
