"""Bitwise fingerprint of the evaluator's output for every order and layout on
fixed inputs (development aid: A/B builds must print identical lines).

    BOYSFN_LIB=... python tools/hash_outputs.py
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def main():
    n = 4_000_037
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 5, 0.0, 40.0)
    xb = torch.empty(1_000_003, dtype=torch.float64, device="cuda")
    pkg.generate_boundary(xb, 6)
    h = hashlib.sha256()
    for xs in (x, xb):
        out = torch.empty(xs.numel() * 33, dtype=torch.float64, device="cuda")
        for k in range(33):
            for lay in ("soa", "aos"):
                o = out[: xs.numel() * (k + 1)]
                pkg.eval_device(xs, k, o, layout=lay)
                h.update(o.view(torch.int64).cpu().numpy().tobytes())
    print(os.environ.get("BOYSFN_LIB", "product"), h.hexdigest())


if __name__ == "__main__":
    main()
