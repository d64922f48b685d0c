"""Host<->device ceilings for the e2e number (development aid).

Pinned H2D / D2H bandwidth with CUDA events, and the host API
(boys_batch_many -> boysfn_eval_host) at k = 32 for both layouts with pinned
and pageable buffers, so the e2e figure in bench.py can be read against the
PCIe link it is bound by.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def bw(src, dst, reps=5):
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    return src.numel() * src.element_size() * reps / (a.elapsed_time(b) * 1e-3) / 1e9


def main():
    nbytes = 2 << 30
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    print("pinned H2D %.1f GB/s   D2H %.1f GB/s (2 GiB, one stream)" % (bw(h, d), bw(d, h)))
    n, k = 20_000_000, 32
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0)
    xs_pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xs_pin.copy_(x)
    out_pin = torch.empty(n * (k + 1), dtype=torch.float64, pin_memory=True)
    out_page = np.empty(n * (k + 1))
    s = pkg.embedded_default()
    for lay in ("soa", "aos"):
        for name, xs, out in (("pinned", xs_pin.numpy(), out_pin.numpy()), ("pageable", xs_pin.numpy().copy(), out_page)):
            pkg.boys_batch_many(xs, k, s, out, layout=lay)
            t = time.perf_counter()
            reps = 3
            for _ in range(reps):
                pkg.boys_batch_many(xs, k, s, out, layout=lay)
            el = (time.perf_counter() - t) / reps
            print("host API %s %-8s k=%d n=%d: %.3f s  %.3e values/s  D2H %.1f GB/s"
                  % (lay, name, k, n, el, n * (k + 1) / el, n * (k + 1) * 8 / el / 1e9))


if __name__ == "__main__":
    main()
