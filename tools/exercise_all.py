"""Small end-to-end exercise of every kernel family: all output paths at ragged
sizes, the generic kernel, the region seam, the host pipeline with an error
mid-batch, verify_tables and Algorithm 2.  Run it against the checked build
(python -m paper_2512_10059_b200.build --variant checked BOYSFN_DEVICE_CHECKS,
BOYSFN_LIB=.../variants/checked/libboysfn_b200.so): every shared-memory and
global index the kernels form is then asserted in range on the device
(compute-sanitizer is closed on this GPU pool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402

PATHS = [("soa", "warp"), ("soa", "block"), ("soa", "binned"), ("soa", "blocktma"), ("soa", "blocktmabin"),
         ("aos", "xpose"), ("aos", "binned"), ("aos", "blocktma"), ("aos", "blocktmabin"),
         ("soa", "blockbulk"), ("soa", "blockbulkw"), ("soa", "blockbulkw3")]


def main():
    s = pkg.embedded_default()
    for n in (1, 33, 129, 1000, 4099):
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        pkg.generate_uniform(x, n, 0.0, 45.0)
        for k in (0, 1, 2, 5, 8, 15, 16, 31, 32):
            # SoA with an odd ld and with an output 8 B off a 16-B boundary (bulk store, default path)
            for shift, ld in ((0, n + 1), (1, n), (1, n + 3)):
                buf = torch.empty(shift + (k + 1) * ld, dtype=torch.float64, device="cuda")
                pkg.eval_device(x, k, buf[shift:], layout="soa", ld=ld)
            for lay, path in PATHS:
                os.environ["BOYSFN_SOA_PATH" if lay == "soa" else "BOYSFN_AOS_PATH"] = path
                out = torch.empty(n * (k + 1), dtype=torch.float64, device="cuda")
                pkg.eval_device(x, k, out, layout=lay)
                os.environ.pop("BOYSFN_SOA_PATH", None)
                os.environ.pop("BOYSFN_AOS_PATH", None)
            os.environ["BOYSFN_GENERIC"] = "1"
            out = torch.empty(n * (k + 1), dtype=torch.float64, device="cuda")
            pkg.eval_device(x, k, out, layout="aos")
            os.environ.pop("BOYSFN_GENERIC")
    torch.cuda.synchronize()
    xs = np.random.default_rng(1).uniform(0, 40, 5000)
    xs[3000] = np.nan
    out = np.empty(xs.size * 9)
    try:
        pkg.boys_batch_many(xs, 8, s, out)
    except pkg.domain_error:
        pass
    for r in (pkg.Region.A, pkg.Region.B, pkg.Region.C):
        pkg.boys_batch_region(15.0, 12, s, r)
    pkg.verify_tables(s, 50)
    z = pkg.alg2(torch.rand(300, dtype=torch.float64, device="cuda") * 30,
                 torch.rand(300, dtype=torch.float64, device="cuda"), np.ones(13))
    torch.cuda.synchronize()
    print("exercise done", float(z.sum()))


if __name__ == "__main__":
    main()
