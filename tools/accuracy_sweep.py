"""Accuracy at scale: verify_tables (GPU, double-double oracle) with
samples_per_region x per region (SPEC acceptance 1 uses 1e5) for the embedded
set, printed as one JSON line (profiles/r01_accuracy_sweep.json)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402


def main():
    spr = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    t = time.time()
    r = pkg.verify_tables(pkg.embedded_default(), spr, 200.0, seed)
    el = time.time() - t
    print(json.dumps({"samples_per_region": spr, "seed": seed, "xmax": 200.0, "seconds": el,
                      "max_err": r.max_err, "within_5e-14": r.all_within(5e-14), "worst_x": r.worst_x,
                      "worst_k": r.worst_k, "worst_region": r.worst_region,
                      "max_err_region": r.max_err_region,
                      "per_k": [[e.k, e.max_err_a, e.max_err_b, e.max_err_c] for e in r.per_k]}))


if __name__ == "__main__":
    main()
