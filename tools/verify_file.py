"""verify_tables on the GPU for table files, per order and region (development aid).

    python tools/verify_file.py samples xmax seed file1 [file2 ...]    ('embedded' = Appendix C)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_10059_b200 as pkg  # noqa: E402
from paper_2512_10059_b200 import tables as T  # noqa: E402


def main():
    spr, xmax, seed = int(float(sys.argv[1])), float(sys.argv[2]), int(sys.argv[3])
    for path in sys.argv[4:]:
        t = pkg.embedded_default() if path == "embedded" else T.parse_tables(open(path).read())
        rep = pkg.verify_tables(t, spr, xmax, seed)
        print("%s: max_err %.4e at k=%d region %s x=%.17g" % (path, rep.max_err, rep.worst_k, rep.worst_region,
                                                             rep.worst_x))
        for e in rep.per_k:
            flag = " <-- over %.1e" % t.eps_tol if max(e.max_err_a, e.max_err_b, e.max_err_c) > t.eps_tol else ""
            print("  k=%2d A %.3e B %.3e C %.3e%s" % (e.k, e.max_err_a, e.max_err_b, e.max_err_c, flag))


if __name__ == "__main__":
    main()
