"""Registers per kernel instantiation from build/obj/*.ptxas.log (development aid).

    python tools/ptxas_regs.py [obj_dir] [unit-substring]
"""
import glob
import os
import re
import sys


def main():
    obj = sys.argv[1] if len(sys.argv) > 1 else "build/obj"
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    for f in sorted(glob.glob(os.path.join(obj, "*.ptxas.log"))):
        if sub not in f:
            continue
        cur, out = None, {}
        for line in open(f):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                cur = m.group(1)
            m = re.search(r"Used (\d+) registers", line)
            if m and cur:
                km = re.search(r"kernelILi(\d+)ELi(\d+)E", cur)
                if km and km.group(2) != "23" and "ILi9ELi13ELi6ELi7E" not in cur:  # embedded variant only
                    out[int(km.group(1))] = int(m.group(1))
        if out:
            print(os.path.basename(f).replace(".cu.ptxas.log", ""), " ".join("%d:%d" % kv for kv in sorted(out.items())))


if __name__ == "__main__":
    main()
