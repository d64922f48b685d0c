#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY -- generates the committed golden fixtures under
tests/golden/ in the build container (where /root/reference exists):

  reference_rows.json     outputs of the UNMODIFIED reference hot path
                          (oracle/_ref: eval.cpp/tables*.cpp compiled as-is) on
                          seeded inputs, every double as a hex string (bit-exact)
  mpmath_truth.json       F_0..F_32 from mpmath at 50 digits (lower incomplete
                          gamma closed form), rounded to double once -- pins the
                          binary128 oracle (oracle/boys_hp.c)
  error_cases.json        the reference's status / message / partial rows for
                          invalid inputs (boys_batch_many, eval.cpp:88-96)
  tables_parse_cases.json the reference's parse_tables/emit_tables verdict on
                          well-formed and malformed table texts (tables.cpp:79-160)

    python oracle/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, HERE)
import pyoracle  # noqa: E402


def hexs(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def ulps(b, j):
    v = b
    step = np.inf if j > 0 else -np.inf
    for _ in range(abs(j)):
        v = np.nextafter(v, step)
    return float(v)


def boundary_set(x0, x1):
    xs = [0.0, 5e-324, 1e-300, 1e-30, 1e-12, 1e-6, 1e-3, 0.5, 1.0, 2.0, 5.0, 10.0, 15.0, 20.0, 28.0,
          29.0, 30.0, 35.0, 40.0, 50.0, 100.0, 200.0, 1e3, 7331.0, 1e4, 1e6, 1e300]
    for b in (x0, x1):
        xs += [ulps(b, j) for j in range(-8, 9)]
        xs += [b - 1e-9, b + 1e-9, b - 1e-6, b + 1e-6]
    return np.array(xs)


def reference_rows(port, ref):
    sets = {}
    # configs[0] shape: F_0..F_8 of uniform x in [0, 50] (the survey's splitmix stream, seed 1)
    x = port.gen_uniform(512, 1, 0.0, 50.0)
    sets["cfg0_uniform50_k8"] = (x, 8)
    sets["boundary_k32"] = (boundary_set(port.x0, port.x1), 32)
    u = port.gen_uniform(256, 3, 0.0, 1.0)
    sets["logu_k16"] = (10.0 ** (-12.0 + 16.0 * u), 16)
    out = {}
    for name, (xs, k) in sets.items():
        st, msg, o = ref.boys_batch_many(xs, k)
        assert st == 0, (name, msg)
        out[name] = {"k": k, "x": hexs(xs), "F": hexs(o)}
    # every order 0..32 on a mixed A/B/C sample
    for k in range(33):
        xs = port.gen_uniform(48, 100 + k, 0.0, 45.0)
        st, msg, o = ref.boys_batch_many(xs, k)
        assert st == 0
        out["sweep_k%d" % k] = {"k": k, "x": hexs(xs), "F": hexs(o)}
    # forced regions at the boundaries (the boys_batch_region seam)
    seam = []
    for b in (port.x0, port.x1):
        for x in (b - 1e-9, b, b + 1e-9):
            for reg in (0, 1, 2):
                for k in (0, 12, 32):
                    st, msg, o = ref.boys_batch_region(x, k, reg)
                    seam.append({"x": float(x).hex(), "k": k, "region": reg, "status": st, "F": hexs(o)})
    out["_region_seam"] = seam
    return out


def mpmath_truth(port):
    import mpmath as mp
    mp.mp.dps = 50
    xs = list(boundary_set(port.x0, port.x1))
    xs = [x for x in xs if x <= 1e4]
    xs += list(port.gen_uniform(40, 11, 0.0, 60.0))
    rows = []
    for x in xs:
        X = mp.mpf(x)
        vals = []
        for l in range(33):
            if x == 0:
                v = mp.mpf(1) / (2 * l + 1)
            else:
                a = l + mp.mpf(1) / 2
                v = mp.gammainc(a, 0, X) / (2 * X ** a)
            vals.append(float(v))
        rows.append({"x": float(x).hex(), "F": hexs(vals)})
    return {"dps": 50, "formula": "F_l(x) = gammainc(l+1/2, 0, x) / (2 x^(l+1/2)); F_l(0) = 1/(2l+1)",
            "rows": rows}


def error_cases(port, ref):
    cases = []
    good = port.gen_uniform(64, 5, 0.0, 40.0)

    def run(name, xs, k, out_len=None):
        xs = np.asarray(xs, dtype=np.float64)
        n_out = out_len if out_len is not None else max(xs.size * (k + 1), 0)
        o = np.full(max(n_out, 1), -7.0)
        st, msg, o = ref.boys_batch_many(xs, k, out=o, out_len=n_out)
        cases.append({"name": name, "x": hexs(xs), "k": k, "out_len": n_out, "status": st, "message": msg,
                      "out": hexs(o[:n_out]) if n_out > 0 else []})

    for pos, bad in ((0, np.nan), (5, -1.0), (17, np.inf), (63, -np.inf), (30, -0.0), (40, -1e-300)):
        xs = good.copy()
        xs[pos] = bad
        run("bad_%s_at_%d" % (repr(float(bad)), pos), xs, 6)
    run("k_too_large", good[:8], 33)
    run("k_negative", good[:8], -1)
    run("k_too_large_bad_x_first", np.concatenate([[np.nan], good[:4]]), 40)
    run("size_mismatch", good[:8], 4, out_len=8 * 5 - 1)
    run("empty_ok", np.zeros(0), 4)
    run("empty_bad_k", np.zeros(0), 99)
    run("x_zero", np.zeros(3), 32)
    return cases


PARSE_CASES = {
    "empty": "",
    "comments_only": "# nothing\n   \n",
    "bad_header": "boys-minimax v2 kmax=0 eps=1e-8 x0=1 x1=2\n",
    "negative_kmax": "boys-minimax v1 kmax=-1 eps=1e-8 x0=1 x1=2\n",
    "bad_eps": "boys-minimax v1 kmax=0 eps=abc x0=1 x1=2\n",
    "nonfinite_eps": "boys-minimax v1 kmax=0 eps=inf x0=1 x1=2\n",
    "minimal_ok": ("boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\n# B\ntable B k=0 n=0 m=0\n0.5\n1\n"
                   "table A k=0 n=1 m=1\n1.0\n-0.25\n2.0\n1.0\n"),
    "missing_B": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable A k=0 n=0 m=0\n1\n1\n",
    "missing_A": "boys-minimax v1 kmax=1 eps=1e-8 x0=1 x1=2\ntable B k=0 n=0 m=0\n1\n1\ntable A k=0 n=0 m=0\n1\n1\n",
    "non_monic": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=0 n=0 m=1\n1\n2\n0.99\n",
    "ended_early": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=0 n=1 m=1\n1\n2\n\n\n",
    "next_table_too_soon": ("boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=0 n=1 m=1\n1\n2\n"
                            "table A k=0 n=0 m=0\n1\n1\n"),
    "bad_coefficient": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=0 n=0 m=0\n1.0x\n1\n",
    "nan_coefficient": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=0 n=0 m=0\nnan\n1\n",
    "bad_table_header": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable C k=0 n=0 m=0\n1\n1\n",
    "negative_degree": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=0 n=-1 m=0\n1\n",
    "B_with_k1": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=1 n=0 m=0\n1\n1\n",
    "duplicate_B": ("boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable B k=0 n=0 m=0\n1\n1\n"
                    "table B k=0 n=0 m=0\n1\n1\n"),
    "A_out_of_range": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable A k=3 n=0 m=0\n1\n1\n",
    "duplicate_A": ("boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\ntable A k=0 n=0 m=0\n1\n1\n"
                    "table A k=0 n=0 m=0\n1\n1\n"),
    "x0_ge_x1": "boys-minimax v1 kmax=0 eps=1e-8 x0=3 x1=2\ntable B k=0 n=0 m=0\n1\n1\ntable A k=0 n=0 m=0\n1\n1\n",
    "hex_and_comments": ("# header follows\nboys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2  # trailing\n"
                         "table B k=0 n=0 m=0\n 0x1.8p-1 \t\n1\ntable A k=0 n=0 m=0\n+2.5e0\n1.0\n"),
    "crlf": "boys-minimax v1 kmax=0 eps=1e-8 x0=1 x1=2\r\ntable B k=0 n=0 m=0\r\n1\r\n1\r\ntable A k=0 n=0 m=0\r\n1\r\n1",
}


def parse_cases(ref):
    out = []
    for name, text in PARSE_CASES.items():
        st, res = ref.parse_emit(text)
        out.append({"name": name, "text": text, "status": st, "result": res})
    emb = ref.emit_embedded()
    st, res = ref.parse_emit(emb)
    out.append({"name": "embedded_round_trip", "text": emb, "status": st, "result": res})
    return out


def main():
    if not pyoracle.Ref.available():
        sys.exit("needs oracle/_ref (make -C oracle in the container with /root/reference)")
    port, ref = pyoracle.Port(), pyoracle.Ref()
    os.makedirs(GOLD, exist_ok=True)
    for fname, data in (("reference_rows.json", reference_rows(port, ref)),
                        ("error_cases.json", error_cases(port, ref)),
                        ("tables_parse_cases.json", parse_cases(ref)),
                        ("mpmath_truth.json", mpmath_truth(port))):
        with open(os.path.join(GOLD, fname), "w") as f:
            json.dump(data, f, indent=0)
        print("wrote", fname)


if __name__ == "__main__":
    main()
