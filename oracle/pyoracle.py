"""TEST INFRASTRUCTURE ONLY -- Python access to the CPU checkers.

  Port      oracle/_build/libboys_oracle.so  C restatement of eval.cpp (Algorithm 1),
            bit-identical to the reference; plus the binary128 oracle (boys_hp.c).
  Ref       oracle/_ref/libboysfn_ref.so     the reference's own eval.cpp/tables*.cpp
            compiled unmodified (present when built in the container that has
            /root/reference; the prebuilt file travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
`--impl reference` arm) import this module.  It never imports the product
package; the coefficient set is read from the committed data file, which
tools/extract_appendix_c.py pinned bit-identical to the reference.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PORT_SO = os.path.join(HERE, "_build", "libboys_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libboysfn_ref.so")
TABLES_TXT = os.path.join(ROOT, "paper_2512_10059_b200", "data", "boys_minimax_k32.txt")

_dp = ctypes.POINTER(ctypes.c_double)


class _Rational(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("m", ctypes.c_int), ("numer", _dp), ("denom", _dp)]


class _Tables(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("x1", ctypes.c_double), ("k_max", ctypes.c_int),
                ("eps_tol", ctypes.c_double), ("r_B", _Rational), ("r_A", ctypes.POINTER(_Rational))]


def _read_tables(path=TABLES_TXT):
    """Minimal reader of the committed `boys-minimax v1` file (well-formed input)."""
    lines = [l.split("#")[0].strip() for l in open(path)]
    lines = [l for l in lines if l]
    head = dict(kv.split("=") for kv in lines[0].split()[2:])
    out = {"x0": float(head["x0"]), "x1": float(head["x1"]), "k_max": int(head["kmax"]),
           "eps": float(head["eps"]), "A": {}, "B": None}
    i = 1
    while i < len(lines):
        f = lines[i].split()
        kind, k, n, m = f[1], int(f[2][2:]), int(f[3][2:]), int(f[4][2:])
        vals = [float(v) for v in lines[i + 1:i + 1 + n + m + 2]]
        r = (np.array(vals[:n + 1]), np.array(vals[n + 1:]))
        if kind == "B":
            out["B"] = r
        else:
            out["A"][k] = r
        i += 1 + n + m + 2
    return out


class Port:
    """The C restatement (boys_port.c) and the binary128 oracle (boys_hp.c)."""

    def __init__(self):
        if not os.path.exists(PORT_SO):
            raise RuntimeError("oracle not built: run `make -C oracle`")
        L = ctypes.CDLL(PORT_SO)
        L.oracle_boys_batch_many.argtypes = [_dp, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_Tables), _dp,
                                             ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.oracle_boys_batch_many_mt.argtypes = [_dp, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_Tables),
                                                _dp, ctypes.c_int]
        L.oracle_boys_batch_region.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.POINTER(_Tables),
                                               ctypes.c_int, _dp]
        L.oracle_classify_region.argtypes = [ctypes.c_double, ctypes.POINTER(_Tables)]
        L.oracle_gen_uniform.argtypes = [_dp, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_double, ctypes.c_double]
        L.oracle_gen_loguniform.argtypes = L.oracle_gen_uniform.argtypes
        L.oracle_compare_output.argtypes = [_dp, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_Tables), _dp,
                                            ctypes.c_int, ctypes.c_size_t, ctypes.c_double, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_size_t),
                                            ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]
        L.oracle_gen_boundary.argtypes = L.oracle_gen_uniform.argtypes
        L.oracle_mt64_nth.argtypes = [ctypes.c_uint64, ctypes.c_size_t]
        L.oracle_mt64_nth.restype = ctypes.c_uint64
        L.oracle_verify_samples.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_size_t,
                                            ctypes.c_uint64, _dp]
        L.oracle_alg2_direct.argtypes = [_dp, _dp, ctypes.c_size_t, ctypes.c_int, _dp, ctypes.POINTER(_Tables), _dp,
                                         _dp, ctypes.c_int]
        L.oracle_hp_boys_batch_many.argtypes = [ctypes.c_int, _dp, ctypes.c_size_t, _dp, ctypes.c_int]
        L.oracle_hp_boys_batch.argtypes = [ctypes.c_int, ctypes.c_double, _dp]
        L.oracle_hp_series.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int]
        L.oracle_hp_series.restype = ctypes.c_double
        L.oracle_hp_closed_form.argtypes = [ctypes.c_int, ctypes.c_double]
        L.oracle_hp_closed_form.restype = ctypes.c_double
        L.oracle_hp_terms_for.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.oracle_hp_truncation_bound.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int]
        L.oracle_hp_truncation_bound.restype = ctypes.c_double
        self.L = L
        t = _read_tables()
        self._keep = []

        def rat(nd):
            nu, de = (np.ascontiguousarray(a, dtype=np.float64) for a in nd)
            self._keep.extend((nu, de))
            return _Rational(len(nu) - 1, len(de) - 1, nu.ctypes.data_as(_dp), de.ctypes.data_as(_dp))
        ra = (_Rational * (t["k_max"] + 1))(*[rat(t["A"][k]) for k in range(t["k_max"] + 1)])
        self._keep.append(ra)
        self.tables = _Tables(t["x0"], t["x1"], t["k_max"], t["eps"], rat(t["B"]), ra)
        self.x0, self.x1, self.k_max = t["x0"], t["x1"], t["k_max"]

    def boys_batch_many(self, xs, k, threads=1):
        """AoS (N, k+1) array, bit-identical to the reference; raises on bad input."""
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        out = np.zeros((xs.size, k + 1), dtype=np.float64)
        if threads > 1:
            st = self.L.oracle_boys_batch_many_mt(xs.ctypes.data_as(_dp), xs.size, k, ctypes.byref(self.tables),
                                                  out.ctypes.data_as(_dp), threads)
            bad = None
        else:
            badv = ctypes.c_size_t(0)
            st = self.L.oracle_boys_batch_many(xs.ctypes.data_as(_dp), xs.size, k, ctypes.byref(self.tables),
                                               out.ctypes.data_as(_dp), out.size, ctypes.byref(badv))
            bad = badv.value
        if st != 0:
            e = RuntimeError("oracle status %d" % st)
            e.status, e.first_bad, e.partial = st, bad, out
            raise e
        return out

    def boys_batch_region(self, x, k, region):
        out = np.zeros(k + 1)
        st = self.L.oracle_boys_batch_region(float(x), k, ctypes.byref(self.tables), int(region),
                                             out.ctypes.data_as(_dp))
        if st:
            raise RuntimeError("oracle status %d" % st)
        return out

    def classify(self, x):
        return self.L.oracle_classify_region(float(x), ctypes.byref(self.tables))

    def gen_uniform(self, n, seed, lo, hi, offset=0):
        x = np.empty(n, dtype=np.float64)
        self.L.oracle_gen_uniform(x.ctypes.data_as(_dp), n, seed, offset, lo, hi)
        return x

    def gen_loguniform(self, n, seed, log10_lo, log10_hi, offset=0):
        x = np.empty(n, dtype=np.float64)
        self.L.oracle_gen_loguniform(x.ctypes.data_as(_dp), n, seed, offset, log10_lo, log10_hi)
        return x

    def gen_boundary(self, n, seed, offset=0):
        x = np.empty(n, dtype=np.float64)
        self.L.oracle_gen_boundary(x.ctypes.data_as(_dp), n, seed, offset, self.x0, self.x1)
        return x

    def compare_output(self, xs, k, out, soa, ld=None, tol=5e-14, threads=None):
        """Every value of out (AoS, or SoA with row stride ld) against the
        restatement: (max |out - ref|, values above tol, region-C values that
        differ in any bit, region-C values checked)."""
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        assert out.dtype == np.float64 and out.flags.c_contiguous
        md, ot, cm, cv = ctypes.c_double(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        st = self.L.oracle_compare_output(xs.ctypes.data_as(_dp), xs.size, k, ctypes.byref(self.tables),
                                          out.ctypes.data_as(_dp), 1 if soa else 0, ld or xs.size, tol,
                                          threads or os.cpu_count() or 1, ctypes.byref(md), ctypes.byref(ot),
                                          ctypes.byref(cm), ctypes.byref(cv))
        if st:
            raise RuntimeError("compare status %d" % st)
        return md.value, ot.value, cm.value, cv.value

    def verify_samples(self, per_region, xmax=200.0, seed=1, x0=None, x1=None):
        """The x verify_tables draws (verify.cpp:23-33), regions A, B, C in order."""
        xs = np.empty(3 * per_region)
        self.L.oracle_verify_samples(self.x0 if x0 is None else x0, self.x1 if x1 is None else x1, xmax,
                                     per_region, seed, xs.ctypes.data_as(_dp))
        return xs

    def alg2(self, x, y, c, threads=None):
        """Algorithm 2 by direct summation: (z, sum_j |y_j w_ij|)."""
        x, y, c = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, y, c))
        z, za = np.zeros(x.size), np.zeros(x.size)
        st = self.L.oracle_alg2_direct(x.ctypes.data_as(_dp), y.ctypes.data_as(_dp), x.size, c.size - 1,
                                       c.ctypes.data_as(_dp), ctypes.byref(self.tables), z.ctypes.data_as(_dp),
                                       za.ctypes.data_as(_dp), threads or os.cpu_count() or 1)
        if st:
            raise RuntimeError("alg2 oracle status %d" % st)
        return z, za

    def hp(self, xs, kmax, threads=None):
        """Extended-precision F_0..F_kmax rounded to double, shape (N, kmax+1)."""
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        out = np.zeros((xs.size, kmax + 1))
        threads = threads or os.cpu_count() or 1
        st = self.L.oracle_hp_boys_batch_many(kmax, xs.ctypes.data_as(_dp), xs.size, out.ctypes.data_as(_dp),
                                              threads)
        if st:
            raise RuntimeError("hp oracle status %d" % st)
        return out


class Ref:
    """The compiled, unmodified reference (oracle/_ref/libboysfn_ref.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise RuntimeError("reference not built (needs /root/reference at build time)")
        L = ctypes.CDLL(REF_SO)
        L.ref_boys_batch_many.argtypes = [_dp, ctypes.c_size_t, ctypes.c_int, _dp, ctypes.c_size_t,
                                          ctypes.c_char_p, ctypes.c_size_t]
        L.ref_boys_batch_many_mt.argtypes = [_dp, ctypes.c_size_t, ctypes.c_int, _dp, ctypes.c_int]
        L.ref_boys_batch_region.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_char_p,
                                            ctypes.c_size_t]
        L.ref_classify_region.argtypes = [ctypes.c_double]
        L.ref_emit_embedded.restype = ctypes.c_size_t
        L.ref_parse_emit.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]
        self.L = L

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def boys_batch_many(self, xs, k, out=None, out_len=None):
        """Returns (status, message, out); out keeps the reference's partial rows."""
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        if out is None:
            out = np.zeros(max(xs.size * (k + 1), 0))
        msg = ctypes.create_string_buffer(256)
        st = self.L.ref_boys_batch_many(xs.ctypes.data_as(_dp), xs.size, k, out.ctypes.data_as(_dp),
                                        out.size if out_len is None else out_len, msg, 256)
        return st, msg.value.decode(), out

    def boys_batch_many_mt(self, xs, k, threads, out=None):
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        if out is None:
            out = np.empty(xs.size * (k + 1))
        st = self.L.ref_boys_batch_many_mt(xs.ctypes.data_as(_dp), xs.size, k, out.ctypes.data_as(_dp), threads)
        if st:
            raise RuntimeError("reference status %d" % st)
        return out

    def boys_batch_region(self, x, k, region):
        out = np.zeros(k + 1)
        msg = ctypes.create_string_buffer(256)
        st = self.L.ref_boys_batch_region(float(x), k, int(region), out.ctypes.data_as(_dp), msg, 256)
        return st, msg.value.decode(), out

    def parse_emit(self, text):
        buf = ctypes.create_string_buffer(1 << 20)
        st = self.L.ref_parse_emit(text.encode(), buf, len(buf))
        return st, buf.value.decode()

    def emit_embedded(self):
        n = self.L.ref_emit_embedded(None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        self.L.ref_emit_embedded(buf, n + 1)
        return buf.value.decode()
