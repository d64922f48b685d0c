"""Coefficient-set data model, Python mirror of the reference's tables.hpp.

RationalApproximant / CoefficientTableSet / TableParseError / embedded_default /
validate_tables / parse_tables / emit_tables keep the names, members, checks,
diagnostics and the `boys-minimax v1` text format of
/root/reference/proj/core/include/boysfn/tables.hpp:12-49 and
/root/reference/proj/core/src/tables.cpp:14-160.  The embedded set is the
paper's Appendix C, shipped as data/boys_minimax_k32.txt (bit-identical to the
reference's embedded_default(), tables_data.cpp:8-412; see
tools/extract_appendix_c.py).  Host-side plumbing only: evaluation lives in the
CUDA library (eval.py).
"""
import math
import os
import re
from dataclasses import dataclass, field
from typing import List

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "boys_minimax_k32.txt")


@dataclass
class RationalApproximant:
    """p(x)/q(x), ascending degree, monic q (tables.hpp:12-17)."""
    numer: List[float] = field(default_factory=list)
    denom: List[float] = field(default_factory=list)

    def degree_n(self):
        return len(self.numer) - 1

    def degree_m(self):
        return len(self.denom) - 1


@dataclass
class CoefficientTableSet:
    """x0, x1, k_max, eps_tol, r_B, r_A[0..k_max] (tables.hpp:21-28)."""
    x0: float = 0.0
    x1: float = 0.0
    k_max: int = 0
    eps_tol: float = 0.0
    r_B: RationalApproximant = field(default_factory=RationalApproximant)
    r_A: List[RationalApproximant] = field(default_factory=list)


class TableParseError(RuntimeError):
    """tables.hpp:30-34: message 'line N: ...' and the line number."""

    def __init__(self, line, message):
        super().__init__("line %d: %s" % (line, message))
        self.line = line


def validate_tables(s):
    """tables.cpp:14-32; raises ValueError (std::invalid_argument) with the
    reference's messages, in the reference's order."""
    def bad(m):
        raise ValueError("tables: " + m)
    if s.k_max < 0:
        bad("k_max must be non-negative")
    if not (s.eps_tol > 0):
        bad("eps_tol must be positive")
    if not (s.x0 > 0 and s.x0 < s.x1):
        bad("need 0 < x0 < x1")
    if len(s.r_A) != s.k_max + 1:
        bad("need exactly k_max+1 region-A tables")

    def one(r, name):
        if not r.numer or not r.denom:
            bad("empty coefficient vector in " + name)
        if not all(math.isfinite(c) for c in list(r.numer) + list(r.denom)):
            bad("non-finite value in " + name)
        if r.denom[-1] != 1.0:
            bad("non-monic denominator in " + name)
    one(s.r_B, "r_B")
    for k, r in enumerate(s.r_A):
        one(r, "r_A[%d]" % k)


def _lines(text):
    """(line_no, content) of non-empty logical lines; '#' comments stripped,
    every physical line counted (the numbering of tables.cpp:42-63)."""
    parts = text.split("\n")
    if parts and parts[-1] == "":
        parts.pop()
    for no, raw in enumerate(parts, 1):
        body = raw.split("#", 1)[0].strip(" \t\r")
        if body:
            yield no, body


_C_INT = r"[ \t\n\r\f\v]*[-+]?\d+"


def _strtod(tok, line):
    """strtod over the whole token (tables.cpp:65-73)."""
    t = tok
    if not re.fullmatch(r"[-+]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?|inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?"
                        r"|0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][-+]?\d+)?)", t,
                        re.IGNORECASE):
        raise TableParseError(line, "expected a coefficient, got '%s'" % tok)
    low = t.lower().lstrip("+-")
    v = float.fromhex(t) if low.startswith("0x") else float(t)
    if not math.isfinite(v):
        raise TableParseError(line, "non-finite value '%s'" % tok)
    return v


def parse_tables(text):
    """`boys-minimax v1` text -> CoefficientTableSet (tables.cpp:79-144)."""
    it = iter(_lines(text))
    last = [0]

    def nxt():
        try:
            no, body = next(it)
        except StopIteration:
            return None
        last[0] = no
        return body

    # Physical line count for diagnostics raised at end of input.
    def eof_line():
        parts = text.split("\n")
        return len(parts) - 1 if parts and parts[-1] == "" else len(parts)

    hdr = nxt()
    if hdr is None:
        raise TableParseError(0, "empty input")
    # sscanf("boys-minimax v1 kmax=%d eps=%63s x0=%63s x1=%63s"): a blank in the
    # format matches any run of whitespace, including none.
    m = re.match(r"boys-minimax\s*v1\s*kmax=(%s)\s*eps=(\S{1,63})\s*x0=(\S{1,63})\s*x1=(\S{1,63})"
                 % _C_INT, hdr)
    if not m:
        raise TableParseError(last[0], "malformed header '%s'" % hdr)
    s = CoefficientTableSet()
    s.k_max = int(m.group(1))
    s.eps_tol = _strtod(m.group(2), last[0])
    s.x0 = _strtod(m.group(3), last[0])
    s.x1 = _strtod(m.group(4), last[0])
    if s.k_max < 0:
        raise TableParseError(last[0], "kmax must be non-negative")
    s.r_A = [RationalApproximant() for _ in range(s.k_max + 1)]
    seen_a = [False] * (s.k_max + 1)
    seen_b = False
    while True:
        line = nxt()
        if line is None:
            break
        th = re.match(r"table\s*(\S)\s*k=(%s)\s*n=(%s)\s*m=(%s)" % (_C_INT, _C_INT, _C_INT), line)
        if not th or th.group(1) not in "AB":
            raise TableParseError(last[0], "expected a table header, got '%s'" % line)
        kind, k, n, mm = th.group(1), int(th.group(2)), int(th.group(3)), int(th.group(4))
        if n < 0 or mm < 0:
            raise TableParseError(last[0], "negative degree")
        r = RationalApproximant()
        for i in range(n + mm + 2):
            c = nxt()
            if c is None:
                raise TableParseError(eof_line(), "wrong coefficient count: table ended early")
            if c.startswith("table "):
                raise TableParseError(last[0], "wrong coefficient count: next table too soon")
            (r.numer if i <= n else r.denom).append(_strtod(c, last[0]))
        if r.denom[-1] != 1.0:
            raise TableParseError(last[0], "non-monic denominator (top coefficient must be 1)")
        if kind == "B":
            if k != 0:
                raise TableParseError(last[0], "table B must have k=0")
            if seen_b:
                raise TableParseError(last[0], "duplicate table B")
            seen_b = True
            s.r_B = r
        else:
            if k < 0 or k > s.k_max:
                raise TableParseError(last[0], "table A k out of range")
            if seen_a[k]:
                raise TableParseError(last[0], "duplicate table A k=%d" % k)
            seen_a[k] = True
            s.r_A[k] = r
    if not seen_b:
        raise TableParseError(eof_line(), "missing table B")
    for k in range(s.k_max + 1):
        if not seen_a[k]:
            raise TableParseError(eof_line(), "missing table A k=%d" % k)
    validate_tables(s)
    return s


def _e17(v):
    return "%.16e" % v


def emit_tables(s):
    """CoefficientTableSet -> text, 17 significant digits (tables.cpp:146-160)."""
    validate_tables(s)
    out = ["boys-minimax v1 kmax=%d eps=%s x0=%s x1=%s" % (s.k_max, _e17(s.eps_tol), _e17(s.x0), _e17(s.x1))]

    def one(kind, k, r):
        out.append("table %s k=%d n=%d m=%d" % (kind, k, r.degree_n(), r.degree_m()))
        out.extend(_e17(c) for c in r.numer)
        out.extend(_e17(c) for c in r.denom)
    one("B", 0, s.r_B)
    for k in range(s.k_max + 1):
        one("A", k, s.r_A[k])
    return "\n".join(out) + "\n"


_EMBEDDED = None


def embedded_default():
    """The Appendix-C set (k_max=32, eps 5e-14), one shared immutable-by-convention
    instance (tables_data.cpp:8-412)."""
    global _EMBEDDED
    if _EMBEDDED is None:
        with open(_DATA) as f:
            _EMBEDDED = parse_tables(f.read())
    return _EMBEDDED
