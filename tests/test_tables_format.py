"""CPU tests of the coefficient-set plumbing (no GPU): the Python mirror
(paper_2512_10059_b200/tables.py) and the C++ shim (cpp/src/shim_tables.cpp)
against the reference's own parse_tables/emit_tables verdicts recorded in
tests/golden/tables_parse_cases.json (tables.cpp:14-160), and the embedded set
against the reference's embedded_default() (tables_data.cpp:8-412)."""
import os
import subprocess
import tempfile

import pytest

import paper_2512_10059_b200 as pkg
from conftest import ROOT, load_golden

CASES = load_golden("tables_parse_cases.json")


def _python_verdict(text):
    try:
        return 0, pkg.emit_tables(pkg.parse_tables(text))
    except pkg.TableParseError as e:
        return 8, str(e)
    except ValueError as e:
        return 4, str(e)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_python_parse_matches_reference(case):
    st, res = _python_verdict(case["text"])
    assert (st, res) == (case["status"], case["result"])


@pytest.fixture(scope="module")
def shim_test():
    from paper_2512_10059_b200 import build
    build.build_library(verbose=False)
    exe = build.build_shim_test()
    if exe is None:
        pytest.skip("no shim test source")
    return exe


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_cpp_shim_parse_matches_reference(case, shim_test):
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write(case["text"])
    try:
        out = subprocess.run([shim_test, "parse", f.name], capture_output=True, text=True, check=True).stdout
    finally:
        os.unlink(f.name)
    head, _, body = out.partition("\n")
    st = 0 if head == "OK" else int(head.split()[1])
    assert (st, body) == (case["status"], case["result"])


def test_embedded_default_matches_reference():
    emb = [c for c in CASES if c["name"] == "embedded_round_trip"][0]
    assert pkg.emit_tables(pkg.embedded_default()) == emb["text"]
    s = pkg.embedded_default()
    assert (s.k_max, s.eps_tol, s.x0, s.x1) == (32, 5e-14, 11.899848152108484, 28.98933773882074)
    assert [(r.degree_n(), r.degree_m()) for r in [s.r_B] + s.r_A][:5] == [(5, 6), (6, 9), (6, 10), (6, 10), (4, 12)]
    assert s.r_A[0].denom[0] == 4.59649054199579770e11
    assert all(r.denom[-1] == 1.0 for r in s.r_A)


def test_round_trip_is_bit_exact():
    s = pkg.embedded_default()
    t = pkg.parse_tables(pkg.emit_tables(s))
    assert t == s


def test_validate_tables_messages():
    import copy
    s = copy.deepcopy(pkg.embedded_default())
    s.r_A[7].denom[-1] = 0.99
    with pytest.raises(ValueError, match=r"tables: non-monic denominator in r_A\[7\]"):
        pkg.validate_tables(s)
    s = copy.deepcopy(pkg.embedded_default())
    s.r_A.pop()
    with pytest.raises(ValueError, match="need exactly k_max\\+1 region-A tables"):
        pkg.validate_tables(s)
    s = copy.deepcopy(pkg.embedded_default())
    s.x0 = 40.0
    with pytest.raises(ValueError, match="need 0 < x0 < x1"):
        pkg.validate_tables(s)


def test_data_file_is_the_committed_extraction():
    """The shipped data file is the one tools/extract_appendix_c.py wrote."""
    path = os.path.join(ROOT, "paper_2512_10059_b200", "data", "boys_minimax_k32.txt")
    emb = [c for c in CASES if c["name"] == "embedded_round_trip"][0]
    assert open(path).read() == emb["text"]
