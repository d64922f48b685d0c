"""CPU tests of the C-ABI library (no GPU): it loads, exports every entry point
include/boysfn_b200.h declares, validates table sets like validate_tables
(tables.cpp:14-32) on the host, and -- with no device -- refuses to evaluate
(BOYSFN_ERR_CUDA) instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2512_10059_b200 as pkg
from paper_2512_10059_b200 import _capi
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "boysfn_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(boysfn_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_bound_api():
    assert declared_functions() == sorted(_capi.exported_names())


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    nm = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (\w+)", nm))
    for name in declared_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_cpp_shim_symbols_exported():
    nm = subprocess.run(["nm", "-DC", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ("boysfn::boys_batch_many(std::span<double const", "boysfn::boys_batch(double, int",
                "boysfn::boys_batch_region(double, int", "boysfn::classify_region(double",
                "boysfn::embedded_default()", "boysfn::parse_tables(", "boysfn::emit_tables",
                "boysfn::validate_tables("):
        assert sym in nm, sym


def test_no_cudart_symbols_leak():
    """cudart is linked statically and kept local (build.py), so the library
    never binds to the libcudart another module (torch) loaded."""
    nm = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert not re.search(r"\bT cuda[A-Z]", nm)


def test_abi_and_status_strings():
    lib = _capi.lib()
    assert lib.boysfn_abi_version() == 2
    for st in range(8):
        assert lib.boysfn_status_string(st)


def test_embedded_handle_info():
    lib = _capi.lib()
    h = ctypes.c_void_p()
    assert lib.boysfn_tables_embedded(ctypes.byref(h)) == 0
    x0, x1, eps, km = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    assert lib.boysfn_tables_info(h, ctypes.byref(x0), ctypes.byref(x1), ctypes.byref(km), ctypes.byref(eps)) == 0
    s = pkg.embedded_default()
    assert (x0.value, x1.value, km.value, eps.value) == (s.x0, s.x1, s.k_max, s.eps_tol)


def test_tables_create_checks_only_what_the_device_needs():
    """eval.cpp never validates: a set it evaluates (non-monic denominator,
    eps_tol 0, x0 >= x1) loads; non-finite or empty coefficients do not.
    boysfn_tables_validate is validate_tables (tables.cpp:14-32)."""
    import copy
    lib = _capi.lib()
    h = pkg.DeviceTables(copy.deepcopy(pkg.embedded_default()))  # host-only: no device allocation
    h.close()
    bad = copy.deepcopy(pkg.embedded_default())
    bad.r_B.numer[2] = float("inf")
    with pytest.raises(ValueError, match="tables: non-finite value in r_B"):
        pkg.DeviceTables(bad)
    odd = copy.deepcopy(pkg.embedded_default())
    odd.eps_tol = 0.0
    odd.r_A[3].denom[-1] = 2.0
    pkg.DeviceTables(odd).close()
    nu = (ctypes.c_double * 1)(1.0)
    de = (ctypes.c_double * 1)(0.5)
    r = _capi.RationalDesc(0, 0, nu, de)
    ra = (_capi.RationalDesc * 1)(r)
    d = _capi.TableDesc(1.0, 2.0, 0, 1e-8, r, ra)
    out = ctypes.c_void_p()
    assert lib.boysfn_tables_create(ctypes.byref(d), ctypes.byref(out)) == 0
    lib.boysfn_tables_destroy(out)
    # validate_tables itself, through the C ABI: the reference's message
    assert lib.boysfn_tables_validate(ctypes.byref(d)) == _capi.ERR_TABLES
    assert _capi.last_error() == "tables: non-monic denominator in r_B"
    # verify_tables validates first (verify.cpp:14), before any device work
    with pytest.raises(ValueError, match="tables: eps_tol must be positive"):
        pkg.verify_tables(odd, 10)


def test_eval_device_size_check_needs_no_device():
    """boysfn_eval_device refuses an output shorter than the layout needs
    (AoS n(k+1), SoA k*ld+n) before touching the device."""
    lib = _capi.lib()
    h = ctypes.c_void_p()
    assert lib.boysfn_tables_embedded(ctypes.byref(h)) == 0
    fake = ctypes.c_void_p(1 << 20)  # never dereferenced: the check comes first
    n, k = 1000, 8
    assert lib.boysfn_eval_device(h, fake, n, k, fake, n * (k + 1) - 1, _capi.LAYOUT_AOS, 0, None, None) \
        == _capi.ERR_SIZE
    assert _capi.last_error() == "boys_batch_many: output span has wrong size"
    assert lib.boysfn_eval_device(h, fake, n, k, fake, k * 1024 + n - 1, _capi.LAYOUT_SOA, 1024, None, None) \
        == _capi.ERR_SIZE
    import torch
    x = torch.zeros(n, dtype=torch.float64)
    with pytest.raises(pkg.invalid_argument, match="CUDA"):
        pkg.eval_device(x, k, torch.zeros(n * (k + 1), dtype=torch.float64))
    with pytest.raises(pkg.invalid_argument, match="float64"):
        pkg.eval_device(x.float(), k, torch.zeros(n * (k + 1), dtype=torch.float64))


def test_host_side_argument_checks_need_no_device():
    """eval.cpp:88-96 ordering: the size check precedes everything and an empty
    batch returns before any device work, even with a bad k."""
    s = pkg.embedded_default()
    with pytest.raises(pkg.invalid_argument, match="boys_batch_many: output span has wrong size"):
        pkg.boys_batch_many(np.zeros(4), 3, s, np.zeros(15))
    pkg.boys_batch_many(np.zeros(0), 99, s, np.zeros(0))  # no throw, like the reference


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="a device is present")
def test_no_cpu_fallback_without_device():
    s = pkg.embedded_default()
    with pytest.raises(pkg.cuda_error):
        pkg.boys_batch_many(np.ones(8), 4, s, np.zeros(40))
