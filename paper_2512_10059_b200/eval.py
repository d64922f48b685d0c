"""Evaluation API, Python mirror of the reference's eval.hpp, on the GPU.

Same names and semantics as /root/reference/proj/core/include/boysfn/eval.hpp:
  boys_batch_many(xs, k, tables, out)   eval.hpp:43-45 / eval.cpp:88-96
  boys_batch(x, k, tables)              eval.hpp:37    / eval.cpp:83-86
  boys_batch_region(x, k, tables, r)    eval.hpp:39-41 / eval.cpp:59-81
  classify_region(x, tables)            eval.hpp:23    / eval.cpp:22-26
Exceptions mirror the reference's C++ types (invalid_argument, domain_error,
out_of_range) with its messages; rows before the first bad x are written and
later rows untouched.  Every value is computed by the sm_100a kernels of
libboysfn_b200.so through the C ABI (include/boysfn_b200.h); there is no CPU
fallback.  `eval_device` is the HBM-resident entry point (torch CUDA tensors).
"""
import ctypes
import enum
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _capi
from .tables import CoefficientTableSet, embedded_default, validate_tables


class invalid_argument(ValueError):
    """std::invalid_argument."""


class domain_error(ValueError):
    """std::domain_error."""


class out_of_range(IndexError):
    """std::out_of_range."""


class cuda_error(RuntimeError):
    """A CUDA runtime failure (no reference equivalent)."""


class unsupported(RuntimeError):
    """A table degree the device image cannot hold (> 23), or Algorithm 2 with k > 32."""


def _raise(status, first_bad=None):
    if status == _capi.OK:
        return
    msg = _capi.last_error()
    exc = {
        _capi.ERR_SIZE: invalid_argument,
        _capi.ERR_DOMAIN: domain_error,
        _capi.ERR_RANGE: out_of_range,
        _capi.ERR_TABLES: invalid_argument,
        _capi.ERR_CUDA: cuda_error,
        _capi.ERR_ARG: invalid_argument,
        _capi.ERR_UNSUPPORTED: unsupported,
        _capi.ERR_INVALID: invalid_argument,
    }.get(status, RuntimeError)(msg)
    if first_bad is not None:
        exc.first_bad = first_bad
    raise exc


class Region(enum.IntEnum):
    """eval.hpp:17."""
    A = 0
    B = 1
    C = 2


@dataclass
class BoysBatch:
    """eval.hpp:11-15."""
    x: float = 0.0
    k: int = 0
    values: List[float] = field(default_factory=list)


class DeviceTables:
    """Device table handle for a CoefficientTableSet (boysfn_tables_t)."""

    def __init__(self, tables):
        L = _capi.lib()
        self._h = ctypes.c_void_p()
        self._owned = tables is not embedded_default()
        if not self._owned:
            _raise(L.boysfn_tables_embedded(ctypes.byref(self._h)))
            return
        # eval.cpp evaluates any set it is given; the device image needs only
        # k_max+1 region-A tables with finite coefficients (checked by
        # boysfn_tables_create).  Extra r_A entries are ignored.
        if len(tables.r_A) < tables.k_max + 1:
            raise invalid_argument("tables: need exactly k_max+1 region-A tables")
        keep = []

        def desc(r):
            nu = np.ascontiguousarray(r.numer, dtype=np.float64)
            de = np.ascontiguousarray(r.denom, dtype=np.float64)
            keep.extend((nu, de))
            return _capi.RationalDesc(len(nu) - 1, len(de) - 1,
                                      nu.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      de.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        ra = (_capi.RationalDesc * (tables.k_max + 1))(*[desc(r) for r in tables.r_A[: tables.k_max + 1]])
        d = _capi.TableDesc(tables.x0, tables.x1, tables.k_max, tables.eps_tol, desc(tables.r_B), ra)
        _raise(L.boysfn_tables_create(ctypes.byref(d), ctypes.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h and self._owned:
            _capi.lib().boysfn_tables_destroy(self._h)
        self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_EMB_HANDLE = None


def _handle(tables):
    global _EMB_HANDLE
    if tables is embedded_default():
        if _EMB_HANDLE is None:
            _EMB_HANDLE = DeviceTables(tables)
        return _EMB_HANDLE
    return DeviceTables(tables)


def classify_region(x, tables):
    """Half-open [0,x0)->A, [x0,x1)->B, [x1,inf)->C (eval.cpp:22-26)."""
    if x < tables.x0:
        return Region.A
    if x < tables.x1:
        return Region.B
    return Region.C


def boys_batch_many(xs, k, tables, out, layout="aos", ld=None):
    """Host-buffer bulk entry (eval.cpp:88-96).  xs: float64 array of N x;
    out: writable float64 array of N*(k+1) (AoS, row i = F_0..F_k(x_i)) or,
    with layout="soa", ld*(k+1) doubles laid out out[l*ld+i]."""
    L = _capi.lib()
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous):
        raise invalid_argument("out must be a C-contiguous float64 numpy array")
    lay = _capi.LAYOUT_SOA if layout == "soa" else _capi.LAYOUT_AOS
    h = _handle(tables)
    bad = ctypes.c_size_t(0)
    st = L.boysfn_eval_host(h.handle, xs.ctypes.data, xs.size, int(k), out.ctypes.data, out.size, lay,
                            int(ld if ld is not None else xs.size), ctypes.byref(bad))
    _raise(st, bad.value if st == _capi.ERR_DOMAIN else None)


class _PinnedBlock:
    """Owner of one boysfn_host_alloc block; freed when the last view dies."""

    def __init__(self, nbytes):
        self.ptr = ctypes.c_void_p()
        _raise(_capi.lib().boysfn_host_alloc(nbytes, ctypes.byref(self.ptr)))

    def __del__(self):
        try:
            if self.ptr:
                _capi.lib().boysfn_host_free(self.ptr)
        except Exception:
            pass


class PinnedArray(np.ndarray):
    """numpy view of a boysfn_host_alloc block; the block is freed when the
    array and every view of it are gone."""


def host_empty(n):
    """An uninitialised float64 numpy array of n elements in page-locked host
    memory (boysfn_host_alloc): boys_batch_many reads and writes it with the
    copy engines directly instead of through pinned staging."""
    n = int(n)
    if n <= 0:
        return np.empty(0)
    blk = _PinnedBlock(n * 8)
    arr = np.frombuffer((ctypes.c_double * n).from_address(blk.ptr.value), dtype=np.float64).view(PinnedArray)
    arr._block = blk  # views keep `arr` (their base) and so the block alive
    return arr


def set_devices(devices=None):
    """Spread large boys_batch_many calls over these CUDA devices (contiguous
    shards, one host thread and staging pipeline each); None or [] restores
    the calling thread's current device only (boysfn_set_devices)."""
    devs = list(devices or [])
    arr = (ctypes.c_int * max(len(devs), 1))(*devs)
    _raise(_capi.lib().boysfn_set_devices(arr, len(devs)))


def boys_batch(x, k, tables):
    """One argument (eval.cpp:83-86)."""
    out = np.empty(max(int(k) + 1, 0), dtype=np.float64)
    if k < 0 or k > tables.k_max:
        # same order of checks as check_input: x first, then k
        boys_batch_many(np.array([x], dtype=np.float64), k, tables,
                        np.empty(int(k) + 1 if k >= 0 else 0, dtype=np.float64))
    boys_batch_many(np.array([x], dtype=np.float64), k, tables, out)
    return BoysBatch(float(x), int(k), out.tolist())


def boys_batch_region(x, k, tables, region):
    """Forced region (eval.cpp:59-81), evaluated by the device kernel."""
    L = _capi.lib()
    out = np.empty(max(int(k) + 1, 1), dtype=np.float64)
    h = _handle(tables)
    _raise(L.boysfn_eval_region_host(h.handle, float(x), int(k), int(region), out.ctypes.data))
    return BoysBatch(float(x), int(k), out[: int(k) + 1].tolist())


def _check_device_tensor(name, t, dtype, device=None):
    """A tensor handed to the C ABI as a raw device pointer: right dtype,
    contiguous, on a CUDA device (the same one as x)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise invalid_argument("%s must be a torch CUDA tensor" % name)
    if t.dtype != dtype:
        raise invalid_argument("%s must be %s, got %s" % (name, dtype, t.dtype))
    if not t.is_cuda:
        raise invalid_argument("%s must be on a CUDA device" % name)
    if device is not None and t.device != device:
        raise invalid_argument("%s is on %s, x on %s" % (name, t.device, device))
    if not t.is_contiguous():
        raise invalid_argument("%s must be contiguous" % name)


def eval_device(x, k, out, tables=None, layout="soa", ld=None, stream=None, first_bad=None):
    """HBM-resident entry point: x a CUDA float64 tensor of N arguments, out a
    CUDA float64 tensor (at least k*ld+N doubles for SoA, N*(k+1) for AoS;
    boysfn_eval_device checks the size).  Enqueued on `stream` (default:
    torch's current stream), asynchronous.  first_bad: an optional CUDA int64
    tensor lowered to the smallest invalid index."""
    import torch
    if layout not in ("soa", "aos"):
        raise invalid_argument("layout must be 'soa' or 'aos'")
    _check_device_tensor("x", x, torch.float64)
    _check_device_tensor("out", out, torch.float64, x.device)
    if first_bad is not None:
        _check_device_tensor("first_bad", first_bad, torch.int64, x.device)
        if first_bad.numel() < 1:
            raise invalid_argument("first_bad must hold one element")
    L = _capi.lib()
    tables = tables if tables is not None else embedded_default()
    h = _handle(tables)
    n = x.numel()
    lay = _capi.LAYOUT_SOA if layout == "soa" else _capi.LAYOUT_AOS
    ld = n if ld is None else int(ld)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    st = L.boysfn_eval_device(h.handle, x.data_ptr(), n, int(k), out.data_ptr(), out.numel(), lay, ld,
                              ctypes.c_void_p(s.cuda_stream),
                              first_bad.data_ptr() if first_bad is not None else None)
    _raise(st)


def generate_uniform(x, seed, lo, hi, offset=0, stream=None):
    """Fill CUDA tensor x with the splitmix64 uniform stream (boysfn_b200.h)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    _raise(_capi.lib().boysfn_generate_uniform(x.data_ptr(), x.numel(), seed, offset, lo, hi,
                                               ctypes.c_void_p(s.cuda_stream)))


def generate_loguniform(x, seed, log10_lo, log10_hi, offset=0, stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    _raise(_capi.lib().boysfn_generate_loguniform(x.data_ptr(), x.numel(), seed, offset, log10_lo,
                                                  log10_hi, ctypes.c_void_p(s.cuda_stream)))


def generate_boundary(x, seed, offset=0, tables=None, stream=None):
    """configs[2] boundary-stress stream around 0+, x0 and x1 (boysfn_b200.h)."""
    import torch
    t = tables if tables is not None else embedded_default()
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    _raise(_capi.lib().boysfn_generate_boundary(x.data_ptr(), x.numel(), seed, offset, t.x0, t.x1,
                                                ctypes.c_void_p(s.cuda_stream)))


def alg2(x, y, c, k=None, z=None, tables=None, stream=None):
    """Algorithm 2: z_i = sum_l c_l sum_j F_l(x_i + x_j) y_j on
    the device.  x, y: CUDA float64 tensors of n; c: k+1 host floats; returns
    z (a new CUDA tensor unless given).  Asynchronous on `stream`."""
    import torch
    c = np.ascontiguousarray(c, dtype=np.float64).ravel()
    k = len(c) - 1 if k is None else int(k)
    if k < 0 or len(c) < k + 1:
        raise invalid_argument("alg2: c needs k+1 = %d coefficients, got %d" % (k + 1, len(c)))
    _check_device_tensor("x", x, torch.float64)
    _check_device_tensor("y", y, torch.float64, x.device)
    if y.numel() != x.numel():
        raise invalid_argument("alg2: y must have as many elements as x")
    if z is None:
        z = torch.empty_like(x)
    _check_device_tensor("z", z, torch.float64, x.device)
    if z.numel() != x.numel():
        raise invalid_argument("alg2: z must have as many elements as x")
    tables = tables if tables is not None else embedded_default()
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    h = _handle(tables)  # keep the handle alive across the call
    _raise(_capi.lib().boysfn_alg2_device(h.handle, x.data_ptr(), y.data_ptr(), x.numel(), k,
                                          c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), z.data_ptr(),
                                          ctypes.c_void_p(s.cuda_stream)))
    return z


@dataclass
class VerifyEntry:
    """verify.hpp:12-17."""
    k: int = 0
    max_err_a: float = 0.0
    max_err_b: float = 0.0
    max_err_c: float = 0.0


@dataclass
class VerifyReport:
    """verify.hpp:19-28."""
    per_k: List[VerifyEntry] = field(default_factory=list)
    max_err: float = 0.0
    worst_x: float = 0.0
    worst_k: int = 0
    worst_region: str = "-"
    max_err_region: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])

    def all_within(self, eps):
        return self.max_err <= eps


def verify_tables(tables, samples_per_region, xmax=200.0, seed=1):
    """verify_tables (verify.hpp:34-35) on the GPU: the reference's sampling,
    every order, a double-double oracle; same report fields."""
    validate_tables(tables)  # verify.cpp:14
    per_k = (ctypes.c_double * ((tables.k_max + 1) * 3))()
    rep = _capi.VerifyReportC()
    rep.per_k = per_k
    h = _handle(tables)  # keep the handle alive across the call
    _raise(_capi.lib().boysfn_verify_tables(h.handle, int(samples_per_region), float(xmax),
                                            int(seed), ctypes.byref(rep)))
    return VerifyReport(
        per_k=[VerifyEntry(k, per_k[3 * k], per_k[3 * k + 1], per_k[3 * k + 2]) for k in range(tables.k_max + 1)],
        max_err=rep.max_err, worst_x=rep.worst_x, worst_k=rep.worst_k, worst_region=rep.worst_region.decode(),
        max_err_region=list(rep.max_err_region))


def kernel_launch_count():
    return int(_capi.lib().boysfn_kernel_launch_count())
