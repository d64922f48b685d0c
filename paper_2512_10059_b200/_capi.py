"""ctypes binding of the C ABI in include/boysfn_b200.h (libboysfn_b200.so).

The library is the product: there is no Python or CPU fallback.  Loading fails
loudly if the in-tree build (python -m paper_2512_10059_b200.build) is missing.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BOYSFN_LIB points at an alternative in-tree build (development experiments).
LIB_PATH = os.environ.get("BOYSFN_LIB") or os.path.join(_HERE, "_lib", "libboysfn_b200.so")

# include/boysfn_b200.h: boysfn_status
OK, ERR_SIZE, ERR_DOMAIN, ERR_RANGE, ERR_TABLES, ERR_CUDA, ERR_ARG, ERR_UNSUPPORTED, ERR_INVALID = range(9)
LAYOUT_AOS, LAYOUT_SOA = 0, 1
REGION_A, REGION_B, REGION_C = 0, 1, 2
DEVICE_KMAX = 32
DEVICE_MAX_DEGREE = 23


class RationalDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("m", ctypes.c_int),
                ("numer", ctypes.POINTER(ctypes.c_double)),
                ("denom", ctypes.POINTER(ctypes.c_double))]


class TableDesc(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("x1", ctypes.c_double), ("k_max", ctypes.c_int),
                ("eps_tol", ctypes.c_double), ("r_B", RationalDesc),
                ("r_A", ctypes.POINTER(RationalDesc))]


class VerifyReportC(ctypes.Structure):
    _fields_ = [("max_err", ctypes.c_double), ("worst_x", ctypes.c_double), ("worst_k", ctypes.c_int),
                ("worst_region", ctypes.c_char), ("max_err_region", ctypes.c_double * 3),
                ("per_k", ctypes.POINTER(ctypes.c_double))]


# (name, restype, argtypes) for every entry point the header declares.
_SIGNATURES = [
    ("boysfn_abi_version", ctypes.c_int, []),
    ("boysfn_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("boysfn_last_error", ctypes.c_char_p, []),
    ("boysfn_tables_create", ctypes.c_int, [ctypes.POINTER(TableDesc), ctypes.POINTER(ctypes.c_void_p)]),
    ("boysfn_tables_embedded", ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p)]),
    ("boysfn_tables_validate", ctypes.c_int, [ctypes.POINTER(TableDesc)]),
    ("boysfn_tables_destroy", ctypes.c_int, [ctypes.c_void_p]),
    ("boysfn_tables_info", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int),
                                          ctypes.POINTER(ctypes.c_double)]),
    ("boysfn_eval_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    ("boysfn_eval_host", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t,
                                        ctypes.POINTER(ctypes.c_size_t)]),
    ("boysfn_set_devices", ctypes.c_int, [ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
    ("boysfn_host_alloc", ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    ("boysfn_host_free", ctypes.c_int, [ctypes.c_void_p]),
    ("boysfn_eval_region_host", ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_void_p]),
    ("boysfn_generate_uniform", ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64,
                                               ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                               ctypes.c_void_p]),
    ("boysfn_generate_loguniform", ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64,
                                                  ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                                  ctypes.c_void_p]),
    ("boysfn_generate_boundary", ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64,
                                                ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                                ctypes.c_void_p]),
    ("boysfn_verify_tables", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                            ctypes.POINTER(VerifyReportC)]),
    ("boysfn_alg2_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                          ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p,
                                          ctypes.c_void_p]),
    ("boysfn_gen_error_scan", ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    ("boysfn_gen_boys_dd", ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    ("boysfn_kernel_launch_count", ctypes.c_ulonglong, []),
]

_lib = None


def lib():
    """The loaded library (loaded once).  Raises if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libboysfn_b200.so is not built (%s); run "
                              "`python -m paper_2512_10059_b200.build` -- there is no CPU fallback"
                              % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in _SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_names():
    return [name for name, _, _ in _SIGNATURES]


def last_error():
    return lib().boysfn_last_error().decode()
