"""B200-native batched Boys-function evaluator (arXiv 2512.10059, Algorithm 1).

Drop-in for the reference's evaluation API (boysfn::boys_batch_many & co.,
/root/reference/proj/core/include/boysfn/eval.hpp): the C ABI is
include/boysfn_b200.h, the C++ shim paper_2512_10059_b200/cpp/, and this
package is the Python mirror.  All evaluation runs in hand-written sm_100a
FP64 kernels (csrc/); see DESIGN.md.
"""
from .tables import (CoefficientTableSet, RationalApproximant, TableParseError, embedded_default,
                     emit_tables, parse_tables, validate_tables)
from .eval import (BoysBatch, alg2, DeviceTables, Region, boys_batch, boys_batch_many, boys_batch_region,
                   classify_region, cuda_error, domain_error, eval_device, generate_boundary, generate_loguniform,
                   generate_uniform, host_empty, invalid_argument, kernel_launch_count, out_of_range, set_devices,
                   unsupported, VerifyEntry, VerifyReport, verify_tables)

__all__ = [
    "CoefficientTableSet", "RationalApproximant", "TableParseError", "embedded_default", "emit_tables",
    "parse_tables", "validate_tables", "alg2", "BoysBatch", "DeviceTables", "Region", "boys_batch",
    "boys_batch_many", "boys_batch_region", "classify_region", "cuda_error", "domain_error",
    "eval_device", "host_empty", "set_devices", "generate_boundary", "generate_loguniform", "generate_uniform", "invalid_argument",
    "kernel_launch_count", "out_of_range", "unsupported", "VerifyEntry", "VerifyReport", "verify_tables",
]
