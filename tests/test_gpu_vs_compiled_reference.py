"""The device output against the COMPILED, unmodified reference
(oracle/_ref/libboysfn_ref.so, built by oracle/Makefile from the reference's
own eval.cpp / tables sources) on the bench's own inputs: region C bit for
bit, every other value within EPS_TOL absolute.  The other GPU parity tests
go through the bit-faithful restatement (oracle/boys_port.c, itself pinned
bit for bit to this library on the CPU side); this closes the chain on the
GPU box directly."""
import os

import numpy as np
import pytest

import paper_2512_10059_b200 as pkg
from conftest import EPS_TOL, bits

pytestmark = pytest.mark.gpu

THREADS = max(1, min(16, os.cpu_count() or 1))


def compare(xs, k, got, want, x1):
    inC = xs >= x1
    g, w = got.reshape(-1, k + 1), want.reshape(-1, k + 1)
    assert np.array_equal(bits(g[inC]), bits(w[inC])), "region C not bit-identical to the compiled reference"
    dev = float(np.max(np.abs(g - w)))
    assert dev <= EPS_TOL, dev
    return dev


@pytest.mark.parametrize("case", ["cfg1_uniform_k32_soa", "cfg3_logu_k16_aos", "cfg2_boundary_all_k"])
def test_device_vs_compiled_reference(cuda, ref, case):
    torch = cuda
    s = pkg.embedded_default()
    n = 2_000_000 if case != "cfg2_boundary_all_k" else 300_000
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    if case.startswith("cfg1"):
        pkg.generate_uniform(x, 2, 0.0, 100.0)
        ks, layout = (32,), "soa"
    elif case.startswith("cfg3"):
        pkg.generate_loguniform(x, 4, -12.0, 4.0)
        ks, layout = (16,), "aos"
    else:
        pkg.generate_boundary(x, 3)
        ks, layout = range(33), "soa"
    xs = x.cpu().numpy()
    for k in ks:
        out = torch.empty(n * (k + 1), dtype=torch.float64, device="cuda")
        pkg.eval_device(x, k, out, layout=layout)
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        got = o.reshape(k + 1, n).T if layout == "soa" else o.reshape(n, k + 1)
        want = ref.boys_batch_many_mt(xs, k, THREADS)
        compare(xs, k, np.ascontiguousarray(got), want, s.x1)


def test_host_api_vs_compiled_reference_cfg0(cuda, ref):
    """configs[0] (1e6 U[0,50], k = 8, AoS) through the drop-in host API with
    plain NumPy buffers, against the compiled reference's boys_batch_many."""
    torch = cuda
    s = pkg.embedded_default()
    n, k = 1_000_000, 8
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 1, 0.0, 50.0)
    xs = x.cpu().numpy()
    out = np.empty(n * (k + 1))
    pkg.boys_batch_many(xs, k, s, out)
    st, msg, want = ref.boys_batch_many(xs, k)
    assert st == 0, msg
    compare(xs, k, out, want, s.x1)
