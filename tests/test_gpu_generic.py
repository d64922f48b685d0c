"""The run-time-k kernels (boys_eval_generic_tma_kernel, and the per-warp
boys_eval_generic_kernel where no tensor map applies): bit-identical to the
templated kernels for every k <= 32 (BOYSFN_GENERIC=1 routes all orders to the
run-time-k kernels, =2 to the per-warp one, =3 to the staged block kernel, =4 to
the register-buffered block kernel),
and the evaluator for table sets with k_max > 32 -- the reference's gen path
allows k_max <= 64 -- checked against the C restatement of
eval.cpp, which takes any k."""
import copy
import ctypes

import numpy as np
import pytest

import paper_2512_10059_b200 as pkg
from conftest import bits

pytestmark = pytest.mark.gpu


def dev(torch, xs, k, layout, tables=None):
    """F on the device; the 4 KB past the output must stay untouched (the
    tensor stores clip rows >= n and the AoS stage's pad columns)."""
    x = torch.from_numpy(np.ascontiguousarray(xs)).cuda()
    n = xs.size
    buf = torch.full((n * (k + 1) + 512,), 7.25, dtype=torch.float64, device="cuda")
    out = buf[: n * (k + 1)]
    pkg.eval_device(x, k, out, tables=tables, layout=layout)
    torch.cuda.synchronize()
    assert bool((buf[n * (k + 1):] == 7.25).all()), "write past the output"
    o = out.cpu().numpy()
    return o.reshape(k + 1, n).T.copy() if layout == "soa" else o.reshape(n, k + 1)


def test_generic_bit_identical_to_templated(cuda, port, monkeypatch):
    xs = np.concatenate([port.gen_uniform(4099, 5, 0.0, 45.0), [0.0, port.x0, port.x1, 1e4]])
    for k in range(33):
        for layout in ("soa", "aos"):
            a = dev(cuda, xs, k, layout)
            for mode in ("1", "2", "3", "4"):
                monkeypatch.setenv("BOYSFN_GENERIC", mode)
                b = dev(cuda, xs, k, layout)
                monkeypatch.delenv("BOYSFN_GENERIC")
                assert np.array_equal(bits(a), bits(b)), (k, layout, mode)


def test_generic_block_tma_equals_per_warp_above_32(cuda, port, monkeypatch):
    """Orders above 32: the block-TMA kernels (region-sorted tiles; F staged as
    produced, or held in registers while the previous tile drains) and the
    per-warp kernel agree bit for bit on ragged sizes, and the first bad x is
    reported identically."""
    t = table_k64()
    for n in (1, 127, 128, 129, 20011):
        xs = port.gen_uniform(n, 40 + n % 7, 0.0, 60.0)
        for k in (33, 35, 40, 47, 63, 64):  # even k+1: the padded AoS stage
            for layout in ("soa", "aos"):
                a = dev(cuda, xs, k, layout, tables=t)
                # "4r": the padded AoS stage's per-row bulk copies instead of
                # its one clipped tensor store (BOYSFN_GENERIC_AOS_ROWS)
                for mode in ("2", "3", "4", "4r"):
                    monkeypatch.setenv("BOYSFN_GENERIC", mode[0])
                    if mode == "4r":
                        monkeypatch.setenv("BOYSFN_GENERIC_AOS_ROWS", "1")
                    b = dev(cuda, xs, k, layout, tables=t)
                    monkeypatch.delenv("BOYSFN_GENERIC")
                    monkeypatch.delenv("BOYSFN_GENERIC_AOS_ROWS", raising=False)
                    assert np.array_equal(bits(a), bits(b)), (n, k, layout, mode)
    xs = port.gen_uniform(5000, 3, 0.0, 60.0)
    xs[[4001, 777]] = (np.nan, -2.0)
    for mode in (None, "2", "3", "4"):
        if mode:
            monkeypatch.setenv("BOYSFN_GENERIC", mode)
        o = np.full(xs.size * 41, 1.5)
        with pytest.raises(pkg.domain_error) as ei:
            pkg.boys_batch_many(xs, 40, t, o)
        monkeypatch.delenv("BOYSFN_GENERIC", raising=False)
        assert ei.value.first_bad == 777


def table_k64():
    """Appendix C extended to k_max = 64: r_A[k > 32] reuse r_A[32] (a seed of
    the right magnitude; the values are not Boys functions above 32, but the
    arithmetic is fully defined and the oracle restates it exactly)."""
    t = copy.deepcopy(pkg.embedded_default())
    t.k_max = 64
    t.r_A += [copy.deepcopy(t.r_A[32]) for _ in range(32)]
    pkg.validate_tables(t)
    return t


def oracle_tables(port, t):
    """The port's view of a custom table set (pyoracle's structs)."""
    import pyoracle
    keep = []

    def rat(r):
        nu, de = np.ascontiguousarray(r.numer), np.ascontiguousarray(r.denom)
        keep.extend((nu, de))
        return pyoracle._Rational(len(nu) - 1, len(de) - 1, nu.ctypes.data_as(pyoracle._dp),
                                  de.ctypes.data_as(pyoracle._dp))
    ra = (pyoracle._Rational * len(t.r_A))(*[rat(r) for r in t.r_A])
    keep.append(ra)
    return pyoracle._Tables(t.x0, t.x1, t.k_max, t.eps_tol, rat(t.r_B), ra), keep


def test_orders_above_32_match_reference_arithmetic(cuda, port):
    t = table_k64()
    ot, keep = oracle_tables(port, t)
    xs = np.concatenate([port.gen_uniform(3001, 6, 0.0, 45.0), port.gen_uniform(64, 7, 28.9, 31.0)])
    for k in (33, 40, 63, 64):
        want = np.zeros((xs.size, k + 1))
        bad = ctypes.c_size_t()
        import pyoracle
        st = port.L.oracle_boys_batch_many(xs.ctypes.data_as(pyoracle._dp), xs.size, k, ctypes.byref(ot),
                                           want.ctypes.data_as(pyoracle._dp), want.size, ctypes.byref(bad))
        assert st == 0
        for layout in ("soa", "aos"):
            got = dev(cuda, xs, k, layout, tables=t)
            inA, inC = xs < t.x0, xs >= t.x1
            assert np.array_equal(bits(got[inC]), bits(want[inC])), (k, layout)  # region C exact
            rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
            # region A: the downward chain is stable at every order
            assert np.max(rel[inA]) <= 1e-12, (k, layout, np.max(rel[inA]))
            # region B: the upward chain is only conditioned up to the order x1 was
            # sized for (32 here; a genuine k_max = 64 set moves x0/x1)
            inB = ~inA & ~inC
            dev_b = np.abs(got - want)[inB][:, :33]
            assert np.max(dev_b) <= 5e-14, (k, layout, np.max(dev_b))  # the absolute budget
            assert np.all(np.isfinite(got))
        # the host (drop-in) API on the same table set
        host = np.empty(xs.size * (k + 1))
        pkg.boys_batch_many(xs, k, t, host)
        assert np.array_equal(bits(host.reshape(-1, k + 1)), bits(dev(cuda, xs, k, "aos", tables=t)))
    del keep


def test_region_seam_above_32(cuda, port):
    t = table_k64()
    for r in (pkg.Region.A, pkg.Region.B, pkg.Region.C):
        x = {pkg.Region.A: t.x0 - 1e-9, pkg.Region.B: t.x0 + 1e-9, pkg.Region.C: t.x1 + 1e-9}[r]
        v = np.array(pkg.boys_batch_region(x, 48, t, r).values)
        assert v.shape == (49,) and np.all(np.isfinite(v))
    with pytest.raises(pkg.out_of_range):
        pkg.boys_batch(1.0, 65, t)
