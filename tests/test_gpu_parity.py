"""GPU parity tests: the sm_100a kernels (through the C ABI) against the CPU
oracle on the same inputs.

Bar:
  * region C (x >= x1) BIT-IDENTICAL to the reference (eval.cpp:73-77) -- at
    x1+ with l = 32 the reference itself sits at the 5e-14 budget;
  * regions A and B within EPS_TOL = 5e-14 absolute per value of the reference
    (the kernels use FMA Horner and reciprocal multiplies; the reference
    rounds mul and add separately and divides);
  * every value within 5e-14 absolute of the binary128 oracle (SPEC.md:432,
    acceptance 1 at SPEC.md:523), the reference's own accuracy contract.
"""
import copy

import numpy as np
import pytest

import paper_2512_10059_b200 as pkg
from conftest import EPS_TOL, bits, load_golden, unhex

pytestmark = pytest.mark.gpu


def device_eval(torch, xs, k, layout="soa", tables=None, misalign=False):
    """Evaluate on the device; returns an (N, k+1) host array."""
    n = xs.size
    x = torch.from_numpy(np.ascontiguousarray(xs)).cuda()
    if misalign:  # 8-B aligned, not 16-B aligned output: forces the transpose path
        buf = torch.empty(n * (k + 1) + 1, dtype=torch.float64, device="cuda")
        out = buf[1:]
    else:
        out = torch.empty(max(n * (k + 1), 1), dtype=torch.float64, device="cuda")
    pkg.eval_device(x, k, out, tables=tables, layout=layout)
    torch.cuda.synchronize()
    o = out[: n * (k + 1)].cpu().numpy()
    return o.reshape(k + 1, n).T.copy() if layout == "soa" else o.reshape(n, k + 1)


def check_against_reference(xs, k, got, want, x1):
    inC = xs >= x1
    assert np.array_equal(bits(got[inC]), bits(want[inC])), "region C not bit-identical"
    dev = float(np.max(np.abs(got - want))) if got.size else 0.0
    assert dev <= EPS_TOL, dev
    return dev


def test_golden_reference_rows(cuda, port):
    """Every golden set (reference outputs) through both layouts and the host API."""
    gold = load_golden("reference_rows.json")
    s = pkg.embedded_default()
    for name, g in gold.items():
        if name.startswith("_"):
            continue
        xs, k = unhex(g["x"]), g["k"]
        want = unhex(g["F"]).reshape(-1, k + 1)
        for layout in ("soa", "aos"):
            check_against_reference(xs, k, device_eval(cuda, xs, k, layout), want, s.x1)
        host = np.empty(xs.size * (k + 1))
        pkg.boys_batch_many(xs, k, s, host)
        check_against_reference(xs, k, host.reshape(-1, k + 1), want, s.x1)


def test_all_orders_vs_reference_and_oracle(cuda, port):
    """k = 0..32 on a mixed A/B/C sample: parity with the reference and accuracy
    against the binary128 oracle, both layouts."""
    xs = np.concatenate([port.gen_uniform(30000, 21, 0.0, 45.0), port.gen_uniform(3000, 22, 0.0, 1e-3),
                         port.gen_uniform(3000, 23, 45.0, 1e4)])
    hp = port.hp(xs, 32)
    worst_ref, worst_hp = 0.0, 0.0
    for k in range(33):
        want = port.boys_batch_many(xs, k)
        for layout in ("soa", "aos"):
            got = device_eval(cuda, xs, k, layout)
            worst_ref = max(worst_ref, check_against_reference(xs, k, got, want, port.x1))
            e = float(np.max(np.abs(got - hp[:, :k + 1])))
            assert e <= EPS_TOL, (k, layout, e)
            worst_hp = max(worst_hp, e)
    print("max |gpu-ref| %.3g  max |gpu-oracle| %.3g" % (worst_ref, worst_hp))


def test_acceptance_accuracy_sweep(cuda, port):
    """SPEC acceptance 1: 1e5 uniform x per region (A [0,x0),
    B [x0,x1), C [x1,200]), every k <= 32, max |F - oracle| <= 5e-14."""
    xs = np.concatenate([port.gen_uniform(100000, 31, 0.0, port.x0),
                         port.gen_uniform(100000, 32, port.x0, port.x1),
                         port.gen_uniform(100000, 33, port.x1, 200.0)])
    hp = port.hp(xs, 32)
    per_region = np.zeros(3)
    for k in range(33):
        got = device_eval(cuda, xs, k, "soa")
        err = np.abs(got - hp[:, :k + 1]).max(axis=1)
        for r in range(3):
            per_region[r] = max(per_region[r], err[r * 100000:(r + 1) * 100000].max())
    print("max err per region A/B/C:", per_region)
    assert np.all(per_region <= EPS_TOL), per_region


def test_region_c_knife_edge_bit_exact(cuda, port):
    """x1 + j ulps, j = 0..64, k = 32: the reference is at exactly 5e-14 there;
    the kernel must reproduce it bit for bit (hard parts)."""
    xs = [port.x1]
    for _ in range(64):
        xs.append(np.nextafter(xs[-1], np.inf))
    xs = np.array(xs)
    want = port.boys_batch_many(xs, 32)
    for layout in ("soa", "aos"):
        got = device_eval(cuda, xs, 32, layout)
        assert np.array_equal(bits(got), bits(want))
    assert np.max(np.abs(want - port.hp(xs, 32))) <= EPS_TOL


def test_boundaries_and_special_values(cuda, port):
    """Half-open regions: boundary doubles go right; x0/x1 +- ulps,
    0, subnormals, tiny and huge x."""
    xs = [0.0, 5e-324, 1e-310, 1e-300, 1e-15, 1e-8, 7331.0, 1e4, 1e6, 1e15, 1e300, 1.7976931348623157e308]
    for b in (port.x0, port.x1):
        v = b
        for _ in range(40):
            v = np.nextafter(v, 0.0)
        for _ in range(81):
            xs.append(v)
            v = np.nextafter(v, np.inf)
    xs = np.array(xs)
    for k in (0, 1, 2, 8, 16, 31, 32):
        want = port.boys_batch_many(xs, k)
        for layout in ("soa", "aos"):
            check_against_reference(xs, k, device_eval(cuda, xs, k, layout), want, port.x1)
    assert port.classify(port.x0) == 1 and port.classify(np.nextafter(port.x0, 0)) == 0
    assert port.classify(port.x1) == 2


def test_region_c_fast_path_range_end(cuda, port, monkeypatch):
    """Region C's sqrt/division fast paths apply for x < 2^1022 and the IEEE
    operations above (boys_device.cuh: in_bc_fast_range).  Around that switch
    and at the top of the double range every output path is bit-identical to
    the reference for every order."""
    xs = [2.0 ** 1021, 1e300, 1.7976931348623157e308, np.nextafter(np.inf, 0)]
    v = 2.0 ** 1022
    for _ in range(6):
        v = np.nextafter(v, 0.0)
    for _ in range(13):
        xs.append(v)
        v = np.nextafter(v, np.inf)
    xs = np.array(xs)
    paths = [("soa", p) for p in ("warp", "block", "binned", "blocktma", "blocktmabin")] + \
            [("aos", p) for p in ("xpose", "binned", "blocktma", "blocktmabin")]
    for k in range(33):
        want = port.boys_batch_many(xs, k)
        for layout, path in paths:
            monkeypatch.setenv("BOYSFN_SOA_PATH" if layout == "soa" else "BOYSFN_AOS_PATH", path)
            got = device_eval(cuda, xs, k, layout)
            monkeypatch.delenv("BOYSFN_SOA_PATH", raising=False)
            monkeypatch.delenv("BOYSFN_AOS_PATH", raising=False)
            assert np.array_equal(bits(got), bits(want)), (k, layout, path)


def test_branch_consistency_at_boundaries(cuda, port):
    """at x0 +- 1e-9 and x1 +- 1e-9 adjacent branches agree within
    1e-13 -- checked through the forced-region seam (boys_batch_region)."""
    s = pkg.embedded_default()
    for b, (ra, rb) in ((s.x0, (pkg.Region.A, pkg.Region.B)), (s.x1, (pkg.Region.B, pkg.Region.C))):
        for x in (b - 1e-9, b, b + 1e-9):
            for k in (0, 8, 16, 32):
                fa = np.array(pkg.boys_batch_region(x, k, s, ra).values)
                fb = np.array(pkg.boys_batch_region(x, k, s, rb).values)
                assert np.max(np.abs(fa - fb)) <= 1e-13, (b, x, k)


def test_region_seam_vs_golden(cuda, port):
    s = pkg.embedded_default()
    for c in load_golden("reference_rows.json")["_region_seam"]:
        x, k, r = float.fromhex(c["x"]), c["k"], c["region"]
        got = np.array(pkg.boys_batch_region(x, k, s, pkg.Region(r)).values)
        want = unhex(c["F"])
        if r == 2:
            assert np.array_equal(bits(got), bits(want)), c
        elif r == 0 and x > s.x0 + 1.0:
            continue  # r_A extrapolated 17 units past its interval: not a parity point
        else:
            assert np.max(np.abs(got - want)) <= EPS_TOL, c


def test_error_semantics_vs_reference(cuda):
    """eval.cpp:88-96 through the host API: same exception type and message,
    rows before the first bad x written, later rows untouched."""
    s = pkg.embedded_default()
    exc = {1: pkg.invalid_argument, 2: pkg.domain_error, 3: pkg.out_of_range}
    for c in load_golden("error_cases.json"):
        xs, k, n_out = unhex(c["x"]), c["k"], c["out_len"]
        out = np.full(max(n_out, 0), -7.0)
        if c["status"] == 0:
            pkg.boys_batch_many(xs, k, s, out)
            if n_out:
                assert np.max(np.abs(out - unhex(c["out"]))) <= EPS_TOL
            continue
        with pytest.raises(exc[c["status"]]) as e:
            pkg.boys_batch_many(xs, k, s, out)
        assert str(e.value) == c["message"], c["name"]
        gold = unhex(c["out"])
        written = gold != -7.0
        assert np.all(out[~written] == -7.0), c["name"]
        if written.any():
            assert np.max(np.abs(out[written] - gold[written])) <= EPS_TOL


def test_host_path_error_in_later_chunk(cuda, port):
    """A bad x deep inside a multi-chunk host call: exact first_bad, earlier
    chunks written, later rows untouched (chunks hold ~1/16 of the output)."""
    s = pkg.embedded_default()
    k = 32
    n = 1_500_000  # 16 chunks of ~25 MB of output at k = 32
    xs = port.gen_uniform(n, 77, 0.0, 60.0)
    bad_at = 1_234_567
    xs[bad_at] = np.nan
    out = np.full(n * (k + 1), -7.0)
    with pytest.raises(pkg.domain_error) as e:
        pkg.boys_batch_many(xs, k, s, out)
    assert e.value.first_bad == bad_at
    o = out.reshape(n, k + 1)
    assert np.all(o[bad_at:] == -7.0)
    idx = np.arange(0, bad_at, 997)
    want = port.boys_batch_many(xs[idx], k)
    check_against_reference(xs[idx], k, o[idx], want, port.x1)


def test_ragged_sizes_and_layout_paths(cuda, port):
    """Tile edges (32 x per warp tile), empty input, both AoS paths (TMA bulk
    store on a 16-B aligned output, shared-memory transpose otherwise)."""
    for n in (1, 2, 31, 32, 33, 63, 65, 257, 1000, 4097):
        xs = port.gen_uniform(n, 1000 + n, 0.0, 40.0)
        for k in (0, 3, 8, 15, 16, 32):
            want = port.boys_batch_many(xs, k)
            a = device_eval(cuda, xs, k, "aos")
            b = device_eval(cuda, xs, k, "aos", misalign=True)
            c = device_eval(cuda, xs, k, "soa")
            assert np.array_equal(bits(a), bits(b)) and np.array_equal(bits(a), bits(c)), (n, k)
            check_against_reference(xs, k, a, want, port.x1)
    got = device_eval(cuda, np.zeros(0), 4, "aos")
    assert got.size == 0


@pytest.mark.parametrize("extra", [1, 3])
def test_custom_table_set_compact_and_padded_kernels(cuda, port, extra):
    """A caller-built CoefficientTableSet whose degrees differ from Appendix C
    takes the compact kernels (r_A <= (9, 13), r_B <= (6, 7); extra = 1 zero
    appended to every numerator) or the 23/23 padded ones (extra = 3 pushes
    most r_A numerators past 9); zero leading coefficients are exact under
    Horner-FMA, so both are bit-identical to the embedded kernels."""
    s = pkg.embedded_default()
    t = copy.deepcopy(s)
    t.r_B.numer.extend([0.0] * extra)
    for r in t.r_A:
        r.numer.extend([0.0] * extra)
    xs = port.gen_uniform(20000, 5, 0.0, 50.0)
    for k in (0, 7, 16, 32):
        a = device_eval(cuda, xs, k, "soa")
        b = device_eval(cuda, xs, k, "soa", tables=t)
        assert np.array_equal(bits(a), bits(b)), k
        hb = np.empty(xs.size * (k + 1))
        pkg.boys_batch_many(xs, k, t, hb)
        assert np.array_equal(bits(hb.reshape(-1, k + 1)), bits(device_eval(cuda, xs, k, "aos"))), k


def test_determinism_and_streams(cuda, port):
    """Bit-identical reruns, also when two streams run at once."""
    torch = cuda
    n, k = 2_000_000, 16
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 4, 0.0, 80.0)
    outs = [torch.empty(n * (k + 1), dtype=torch.float64, device="cuda") for _ in range(3)]
    pkg.eval_device(x, k, outs[0])
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        pkg.eval_device(x, k, outs[1])
    with torch.cuda.stream(s2):
        pkg.eval_device(x, k, outs[2])
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int64), outs[1].view(torch.int64))
    assert torch.equal(outs[0].view(torch.int64), outs[2].view(torch.int64))


def test_device_generator_matches_oracle_stream(cuda, port):
    torch = cuda
    x = torch.empty(100000, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 2, 0.0, 100.0, offset=5_000_000)
    assert np.array_equal(bits(x.cpu().numpy()), bits(port.gen_uniform(100000, 2, 0.0, 100.0, offset=5_000_000)))


def test_first_bad_device_flag(cuda, port):
    torch = cuda
    xs = port.gen_uniform(100000, 8, 0.0, 30.0)
    for pos in (77777, 99999, 5):
        xs[pos] = -1.0
    x = torch.from_numpy(xs).cuda()
    out = torch.empty(xs.size * 9, dtype=torch.float64, device="cuda")
    fb = torch.full((1,), -1, dtype=torch.int64, device="cuda")  # all ones = UINT64_MAX
    pkg.eval_device(x, 8, out, first_bad=fb)
    assert int(fb.item()) == 5


def test_cpp_shim_drop_in(cuda):
    """The C++ drop-in (boysfn::boys_batch_many & co.) as reference code calls it."""
    import subprocess
    from paper_2512_10059_b200 import build
    exe = build.build_shim_test()
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cuda_graph_capture_and_replay(cuda, port):
    """The device entry point is stream-ordered end to end (per-launch scratch
    from the stream-ordered pool), so it captures into a CUDA graph; replays
    reproduce the eager result bit for bit, also after the inputs change."""
    torch = cuda
    n, k = 300_000, 16
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pkg.generate_uniform(x, 12, 0.0, 60.0)
    eager = torch.empty(n * (k + 1), dtype=torch.float64, device="cuda")
    out = torch.empty_like(eager)
    pkg.eval_device(x, k, eager, layout="soa")  # warm the per-kernel caches outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pkg.eval_device(x, k, out, layout="soa")
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int64), eager.view(torch.int64))
    pkg.generate_uniform(x, 13, 0.0, 60.0)
    pkg.eval_device(x, k, eager, layout="soa")
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int64), eager.view(torch.int64))


def test_binned_region_c_pairs_with_huge_x(cuda, port, monkeypatch):
    """The binned kernels evaluate all-region-C virtual tiles two at a time
    with the fast sqrt/division paths run unconditionally and the IEEE
    operations re-run for lanes outside the fast range (boys_device.cuh:
    boys_values_c_pair).  Groups made only of region-C x, with x >= 2^1022
    scattered through them (including pairs where only one tile has such an x),
    are bit-identical to the reference at every order the binned kernels run."""
    rng = np.random.default_rng(11)
    n = 4096 + 77  # whole 128- and 256-x groups plus a ragged tail
    xs = rng.uniform(port.x1, 5e3, n)
    huge = [2.0 ** 1022, np.nextafter(2.0 ** 1022, 0.0), 1e308, 1.7976931348623157e308]
    for i, pos in enumerate((5, 70, 300, 301, 1000, 2050, 4100)):
        xs[pos] = huge[i % len(huge)]
    for k in range(7):
        want = port.boys_batch_many(xs, k)
        for layout in ("soa", "aos"):
            monkeypatch.setenv("BOYSFN_SOA_PATH" if layout == "soa" else "BOYSFN_AOS_PATH", "binned")
            got = device_eval(cuda, xs, k, layout)
            monkeypatch.delenv("BOYSFN_SOA_PATH", raising=False)
            monkeypatch.delenv("BOYSFN_AOS_PATH", raising=False)
            assert np.array_equal(bits(got), bits(want)), (k, layout)
