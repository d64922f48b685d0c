"""verify_tables on the GPU (verify.cpp:12-63): the reference's sampling
(std::mt19937_64, restated in oracle/boys_port.c and checked against the C++
standard's 10000th output), a device double-double oracle, and the reference's
report.  Cross-checked against the same report built on the CPU from the
binary128 oracle and the device evaluator's values."""
import copy

import numpy as np
import pytest

import paper_2512_10059_b200 as pkg

pytestmark = pytest.mark.gpu


def cpu_report(torch, port, tables, spr, xmax=200.0, seed=1):
    xs = port.verify_samples(spr, xmax, seed, tables.x0, tables.x1)
    hp = port.hp(xs, tables.k_max)
    x = torch.from_numpy(xs).cuda()
    per_k = np.zeros((tables.k_max + 1, 3))
    for k in range(tables.k_max + 1):
        out = torch.empty(xs.size * (k + 1), dtype=torch.float64, device="cuda")
        pkg.eval_device(x, k, out, tables=tables, layout="aos")
        err = np.abs(out.cpu().numpy().reshape(-1, k + 1) - hp[:, :k + 1]).max(axis=1)
        per_k[k] = err.reshape(3, spr).max(axis=1)
    return xs, per_k


def test_mt19937_64_restatement(port):
    # [rand.predef]: the 10000th invocation of a default-constructed mt19937_64
    assert port.L.oracle_mt64_nth(5489, 10000) == 9981545732273789042


def test_verify_embedded_tables(cuda, port):
    spr = 20000
    r = pkg.verify_tables(pkg.embedded_default(), spr)
    assert r.all_within(5e-14), r.max_err
    xs, per_k = cpu_report(cuda, port, pkg.embedded_default(), spr)
    got = np.array([[e.max_err_a, e.max_err_b, e.max_err_c] for e in r.per_k])
    assert np.all(np.abs(got - per_k) <= 2e-16), np.max(np.abs(got - per_k))
    assert r.max_err == pytest.approx(per_k.max(), abs=2e-16)
    assert r.worst_region in "ABC" and r.worst_x in xs
    assert r.max_err_region == pytest.approx(list(per_k.max(axis=0)), abs=2e-16)


def test_verify_detects_a_perturbed_coefficient(cuda):
    """one coefficient perturbed by 1e-6 relative -> failure reported
    for the affected k."""
    t = copy.deepcopy(pkg.embedded_default())
    t.r_A[7].numer[2] *= 1 + 1e-6
    r = pkg.verify_tables(t, 3000)
    assert not r.all_within(5e-14)
    bad = [e.k for e in r.per_k if max(e.max_err_a, e.max_err_b, e.max_err_c) > 5e-14]
    assert bad == [7], bad
    assert r.worst_k == 7 and r.worst_region == "A"


def test_verify_argument_errors(cuda):
    s = pkg.embedded_default()
    with pytest.raises(pkg.invalid_argument, match="verify_tables: need at least one sample per region"):
        pkg.verify_tables(s, 0)
    with pytest.raises(pkg.invalid_argument, match="verify_tables: xmax must exceed x1"):
        pkg.verify_tables(s, 10, xmax=20.0)
