"""The generator's B200 extremum scan and the gen pipeline on the GPU
(SPEC.md acceptance 3 and cmd_gen)."""
import numpy as np
import pytest
from mpmath import mpf

import paper_2512_10059_b200 as pkg
import genport as gen
from paper_2512_10059_b200 import tables as T
from genport import hp, scan
from genport.generate import generate_tables, search_table

pytestmark = pytest.mark.gpu


def _mp(coeffs):
    return [mpf(c) for c in coeffs]


@pytest.mark.parametrize("k,weight", [(0, "one"), (12, "rho_A"), (32, "rho_A")])
def test_error_scan_matches_working_precision(cuda, k, weight):
    emb = pkg.embedded_default()
    r = emb.r_B if weight == "one" else emb.r_A[k]
    a, b = (emb.x0, emb.x1) if weight == "one" else (0.0, emb.x0)
    xs = np.concatenate(([a, b], np.random.default_rng(k).uniform(a, b, 40)))
    e = scan.error_scan(k, weight, _mp(r.numer), _mp(r.denom), xs)
    with hp.precision():
        f = hp.boys_target(k)
        for x, ev in zip(xs, e):
            rho = gen.weight_rho_A(k, x) if weight == "rho_A" else 1
            want = rho * (f(mpf(x)) - gen.poly_eval(_mp(r.numer), mpf(x)) / gen.poly_eval(_mp(r.denom), mpf(x)))
            assert abs(float(want) - ev) <= 1e-26 + 1e-12 * abs(float(want)), (x, float(want), ev)


def test_boys_dd_matches_the_series(cuda):
    xs = np.array([0.0, 1e-9, 0.5, 3.0, 11.9, 17.0, 28.9, 45.0])
    for k in (0, 7, 32, 64):
        hi, lo = scan.boys_dd(k, xs)
        with hp.precision():
            for x, h, l in zip(xs, hi, lo):
                want = hp.boys_reference(k, mpf(x), hp.reference_terms_for(k, x, 1e-40) if x > 0 else 150)
                assert abs((mpf(h) + mpf(l)) / want - 1) < mpf("1e-29"), (k, x)


def test_table_reproduction_r_B(cuda):
    """Acceptance 3: remez_solve for F_0 on [x0, x1], rho = 1, (5, 6) converges
    with 13 equioscillation nodes and matches the embedded r_B within 1e-12
    relative on 1000 points."""
    emb = pkg.embedded_default()
    with hp.precision():
        x0, x1 = gen.compute_x0(32), gen.compute_x1(32, 5e-14)
        res = gen.remez_solve(gen.RemezProblem(f=hp.boys_target(0), a=x0, b=x1, n=5, m=6, eps_conv=mpf("5e-16"),
                                               scan=scan.GpuScan(0, "one")))
        assert res.status == gen.RemezStatus.Converged and res.alternation_count == 13
        assert res.sup_error <= mpf("5e-14")
        worst = 0
        for x in np.linspace(float(x0), float(x1), 1000):
            ref = gen.poly_eval(_mp(emb.r_B.numer), mpf(x)) / gen.poly_eval(_mp(emb.r_B.denom), mpf(x))
            worst = max(worst, abs(float(res.approximant.eval(mpf(x)) / ref - 1)))
    assert worst <= 1e-12, worst


def test_walsh_search_selects_the_paper_degrees_for_r_B(cuda):
    """Acceptance 3: walsh_search at 5e-14 selects n+m <= 11 -- (5, 6), Table I."""
    with hp.precision():
        x0, x1 = gen.compute_x0(32), gen.compute_x1(32, 5e-14)
    res, rep = search_table(0, "B", x0, x1, 5e-14, 12)
    assert res.met_tolerance and (res.n, res.m) == (5, 6) and res.sup_error <= mpf("5e-14")


def test_generate_small_set_self_verifies(cuda):
    """cmd_gen for k_max = 2 at 1e-8: every table meets the tolerance, the text
    round-trips, and verify_tables on the GPU passes (SPEC.md: gen output always
    passes verify)."""
    res = generate_tables(2, 1e-8, max_total_degree=16)
    assert all(r.met_tolerance for r in res.reports)
    text = T.emit_tables(res.tables)
    back = T.parse_tables(text)
    assert T.emit_tables(back) == text
    rep = pkg.verify_tables(back, 4000, 60.0, 3)
    assert rep.max_err <= 1e-8, (rep.max_err, rep.worst_k, rep.worst_region)


def test_generated_k32_set_passes_verify(cuda):
    """The certified generated set meets eps_tol on the GPU verify (1e4/region)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "generated_k32_tables.txt")
    t = T.parse_tables(open(path).read())
    rep = pkg.verify_tables(t, 10000, 200.0, 11)
    assert rep.max_err <= t.eps_tol, (rep.max_err, rep.worst_k, rep.worst_region)


def test_native_generator_reproduces_r_B_and_a_small_set(cuda, tmp_path):
    """boysfn_gen (binary128 + GPU scan): r_B (5, 6) matches the embedded table
    within 1e-12 relative on 1000 points; `gen` for k_max = 2 at 1e-8 writes a
    set that parses and passes verify_tables."""
    import subprocess
    from paper_2512_10059_b200 import build
    r = subprocess.run([build.GEN, "remez", "--region", "B", "--n", "5", "--m", "6"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert "alternation=13" in lines[0]
    num = [float(l.split()[1]) for l in lines if l.startswith("numer")]
    den = [float(l.split()[1]) for l in lines if l.startswith("denom")]
    emb = pkg.embedded_default()
    xs = np.linspace(emb.x0, emb.x1, 1000)
    mine = np.polyval(num[::-1], xs) / np.polyval(den[::-1], xs)
    ref = np.polyval(emb.r_B.numer[::-1], xs) / np.polyval(emb.r_B.denom[::-1], xs)
    assert np.abs(mine / ref - 1).max() <= 1e-12
    out = tmp_path / "k2.txt"
    r = subprocess.run([build.GEN, "gen", "--kmax", "2", "--eps", "1e-8", "--out", str(out), "--max-degree", "16"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    t = T.parse_tables(out.read_text())
    assert t.k_max == 2 and pkg.verify_tables(t, 4000, 60.0, 5).max_err <= 1e-8
