"""The coefficient generator's restated pieces on the CPU (SURVEY.md section
8(f) rank 4; SPEC.md acceptance 2 and 6 and the module examples of
SPEC.md:157-330).  Working precision 50+12 digits, mpmath."""
import math
import random

import mpmath
import numpy as np
import pytest
from mpmath import mpf

import genport as gen
from genport import hp, remez


@pytest.fixture(autouse=True)
def _prec():
    with hp.precision():
        yield


def test_region_constants_match_appendix_c():
    """Acceptance 2: compute_x0(32) and compute_x1(32, 5e-14) to all 17 digits."""
    assert "%.17g" % float(gen.compute_x0(32)) == "11.899848152108484"
    assert float(gen.compute_x1(32, 5e-14)) == float("28.989337738820740")
    assert gen.compute_x0(1) == 1 and gen.compute_x0(2) == 1


def test_x1_residual_monotonicity_and_k0_bisection():
    eps = mpf("5e-14")
    x1 = gen.compute_x1(32, eps)
    s = mpf(32) + mpf("0.5")
    resid = gen.upper_gamma_half(32, x1) / (2 * mpmath.power(x1, s)) - eps
    assert abs(resid) <= eps * mpf(10) ** -20
    assert gen.compute_x1(16, 1e-14) > gen.compute_x1(16, 1e-10)
    # k = 0: sqrt(pi) erfc(sqrt x) / (2 sqrt x) = eps by an independent bisection
    g = lambda x: mpmath.sqrt(mp_pi()) * mpmath.erfc(mpmath.sqrt(x)) / (2 * mpmath.sqrt(x)) - mpf(5e-14)  # noqa: E731
    root = mpmath.findroot(g, (mpf(20), mpf(40)), solver="bisect", tol=mpf(10) ** -40)
    # Newton stops at a residual of eps*1e-21 (regions.cpp:55), i.e. x to ~1e-20
    assert abs(gen.compute_x1(0, 5e-14) - root) < mpf(10) ** -18


def mp_pi():
    return mpmath.mp.pi


def test_weight_rho_A():
    assert gen.weight_rho_A(0, 7) == 1 and gen.weight_rho_A(9, 0) == 1
    assert gen.weight_rho_A(2, 3) == 12
    xs = sorted(random.Random(3).uniform(0, 12) for _ in range(50))
    for k in (1, 5, 17, 32):
        w = [gen.weight_rho_A(k, x) for x in xs]
        assert all(b >= a for a, b in zip(w, w[1:]))


def test_mt19937_64_matches_the_standard():
    g = remez.MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_highprec_kernels():
    assert abs(gen.erfc(1) - mpf("0.15729920705028513065877936491739074070393300203369719")) < mpf(10) ** -48
    for x in (mpf("0.3"), mpf("1.7"), mpf("2.5"), mpf("6")):
        assert abs(gen.erf(x) + gen.erfc(x) - 1) < mpf(10) ** -47
    for k, x in ((0, mpf(3)), (5, mpf("0.7")), (12, mpf(20)), (32, mpf(29))):
        ref = mpmath.gammainc(k + mpf("0.5"), x)
        assert abs(gen.upper_gamma_half(k, x) / ref - 1) < mpf(10) ** -45
    assert gen.boys_reference(0, 0) == 1
    assert abs(gen.boys_reference(5, 0) - mpf(1) / 11) < mpf(10) ** -55
    assert abs(gen.boys_reference(0, 1) - mpf("0.74682413281242702539946743613185300535449968681260632902")) \
        < mpf(10) ** -48
    assert gen.truncation_bound(4, 0, 150) == 0


def test_two_truncation_residual_respects_the_bound():
    """Acceptance 5 (empirical part): |F(L=150) - F(L=200)| / F <= bound(150)."""
    rng = random.Random(5)
    for _ in range(20):
        k, x = rng.randint(0, 32), mpf(rng.uniform(0, 30))
        a, b = gen.boys_reference(k, x, 150), gen.boys_reference(k, x, 200)
        assert abs(a - b) / b <= gen.truncation_bound(k, x, 150) * (1 + mpf(10) ** -10) + mpf(10) ** -55


def test_sturm_root_count():
    assert gen.sturm_root_count([mpf(-1), 0, 1], 0, 2) == 1
    assert gen.sturm_root_count([mpf(1), 0, 1], -10, 10) == 0
    rng = random.Random(11)
    for _ in range(40):
        roots = sorted({round(rng.uniform(-5, 5), 3) for _ in range(rng.randint(1, 8))})
        p = [mpf(1)]
        for r in roots:  # p *= (x - r)
            p = [(p[i - 1] if i > 0 else 0) - mpf(r) * (p[i] if i < len(p) else 0) for i in range(len(p) + 1)]
        a, b = rng.uniform(-6, 0), rng.uniform(0, 6)
        want = sum(1 for r in roots if a < r <= b)
        assert gen.sturm_root_count(p, mpf(a), mpf(b)) == want, (roots, a, b)


def test_newton_interpolate_and_leja():
    xs = [mpf(v) for v in (0.1, -0.7, 1.3, 2.2, -1.9)]
    coef = [mpf(v) for v in (1.5, -2, 0.25, 3, -0.5)]
    ys = [gen.poly_eval(coef, x) for x in xs]
    got = gen.newton_interpolate(xs, ys)
    assert max(abs(a - b) for a, b in zip(got, coef)) < mpf(10) ** -50
    order = gen.leja_order(xs)
    assert sorted(order) == list(range(len(xs))) and order[0] == 3  # largest |x| first


def test_jacobi_matches_numpy():
    rng = np.random.default_rng(2)
    a = rng.normal(size=(6, 6))
    a = a + a.T
    vals, vecs = gen.jacobi_eigensolve([[mpf(float(v)) for v in row] for row in a])
    assert np.allclose(sorted(float(v) for v in vals), np.linalg.eigvalsh(a), atol=1e-12)
    for lam, v in zip(vals, vecs):
        r = np.array(a) @ np.array([float(c) for c in v]) - float(lam) * np.array([float(c) for c in v])
        assert np.abs(r).max() < 1e-12


def test_golden_section_fixtures():
    assert abs(gen.golden_section_max(lambda x: -(x - 1) ** 2, 0, 2, mpf("1e-12")) - 1) < mpf("1e-11")
    assert abs(gen.golden_section_max(lambda x: x, 0, 2, mpf("1e-12")) - 2) < mpf("1e-11")
    assert abs(gen.golden_section_max(mpmath.sin, 0, 3, mpf("1e-10")) - mpmath.pi / 2) < mpf("1e-9")


def test_solve_fixed_nodes_examples():
    nodes = [mpf(0), mpf(1) / 3, mpf(2) / 3]
    c = gen.solve_fixed_nodes(nodes, list(nodes), [mpf(1)] * 3, 1, 0)
    assert c and abs(c[0].levelled_error) < mpf(10) ** -50
    q0 = c[0].denom[0]  # m = 0: q is the constant q0, p = q0 * x
    assert max(abs(a / q0 - b) for a, b in zip(c[0].numer, [0, 1])) < mpf(10) ** -45
    c = gen.solve_fixed_nodes([mpf(0), mpf(1)], [mpf(0), mpf(1)], [mpf(1)] * 2, 0, 0)
    assert c and abs(abs(c[0].levelled_error) - mpf("0.5")) < mpf(10) ** -50
    cst = gen.solve_fixed_nodes([mpf(v) for v in (0, 0.2, 0.5, 0.7, 1)], [mpf(3)] * 5, [mpf(1)] * 5, 2, 1)
    assert all(abs(cc.levelled_error) < mpf(10) ** -45 for cc in cst)


def test_select_pole_free_rejects_planted_poles():
    good = remez.FixedNodeCandidate([mpf(1)], [mpf(2), mpf(1)], [], mpf(0), mpf(1e-60))  # root at -2
    bad = remez.FixedNodeCandidate([mpf(1)], [mpf("-0.5"), mpf(1)], [], mpf(0), mpf(0))  # root at 0.5
    assert gen.select_pole_free([bad, good], 0, 1) is good
    assert gen.select_pole_free([bad], 0, 1) is None


def test_remez_classical_fixtures():
    """Acceptance 6: x^2 by (1,0) on [0,1] -> x - 1/8 with sup 1/8; alternation n+m+2;
    the levelled error never exceeds the sup error (asserted every iteration)."""
    res = gen.remez_solve(gen.RemezProblem(f=lambda x: x * x, a=0, b=1, n=1, m=0, eps_conv=mpf("1e-30")))
    assert res.status == gen.RemezStatus.Converged
    assert abs(res.sup_error - mpf(1) / 8) < mpf("1e-12") and res.alternation_count == 3
    assert abs(res.approximant.numer[0] + mpf(1) / 8) < mpf("1e-12") and abs(res.approximant.numer[1] - 1) < 1e-12
    assert all(h.levelled_error_abs <= h.sup_error * (1 + mpf(10) ** -10) for h in res.history)
    lin = gen.remez_solve(gen.RemezProblem(f=lambda x: 3 * x + 2, a=0, b=1, n=1, m=0, eps_conv=mpf("1e-30")))
    assert lin.status == gen.RemezStatus.Converged and lin.sup_error < mpf(10) ** -40


def test_remez_weight_scaling_invariance():
    f = lambda x: mpmath.exp(-x)  # noqa: E731
    r1 = gen.remez_solve(gen.RemezProblem(f=f, a=0, b=1, n=2, m=2, eps_conv=mpf("1e-14"))).approximant
    r2 = gen.remez_solve(gen.RemezProblem(f=f, rho=lambda x: mpf(7), a=0, b=1, n=2, m=2,
                                          eps_conv=mpf("7e-14"))).approximant
    for x in np.linspace(0, 1, 50):
        assert abs(r1.eval(mpf(x)) / r2.eval(mpf(x)) - 1) < 1e-12


def test_walsh_search_minimal_degree():
    """e^{-x} on [0, 1] at 1e-6: the selected anti-diagonal is the first with a
    cell meeting the tolerance, and every cell below it failed."""
    res = gen.walsh_search(lambda x: mpmath.exp(-x), None, 0, 1, 1e-6, 8)
    assert res.met_tolerance and res.sup_error <= mpf("1e-6")
    d = res.n + res.m
    for c in res.cells:
        if c.n + c.m < d:
            assert c.status != gen.RemezStatus.Converged or c.sup_error > mpf("1e-6")


def test_rho_A_is_the_downward_amplification():
    """a seed perturbation delta at order k, carried down the
    recurrence F_l = (2x F_{l+1} + e^-x)/(2l+1), is amplified at most by
    rho_A,k(x) over l = 0..k (equality at the worst order)."""
    rng = random.Random(8)
    x0 = float(gen.compute_x0(32))
    for _ in range(12):
        k, x = rng.randint(1, 32), mpf(rng.uniform(0, x0))
        e = mpmath.exp(-x)
        delta = mpf("1e-16")
        a, b = gen.boys_reference(k, x), gen.boys_reference(k, x) + delta
        amp = mpf(1)
        for l in range(k - 1, -1, -1):
            a = (2 * x * a + e) / (2 * l + 1)
            b = (2 * x * b + e) / (2 * l + 1)
            amp = max(amp, abs(b - a) / delta)
        rho = gen.weight_rho_A(k, x)
        assert abs(amp / rho - 1) < mpf("1e-6"), (k, x)


def test_generated_k32_set_matches_appendix_c_shape():
    """The set written by `gen --kmax 32 --eps 5e-14` on the B200 box
    (tests/golden/generated_k32_tables.txt, profiles/r01_gen_full_k32.txt):
    same x0, x1 and, table by table, the same total degree n+m as Appendix C."""
    import os
    import paper_2512_10059_b200 as pkg
    from paper_2512_10059_b200 import tables as T
    path = os.path.join(os.path.dirname(__file__), "golden", "generated_k32_tables.txt")
    g = T.parse_tables(open(path).read())
    e = pkg.embedded_default()
    assert (g.x0, g.x1, g.k_max, g.eps_tol) == (e.x0, e.x1, e.k_max, e.eps_tol)
    assert (g.r_B.degree_n(), g.r_B.degree_m()) == (5, 6)
    for a, b in zip(g.r_A, e.r_A):
        assert a.degree_n() + a.degree_m() == b.degree_n() + b.degree_m()


def _gen_binary():
    import os
    import subprocess
    from paper_2512_10059_b200 import build
    path = build.GEN
    if not os.path.exists(path):
        pytest.skip("boysfn_gen not built")
    return path, subprocess


def test_native_generator_selftest_and_regions():
    """The native (binary128) generator: SPEC acceptance 2 and 6 fixtures, and
    the `regions` subcommand."""
    path, sp = _gen_binary()
    r = sp.run([path, "selftest"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    r = sp.run([path, "regions", "--kmax", "32", "--eps", "5e-14"], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "x0=11.899848152108484 x1=28.98933773882074"
    r = sp.run([path, "regions", "--kmax", "32"], capture_output=True, text=True)
    assert r.returncode == 1  # input error: missing flag


def test_native_generator_matches_the_mpmath_restatement_cpu():
    """r_B by the reference's golden-section search on the CPU: the binary128
    and the 50-digit mpmath restatements take the same exchange path (same
    iteration count) to the same minimax error."""
    path, sp = _gen_binary()
    r = sp.run([path, "remez", "--region", "B", "--n", "5", "--m", "6", "--mp"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    head = dict(kv.split("=") for kv in r.stdout.splitlines()[0].split())
    assert int(head["alternation"]) == 13
    assert abs(float(head["sup"]) - 9.50270970198117e-15) < 1e-19  # mpmath backend, DESIGN.md 3.4
