"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the pin of SURVEY.md §8(c) / DESIGN.md §4 it implements.  None of them
re-types the oracle's own formula: they compare against library routines (numpy
leggauss, scipy BSpline/quad/eigh), closed forms (cardinal B-splines, integrals of the
weight), invariants (partition of unity, symmetry, S.1 = 0), worked examples printed in
SPEC.md, and brute force (np.kron of independently checked 1D Grams).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.filterwarnings("ignore::scipy.integrate.IntegrationWarning")

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _frac(s):
    return float(Fraction(s))


# --------------------------------------------------------------------------- Gauss rule
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 9])
def test_gauss_matches_numpy_leggauss(m):
    x, w = oracle.gauss_legendre(m)
    xr, wr = np.polynomial.legendre.leggauss(m)
    assert np.allclose(x, xr, atol=2e-16, rtol=0)
    assert np.allclose(w, wr, atol=1e-15, rtol=0)  # a few ulp (G2)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5])
def test_gauss_exact_to_degree_2m_minus_1(m):
    """P11: m points integrate x^j exactly for j <= 2m-1."""
    x, w = oracle.gauss_legendre(m)
    for j in range(2 * m):
        exact = 0.0 if j % 2 else 2.0 / (j + 1)
        assert abs(np.dot(w, x ** j) - exact) < 1e-15
    j = 2 * m  # first non-exact degree
    assert abs(np.dot(w, x ** j) - 2.0 / (j + 1)) > 1e-6


def test_gauss_spec_examples_on_unit_interval():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["gauss_01"]
    for case in ex:
        x, w = oracle.gauss_legendre(case["m"])
        nodes = [eval(v, {"sqrt": math.sqrt}) if isinstance(v, str) else v for v in case["nodes"]]
        assert np.allclose(0.5 * (x + 1), nodes, atol=1e-16)
        assert np.allclose(0.5 * w, case["weights"], atol=1e-16)
    # int_0^1 x^3 = 1/4 with m = 2
    x, w = oracle.gauss_legendre(2)
    assert abs(np.dot(0.5 * w, (0.5 * (x + 1)) ** 3) - 0.25) < 1e-16


# --------------------------------------------------------------------------- basis
def test_basis_spec_examples():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["basis"]
    for case in ex:
        v, d = oracle.basis_all(case["knots"], case["p"], case["t"])
        if "vals" in case:
            assert np.allclose(v, case["vals"], atol=1e-15)
        if "ders" in case:
            assert np.allclose(d, case["ders"], atol=1e-14)


def _random_open_knots(rng, n, p, repeat=False):
    inner = np.sort(rng.uniform(0.02, 0.98, n - p - 1))
    if repeat and n - p - 1 >= 3:
        inner[1] = inner[2]  # one double interior knot (multiplicity <= p)
    return np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)])


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("repeat", [False, True])
def test_basis_matches_scipy_bspline(p, repeat):
    """Cox-de Boor values/derivatives vs scipy.interpolate.BSpline (library routine)."""
    from scipy.interpolate import BSpline
    rng = np.random.default_rng(100 + p)
    n = p + 7
    k = _random_open_knots(rng, n, p, repeat and p >= 2)
    for t in rng.uniform(0, 1, 25):
        v, d = oracle.basis_all(k, p, t)
        for i in range(n):
            c = np.zeros(n)
            c[i] = 1.0
            b = BSpline(k, c, p, extrapolate=False)
            assert abs(v[i] - b(t)) < 1e-14
            assert abs(d[i] - b.derivative()(t)) < 1e-11 * max(1, abs(d[i]))
        assert abs(v.sum() - 1) < 1e-14          # partition of unity
        assert abs(d.sum()) < 1e-11 * n           # derivatives sum to 0


def test_basis_right_endpoint():
    k = synth.uniform_open_knots(6, 3)
    v, _ = oracle.basis_all(k, 3, 1.0)
    assert v[-1] == 1.0 and abs(v[:-1]).max() == 0.0


# --------------------------------------------------------------------------- 1D Grams
def _cardinal(m_deg, x):
    """Centred cardinal B-spline of degree m_deg at x (exact Fractions):
    N_m(x) = 1/(m-1)! sum_j (-1)^j C(m,j) (x - j)_+^{m-1}, order m = deg+1, centred."""
    m = m_deg + 1
    xs = Fraction(x) + Fraction(m, 2)
    s = Fraction(0)
    for j in range(m + 1):
        t = xs - j
        if t > 0:
            s += (-1) ** j * math.comb(m, j) * t ** (m - 1)
    return s / math.factorial(m - 1)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_p1_uniform_interior_rows_closed_form(p):
    """P1: interior rows of w==1 Grams on uniform knots equal cardinal B-spline values
    (golden rationals, and re-derived here from the cardinal B-spline formula)."""
    g = json.load(open(os.path.join(GOLD, "p1_uniform_gram.json")))
    mass = [_frac(s) for s in g["mass_over_h"][str(p)]]
    stiff = [_frac(s) for s in g["stiff_times_h"][str(p)]]
    for k in range(p + 1):
        assert abs(float(_cardinal(2 * p + 1, k)) - mass[k]) < 1e-17
        c = lambda j: _cardinal(2 * p - 1, j)
        assert abs(float(2 * c(k) - c(k - 1) - c(k + 1)) - stiff[k]) < 1e-16
    n = 4 * p + 8
    kn = synth.uniform_open_knots(n, p)
    h = 1.0 / (n - p)
    M = oracle.gram_1d(kn, p, p + 1, 0.0, 1.0, 0.0, 0, 0)
    K = oracle.gram_1d(kn, p, p + 1, 0.0, 1.0, 0.0, 1, 1)
    for i in range(2 * p, n - 2 * p):
        for k in range(p + 1):
            assert abs(M[i, i + k] / h - mass[k]) < 1e-14
            assert abs(K[i, i + k] * h - stiff[k]) < 1e-13
        assert np.all(M[i, i + p + 1:] == 0) and np.all(K[i, i + p + 1:] == 0)  # band zeros exact


def test_p1_boundary_p1():
    n, p = 9, 1
    kn = synth.uniform_open_knots(n, p)
    h = 1.0 / (n - p)
    M = oracle.gram_1d(kn, p, 2, 0.0, 1.0, 0.0, 0, 0)
    K = oracle.gram_1d(kn, p, 2, 0.0, 1.0, 0.0, 1, 1)
    assert abs(M[0, 0] - h / 3) < 1e-16 and abs(M[-1, -1] - h / 3) < 1e-16
    assert abs(K[0, 0] - 1 / h) < 1e-13


def test_p2_single_span():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["gram_single_span_p1"]
    M = oracle.gram_1d(g["knots"], 1, 2, 0.0, 1.0, 0.0, 0, 0)
    K = oracle.gram_1d(g["knots"], 1, 2, 0.0, 1.0, 0.0, 1, 1)
    assert np.allclose(M, [[_frac(v) for v in r] for r in g["mass"]], atol=1e-16)
    assert np.allclose(K, [[_frac(v) for v in r] for r in g["stiff"]], atol=1e-15)
    # w == 0 gives exactly zero (amp=-1, k=0, phi=pi/2 -> 1 - sin(pi/2) = 0)
    Z = oracle.gram_1d(g["knots"], 1, 2, -1.0, 0.0, math.pi / 2, 0, 0)
    assert np.all(Z == 0)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_gram_weighted_vs_scipy_quad(p):
    """Weighted Gram with the sine weight vs adaptive quadrature of scipy BSpline products
    (library routines); our rule uses many points per span so the rule error vanishes."""
    from scipy.integrate import quad
    from scipy.interpolate import BSpline
    n = p + 5
    kn = synth.uniform_open_knots(n, p)
    amp, kk, phi = 0.5, 3.0, 1.2
    for a, b in [(0, 0), (1, 1), (1, 0), (0, 1)]:
        G = oracle.gram_1d(kn, p, 12, amp, kk, phi, a, b)
        bs = []
        for i in range(n):
            c = np.zeros(n)
            c[i] = 1
            s = BSpline(kn, c, p, extrapolate=False)
            bs.append(s.derivative() if False else s)
        for i in range(n):
            for j in range(n):
                fi = bs[i].derivative() if a else bs[i]
                fj = bs[j].derivative() if b else bs[j]
                f = lambda t: np.nan_to_num(fi(t)) * np.nan_to_num(fj(t)) * (1 + amp * math.sin(kk * math.pi * t + phi))
                ref = sum(quad(f, kn[s], kn[s + 1], epsabs=1e-15, epsrel=1e-14)[0]
                          for s in range(len(kn) - 1) if kn[s] < kn[s + 1])
                assert abs(G[i, j] - ref) < 1e-12 * max(1.0, abs(ref))


def test_gram_transpose_and_spd():
    """T = E^T and SPD mass for a positive weight."""
    kn = synth.uniform_open_knots(11, 3)
    T = oracle.gram_1d(kn, 3, 4, 0.5, 2.0, 0.3, 1, 0)
    E = oracle.gram_1d(kn, 3, 4, 0.5, 2.0, 0.3, 0, 1)
    assert np.abs(T - E.T).max() < 1e-15 * np.abs(T).max()  # equal up to product order
    M = oracle.gram_1d(kn, 3, 4, 0.5, 2.0, 0.3, 0, 0)
    assert np.linalg.eigvalsh(M).min() > 0


# --------------------------------------------------------------------------- 3D problems
def _tiny(n=5, p=2, R=2, seed=7, dirichlet=False, nq=None):
    """Anisotropic reading-A weights (G6) on a tiny mesh."""
    cfg = synth.Config(99, "tiny", n=n, p=p, R=R, batch=1, dirichlet=dirichlet)
    w = synth.draw_weights(cfg, np.random.default_rng(seed))
    return cfg, w, oracle.problem_from_config(cfg, w, nq=nq)


def _kron_bruteforce(cfg, w, nq):
    """P10: sum_r (x)_d of independently pinned 1D Grams, densified with np.kron
    (z slowest).  Mass: M^{(d)}(w_r^{(d)}); stiffness block (k,l) dir d: pattern
    (row deriv [l==d], col deriv [k==d])."""
    kn = synth.uniform_open_knots(cfg.n, cfg.p)
    p = cfg.p
    N = cfg.n ** 3
    M = np.zeros((N, N))
    S = np.zeros((N, N))
    for r in range(w.mass.shape[0]):
        fac = [oracle.gram_1d(kn, p, nq, *w.mass[r, 1 + 3 * d:4 + 3 * d], 0, 0) for d in range(3)]
        M += w.mass[r, 0] * np.kron(fac[2], np.kron(fac[1], fac[0]))
    for k in range(3):
        for l in range(3):
            for r in range(w.v.shape[0]):
                fac = [oracle.gram_1d(kn, p, nq, *w.v[r, d], int(l == d), int(k == d)) for d in range(3)]
                S += w.A[r, k, l] * np.kron(fac[2], np.kron(fac[1], fac[0]))
    return M, S


@pytest.mark.parametrize("n,p,R", [(5, 2, 2), (6, 3, 1), (4, 1, 3)])
def test_p10_bruteforce_kron_equals_3d_assembly(n, p, R):
    """Separable weight + tensor Gauss rule => the Kronecker sum EQUALS the 3D assembly
    (SURVEY finding 2).  Entrywise <= 1e-14 and Frobenius diff."""
    cfg, w, P = _tiny(n, p, R)
    M, S = oracle.assemble_csr(P)
    Mk, Sk = _kron_bruteforce(cfg, w, p + 1)
    Md, Sd = M.toarray(), S.toarray()
    assert np.abs(Md - Mk).max() < 1e-14 * np.abs(Mk).max() * 10
    assert np.abs(Sd - Sk).max() < 1e-13 * np.abs(Sk).max()
    assert np.linalg.norm(Sd - Sk) / np.linalg.norm(Sk) < 1e-14
    # CSR pattern contains every nonzero of the brute force
    assert np.all((Mk != 0) <= (Md != 0) | (np.abs(Mk) < 1e-300))


def test_p3_kron_vec_identity():
    """P3: (A (x) B) vec(X) = vec(B X A^T) for the layout used by the
    oracle's brute force (C order, x fastest)."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((4, 4))
    B = rng.standard_normal((5, 5))
    X = rng.standard_normal((4, 5))  # [slow, fast]
    assert np.allclose(np.kron(A, B) @ X.reshape(-1), (A @ X @ B.T).reshape(-1), atol=1e-13)


def _omega_integral(mass_terms):
    """closed-form int_[0,1]^3 omega = sum_r coef prod_d (1 + amp (cos phi - cos(k pi + phi))/(k pi))"""
    tot = 0.0
    for T in mass_terms:
        f = T[0]
        for d in range(3):
            amp, k, ph = T[1 + 3 * d:4 + 3 * d]
            f *= 1 + amp * (math.cos(ph) - math.cos(k * math.pi + ph)) / (k * math.pi)
        tot += f
    return tot


@pytest.mark.parametrize("cfgname", ["c1", "c2", "c3", "c5"])
def test_p4_partition_of_unity_mass(cfgname):
    """P4: 1^T M 1 = int omega (partition of unity) with each config's
    weights, on a small mesh with a rule accurate to rounding (nq=10)."""
    cfg = synth.CONFIGS[cfgname]
    w = synth.draw_weights(cfg)
    P = oracle.problem_from_config(cfg, w, n=cfg.p + 4, nq=10)
    one = np.ones(P.ndof)
    rows = np.arange(P.ndof)
    yM, yS = oracle.apply_rows(P, one, rows)
    assert abs(yM.sum() - _omega_integral(w.mass)) < 1e-13 * abs(_omega_integral(w.mass))
    # P5: S 1 = 0 (every term carries a derivative on the column function)
    assert np.abs(yS).max() < 1e-13 * max(1.0, np.abs(w.A).max())


def test_p4_c1_exact():
    cfg = synth.CONFIGS["c1"]
    knots, w, x = synth.draw_problem(cfg)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    one = np.ones(P.ndof)
    assert abs(one @ oracle.spmv(M, one) - 1.0) < 1e-14
    assert np.abs(oracle.spmv(S, one)).max() < 1e-14


def test_p6_symmetry_and_definiteness():
    cfg, w, P = _tiny(6, 2, 2, seed=11)
    M, S = oracle.assemble_csr(P)
    Md, Sd = M.toarray(), S.toarray()
    assert np.abs(Md - Md.T).max() < 1e-16
    assert np.abs(Sd - Sd.T).max() < 1e-15
    assert np.linalg.eigvalsh(Md).min() > 0
    ev = np.linalg.eigvalsh(Sd)
    assert ev.min() > -1e-13 and abs(ev.min()) < 1e-12  # semidefinite, kernel = constants
    cfgd, wd, Pd = _tiny(7, 2, 2, seed=11, dirichlet=True)
    Md2, Sd2 = (A.toarray() for A in oracle.assemble_csr(Pd))
    assert np.linalg.eigvalsh(Sd2).min() > 1e-6  # SPD with Dirichlet


def test_dirichlet_equals_deleting_boundary_rows_cols():
    """A4 / SPEC.md:325-328: eliminating boundary DoFs = deleting rows & columns."""
    _, w, P = _tiny(7, 3, 2, seed=5)
    _, _, Pd = _tiny(7, 3, 2, seed=5, dirichlet=True)
    M, S = (A.toarray() for A in oracle.assemble_csr(P))
    Md, Sd = (A.toarray() for A in oracle.assemble_csr(Pd))
    n = 7
    keep = [((iz * n) + iy) * n + ix for iz in range(1, n - 1) for iy in range(1, n - 1) for ix in range(1, n - 1)]
    assert np.array_equal(M[np.ix_(keep, keep)], Md)
    assert np.array_equal(S[np.ix_(keep, keep)], Sd)


def test_p7_c1_generalised_eigen():
    """P7: w==1, Q=I: S(v_a (x) v_b (x) v_c) = (mu_a+mu_b+mu_c) M(v_a (x) v_b (x) v_c)
    with 1D pairs K1 v = mu M1 v from scipy.linalg.eigh (library routine)."""
    import scipy.linalg
    cfg = synth.CONFIGS["c1"]
    _, w, _ = synth.draw_problem(cfg)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    kn = synth.uniform_open_knots(cfg.n, cfg.p)
    M1 = oracle.gram_1d(kn, cfg.p, cfg.p + 1, 0, 1, 0, 0, 0)
    K1 = oracle.gram_1d(kn, cfg.p, cfg.p + 1, 0, 1, 0, 1, 1)
    mu, V = scipy.linalg.eigh(K1, M1)
    for (a, b, c) in [(0, 0, 0), (1, 2, 3), (7, 0, 5), (4, 4, 4), (7, 7, 6)]:
        v = np.kron(V[:, c], np.kron(V[:, b], V[:, a]))
        lhs = oracle.spmv(S, v)
        rhs = (mu[a] + mu[b] + mu[c]) * oracle.spmv(M, v)
        assert np.abs(lhs - rhs).max() < 1e-11 * max(1.0, np.abs(rhs).max())


def test_p8_c1_linear_reproduction():
    """P8: Greville coordinates g reproduce x: 1'Mg = 1/2, g'Mg = 1/3,
    (Sg)_i = (int d_x beta_ix)(int beta_iy)(int beta_iz) with int d_x beta = beta(1)-beta(0)."""
    cfg = synth.CONFIGS["c1"]
    _, w, _ = synth.draw_problem(cfg)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    n, p = cfg.n, cfg.p
    kn = synth.uniform_open_knots(n, p)
    gre = np.array([kn[i + 1:i + p + 1].mean() for i in range(n)])
    g = np.tile(gre, n * n)  # x-coordinate, x fastest
    one = np.ones(n ** 3)
    assert abs(one @ oracle.spmv(M, g) - 0.5) < 1e-14
    assert abs(g @ oracle.spmv(M, g) - 1.0 / 3.0) < 1e-14
    ib = np.array([(kn[i + p + 1] - kn[i]) / (p + 1) for i in range(n)])  # int beta_i
    dx = np.zeros(n)
    dx[0], dx[-1] = -1.0, 1.0
    ref = np.kron(ib, np.kron(ib, dx))
    assert np.abs(oracle.spmv(S, g) - ref).max() < 1e-14


@pytest.mark.parametrize("dirichlet", [False, True])
def test_p12_three_routes_agree(dirichlet):
    """P12: CSR+SpMV, element-loop and row-restricted bilinear form agree <= 1e-13."""
    cfg, w, P = _tiny(9, 3, 3, seed=21, dirichlet=dirichlet)
    M, S = oracle.assemble_csr(P)
    x = np.random.default_rng(2).standard_normal((2,) + tuple(P.dims[::-1]))
    yM, yS = oracle.apply_matfree(P, x)
    for b in range(2):
        rm = oracle.spmv(M, x[b])
        rs = oracle.spmv(S, x[b])
        assert np.abs(yM[b].ravel() - rm).max() < 1e-13 * np.abs(rm).max()
        assert np.abs(yS[b].ravel() - rs).max() < 1e-13 * np.abs(rs).max()
        rows = np.arange(0, P.ndof, 7)
        am, as_ = oracle.apply_rows(P, x[b], rows)
        assert np.abs(am - rm[rows]).max() < 1e-13 * np.abs(rm).max()
        assert np.abs(as_ - rs[rows]).max() < 1e-13 * np.abs(rs).max()


def test_nonuniform_and_repeated_knots_bruteforce():
    """Non-uniform knots with a double interior knot (C^{p-2}): 3D assembly still equals
    the np.kron of 1D Grams (reading A weights)."""
    rng = np.random.default_rng(9)
    p = 3
    kn = [_random_open_knots(rng, 8, p, repeat=True) for _ in range(3)]
    cfg = synth.Config(98, "nonuni", n=8, p=p, R=1, batch=1)
    w = synth.draw_weights(cfg, np.random.default_rng(4))
    P = oracle.Problem(knots=kn, p=[p] * 3, nq=p + 1, mass_terms=w.mass, q_terms=w.q_block_terms())
    M, S = (A.toarray() for A in oracle.assemble_csr(P))
    facM = [oracle.gram_1d(kn[d], p, p + 1, *w.mass[0, 1 + 3 * d:4 + 3 * d], 0, 0) for d in range(3)]
    Mk = np.kron(facM[2], np.kron(facM[1], facM[0]))
    Sk = 0
    for k in range(3):
        for l in range(3):
            fac = [oracle.gram_1d(kn[d], p, p + 1, *w.v[0, d], int(l == d), int(k == d)) for d in range(3)]
            Sk = Sk + w.A[0, k, l] * np.kron(fac[2], np.kron(fac[1], fac[0]))
    assert np.abs(M - Mk).max() < 1e-14 * np.abs(Mk).max() * 10
    assert np.abs(S - Sk).max() < 1e-13 * np.abs(Sk).max()


# --------------------------------------------------------------------------- KKT
def _kkt_small(nt=3, n=6, seed=1):
    cfg = synth.Config(97, "kkt", n=n, p=2, R=2, batch=1, dirichlet=True, n_t=nt, tau=1.0 / nt, beta=1e-2)
    w = synth.draw_weights(cfg, np.random.default_rng(seed))
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    return cfg, P, M, S


def test_p9_kkt_symmetric_indefinite():
    """P9/P6: the KKT operator of Eq. (KKTSystem) is symmetric and indefinite
    (saddle point); a sign or time-index error breaks symmetry."""
    cfg, P, M, S = _kkt_small()
    N = P.ndof
    dim = 3 * cfg.n_t * N
    K = np.zeros((dim, dim))
    for c in range(dim):
        e = np.zeros(dim)
        e[c] = 1
        K[:, c] = oracle.kkt_apply_csr(M, S, e.reshape(3, cfg.n_t, N), cfg.tau, cfg.beta).ravel()
    assert np.abs(K - K.T).max() < 1e-15 * np.abs(K).max() * 10
    ev = np.linalg.eigvalsh(0.5 * (K + K.T))
    assert ev.min() < 0 < ev.max()


def test_p9_kkt_special_cases():
    cfg, P, M, S = _kkt_small(nt=4)
    N = P.ndof
    rng = np.random.default_rng(5)
    tau, beta = cfg.tau, cfg.beta
    # u = lambda / beta  =>  r_u = 0
    X = rng.standard_normal((3, cfg.n_t, N))
    X[1] = X[2] / beta
    out = oracle.kkt_apply_csr(M, S, X, tau, beta)
    assert np.abs(out[1]).max() < 1e-13 * np.abs(out).max()
    # constant-in-time y, u = lambda = 0: r_lam[1] = (M + tau S) y, r_lam[k>1] = tau S y
    y = rng.standard_normal(N)
    X = np.zeros((3, cfg.n_t, N))
    X[0, :] = y
    out = oracle.kkt_apply_csr(M, S, X, tau, beta)
    My, Sy = M @ y, S @ y
    assert np.allclose(out[2, 0], My + tau * Sy, atol=1e-14)
    for k in range(1, cfg.n_t):
        assert np.allclose(out[2, k], tau * Sy, atol=1e-14)
    assert np.allclose(out[1], 0, atol=0)
    # r_y = tau M y_k (lambda = 0)
    assert np.allclose(out[0], tau * My[None], atol=1e-15)


def test_p9_kkt_time_matrix_c():
    """C . 1 = e_1: with y_k = v for all k, u = lam = 0, the constraint rows
    of the M-part telescope: sum over the C (x) M block = M v at step 1 only."""
    cfg, P, M, S = _kkt_small(nt=5)
    N = P.ndof
    v = np.random.default_rng(8).standard_normal(N)
    X = np.zeros((3, cfg.n_t, N))
    X[0, :] = v
    S0 = S * 0.0
    out = oracle.kkt_apply_csr(M, S0, X, cfg.tau, cfg.beta)  # K = 0 => r_lam = (C (x) M) y
    assert np.allclose(out[2, 0], M @ v, atol=1e-15)
    assert np.abs(out[2, 1:]).max() < 1e-15


def test_kkt_rows_matches_full():
    cfg, P, M, S = _kkt_small(nt=3, n=7)
    N = P.ndof
    X = np.random.default_rng(6).standard_normal((3, cfg.n_t, N))
    full = oracle.kkt_apply_csr(M, S, X, cfg.tau, cfg.beta)
    rows = np.array([0, 3, N // 2, N - 1])
    steps = [0, 1, 2]
    samp = oracle.kkt_rows(P, X, cfg.tau, cfg.beta, steps, rows)
    for j, k in enumerate(steps):
        assert np.abs(samp[:, j] - full[:, k][:, rows]).max() < 1e-13 * np.abs(full).max()


def test_kkt_nt1_reduces_to_single_step():
    cfg, P, M, S = _kkt_small(nt=1)
    N = P.ndof
    X = np.random.default_rng(2).standard_normal((3, 1, N))
    out = oracle.kkt_apply_csr(M, S, X, cfg.tau, cfg.beta)
    y, u, lam = X[0, 0], X[1, 0], X[2, 0]
    t, b = cfg.tau, cfg.beta
    # single step: [tau M, 0, (M + tau K)^T; 0, tau b M, -tau M; M + tau K, -tau M, 0]
    A = (M + t * S).toarray()
    Md = M.toarray()
    assert np.allclose(out[0, 0], t * Md @ y + A.T @ lam, atol=1e-14)
    assert np.allclose(out[1, 0], t * b * Md @ u - t * Md @ lam, atol=1e-15)
    assert np.allclose(out[2, 0], A @ y - t * Md @ u, atol=1e-14)


# ------------------------------------------------------------- general (tabulated) weights
def _tab3(P, fields):
    """A weight field evaluated on the oracle's own tensor quadrature grid."""
    nodes = [oracle.quad_nodes(P.knots[d], P.p[d], P.nq) for d in range(3)]
    return fields(nodes[0], nodes[1], nodes[2])


def test_weights3d_separable_equals_closed_form():
    """The tabulated-weight path (Eqs. (massMatrix)/(stiffnessMatrix), with
    omega and Q given at every 3D point) reproduces the closed-form separable path when the table
    holds the same separable weights."""
    cfg = synth.scaled(synth.CONFIGS["c2"], 7)
    w = synth.draw_weights(cfg)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)

    def sep(terms):
        def f(x, y, z):
            out = np.zeros((len(z), len(y), len(x)))
            for T in np.asarray(terms).reshape(-1, synth.TERM_WIDTH):
                fx, fy, fz = (1.0 + T[1 + 3 * d] * np.sin(T[2 + 3 * d] * np.pi * t + T[3 + 3 * d])
                              for d, t in enumerate((x, y, z)))
                out += T[0] * fz[:, None, None] * fy[None, :, None] * fx[None, None, :]
            return out
        return f

    qb = w.q_block_terms()
    w3 = np.zeros((10,) + _tab3(P, sep(w.mass)).shape)
    w3[0] = _tab3(P, sep(w.mass))
    for b in range(9):
        if qb[b] is not None and len(qb[b]):
            w3[1 + b] = _tab3(P, sep(qb[b]))
    P3 = oracle.Problem(knots=P.knots, p=P.p, nq=P.nq, mass_terms=None, q_terms=None, weights3d=w3)
    M3, S3 = oracle.assemble_csr(P3)
    assert abs(M3 - M).max() <= 1e-15 * abs(M).max()
    assert abs(S3 - S).max() <= 1e-15 * abs(S).max()


def test_weights3d_annulus_volume_and_constants():
    """Quarter annulus with exact geometry weights omega = |det grad G| and
    Q = (grad G^T grad G)^-1 |det grad G|: 1'M1 = physical volume (partition of
    unity; omega is linear in s, so the 5-point rule is exact) and S 1 = 0."""
    from synth.geometry import QuarterAnnulus, refinement_knots
    g = QuarterAnnulus()
    kn = refinement_knots(2, 3)
    P = oracle.Problem(knots=[kn] * 3, p=[2] * 3, nq=5, mass_terms=None, q_terms=None,
                       weights3d=_tab3(oracle.Problem(knots=[kn] * 3, p=[2] * 3, nq=5, mass_terms=None,
                                                      q_terms=None), g.fields))
    M, S = oracle.assemble_csr(P)
    one = np.ones(P.ndof)
    assert abs(one @ (M @ one) - g.volume) <= 1e-13 * g.volume
    assert np.abs(S @ one).max() <= 1e-13 * abs(S).max()


# ------------------------------------------------------------------ TT oracle (NEXT-3)
def _cores(rng, m, R1, R2):
    mz, my, mx = m
    return (rng.standard_normal((mz, R1)), rng.standard_normal((R1, my, R2)), rng.standard_normal((R2, mx)))


def test_tt_full_brute_force():
    rng = np.random.default_rng(1)
    gz, gy, gx = _cores(rng, (3, 4, 2), 2, 3)
    v = oracle.tt_full(gz, gy, gx)
    for iz, iy, ix in [(0, 0, 0), (2, 3, 1), (1, 2, 0)]:
        ref = sum(gz[iz, a] * gy[a, iy, b] * gx[b, ix] for a in range(2) for b in range(3))
        assert abs(v[iz, iy, ix] - ref) <= 1e-14


@pytest.mark.parametrize("site", [0, 1, 2])
def test_tt_frame_linearity(site):
    """Eq. (ttlin): F_{!=d} vec(G_d) is the represented tensor."""
    rng = np.random.default_rng(2 + site)
    gz, gy, gx = _cores(rng, (3, 4, 5), 2, 3)
    F = oracle.tt_frame(gz, gy, gx, site)
    vec = {0: gx.ravel(), 1: gy.ravel(), 2: gz.ravel()}[site]
    assert np.allclose(F @ vec, oracle.tt_full(gz, gy, gx).ravel(), atol=1e-13)


@pytest.mark.parametrize("site", [0, 1, 2])
def test_tt_projection_identity_and_symmetry(site):
    """Orthogonal frames project the identity to the identity (the SVD makes
    the frame orthogonal); a symmetric operator projects to a symmetric matrix."""
    rng = np.random.default_rng(7)
    m = (4, 5, 3)
    gz, gy, gx = _cores(rng, m, 2, 3)
    # orthogonalise the cores away from the site: left cores left-orthogonal, right ones right-orthogonal
    if site in (0, 1):
        gz = np.linalg.qr(gz)[0]
    if site == 0:
        q = np.linalg.qr(gy.reshape(-1, gy.shape[2]))[0]
        gy = q.reshape(gy.shape)
    if site in (1, 2):
        gx = np.linalg.qr(gx.T)[0].T
    if site == 2:
        q = np.linalg.qr(gy.reshape(gy.shape[0], -1).T)[0].T
        gy = q.reshape(gy.shape)
    N = m[0] * m[1] * m[2]
    P = oracle.tt_project(np.eye(N), gz, gy, gx, site)
    assert np.allclose(P, np.eye(P.shape[0]), atol=1e-12)
    B = rng.standard_normal((N, N))
    Ps = oracle.tt_project(B + B.T, gz, gy, gx, site)
    assert np.allclose(Ps, Ps.T, atol=1e-12)


# ------------------------------------------------------- KKT with a non-symmetric stiffness
def _kkt_small_nonsym(nt=3, n=6, seed=11):
    """Every q_kl is approximated on its own, so q_kl != q_lk is a valid
    input and K need not be symmetric: scale the (x,y) and (y,z) blocks of A_r only."""
    cfg = synth.Config(96, "kkt_nonsym", n=n, p=2, R=2, batch=1, dirichlet=True, n_t=nt, tau=1.0 / nt, beta=1e-2)
    w = synth.draw_weights(cfg, np.random.default_rng(seed))
    w.A[:, 0, 1] *= 1.7
    w.A[:, 1, 2] *= -0.5
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    return cfg, P, M, S


def test_nonsym_stiffness_is_nonsymmetric_and_transpose_problem_is_its_transpose():
    """Eq. (stiffnessMatrix) PAPER.md:140-143 with Q^T gives K^T (definition, entry by entry)."""
    cfg, P, M, S = _kkt_small_nonsym()
    Sd = S.toarray()
    assert np.abs(Sd - Sd.T).max() > 1e-3 * np.abs(Sd).max()
    _, ST = oracle.assemble_csr(oracle.transpose_problem(P))
    assert np.abs(ST.toarray() - Sd.T).max() < 1e-15 * np.abs(Sd).max() * 10
    # transposing twice is the identity on the problem
    _, S2 = oracle.assemble_csr(oracle.transpose_problem(oracle.transpose_problem(P)))
    assert np.abs(S2.toarray() - Sd).max() == 0.0


def test_p9_kkt_symmetric_with_nonsymmetric_stiffness():
    """Eq. (KKTSystem) PAPER.md:313-319 has calK^T in the first block row, so the KKT matrix
    is symmetric for ANY K; applying K (instead of K^T) to lambda in the y-row breaks it."""
    cfg, P, M, S = _kkt_small_nonsym()
    N = P.ndof
    dim = 3 * cfg.n_t * N
    K = np.zeros((dim, dim))
    for c in range(dim):
        e = np.zeros(dim)
        e[c] = 1
        K[:, c] = oracle.kkt_apply_csr(M, S, e.reshape(3, cfg.n_t, N), cfg.tau, cfg.beta).ravel()
    assert np.abs(K - K.T).max() < 1e-14 * np.abs(K).max()
    # ... and equals the block matrix assembled from calK = I (x) tau K + C (x) M (kkt_dense)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, cfg.beta)
    assert np.abs(K - A).max() < 1e-14 * np.abs(A).max()


def test_kkt_apply_equals_dense_nonsym():
    cfg, P, M, S = _kkt_small_nonsym(nt=4, n=7)
    N = P.ndof
    X = np.random.default_rng(12).standard_normal((3, cfg.n_t, N))
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, cfg.beta)
    out = oracle.kkt_apply_csr(M, S, X, cfg.tau, cfg.beta)
    ref = A @ X.ravel()
    assert np.linalg.norm(out.ravel() - ref) < 1e-14 * np.linalg.norm(ref)
    # the y-row carries K^T lambda: with y = u = 0 it is (M + tau K)^T lambda_k - M lambda_{k+1}
    X0 = np.zeros_like(X)
    X0[2] = X[2]
    o0 = oracle.kkt_apply_csr(M, S, X0, cfg.tau, cfg.beta)
    At = (M + cfg.tau * S).toarray().T
    for k in range(cfg.n_t):
        nxt = M @ X[2, k + 1] if k + 1 < cfg.n_t else 0.0
        assert np.allclose(o0[0, k], At @ X[2, k] - nxt, atol=1e-14)


def test_kkt_rows_matches_full_nonsym():
    cfg, P, M, S = _kkt_small_nonsym(nt=3, n=7)
    N = P.ndof
    X = np.random.default_rng(13).standard_normal((3, cfg.n_t, N))
    full = oracle.kkt_apply_csr(M, S, X, cfg.tau, cfg.beta)
    rows = np.array([0, 5, N // 2, N - 1])
    steps = [0, 1, 2]
    samp = oracle.kkt_rows(P, X, cfg.tau, cfg.beta, steps, rows)
    for j, k in enumerate(steps):
        assert np.abs(samp[:, j] - full[:, k][:, rows]).max() < 1e-13 * np.abs(full).max()


def test_csr_row_range_assembly_matches_full():
    """P12-style self-consistency: the row-range assembly (bench samples of full-size CSR) is the
    full assembly's rows, entry for entry, including Dirichlet problems."""
    for dirichlet in (False, True):
        cfg = synth.Config(95, "rows", n=9, p=3, R=2, batch=1, dirichlet=dirichlet)
        w = synth.draw_weights(cfg, np.random.default_rng(9))
        P = oracle.problem_from_config(cfg, w)
        M, S = oracle.assemble_csr(P)
        N = P.ndof
        for r0, r1 in [(0, 7), (N // 3, N // 3 + 50), (N - 13, N), (0, N)]:
            Mr, Sr = oracle.assemble_csr_rows(P, r0, r1)
            assert (abs(Mr - M[r0:r1]).max() == 0.0) and (abs(Sr - S[r0:r1]).max() == 0.0)
            x = np.random.default_rng(r0).standard_normal(N)
            assert np.array_equal(oracle.spmv(Sr, x), oracle.spmv(S, x)[r0:r1])
