"""CPU pins of the NEXT-1 oracle pieces: the dense KKT matrix and the MINRES recurrence.

kkt_dense is pinned against the paper's gradient rows (oracle.kkt_apply, an
independent formulation); minres is pinned against closed forms (the first MINRES iterate),
the minimum-residual property, a library routine (scipy.sparse.linalg.minres) and dense LU;
the KKT solutions are pinned against PAPER.md:307 (u = lambda / beta) and the paper's
observation that the control magnitude decreases as beta grows.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as sla

import oracle
import synth


def small_kkt(n=7, n_t=3, beta=None):
    cfg = synth.scaled(synth.CONFIGS["c4"], n, n_t=n_t)
    w = synth.draw_weights(cfg)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    b = cfg.beta if beta is None else beta
    return cfg, M, S, b


def rhs_tracking(M, n_t, tau, seed=5):
    """[tau calM yhat; 0; 0] for a seeded desired state yhat (Eq. (KKTSystem) right-hand side)."""
    N = M.shape[0]
    yhat = np.random.default_rng(seed).standard_normal((n_t, N))
    top = np.stack([tau * oracle.spmv(M, yhat[k]) for k in range(n_t)])
    return np.concatenate([top.ravel(), np.zeros(2 * n_t * N)]), yhat


def test_kkt_dense_matches_gradient_rows():
    cfg, M, S, beta = small_kkt()
    N = M.shape[0]
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    X = np.random.default_rng(1).standard_normal((3, cfg.n_t, N))
    ref = oracle.kkt_apply_csr(M, S, X, cfg.tau, beta)
    got = (A @ X.ravel()).reshape(X.shape)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    assert np.allclose(A, A.T, rtol=0, atol=1e-15 * np.abs(A).max())  # saddle-point matrix is symmetric


def test_minres_first_iterate_closed_form():
    # x_1 minimises |b - A x| over span{b}:  x_1 = (b'Ab / |Ab|^2) b
    cfg, M, S, beta = small_kkt(n=6, n_t=2)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    b = np.random.default_rng(2).standard_normal(A.shape[0])
    x1, it, _, _ = oracle.minres(lambda v: A @ v, b, maxit=1, rtol=0.0)
    Ab = A @ b
    ref = (b @ Ab) / (Ab @ Ab) * b
    assert it == 1
    assert np.linalg.norm(x1 - ref) <= 1e-13 * np.linalg.norm(ref)


def test_minres_residual_recurrence_and_monotone():
    cfg, M, S, beta = small_kkt(n=6, n_t=2)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    b = np.random.default_rng(3).standard_normal(A.shape[0])
    prev = np.linalg.norm(b)
    for k in range(1, 25):
        xk, it, relres, res0 = oracle.minres(lambda v: A @ v, b, maxit=k, rtol=0.0)
        true = np.linalg.norm(b - A @ xk)
        assert true <= prev * (1 + 1e-12)  # minimum residual over nested Krylov spaces
        assert abs(true - relres * res0) <= 1e-9 * res0  # |eta| is the residual norm
        prev = true


@pytest.mark.parametrize("k", [1, 2, 5, 10, 20])
def test_minres_iterates_match_scipy(k):
    # the same Krylov iterates as the library MINRES (before loss of orthogonality matters)
    cfg, M, S, beta = small_kkt(n=6, n_t=2, beta=1e-2)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    b = np.random.default_rng(3).standard_normal(A.shape[0])
    x, it, _, _ = oracle.minres(lambda v: A @ v, b, maxit=k, rtol=0.0)
    xl, _ = sla.minres(A, b, rtol=1e-300, maxiter=k)
    assert it == k
    assert np.linalg.norm(x - xl) <= 1e-11 * np.linalg.norm(xl)


def test_minres_converges_to_dense_lu():
    # a small, well-conditioned KKT system (cond ~ 5e5): |x - x*| <= cond * rtol |x*|
    cfg, M, S, beta = small_kkt(n=5, n_t=1, beta=1.0)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    b, _ = rhs_tracking(M, cfg.n_t, cfg.tau)
    xs = np.linalg.solve(A, b)
    x, it, relres, _ = oracle.minres(lambda v: A @ v, b, maxit=20000, rtol=1e-10)
    assert relres <= 1e-10 and it < 20000
    assert np.linalg.norm(x - xs) <= np.linalg.cond(A) * 1e-10 * np.linalg.norm(xs)


def test_kkt_solution_gradient_rows_and_u_equals_lambda_over_beta():
    # tau beta M u_k - tau M lambda_k = 0  =>  u = lambda / beta (M is SPD)
    cfg, M, S, beta = small_kkt(n=6, n_t=3, beta=1e-3)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    b, _ = rhs_tracking(M, cfg.n_t, cfg.tau)
    xs = np.linalg.solve(A, b)
    X = xs.reshape(3, cfg.n_t, -1)
    assert np.linalg.norm(X[1] - X[2] / beta) <= 1e-9 * np.linalg.norm(X[1])
    # and the three gradient rows vanish at the solution
    G = oracle.kkt_apply_csr(M, S, X, cfg.tau, beta).ravel() - b
    assert np.linalg.norm(G) <= 1e-10 * np.linalg.norm(b)


def test_control_norm_decreases_with_beta():
    # "its magnitude decreases with higher control parameter"
    cfg, M, S, _ = small_kkt(n=6, n_t=3)
    b, yhat = rhs_tracking(M, cfg.n_t, cfg.tau)
    unorm, track = [], []
    for beta in (1e-4, 1e-2, 1.0):
        A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
        X = np.linalg.solve(A, b).reshape(3, cfg.n_t, -1)
        unorm.append(sum(X[1, k] @ oracle.spmv(M, X[1, k]) for k in range(cfg.n_t)))
        track.append(sum((X[0, k] - yhat[k]) @ oracle.spmv(M, X[0, k] - yhat[k]) for k in range(cfg.n_t)))
    assert unorm[0] > unorm[1] > unorm[2] > 0
    assert track[0] < track[1] < track[2]


# ----------------------------------------------------------------------------- preconditioner
def test_matching_schur_bounds():
    # Pearson-Stoll-Wathen: with the exact M, S, the matching approximation Sh of the Schur
    # complement S = (1/tau) K M^-1 K' + (tau/beta) M has eig(Sh^-1 S) in [1/2, 1]
    cfg, M, S, beta = small_kkt(n=6, n_t=3, beta=1e-3)
    P = oracle.problem_from_config(cfg, synth.draw_weights(cfg))
    Pm, _, _, _ = oracle.kkt_prec_dense(P, M, S, cfg.n_t, cfg.tau, beta, exact=True)
    N = M.shape[0]
    nt, tau = cfg.n_t, cfg.tau
    Md, Sd = M.toarray(), S.toarray()
    I = np.eye(nt)
    C = np.eye(nt) - np.eye(nt, k=-1)
    K = np.kron(I, tau * Sd) + np.kron(C, Md)
    calM = np.kron(I, Md)
    Schur = K @ np.linalg.solve(calM, K.T) / tau + (tau / beta) * calM
    Sh = Pm[2 * nt * N:, 2 * nt * N:]
    ev = np.linalg.eigvals(np.linalg.solve(Sh, Schur)).real
    assert ev.min() >= 0.5 - 1e-8 and ev.max() <= 1.0 + 1e-8


def test_kronecker_preconditioner_spd_and_effective():
    cfg, M, S, beta = small_kkt(n=7, n_t=3, beta=1e-4)
    P = oracle.problem_from_config(cfg, synth.draw_weights(cfg))
    Pm, mbar, sbar, lams = oracle.kkt_prec_dense(P, M, S, cfg.n_t, cfg.tau, beta)
    assert np.allclose(Pm, Pm.T, rtol=0, atol=1e-14 * np.abs(Pm).max())
    np.linalg.cholesky(Pm)  # SPD
    assert mbar > 0 and sbar > 0 and all(l.min() > 0 for l in lams)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    ev = np.abs(np.linalg.eigvals(np.linalg.solve(Pm, A)).real)
    assert ev.max() / ev.min() < 50  # vs cond(A) ~ 1e10 unpreconditioned
    b, _ = rhs_tracking(M, cfg.n_t, cfg.tau)
    xs = np.linalg.solve(A, b)
    x, it, relres, _ = oracle.minres(lambda v: A @ v, b, maxit=500, rtol=1e-10,
                                     precond=lambda v: np.linalg.solve(Pm, v))
    assert relres <= 1e-10 and it < 200
    assert np.linalg.norm(x - xs) <= 1e-7 * np.linalg.norm(xs)


def test_preconditioned_minres_first_iterate():
    # x_1 minimises |b - A x|_{P^-1} over span{P^-1 b}:  x_1 = t P^-1 b,
    # t = (b' P^-1 A P^-1 b) / (A P^-1 b)' P^-1 (A P^-1 b)
    cfg, M, S, beta = small_kkt(n=6, n_t=2, beta=1e-2)
    P = oracle.problem_from_config(cfg, synth.draw_weights(cfg))
    Pm, _, _, _ = oracle.kkt_prec_dense(P, M, S, cfg.n_t, cfg.tau, beta)
    A = oracle.kkt_dense(M, S, cfg.n_t, cfg.tau, beta)
    b = np.random.default_rng(4).standard_normal(A.shape[0])
    Pinv = lambda v: np.linalg.solve(Pm, v)
    x1, it, _, _ = oracle.minres(lambda v: A @ v, b, maxit=1, rtol=0.0, precond=Pinv)
    z = Pinv(b)
    Az = A @ z
    t = (b @ Pinv(Az)) / (Az @ Pinv(Az))
    assert it == 1
    assert np.linalg.norm(x1 - t * z) <= 1e-12 * np.linalg.norm(t * z)


# -------------------------------------------------- kkt_prec_dense: the inexact branch pinned
def _prob(n, p, mass_row, A, amp_v=(0.0, 0.0, 0.0), dirichlet=False):
    """Problem on a box with distinct extents per direction (a swapped Kronecker order changes
    the operators) and explicit weights: omega = one term row, Q = v(x) A with v = 1 + amp ..."""
    knots = [synth.uniform_open_knots(n[d], p) for d in range(3)]
    v = [0.0, 1.0, 0.0, 0.0, 1.0, 0.0, 0.0, 1.0, 0.0]
    for d in range(3):
        v[3 * d] = amp_v[d]
        v[3 * d + 1] = d + 1.0
        v[3 * d + 2] = 0.4 * d
    qt = []
    for k in range(3):
        for l in range(3):
            c = float(A[k][l])
            qt.append(np.array([[c] + v]) if c != 0.0 else np.zeros((0, 10)))
    return oracle.Problem(knots=knots, p=[p] * 3, nq=p + 1, mass_terms=np.array([mass_row], dtype=float),
                          q_terms=qt, dirichlet=dirichlet)


@pytest.mark.parametrize("dirichlet", [False, True])
def test_prec_unit_weights_equal_exact(dirichlet):
    """omega = 1, Q = I (c1's weights) on a 5x6x7 box: M0 = M and S0 = S exactly, so mbar =
    sbar = 1 and the Kronecker preconditioner IS the exact matching one (a wrong Kronecker
    order, a wrong pattern or a wrong Dirichlet slice in M0 / S0 breaks the equality)."""
    one = [1.0, 0, 1, 0, 0, 1, 0, 0, 1, 0]
    P = _prob((5, 6, 7), 2, one, np.eye(3), dirichlet=dirichlet)
    M, S = oracle.assemble_csr(P)
    nt, tau, beta = 2, 0.5, 1e-2
    Pi, mbar, sbar, _ = oracle.kkt_prec_dense(P, M, S, nt, tau, beta)
    Pe, _, _, _ = oracle.kkt_prec_dense(P, M, S, nt, tau, beta, exact=True)
    assert abs(mbar - 1.0) < 1e-13 and abs(sbar - 1.0) < 1e-13
    assert np.abs(Pi - Pe).max() <= 1e-12 * np.abs(Pe).max()


def test_prec_constant_weights_scale():
    """omega = c, Q = s I: M = c M0 and S = s S0, so mbar = c and sbar = s for any eigenvector
    choice, and the preconditioner again equals the exact one."""
    c, s = 2.5, 0.75
    P = _prob((5, 6, 4), 3, [c, 0, 1, 0, 0, 1, 0, 0, 1, 0], s * np.eye(3))
    M, S = oracle.assemble_csr(P)
    Pi, mbar, sbar, _ = oracle.kkt_prec_dense(P, M, S, 2, 0.5, 1e-3)
    Pe, _, _, _ = oracle.kkt_prec_dense(P, M, S, 2, 0.5, 1e-3, exact=True)
    assert abs(mbar - c) < 1e-13 * c and abs(sbar - s) < 1e-13 * s
    assert np.abs(Pi - Pe).max() <= 1e-12 * np.abs(Pe).max()


def test_prec_mbar_is_product_of_univariate_rayleigh_quotients():
    """Separable omega = a(x) b(y) c(z): M = Mz (x) My (x) Mx and v1 = e1z (x) e1y (x) e1x, so
    mbar = prod_d (e1d' Md e1d) / (e1d' M0d e1d), with e1d the eigenvector of the smallest
    POSITIVE eigenvalue of K0d v = lam M0d v (computed here with scipy.linalg.eigh on gram_1d).  A wrong
    eigenvector (e.g. the largest) or a direction mix-up changes mbar by O(1)."""
    import scipy.linalg as sla_
    row = [1.0, 0.5, 2.0, 0.3, 0.5, 1.0, 1.1, 0.5, 3.0, 2.0]
    n, p = (6, 7, 8), 2
    P = _prob(n, p, row, np.eye(3))
    M, S = oracle.assemble_csr(P)
    _, mbar, _, lams = oracle.kkt_prec_dense(P, M, S, 1, 0.5, 1e-2)
    prod = 1.0
    for d in range(3):
        kn = synth.uniform_open_knots(n[d], p)
        amp, kk, ph = row[1 + 3 * d:4 + 3 * d]
        Md = oracle.gram_1d(kn, p, p + 1, amp, kk, ph, 0, 0)
        M0 = oracle.gram_1d(kn, p, p + 1, 0.0, 1.0, 0.0, 0, 0)
        K0 = oracle.gram_1d(kn, p, p + 1, 0.0, 1.0, 0.0, 1, 1)
        lam, V = sla_.eigh(K0, M0)  # ascending; lam[0] = 0 (constants) without Dirichlet
        e = V[:, int(np.argmax(lam > 1e-8 * lam.max()))]  # smoothest mode with lam > 0
        prod *= (e @ Md @ e) / (e @ M0 @ e)
        assert np.allclose(np.sort(lams[d]), lam, rtol=1e-12, atol=1e-12)
    assert abs(mbar - prod) <= 1e-12 * prod
