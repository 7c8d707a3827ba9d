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
