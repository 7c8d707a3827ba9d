"""GPU MINRES (iga_kkt_minres, NEXT-1) against the oracle MINRES on the same KKT systems.

MINRES iterates are a deterministic function of (A, b); the CUDA path and oracle.minres run the
same recurrence (Elman-Silvester-Wathen Algorithm 2.4) with matvecs that agree to ~1e-15, so
their k-th iterates agree to rounding amplified by the Krylov process: checked element-wise
(relative l2) for k <= 20.  Convergence is checked against a dense LU solve of Eq. (KKTSystem).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1811_06797_b200 as igalr
    from paper_1811_06797_b200 import workloads
    return torch, igalr, workloads


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def setup(env, n, n_t, beta):
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS["c4"], n, n_t=n_t)
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    m = n - 2
    return cfg, op, M, S, m


@pytest.mark.parametrize("k", [1, 3, 10, 20])
@pytest.mark.parametrize("n,n_t", [(8, 3), (11, 2)])
def test_minres_iterates_vs_oracle(env, n, n_t, k):
    torch = env[0]
    cfg, op, M, S, m = setup(env, n, n_t, 1e-2)
    beta = 1e-2
    b = np.random.default_rng(n * 7 + n_t).standard_normal((3, n_t, m, m, m))
    xo, ito, rro, r0o = oracle.minres(lambda v: oracle.kkt_apply_csr(M, S, v.reshape(b.shape), cfg.tau, beta).ravel(),
                                      b.ravel(), maxit=k, rtol=0.0)
    bd = torch.from_numpy(b).cuda()
    xd = torch.empty_like(bd)
    info = op.kkt_minres(bd, xd, n_t, cfg.tau, beta, rtol=0.0, maxit=k)
    assert info.iters == ito == k
    assert abs(info.res0 - r0o) <= 1e-13 * r0o
    assert abs(info.relres - rro) <= 1e-8 * max(rro, 1e-300) + 1e-14
    assert rel(xd.cpu().numpy(), xo) <= 1e-10


def test_minres_initial_guess_and_convergence(env):
    torch = env[0]
    n, n_t, beta = 5, 1, 1.0
    cfg, op, M, S, m = setup(env, n, n_t, beta)
    A = oracle.kkt_dense(M, S, n_t, cfg.tau, beta)
    b = np.random.default_rng(9).standard_normal(A.shape[0])
    xs = np.linalg.solve(A, b)
    bd = torch.from_numpy(b.reshape(3, n_t, m, m, m)).cuda()
    xd = torch.zeros_like(bd)
    info = op.kkt_minres(bd, xd, n_t, cfg.tau, beta, rtol=1e-10, maxit=20000)
    assert info.converged == 1 and info.relres <= 1e-10
    assert rel(xd.cpu().numpy(), xs) <= np.linalg.cond(A) * 1e-10
    # restart from the solution (IGA_MINRES_X0, maxit 0): r_0 = b - A x is the true residual
    info2 = op.kkt_minres(bd, xd, n_t, cfg.tau, beta, rtol=0.0, maxit=0, x0=True)
    true = np.linalg.norm(b - A @ xd.cpu().numpy().ravel())
    assert info2.iters == 0
    assert abs(info2.res0 - true) <= 1e-6 * np.linalg.norm(b)
    assert info2.res0 <= 1e-6 * np.linalg.norm(b)


def test_minres_c4_full_size_residual(env):
    # BASELINE c4 size: the recurrence residual |eta| equals the true residual |b - A x_k|
    torch = env[0]
    cfg = synth.CONFIGS["c4"]
    torch_, igalr, workloads = env
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    m = cfg.n - 2
    g = torch.Generator(device="cuda").manual_seed(4)
    bd = torch.randn((3, cfg.n_t, m, m, m), dtype=torch.float64, device="cuda", generator=g)
    xd = torch.empty_like(bd)
    info = op.kkt_minres(bd, xd, cfg.n_t, cfg.tau, cfg.beta, rtol=0.0, maxit=8)
    ax = torch.empty_like(bd)
    op.kkt_apply(xd, ax, cfg.n_t, cfg.tau, cfg.beta)
    true = float(torch.linalg.vector_norm(bd - ax))
    assert info.iters == 8
    assert abs(true - info.relres * info.res0) <= 1e-6 * info.res0
    assert info.relres < 1.0


def test_minres_errors(env):
    torch, igalr, workloads = env
    cfg, op, M, S, m = setup(env, 6, 2, 1e-2)
    bd = torch.zeros((3, 2, m, m, m), dtype=torch.float64, device="cuda")
    with pytest.raises(igalr.IgaError):
        op.kkt_minres(bd, bd, 2, cfg.tau, 1e-2)
    with pytest.raises(igalr.IgaError):
        op.kkt_minres(bd, torch.empty_like(bd), 2, cfg.tau, 1e-2, maxit=-1)
    with pytest.raises(igalr.IgaError):
        op.kkt_minres(bd, torch.empty_like(bd), 2, -1.0, 1e-2)
    # zero right-hand side: x = 0, no iterations
    x = torch.full_like(bd, 3.0)
    info = op.kkt_minres(bd, x, 2, cfg.tau, 1e-2)
    assert info.iters == 0 and float(x.abs().max()) == 0.0


# ----------------------------------------------------------------------------- preconditioner
def oracle_prec(cfg, M, S, n_t, beta):
    P = oracle.problem_from_config(cfg, synth.draw_weights(cfg))
    return oracle.kkt_prec_dense(P, M, S, n_t, cfg.tau, beta)


@pytest.mark.parametrize("n,n_t,beta", [(6, 2, 1e-2), (9, 3, 1e-4), (12, 1, 1.0)])
def test_prec_apply_vs_oracle(env, n, n_t, beta):
    torch = env[0]
    cfg, op, M, S, m = setup(env, n, n_t, beta)
    Pm, mbar, sbar, lams = oracle_prec(cfg, M, S, n_t, beta)
    prec = op.kkt_preconditioner(n_t, cfg.tau, beta)
    gm, gs, glam = prec.info()
    assert abs(gm - mbar) <= 1e-12 * mbar and abs(gs - sbar) <= 1e-12 * sbar
    for d in range(3):
        assert np.allclose(np.sort(glam[d]), np.sort(lams[d]), rtol=1e-11, atol=0)
    r = np.random.default_rng(n + n_t).standard_normal((3, n_t, m, m, m))
    ref = np.linalg.solve(Pm, r.ravel())
    out = torch.empty((3, n_t, m, m, m), dtype=torch.float64, device="cuda")
    prec.apply(torch.from_numpy(r).cuda(), out)
    assert rel(out.cpu().numpy(), ref) <= 1e-10


@pytest.mark.parametrize("k", [1, 5, 15])
def test_pminres_iterates_vs_oracle(env, k):
    torch = env[0]
    n, n_t, beta = 8, 3, 1e-4
    cfg, op, M, S, m = setup(env, n, n_t, beta)
    Pm, _, _, _ = oracle_prec(cfg, M, S, n_t, beta)
    A = oracle.kkt_dense(M, S, n_t, cfg.tau, beta)
    b = np.random.default_rng(11).standard_normal(A.shape[0])
    xo, ito, rro, r0o = oracle.minres(lambda v: A @ v, b, maxit=k, rtol=0.0, precond=lambda v: np.linalg.solve(Pm, v))
    prec = op.kkt_preconditioner(n_t, cfg.tau, beta)
    bd = torch.from_numpy(b.reshape(3, n_t, m, m, m)).cuda()
    xd = torch.empty_like(bd)
    info = op.kkt_minres(bd, xd, n_t, cfg.tau, beta, rtol=0.0, maxit=k, prec=prec)
    assert info.iters == ito == k
    assert abs(info.res0 - r0o) <= 1e-10 * r0o
    assert rel(xd.cpu().numpy(), xo) <= 1e-8


def test_pminres_converges_to_dense_lu(env):
    torch = env[0]
    n, n_t, beta = 9, 3, 1e-4
    cfg, op, M, S, m = setup(env, n, n_t, beta)
    A = oracle.kkt_dense(M, S, n_t, cfg.tau, beta)
    yhat = np.random.default_rng(5).standard_normal((n_t, M.shape[0]))
    b = np.concatenate([np.stack([cfg.tau * oracle.spmv(M, yhat[k]) for k in range(n_t)]).ravel(),
                        np.zeros(2 * n_t * M.shape[0])])
    xs = np.linalg.solve(A, b)
    prec = op.kkt_preconditioner(n_t, cfg.tau, beta)
    bd = torch.from_numpy(b.reshape(3, n_t, m, m, m)).cuda()
    xd = torch.zeros_like(bd)
    info = op.kkt_minres(bd, xd, n_t, cfg.tau, beta, rtol=1e-11, maxit=1000, prec=prec)
    assert info.converged == 1 and info.iters < 300
    assert rel(xd.cpu().numpy(), xs) <= 1e-8
    X = xd.cpu().numpy()
    assert rel(X[1], X[2] / beta) <= 1e-7  # u = lambda / beta at the optimum


def test_pminres_c4_full_size(env):
    # BASELINE c4 (46^3 interior x 64 steps, beta 1e-4): converges; true residual small
    torch = env[0]
    torch_, igalr, workloads = env
    cfg = synth.CONFIGS["c4"]
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    m = cfg.n - 2
    g = torch.Generator(device="cuda").manual_seed(7)
    yhat = torch.randn((1, cfg.n_t, m, m, m), dtype=torch.float64, device="cuda", generator=g)
    b = torch.zeros((3, cfg.n_t, m, m, m), dtype=torch.float64, device="cuda")
    ym = torch.empty_like(yhat[0])
    op.apply(yhat[0], ym, None)  # M yhat_k (mass only) for every step
    b[0] = cfg.tau * ym
    prec = op.kkt_preconditioner(cfg.n_t, cfg.tau, cfg.beta)
    x = torch.empty_like(b)
    # (rtol is relative in the P^{-1} norm; 1e-10 there gives ~1e-6 in the 2-norm here)
    info = op.kkt_minres(b, x, cfg.n_t, cfg.tau, cfg.beta, rtol=1e-10, maxit=2000, prec=prec)
    assert info.converged == 1 and info.iters < 1000
    ax = torch.empty_like(b)
    op.kkt_apply(x, ax, cfg.n_t, cfg.tau, cfg.beta)
    assert float(torch.linalg.vector_norm(b - ax) / torch.linalg.vector_norm(b)) <= 1e-5
    assert float(torch.linalg.vector_norm(x[1] - x[2] / cfg.beta) / torch.linalg.vector_norm(x[1])) <= 1e-4


def test_prec_errors(env):
    torch, igalr, workloads = env
    cfg, op, M, S, m = setup(env, 6, 2, 1e-2)
    with pytest.raises(igalr.IgaError):
        op.kkt_preconditioner(0, cfg.tau, 1e-2)
    prec = op.kkt_preconditioner(2, cfg.tau, 1e-2)
    bd = torch.ones((3, 2, m, m, m), dtype=torch.float64, device="cuda")
    with pytest.raises(igalr.IgaError):  # built for another beta
        op.kkt_minres(bd, torch.empty_like(bd), 2, cfg.tau, 1e-3, prec=prec)
    with pytest.raises(igalr.IgaError):
        prec.apply(bd, bd)
