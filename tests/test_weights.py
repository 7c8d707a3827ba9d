"""NEXT-2 (low-rank weights from samples): oracle pins and the host path.

The oracle (oracle.greville / tt_svd / weight_lowrank) is pinned against the linear
reproduction of the Greville abscissae, the TT-SVD error bound, exact separability (rank 1 / 2)
and exact interpolation of polynomial weights.  The library's iga_weight_lowrank (host code,
runs without a GPU) is compared with the oracle on the weight it reconstructs at the quadrature
nodes (sign / rotation ambiguities of the SVD factors cancel there).  The GPU test applies an op
assembled from annulus weights: 1'M1 equals the physical volume.
"""
import numpy as np
import pytest

import oracle
import synth


def grid_eval(tabs):
    """sum_r tab_x[r](x) tab_y[r](y) tab_z[r](z) on the node grid, [z, y, x]."""
    return np.einsum("ri,rj,rk->kji", tabs[0], tabs[1], tabs[2])


@pytest.mark.parametrize("p,n", [(1, 5), (2, 7), (3, 12), (5, 9)])
def test_greville_reproduces_linears(p, n):
    # sum_i xi*_i beta_i(t) = t for every t (Marsden's identity for linears)
    kn = synth.uniform_open_knots(n, p)
    g = oracle.greville(kn, p)
    for t in np.linspace(0.0, 1.0, 17):
        v, _ = oracle.basis_all(kn, p, float(t))
        assert abs(v[:n] @ g - t) <= 1e-14


def test_tt_svd_error_bound_and_exact_ranks():
    rng = np.random.default_rng(3)
    g = np.linspace(0, 1, 9)
    S1 = np.einsum("k,j,i->kji", 1 + g ** 2, np.cos(g), np.exp(g))
    G1, G2, G3 = oracle.tt_svd(S1, 1e-12)
    assert G1.shape[1] == 1 and G3.shape[0] == 1
    S2 = S1 + np.einsum("k,j,i->kji", np.sin(g), g, g ** 3)
    G1, G2, G3 = oracle.tt_svd(S2, 1e-12)
    assert G1.shape[1] == 2 and G3.shape[0] == 2
    for eps in (1e-1, 1e-3):
        S = rng.standard_normal((8, 9, 10)) + 3 * S2[:8, :9, :9].mean()
        G1, G2, G3 = oracle.tt_svd(S, eps)
        R = np.einsum("ka,ajb,bi->kji", G1, G2, G3)
        assert np.linalg.norm(S - R) <= eps * np.linalg.norm(S) * (1 + 1e-12)


def test_polynomial_weight_interpolated_exactly():
    # omega polynomial of degree <= p~ per direction lies in S~: the low-rank weight is exact
    pt, nt = 3, 7
    tk = [synth.uniform_open_knots(nt, pt)] * 3
    gr = [oracle.greville(tk[d], pt) for d in range(3)]
    f = lambda x, y, z: (1 + x + x ** 3) * (2 - y ** 2) + z * x ** 2
    S = f(gr[0][None, None, :], gr[1][None, :, None], gr[2][:, None, None])
    kn = synth.uniform_open_knots(10, 3)
    nodes = [oracle.quad_nodes(kn, 3, 4)] * 3
    tabs, ranks = oracle.weight_lowrank(nodes, tk, [pt] * 3, S, 1e-13)
    assert ranks == (2, 2)
    ref = f(nodes[0][None, None, :], nodes[1][None, :, None], nodes[2][:, None, None])
    assert np.abs(grid_eval(tabs) - ref).max() <= 1e-12 * np.abs(ref).max()


def annulus(pt, nt, r0=1.0, r1=2.0, h=0.5):
    """Quarter annulus extruded in z, G(s,t,u) = (r(s) cos(pi t/2), r(s) sin(pi t/2), h u),
    r(s) = r0 + (r1-r0) s: omega = |det grad G| = (r1-r0)(pi/2) r(s) h (rank 1, degree 1),
    Q = omega (grad G)^-1 (grad G)^-T = diag(omega/(r1-r0)^2, omega/(r pi/2)^2, omega/h^2)."""
    tk = [synth.uniform_open_knots(nt, pt)] * 3
    gr = [oracle.greville(tk[d], pt) for d in range(3)]
    s = gr[0][None, None, :]
    r = r0 + (r1 - r0) * s
    om = (r1 - r0) * (np.pi / 2) * r * h * np.ones((nt, nt, nt))
    q11 = om / (r1 - r0) ** 2
    q22 = om / (r * np.pi / 2) ** 2
    q33 = om / h ** 2
    vol = (np.pi / 4) * (r1 ** 2 - r0 ** 2) * h
    return tk, om, (q11, q22, q33), vol


def test_annulus_weights_rank_one_and_volume():
    tk, om, qs, vol = annulus(3, 6)
    kn = synth.uniform_open_knots(8, 3)
    nodes = [oracle.quad_nodes(kn, 3, 4)] * 3
    tabs, ranks = oracle.weight_lowrank(nodes, tk, [3] * 3, om, 1e-12)
    assert ranks == (1, 1)
    for q in qs:
        _, rq = oracle.weight_lowrank(nodes, tk, [3] * 3, q, 1e-12)
        assert rq == (1, 1)
    # integral of the interpolated omega over [0,1]^3 = physical volume (omega is exact here):
    # integrate each factor with the nodes' Gauss rule, sum_q W_q f(x_q)
    _, gw = oracle.gauss_legendre(4)
    ints = []
    for d in range(3):
        # Gauss weights on each span of kn (uniform, 5 spans) in the same order as quad_nodes
        spans = np.unique(kn)
        W = np.concatenate([0.5 * (b - a) * gw for a, b in zip(spans[:-1], spans[1:])])
        ints.append(tabs[d] @ W)
    total = sum(ints[0][r] * ints[1][r] * ints[2][r] for r in range(len(ints[0])))
    assert abs(total - vol) <= 1e-12 * vol


# ----------------------------------------------------------------------------- the library (host)
@pytest.fixture(scope="module")
def igalr():
    import paper_1811_06797_b200 as m
    return m


@pytest.mark.parametrize("p,n", [(2, 7), (3, 12), (4, 9)])
def test_library_greville_matches_oracle(igalr, p, n):
    kn = synth.uniform_open_knots(n, p)
    assert np.array_equal(igalr.greville(kn, p), oracle.greville(kn, p)) or \
        np.abs(igalr.greville(kn, p) - oracle.greville(kn, p)).max() <= 1e-15


@pytest.mark.parametrize("case", ["poly", "annulus_q22", "random_eps"])
def test_library_weight_lowrank_matches_oracle(igalr, case):
    pt, nt = 3, 8
    tk = [synth.uniform_open_knots(nt, pt)] * 3
    gr = [oracle.greville(tk[d], pt) for d in range(3)]
    eps = 1e-12
    if case == "poly":
        f = lambda x, y, z: (1 + x + x ** 3) * (2 - y ** 2) + z * x ** 2 + 0.5 * y * z
        S = f(gr[0][None, None, :], gr[1][None, :, None], gr[2][:, None, None])
    elif case == "annulus_q22":
        S = annulus(pt, nt)[2][1]
    else:
        rng = np.random.default_rng(7)
        S = 2.0 + rng.standard_normal((nt, nt, nt))
        eps = 0.05
    kn = synth.uniform_open_knots(11, 3)
    sep, ranks, err = igalr.weight_lowrank([kn] * 3, [3] * 3, tk, [pt] * 3, S, eps=eps, max_terms=512)
    nodes = [oracle.quad_nodes(kn, 3, 4)] * 3
    tabs, oranks = oracle.weight_lowrank(nodes, tk, [pt] * 3, S, eps)
    assert ranks == oranks
    ref = grid_eval(tabs)
    got = grid_eval(sep.tabs) * 1.0
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    assert err <= eps * (1 + 1e-9)


def test_library_weight_lowrank_errors(igalr):
    tk = [synth.uniform_open_knots(6, 3)] * 3
    kn = synth.uniform_open_knots(8, 3)
    with pytest.raises(ValueError):
        igalr.weight_lowrank([kn] * 3, [3] * 3, tk, [3] * 3, np.zeros((6, 6, 5)))
    S = np.ones((6, 6, 6))
    S[0, 0, 0] = np.nan
    with pytest.raises(igalr.IgaError):
        igalr.weight_lowrank([kn] * 3, [3] * 3, tk, [3] * 3, S)
    with pytest.raises(igalr.IgaError):
        igalr.weight_lowrank([kn] * 3, [3] * 3, tk, [3] * 3, np.ones((6, 6, 6)), eps=-1.0)


@pytest.mark.gpu
def test_gpu_op_from_annulus_weights(igalr):
    # an op assembled from the library's low-rank annulus weights: 1'M1 = volume, S 1 = 0
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pt, nt = 3, 10
    tk, om, qs, vol = annulus(pt, nt)
    n, p = 24, 3
    kn = synth.uniform_open_knots(n, p)
    omega, _, _ = igalr.weight_lowrank([kn] * 3, [p] * 3, tk, [pt] * 3, om, eps=1e-12)
    q = [None] * 9
    for i, qq in enumerate(qs):
        q[i * 3 + i], _, _ = igalr.weight_lowrank([kn] * 3, [p] * 3, tk, [pt] * 3, qq, eps=1e-12)
    op = igalr.LowRankOperator([kn] * 3, [p] * 3, omega, q)
    one = torch.ones((1, n, n, n), dtype=torch.float64, device="cuda")
    ym, ys = torch.empty_like(one), torch.empty_like(one)
    op.apply(one, ym, ys)
    assert abs(float(ym.sum()) - vol) <= 1e-12 * vol
    assert float(ys.abs().max()) <= 1e-12 * float(ym.abs().max()) * n
    # ... and S x is not trivially zero for a random x
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((1, n, n, n))).cuda()
    op.apply(x, ym, ys)
    assert float(ys.norm()) > 1e-2 * float(x.norm())


@pytest.mark.gpu
def test_gpu_op_from_library_weights_vs_oracle_weights(igalr):
    """NEXT-2 end to end: the op assembled from the LIBRARY's low-rank annulus weights
    (iga_weight_lowrank: TT-SVD + collocation solves) applied on the GPU, against
    the oracle's element-loop forms with the ORACLE's own low-rank weights (oracle.weight_lowrank)
    given at every 3D quadrature point (Problem.weights3d): rel l2 <= 1e-11 for M x and S x."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pt, nt = 3, 10
    tk, om, qs, vol = annulus(pt, nt)
    n, p = 20, 3
    kn = synth.uniform_open_knots(n, p)
    knots = [kn] * 3
    omega, _, _ = igalr.weight_lowrank(knots, [p] * 3, tk, [pt] * 3, om, eps=1e-12)
    q = [None] * 9
    for i, qq in enumerate(qs):
        q[i * 3 + i], _, _ = igalr.weight_lowrank(knots, [p] * 3, tk, [pt] * 3, qq, eps=1e-12)
    op = igalr.LowRankOperator(knots, [p] * 3, omega, q)
    nodes = [oracle.quad_nodes(kn, p, p + 1)] * 3
    w3 = np.zeros((10, len(nodes[2]), len(nodes[1]), len(nodes[0])))
    w3[0] = grid_eval(oracle.weight_lowrank(nodes, tk, [pt] * 3, om, 1e-12)[0])
    for i, qq in enumerate(qs):
        w3[1 + i * 3 + i] = grid_eval(oracle.weight_lowrank(nodes, tk, [pt] * 3, qq, 1e-12)[0])
    P = oracle.Problem(knots=knots, p=[p] * 3, nq=p + 1, mass_terms=None, q_terms=None, weights3d=w3)
    x = np.random.default_rng(11).standard_normal((1, n, n, n))
    rm, rs = oracle.apply_matfree(P, x)
    xd = torch.from_numpy(x).cuda()
    ym, ys = torch.empty_like(xd), torch.empty_like(xd)
    op.apply(xd, ym, ys)
    for got, ref in ((ym, rm), (ys, rs)):
        g = got.cpu().numpy()
        assert np.linalg.norm(g - ref) <= 1e-11 * np.linalg.norm(ref)
