"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerance (BASELINE.json north_star): relative l2 error <= 1e-11 per output array, fp64.
Full-vector parity at sizes the oracle finishes in seconds (several tiles + ragged tails);
BASELINE full sizes (c3, c4, c5) in the launch configuration bench.py times, compared on
sampled rows the oracle computes one by one.  Both kernel paths (fused, unfused) are covered.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-11


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


def gpu_apply(env, op, x, path="auto", mass=True, stiff=True):
    torch = env[0]
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ym = torch.empty_like(xd) if mass else None
    ys = torch.empty_like(xd) if stiff else None
    op.apply(xd, ym, ys, path=path)
    torch.cuda.synchronize()
    return (ym.cpu().numpy() if mass else None), (ys.cpu().numpy() if stiff else None)


def sample_rows(dims, count, seed, p):
    mx, my, mz = dims
    N = mx * my * mz
    rng = np.random.default_rng(seed)
    rows = list(rng.integers(0, N, count))
    # boundary / corner rows and rows next to 32-wide tile edges
    for (ix, iy, iz) in [(0, 0, 0), (mx - 1, my - 1, mz - 1), (p, 0, mz // 2), (mx // 2, my - 1, 0),
                         (31 % mx, 32 % my, 1), (32 % mx, 31 % my, mz - 2), (mx - 1, 0, p)]:
        rows.append((iz * my + iy) * mx + ix)
    return np.unique(np.array(rows, dtype=np.int64))


PATHS = ["unfused", "fused_v1", "fused", "auto"]


# ----------------------------------------------------------------------------- factors
def test_c1_factors_closed_form(env):
    """P1 on the GPU factors: w == 1, uniform knots, interior rows = cardinal B-spline values."""
    import json, os
    from fractions import Fraction
    torch, igalr, workloads = env
    cfg = synth.CONFIGS["c1"]
    w = synth.draw_weights(cfg)
    for p in (1, 2, 3, 4):
        c = synth.Config(1, "p1", n=4 * p + 8, p=p, R=1, batch=1, constant_weight=True)
        op = workloads.build_operator(c, synth.draw_weights(c))
        g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "p1_uniform_gram.json")))
        h = 1.0 / (c.n - p)
        seen = set()
        for fid in range(op.info.n_factors[0]):
            band, pat, _ = op.export_factor(0, fid)
            seen.add(pat)
            if pat == 0:
                ref = [float(Fraction(s)) * h for s in g["mass_over_h"][str(p)]]
            elif pat == 3:
                ref = [float(Fraction(s)) / h for s in g["stiff_times_h"][str(p)]]
            else:
                continue
            for i in range(2 * p, c.n - 2 * p):
                for k in range(p + 1):
                    assert abs(band[i, p + k] - ref[k]) < 1e-13 * max(1, abs(ref[k]))
        assert {0, 3} <= seen


def test_factors_vs_oracle_gram(env):
    """Every exported factor equals one oracle univariate Gram (Eq. (massMatrix1D) and
    K^{(d)}_{k,l}) with the same derivative pattern, c2 weights on a small mesh."""
    torch, igalr, workloads = env
    cfg = synth.CONFIGS["c2"]
    w = synth.draw_weights(cfg)
    n = 13
    op = workloads.build_operator(cfg, w, n=n)
    kn = synth.uniform_open_knots(n, cfg.p)
    p = cfg.p
    for d in range(3):
        cands = [tuple(w.mass[r, 1 + 3 * d:4 + 3 * d]) for r in range(cfg.R)] + [tuple(w.v[r, d]) for r in range(cfg.R)]
        for fid in range(op.info.n_factors[d]):
            band, pat, _ = op.export_factor(d, fid)
            a, b = pat // 2, pat % 2
            dense = np.zeros((n, n))
            for i in range(n):
                for k in range(2 * p + 1):
                    j = i - p + k
                    if 0 <= j < n:
                        dense[i, j] = band[i, k]
                    else:
                        assert band[i, k] == 0.0
            errs = [np.abs(dense - oracle.gram_1d(kn, p, p + 1, *c, a, b)).max() for c in cands]
            assert min(errs) < 1e-14 * max(1.0, np.abs(dense).max())


# ----------------------------------------------------------------------------- apply parity
@pytest.mark.parametrize("path", PATHS)
def test_c1_full_vs_csr(env, path):
    torch, igalr, workloads = env
    cfg = synth.CONFIGS["c1"]
    knots, w, x = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    yM, yS = gpu_apply(env, op, x, path)
    for b in range(cfg.batch):
        assert rel(yM[b], oracle.spmv(M, x[b])) <= TOL
        assert rel(yS[b], oracle.spmv(S, x[b])) <= TOL


@pytest.mark.parametrize("path", PATHS)
def test_c2_full_vs_matfree(env, path):
    torch, igalr, workloads = env
    cfg = synth.CONFIGS["c2"]
    knots, w, x = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    rm, rs = oracle.apply_matfree(P, x)
    yM, yS = gpu_apply(env, op, x, path)
    assert rel(yM, rm) <= TOL and rel(yS, rs) <= TOL


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cfgname,n,batch", [("c2", 37, 3), ("c3", 45, 2), ("c5", 36, 1), ("c2", 70, 1)])
def test_multitile_ragged_full(env, path, cfgname, n, batch):
    """Full-vector parity at sizes spanning several 32-wide tiles with ragged tails."""
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS[cfgname], n, batch=batch)
    w = synth.draw_weights(cfg)
    x = np.random.default_rng(n).standard_normal((batch, n, n, n))
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    rm, rs = oracle.apply_matfree(P, x)
    yM, yS = gpu_apply(env, op, x, path)
    for b in range(batch):
        assert rel(yM[b], rm[b]) <= TOL and rel(yS[b], rs[b]) <= TOL


@pytest.mark.parametrize("cfgname", ["c3", "c5"])
def test_full_size_sampled_rows(env, cfgname):
    """BASELINE full sizes in the bench launch configuration (auto path, full batch):
    sampled outputs vs the oracle's row-restricted bilinear form."""
    torch, igalr, workloads = env
    cfg = synth.CONFIGS[cfgname]
    knots, w, x = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    yM, yS = gpu_apply(env, op, x, "auto")
    for b in range(cfg.batch):
        rows = sample_rows(P.dims, 60 if cfg.batch > 1 else 300, 100 + b, cfg.p)
        rm, rs = oracle.apply_rows(P, x[b], rows)
        gm, gs = yM[b].ravel()[rows], yS[b].ravel()[rows]
        # relative to the full output norm of this vector (per-array metric G12), sampled
        scale_m = np.linalg.norm(yM[b]) / np.sqrt(yM[b].size)
        scale_s = np.linalg.norm(yS[b]) / np.sqrt(yS[b].size)
        assert np.abs(gm - rm).max() <= TOL * scale_m
        assert np.abs(gs - rs).max() <= TOL * scale_s
        assert rel(gm, rm) <= TOL and rel(gs, rs) <= TOL


@pytest.mark.parametrize("minlen", [1, 2, 3, 5])
def test_fixup_table_many_contributors(env, minlen):
    """Persistent-CTA ranges of `minlen` planes (the test-only knob of iga_lr_testing.h) give
    output planes with up to 2P+1 contributors in the table-driven fixup; every setting matches
    the oracle (the summation order, not the result, depends on the split)."""
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS["c3"], 21, batch=2)
    knots, w, x = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    op._test_knobs(minlen=minlen)
    yM, yS = gpu_apply(env, op, x, "auto")
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    for b in range(cfg.batch):
        assert rel(yM[b].ravel(), oracle.spmv(M, x[b])) <= TOL
        assert rel(yS[b].ravel(), oracle.spmv(S, x[b])) <= TOL


@pytest.mark.parametrize("n,batch", [(104, 1), (101, 2)])
def test_p4_26row_tiles_sampled_rows(env, n, batch):
    """p = 4 meshes whose y extent tiles best in 26-row tiles (LW 13, the 9-double TMEM ring):
    n = 104 (4 full tiles) and n = 101 (ragged last tile), sampled rows vs the oracle."""
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS["c5"], n, batch=batch)
    knots, w, x = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    yM, yS = gpu_apply(env, op, x, "auto")
    for b in range(batch):
        rows = sample_rows(P.dims, 200, 300 + b, cfg.p)
        rm, rs = oracle.apply_rows(P, x[b], rows)
        assert rel(yM[b].ravel()[rows], rm) <= TOL and rel(yS[b].ravel()[rows], rs) <= TOL


@pytest.mark.parametrize("cfgname", ["c2", "c3"])
def test_invariants_on_gpu(env, cfgname):
    """P4 (1'M1 = int omega) and P5 (S 1 = 0) on the GPU output, nq = 10 so the rule is exact."""
    import math
    torch, igalr, workloads = env
    cfg = synth.CONFIGS[cfgname]
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w, n=20, nq=10)
    one = np.ones((1, 20, 20, 20))
    yM, yS = gpu_apply(env, op, one)
    tot = 0.0
    for T in w.mass:
        f = T[0]
        for d in range(3):
            amp, k, ph = T[1 + 3 * d:4 + 3 * d]
            f *= 1 + amp * (math.cos(ph) - math.cos(k * math.pi + ph)) / (k * math.pi)
        tot += f
    assert abs(yM.sum() - tot) < 1e-13 * tot
    assert np.abs(yS).max() < 1e-13 * np.abs(w.A).max() * 10


def test_determinism_bitwise(env):
    torch, igalr, workloads = env
    cfg = synth.CONFIGS["c2"]
    knots, w, x = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    a = gpu_apply(env, op, x)
    b = gpu_apply(env, op, x)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("cfgname,n,batch", [("c2", 40, 1), ("c3", 30, 2), ("c5", 24, 1)])
def test_small_grid_concurrent_parts_bitwise(env, cfgname, n, batch):
    """Small meshes run one CTA per (tile, plane) unit (up to 2P+1 contributors per partial plane,
    summed by the table-driven fixup) and the mass part on a side stream beside the stiffness part.
    The combined call must equal the two single-part calls bit for bit (same kernels, same
    summation order), and stay within tolerance of the oracle."""
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS[cfgname], n, batch=batch)
    knots, w, x = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    xd = torch.from_numpy(x).cuda()
    ym, ys = torch.empty_like(xd), torch.empty_like(xd)
    op.apply(xd, ym, ys)
    ym1, ys1 = torch.empty_like(xd), torch.empty_like(xd)
    op.apply(xd, ym1, None)
    op.apply(xd, None, ys1)
    torch.cuda.synchronize()
    assert torch.equal(ym, ym1) and torch.equal(ys, ys1)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    for b in range(batch):
        for got, A in ((ym[b], M), (ys[b], S)):
            ref = oracle.spmv(A, x[b])
            assert rel(got.cpu().numpy().ravel(), ref) <= TOL


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("p,n,nq,dirichlet", [(1, 2, 0, False), (2, 3, 0, False), (3, 4, 0, False),
                                              (2, 3, 0, True), (1, 9, 0, False), (5, 12, 0, False),
                                              (3, 10, 6, False), (4, 9, 2, True), (6, 14, 0, False)])
def test_edge_shapes(env, path, p, n, nq, dirichlet):
    torch, igalr, workloads = env
    cfg = synth.Config(7, "edge", n=n, p=p, R=2, batch=2, dirichlet=dirichlet)
    w = synth.draw_weights(cfg, np.random.default_rng(p * 100 + n))
    op = workloads.build_operator(cfg, w, nq=nq)
    P = oracle.problem_from_config(cfg, w, nq=(nq or p + 1))
    m = n - 2 if dirichlet else n
    x = np.random.default_rng(1).standard_normal((2, m, m, m))
    M, S = oracle.assemble_csr(P)
    if path == "fused_v1" and not op.info_dict()["fused_ok"]:
        pytest.skip("first-generation fused kernel supports p <= 5 only")
    if path == "fused" and not (op.info_dict()["fused2_ok"] or op.info_dict()["fused_ok"]):
        pytest.skip("no fused kernel for this degree")
    yM, yS = gpu_apply(env, op, x, path)
    for b in range(2):
        assert rel(yM[b], oracle.spmv(M, x[b])) <= TOL
        assert rel(yS[b], oracle.spmv(S, x[b])) <= TOL


@pytest.mark.parametrize("path", PATHS)
def test_nonuniform_repeated_knots(env, path):
    torch, igalr, workloads = env
    p = 3
    kn = np.array([0, 0, 0, 0, 0.1, 0.25, 0.25, 0.4, 0.55, 0.7, 0.9, 1, 1, 1, 1.0])
    n = len(kn) - p - 1
    cfg = synth.Config(8, "nonuni", n=n, p=p, R=2, batch=1)
    w = synth.draw_weights(cfg, np.random.default_rng(3))
    op = workloads.build_operator(cfg, w, knots=[kn] * 3)
    P = oracle.Problem(knots=[kn] * 3, p=[p] * 3, nq=p + 1, mass_terms=w.mass, q_terms=w.q_block_terms())
    M, S = oracle.assemble_csr(P)
    x = np.random.default_rng(2).standard_normal((1, n, n, n))
    yM, yS = gpu_apply(env, op, x, path)
    assert rel(yM[0], oracle.spmv(M, x[0])) <= TOL
    assert rel(yS[0], oracle.spmv(S, x[0])) <= TOL


@pytest.mark.parametrize("path", PATHS)
def test_mass_only_stiff_only_and_scaling(env, path):
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS["c2"], 12, batch=2)
    w = synth.draw_weights(cfg)
    x = np.random.default_rng(4).standard_normal((2, 12, 12, 12))
    P = oracle.problem_from_config(cfg, w)
    rm, rs = oracle.apply_matfree(P, x)
    opm = workloads.build_operator(cfg, w, stiff=False)
    ops = workloads.build_operator(cfg, w, mass=False)
    ym, _ = gpu_apply(env, opm, x, path, stiff=False)
    _, ys = gpu_apply(env, ops, x, path, mass=False)
    assert rel(ym, rm) <= TOL and rel(ys, rs) <= TOL
    # summed single output alpha M x + gamma S x, and two-input apply2
    op = workloads.build_operator(cfg, w)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    op.apply(xd, out, out, alpha=0.5, gamma=-2.0, path=path)
    assert rel(out.cpu().numpy(), 0.5 * rm - 2.0 * rs) <= TOL
    x2 = torch.from_numpy(np.ascontiguousarray(x[::-1])).cuda()
    rs2 = rs[::-1]
    op.apply2(xd, x2, out, alpha=1.5, gamma=3.0, path=path)
    assert rel(out.cpu().numpy(), 1.5 * rm + 3.0 * rs2) <= TOL
    with pytest.raises(igalr.IgaError) as ei:
        opm.apply(xd, None, out)
    assert ei.value.status == igalr.IGA_ESTATE


def test_error_codes(env):
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS["c2"], 8, batch=1)
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    x = torch.zeros((1, 8, 8, 8), dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    with pytest.raises(igalr.IgaError) as ei:
        op.apply(x, y, None, batch=0)
    assert ei.value.status == igalr.IGA_EINVAL
    with pytest.raises(igalr.IgaError) as ei:
        op.apply(x, x, None)
    assert ei.value.status == igalr.IGA_EINVAL
    X = torch.zeros((3, 2, 8, 8, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(igalr.IgaError) as ei:
        op.kkt_apply(X, torch.zeros_like(X), 2, -1.0, 1e-4)
    assert ei.value.status == igalr.IGA_EINVAL
    opm = workloads.build_operator(cfg, w, stiff=False)
    with pytest.raises(igalr.IgaError) as ei:
        opm.kkt_apply(X, torch.zeros_like(X), 2, 0.5, 1e-4)
    assert ei.value.status == igalr.IGA_ESTATE


def test_host_entry_points_match_device(env):
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS["c2"], 20, batch=2)
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    x = np.random.default_rng(5).standard_normal((2, 20, 20, 20))
    dm, ds = gpu_apply(env, op, x)
    hm = np.zeros_like(x)
    hs = np.zeros_like(x)
    op.apply_host(x, hm, hs)
    # the host entry point pipelines the batch vector by vector (one apply per vector), so it
    # equals per-vector device applies bit for bit and the batched apply to rounding
    for b in range(2):
        m1, s1 = gpu_apply(env, op, x[b:b + 1])
        assert np.array_equal(hm[b], m1[0]) and np.array_equal(hs[b], s1[0])
    assert rel(hm, dm) <= 1e-14 and rel(hs, ds) <= 1e-14
    # summed output (y_mass_host == y_stiff_host) and mass-only
    hsum = np.zeros_like(x)
    op.apply_host(x, hsum, hsum, alpha=2.0, gamma=0.5)
    assert rel(hsum, 2.0 * dm + 0.5 * ds) <= 1e-14
    hm2 = np.zeros_like(x)
    op.apply_host(x, hm2, None)
    assert np.array_equal(hm2, hm)


# ----------------------------------------------------------------------------- KKT
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n,nt", [(10, 5), (13, 1), (7, 9)])
def test_kkt_full_vs_oracle(env, path, n, nt):
    torch, igalr, workloads = env
    base = synth.CONFIGS["c4"]
    cfg = synth.scaled(base, n, n_t=nt)
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    m = n - 2
    X = np.random.default_rng(n + nt).standard_normal((3, nt, m, m, m))
    ref = oracle.kkt_apply_csr(M, S, X, cfg.tau, cfg.beta)
    Xd = torch.from_numpy(X).cuda()
    out = torch.empty_like(Xd)
    op.kkt_apply(Xd, out, nt, cfg.tau, cfg.beta, path=path)
    got = out.cpu().numpy()
    for blk in range(3):
        assert rel(got[blk], ref[blk]) <= TOL
    assert rel(got, ref) <= TOL


@pytest.mark.parametrize("p,n,nt", [(4, 12, 3), (3, 11, 4)])
def test_kkt_batch_split_and_fallback(env, p, n, nt):
    """The KKT's stiffness part runs as one batch-split launch ([lambda, y] -> [r_y, r_lam]) where a
    split kernel variant exists (p = 3) and as one launch per block otherwise (p = 4): both match
    the oracle's rows of Eq. (KKTSystem)."""
    torch, igalr, workloads = env
    import dataclasses
    cfg = dataclasses.replace(synth.scaled(synth.CONFIGS["c4"], n, n_t=nt), p=p)
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    m = n - 2
    X = np.random.default_rng(7 * n + nt).standard_normal((3, nt, m, m, m))
    ref = oracle.kkt_apply_csr(M, S, X, cfg.tau, cfg.beta)
    Xd = torch.from_numpy(X).cuda()
    out = torch.empty_like(Xd)
    op.kkt_apply(Xd, out, nt, cfg.tau, cfg.beta)
    got = out.cpu().numpy()
    for blk in range(3):
        assert rel(got[blk], ref[blk]) <= TOL


def test_kkt_c4_full_size_sampled(env):
    torch, igalr, workloads = env
    cfg = synth.CONFIGS["c4"]
    knots, w, X = synth.draw_problem(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    Xd = torch.from_numpy(X).cuda()
    out = torch.empty_like(Xd)
    op.kkt_apply(Xd, out, cfg.n_t, cfg.tau, cfg.beta)
    got = out.cpu().numpy().reshape(3, cfg.n_t, -1)
    steps = [0, 1, 31, cfg.n_t - 1]
    rows = sample_rows(P.dims, 40, 9, cfg.p)
    ref = oracle.kkt_rows(P, X, cfg.tau, cfg.beta, steps, rows)
    for blk in range(3):
        g = got[blk][steps][:, rows]
        scale = np.linalg.norm(got[blk]) / np.sqrt(got[blk].size)
        assert np.abs(g - ref[blk]).max() <= TOL * scale
        assert rel(g, ref[blk]) <= TOL
    # host entry point agrees bitwise with the device one
    outh = np.zeros_like(X)
    op.kkt_apply_host(X, outh, cfg.n_t, cfg.tau, cfg.beta)
    assert np.array_equal(outh.reshape(3, cfg.n_t, -1), got)
