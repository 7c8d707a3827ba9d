"""NEXT-3: the Kronecker operators on TT vectors through the C ABI
(iga_lr_terms, iga_tt_kron_apply, iga_tt_interfaces, iga_tt_local_apply) against the oracle's
plain definitions: the dense tensor of Eq. (tt), the assembled M and S, and the dense frame
projection F_{!=d}^T A F_{!=d} of Eqs. (frame)/(KKT_red)."""
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
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def _setup(env, cfgname="c2", n=7, p=None):
    torch, igalr, workloads = env
    cfg = synth.scaled(synth.CONFIGS[cfgname], n)
    if p is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, p=p)
    w = synth.draw_weights(cfg)
    op = workloads.build_operator(cfg, w)
    P = oracle.problem_from_config(cfg, w)
    M, S = oracle.assemble_csr(P)
    return op, (M, S), P.dims


@pytest.mark.parametrize("cfgname,n,R1,R2", [("c2", 7, 3, 4), ("c5", 10, 2, 5), ("c1", 8, 1, 1)])
def test_tt_kron_apply_vs_dense(env, cfgname, n, R1, R2):
    torch, igalr, workloads = env
    op, mats, (mx, my, mz) = _setup(env, cfgname, n)
    rng = np.random.default_rng(n + R1)
    gz, gy, gx = rng.standard_normal((mz, R1)), rng.standard_normal((R1, my, R2)), rng.standard_normal((R2, mx))
    v = oracle.tt_full(gz, gy, gx).ravel()
    dg = [torch.from_numpy(a).cuda() for a in (gz, gy, gx)]
    for part, A in enumerate(mats):
        fid, coef = op.terms(part)
        T = len(coef)
        assert T >= 1 and fid.shape == (T, 3)
        wz = torch.empty((T, mz, R1), dtype=torch.float64, device="cuda")
        wy = torch.empty((T, R1, my, R2), dtype=torch.float64, device="cuda")
        wx = torch.empty((T, R2, mx), dtype=torch.float64, device="cuda")
        op.tt_kron_apply(part, *dg, wz, wy, wx)
        got = np.einsum("tza,tayb,tbx->zyx", wz.cpu().numpy(), wy.cpu().numpy(), wx.cpu().numpy())
        assert rel(got, A @ v) <= TOL


@pytest.mark.parametrize("site", [0, 1, 2])
@pytest.mark.parametrize("cfgname,n,p", [("c2", 7, None), ("c5", 9, None), ("c4", 8, 2)])
def test_tt_projected_local_apply_vs_dense_frame(env, site, cfgname, n, p):
    torch, igalr, workloads = env
    op, mats, (mx, my, mz) = _setup(env, cfgname, n, p)
    R1, R2 = 3, 2
    rng = np.random.default_rng(10 * site + n)
    gz, gy, gx = rng.standard_normal((mz, R1)), rng.standard_normal((R1, my, R2)), rng.standard_normal((R2, mx))
    dg = [torch.from_numpy(a).cuda() for a in (gz, gy, gx)]
    Rl, m, Rr = {0: (R2, mx, 1), 1: (R1, my, R2), 2: (1, mz, R1)}[site]
    x = rng.standard_normal((Rl, m, Rr))
    for part, A in enumerate(mats):
        T = len(op.terms(part)[1])
        L = torch.empty((T, Rl, Rl), dtype=torch.float64, device="cuda")
        R = torch.empty((T, Rr, Rr), dtype=torch.float64, device="cuda")
        op.tt_interfaces(part, site, *dg, L, R)
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        op.tt_local_apply(part, site, L, R, xd, yd)
        ref = oracle.tt_project(A, gz, gy, gx, site) @ x.ravel()
        assert rel(yd.cpu().numpy(), ref) <= TOL, (part, site)


def test_tt_errors(env):
    torch, igalr, workloads = env
    op, mats, (mx, my, mz) = _setup(env, "c2", 6)
    g = [torch.zeros(s, dtype=torch.float64, device="cuda") for s in ((mz, 2), (2, my, 2), (2, mx))]
    L = torch.zeros((64, 4, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(igalr.IgaError) as e:
        op.tt_interfaces(1, 3, *g, L, L)
    assert e.value.status == igalr.IGA_EINVAL
    with pytest.raises(igalr.IgaError) as e:
        op.terms(2)
    assert e.value.status == igalr.IGA_EINVAL
