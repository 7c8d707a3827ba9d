"""NEXT-4: the paper's assembly study (section "Assembly with TT method") on the
extruded quarter annulus, with the CPU oracle standing in for GeoPDEs' full assembly.

Per refinement level (4 knots inserted per span per level: 1, 5, 25 spans) and
5-point Gauss rule in both assemblies:

  * full:     the oracle's 3D tensor-product quadrature assembly of M and S with the exact
              geometry weights omega = |det grad G| and Q at every 3D point;
  * low rank: omega and each Q_kl sampled at the Greville points of a degree-(2p+1) spline space
              (PAPER.md:422), TT-SVD + collocation (iga_weight_lowrank, NEXT-2), univariate factor
              assembly on the GPU (iga_lr_assemble_factors);
  * diff = ||S - S~||_F / ||S||_F, same for M; S~ is read back exactly from
    the GPU operator by colour probing: (2p+1)^3 indicator vectors, one per residue class of the
    index modulo 2p+1 in each direction, separate every band column of a row;
  * storage: bytes of the univariate band factors vs the CSR matrix;
  * time: weight compression + GPU factor assembly vs the oracle's full assembly (its cores).

Test infrastructure (it runs the oracle): driven by tests/test_gpu_assembly_study.py, which also
writes the full table when IGALR_STUDY_OUT is set, e.g.
  IGALR_STUDY_LEVELS=1,5,25 IGALR_STUDY_OUT=profiles/r01c_assembly_study \
      python -m pytest tests/test_gpu_assembly_study.py -m gpu
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth.geometry import QuarterAnnulus, refinement_knots  # noqa: E402

NQ = 5


def probe_matrices(op, p, pattern_rows, pattern_cols, dims):
    """Entries of the GPU operator's M~ and S~ on the given (row, col) pattern, by colour probing."""
    import torch
    mx, my, mz = dims
    w = 2 * p + 1
    C = w ** 3
    iz, iy, ix = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    colour = ((iz % w) * w + (iy % w)) * w + (ix % w)
    X = np.zeros((C, mz, my, mx))
    for c in range(C):
        X[c][colour == c] = 1.0
    xd = torch.from_numpy(X).cuda()
    ym, ys = torch.empty_like(xd), torch.empty_like(xd)
    op.apply(xd, ym, ys)
    torch.cuda.synchronize()
    Ym = ym.cpu().numpy().reshape(C, -1)
    Ys = ys.cpu().numpy().reshape(C, -1)
    cz = pattern_cols // (mx * my)
    cy = (pattern_cols // mx) % my
    cx = pattern_cols % mx
    ccol = ((cz % w) * w + (cy % w)) * w + (cx % w)
    return Ym[ccol, pattern_rows], Ys[ccol, pattern_rows], (xd, ym, ys)


def level(p, spans, geom, eps=1e-10):
    import torch  # noqa: F401
    import paper_1811_06797_b200 as igalr
    kn = refinement_knots(p, spans)
    n = len(kn) - p - 1
    # ---- full assembly (oracle, exact geometry weights at every 3D quadrature point)
    nodes = [oracle.quad_nodes(kn, p, NQ)] * 3
    w3 = geom.fields(nodes[0], nodes[1], nodes[2])
    P = oracle.Problem(knots=[kn] * 3, p=[p] * 3, nq=NQ, mass_terms=None, q_terms=None, weights3d=w3)
    t0 = time.perf_counter()
    M, S = oracle.assemble_csr(P)
    t_full = time.perf_counter() - t0
    # ---- low-rank assembly (NEXT-2 weights, GPU factors)
    pt = 2 * p + 1
    tk = refinement_knots(pt, spans)
    gr = igalr.greville(tk, pt)
    samples = geom.fields(gr, gr, gr)
    t0 = time.perf_counter()
    omega, r_om, _ = igalr.weight_lowrank([kn] * 3, [p] * 3, [tk] * 3, [pt] * 3, samples[0], eps=eps, nq=NQ)
    q = [None] * 9
    ranks = {"omega": r_om}
    for b in range(9):
        if np.abs(samples[1 + b]).max() > 0:
            q[b], rq, _ = igalr.weight_lowrank([kn] * 3, [p] * 3, [tk] * 3, [pt] * 3, samples[1 + b], eps=eps,
                                               nq=NQ)
            ranks["q%d%d" % (b // 3 + 1, b % 3 + 1)] = rq
    t_w = time.perf_counter() - t0
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = igalr.LowRankOperator([kn] * 3, [p] * 3, omega, q, nq=NQ)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    # ---- compare on the band pattern
    Mc = M.tocoo()
    rows, cols = Mc.row.astype(np.int64), Mc.col.astype(np.int64)
    Sv = S.tocoo()
    assert np.array_equal(Sv.row, Mc.row) and np.array_equal(Sv.col, Mc.col)
    mt, st, (xd, ym, ys) = probe_matrices(op, p, rows, cols, op.dims)
    diff_m = float(np.linalg.norm(Mc.data - mt) / np.linalg.norm(Mc.data))
    diff_s = float(np.linalg.norm(Sv.data - st) / np.linalg.norm(Sv.data))
    # probing sanity: the reconstructed S~ applied to a random vector equals the GPU apply
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    x = rng.standard_normal(op.dims[::-1])
    St = sp.csr_matrix((st, (rows, cols)), shape=S.shape)
    xg = torch.from_numpy(x[None]).cuda()
    yg = torch.empty_like(xg)
    op.apply(xg, None, yg)
    torch.cuda.synchronize()
    probe_err = float(np.linalg.norm(St @ x.ravel() - yg.cpu().numpy().ravel()) / np.linalg.norm(St @ x.ravel()))
    info = op.info_dict()
    lowrank_bytes = 8 * sum(info["n_factors"][d] * info["dims"][d] * (2 * p + 1) for d in range(3))
    full_bytes = S.nnz * (8 + 4) + 8 * (S.shape[0] + 1)
    return {"p": p, "spans": spans, "n": n, "N": int(S.shape[0]), "nnz": int(S.nnz), "ranks": ranks,
            "diff_M": diff_m, "diff_S": diff_s, "probe_err": probe_err, "lowrank_bytes": int(lowrank_bytes),
            "full_bytes": int(full_bytes), "storage_ratio": full_bytes / lowrank_bytes,
            "t_full_s": t_full, "t_weights_s": t_w, "t_gpu_assembly_s": t_asm,
            "oracle_cores": len(os.sched_getaffinity(0))}


def table(res):
    lines = ["| spans/dir | n/dir | DoFs | TT ranks (omega; q11, q22, q33) | diff M | diff S | storage full/low-rank |"
             " full assembly s (oracle, %d cores) | weights + GPU factors s |" % res[0]["oracle_cores"],
             "|---|---|---|---|---|---|---|---|---|"]
    for r in res:
        rk = r["ranks"]
        lines.append("| %d | %d | %d | %s; %s, %s, %s | %.2e | %.2e | %.0f | %.3f | %.3f + %.3f |" % (
            r["spans"], r["n"], r["N"], rk["omega"], rk.get("q11"), rk.get("q22"), rk.get("q33"), r["diff_M"],
            r["diff_S"], r["storage_ratio"], r["t_full_s"], r["t_weights_s"], r["t_gpu_assembly_s"]))
    return "\n".join(lines)


def write(res, out, p):
    txt = table(res)
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    with open(out + ".md", "w") as f:
        f.write("# NEXT-4 assembly study (tests/study_assembly.py, p = %d)\n\n" % p)
        f.write("Extruded quarter annulus (PAPER.md:424), 5-point Gauss rule, interpolation degree 2p+1 "
                "(PAPER.md:422). diff = ||A - A~||_F / ||A||_F (PAPER.md:436); the low-rank A~ is read back "
                "from the GPU operator by colour probing (probe consistency <= %.1e).\n\n"
                % max(r["probe_err"] for r in res))
        f.write(txt + "\n")
    return txt


