"""CPU oracle for the low-rank IgA hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_1811_06797_b200`` never imports it, and it never imports the product.  The only
shared module is ``synth`` (seeded input definitions, no method arithmetic).

What it computes (each function cites the passage it follows):

* ``gauss_legendre``      nq-point Gauss-Legendre rule on [-1,1] (reading G1/G2).
* ``basis_all``           all B-spline values / first derivatives, Cox-de Boor,
                          PAPER.md:58-63 (§2).
* ``gram_1d``             univariate weighted Gram int beta_i^(a) beta_j^(b) w,
                          Eq. (massMatrix1D) PAPER.md:192-196 and K^{(d)}_{k,l} PAPER.md:217-220.
* ``assemble_csr``        full 3D matrices M (Eq. massMatrix) and
                          K = S (Eq. stiffnessMatrix) by tensor Gauss quadrature.
* ``apply_matfree``       the same bilinear forms applied element by element.
* ``apply_rows``          the same bilinear forms for selected output rows.
* ``kkt_apply``           Eq. (KKTSystem) PAPER.md:313-319 written as the paper's three
                          gradient rows PAPER.md:306-308 per time step.
* ``kkt_dense``           the KKT matrix of Eq. (KKTSystem) assembled block by block from the
                          CSR M, S with calM = I (x) M, calK = I (x) tau S + C (x) M
                          (PAPER.md:316-318), for small sizes (dense LU solves, pins).
* ``minres``              MINRES (Paige & Saunders), the recurrence of Elman-Silvester-Wathen
                          Algorithm 2.4, step by step (the Krylov method of PAPER.md:399-400;
                          NEXT-1 of SURVEY.md §8(f)); ``kkt_prec_dense`` its block preconditioner.
* ``greville``, ``tt_svd``, ``weight_lowrank``  NEXT-2: samples at Greville points -> TT-SVD ->
                          univariate collocation solves -> canonical terms tabulated at nodes
                          (PAPER.md:177-265).
* ``Problem.weights3d``   NEXT-4: general (non-separable) omega and Q given at every 3D quadrature
                          point, e.g. a geometry's |det grad G| and (grad G^T grad G)^-1 |det grad G|
                          (PAPER.md:127-133), in the same assembly of Eqs. (massMatrix)/(stiffnessMatrix).
* ``tt_full``, ``tt_frame``, ``tt_project``  NEXT-3: the TT tensor of Eq. (tt),
                          the frame matrix of Eq. (frame) and F^T A F of
                          Eq. (KKT_red), dense, desk sizes.

Parity pins: tests/test_oracle_pins.py (P1-P12 of SURVEY.md §8(c)).
Every function here is pinned; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

TERM_WIDTH = 10


def build_oracle(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        D = ctypes.POINTER(ctypes.c_double)
        I = ctypes.POINTER(ctypes.c_int)
        I64 = ctypes.POINTER(ctypes.c_int64)
        I32 = ctypes.POINTER(ctypes.c_int32)
        lib.orc_gauss_legendre.argtypes = [ctypes.c_int, D, D]
        lib.orc_basis_all.argtypes = [D, ctypes.c_int, ctypes.c_int, ctypes.c_double, D, D]
        lib.orc_gram_1d.argtypes = [D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int, D]
        lib.orc_quad_nodes.argtypes = [D, ctypes.c_int, ctypes.c_int, ctypes.c_int, D, I64]
        lib.orc_csr_nnz.argtypes = [I, I, ctypes.c_int]
        lib.orc_csr_nnz.restype = ctypes.c_int64
        common = [I, I, D, D, D, ctypes.c_int, ctypes.c_int, D, I, D, ctypes.c_int, D]
        lib.orc_assemble_csr.argtypes = common + [I64, I32, D, D]
        lib.orc_spmv.argtypes = [ctypes.c_int64, I64, I32, D, D, D]
        lib.orc_assemble_csr_rows.argtypes = common + [ctypes.c_int64, ctypes.c_int64, I64, I32, D, D]
        lib.orc_csr_rows_nnz.argtypes = [I, I, ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        lib.orc_csr_rows_nnz.restype = ctypes.c_int64
        lib.orc_set_threads.argtypes = [ctypes.c_int]
        lib.orc_set_threads.restype = None
        lib.orc_apply_matfree.argtypes = common + [D, D, D]
        lib.orc_apply_rows.argtypes = common + [D, ctypes.c_int64, I64, D, D]
        _lib = lib
    return _lib


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


# ----------------------------------------------------------------------------------- 1D
def gauss_legendre(m: int) -> Tuple[np.ndarray, np.ndarray]:
    x = np.zeros(m)
    w = np.zeros(m)
    if _L().orc_gauss_legendre(m, _dp(x), _dp(w)):
        raise ValueError("bad m")
    return x, w


def basis_all(knots, p: int, t: float) -> Tuple[np.ndarray, np.ndarray]:
    k = np.ascontiguousarray(knots, dtype=np.float64)
    n = len(k) - p - 1
    v = np.zeros(n)
    d = np.zeros(n)
    if _L().orc_basis_all(_dp(k), n, p, float(t), _dp(v), _dp(d)):
        raise ValueError("bad knot vector")
    return v, d


def quad_nodes(knots, p: int, nq: int) -> np.ndarray:
    k = np.ascontiguousarray(knots, dtype=np.float64)
    n = len(k) - p - 1
    cnt = ctypes.c_int64(0)
    if _L().orc_quad_nodes(_dp(k), n, p, nq, None, ctypes.byref(cnt)):
        raise ValueError("bad knot vector")
    out = np.zeros(cnt.value)
    _L().orc_quad_nodes(_dp(k), n, p, nq, _dp(out), ctypes.byref(cnt))
    return out


def gram_1d(knots, p: int, nq: int, amp: float, k: float, phi: float, a: int, b: int) -> np.ndarray:
    """Dense n x n: G[i, j] = int beta_i^(a) beta_j^(b) (1 + amp sin(k pi t + phi)) dt."""
    kn = np.ascontiguousarray(knots, dtype=np.float64)
    n = len(kn) - p - 1
    out = np.zeros((n, n))
    if _L().orc_gram_1d(_dp(kn), n, p, nq, amp, k, phi, a, b, _dp(out)):
        raise ValueError("bad input")
    return out


# ----------------------------------------------------------------------------------- 3D
@dataclass
class Problem:
    """A 3D tensor-product spline space with separable closed-form weights.

    knots: [kx, ky, kz]; p: degree per direction (x, y, z); nq: Gauss points per span.
    mass_terms: [Rm, 10] term rows (synth layout) or None (no mass).
    q_terms:    9 arrays [R_kl, 10] for q_kl (k*3+l, k,l over x,y,z), empty => zero block.
    """
    knots: List[np.ndarray]
    p: Sequence[int]
    nq: int
    mass_terms: Optional[np.ndarray]
    q_terms: Optional[List[np.ndarray]]
    dirichlet: bool = False
    # optional general weights at every tensor quadrature point: [10, Gz, Gy, Gx] (omega, then
    # q_kl at 1 + k*3 + l), G_d = (nonempty spans) * nq along direction d in the order of
    # quad_nodes(); given => used instead of the separable closed-form terms
    weights3d: Optional[np.ndarray] = None
    _c: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self.knots = [np.ascontiguousarray(k, dtype=np.float64) for k in self.knots]
        self.p = [int(v) for v in self.p]
        n = [len(self.knots[d]) - self.p[d] - 1 for d in range(3)]
        self._n = np.array(n, dtype=np.int32)
        self._p = np.array(self.p, dtype=np.int32)
        if self.mass_terms is None or len(self.mass_terms) == 0:
            self._tm = np.zeros((1, TERM_WIDTH))
            self._ntm = 0
        else:
            self._tm = np.ascontiguousarray(self.mass_terms, dtype=np.float64).reshape(-1, TERM_WIDTH)
            self._ntm = self._tm.shape[0]
        qs = self.q_terms if self.q_terms is not None else [np.zeros((0, TERM_WIDTH))] * 9
        assert len(qs) == 9
        self._ntq = np.array([0 if q is None else np.asarray(q).reshape(-1, TERM_WIDTH).shape[0] for q in qs],
                             dtype=np.int32)
        cat = [np.asarray(q, dtype=np.float64).reshape(-1, TERM_WIDTH) for q in qs if q is not None and len(q)]
        self._tq = np.ascontiguousarray(np.concatenate(cat, 0)) if cat else np.zeros((1, TERM_WIDTH))
        if self.weights3d is not None:
            g = [len(quad_nodes(self.knots[d], self.p[d], self.nq)) for d in range(3)]
            w3 = np.ascontiguousarray(self.weights3d, dtype=np.float64)
            assert w3.shape == (10, g[2], g[1], g[0]), (w3.shape, g)
            self._w3 = w3

    @property
    def n(self):
        return [int(v) for v in self._n]

    @property
    def dims(self):
        """kept DoF extents (mx, my, mz)"""
        return [v - 2 if self.dirichlet else v for v in self.n]

    @property
    def ndof(self) -> int:
        mx, my, mz = self.dims
        return mx * my * mz

    def _args(self):
        return (_ip(self._n), _ip(self._p), _dp(self.knots[0]), _dp(self.knots[1]), _dp(self.knots[2]),
                self.nq, self._ntm, _dp(self._tm), _ip(self._ntq), _dp(self._tq), int(self.dirichlet),
                _dp(self._w3) if self.weights3d is not None else None)


def problem_from_config(cfg, weights, n: Optional[int] = None, nq: Optional[int] = None) -> Problem:
    """Oracle problem for a synth config (uniform open knots, reading A weights)."""
    import synth
    nn = cfg.n if n is None else n
    knots = [synth.uniform_open_knots(nn, cfg.p) for _ in range(3)]
    return Problem(knots=knots, p=[cfg.p] * 3, nq=(cfg.p + 1) if nq is None else nq,
                   mass_terms=weights.mass, q_terms=weights.q_block_terms(), dirichlet=cfg.dirichlet)


def assemble_csr(P: Problem, mass: bool = True, stiff: bool = True):
    """(M, S) as scipy.sparse.csr_matrix over the kept DoFs (row-major z,y,x)."""
    import scipy.sparse as sp
    nnz = _L().orc_csr_nnz(_ip(P._n), _ip(P._p), int(P.dirichlet))
    N = P.ndof
    rowptr = np.zeros(N + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int32)
    vm = np.zeros(nnz) if mass else None
    vs = np.zeros(nnz) if stiff else None
    rc = _L().orc_assemble_csr(*P._args(), rowptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                               col.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dp(vm), _dp(vs))
    if rc:
        raise ValueError("oracle assembly failed")
    M = sp.csr_matrix((vm, col, rowptr), shape=(N, N)) if mass else None
    S = sp.csr_matrix((vs, col, rowptr), shape=(N, N)) if stiff else None
    return M, S


def assemble_csr_rows(P: Problem, r0: int, r1: int, mass: bool = True, stiff: bool = True):
    """Rows [r0, r1) of (M, S) as scipy.sparse.csr_matrix of shape (r1-r0, N): the same
    assembly as assemble_csr restricted to a row range (bench samples of full-size matrices)."""
    import scipy.sparse as sp
    N = P.ndof
    nnz = _L().orc_csr_rows_nnz(_ip(P._n), _ip(P._p), int(P.dirichlet), int(r0), int(r1))
    rowptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int32)
    vm = np.zeros(nnz) if mass else None
    vs = np.zeros(nnz) if stiff else None
    rc = _L().orc_assemble_csr_rows(*P._args(), int(r0), int(r1),
                                    rowptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                    col.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dp(vm), _dp(vs))
    if rc:
        raise ValueError("oracle row assembly failed")
    M = sp.csr_matrix((vm, col, rowptr), shape=(r1 - r0, N)) if mass else None
    S = sp.csr_matrix((vs, col, rowptr), shape=(r1 - r0, N)) if stiff else None
    return M, S


def set_threads(t: int = 0):
    """OpenMP threads of the oracle (0 = all cores)."""
    _L().orc_set_threads(int(t))


def spmv(A, x: np.ndarray) -> np.ndarray:
    """naive CSR SpMV (row sums in column order), the oracle's y = A x."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    y = np.zeros(A.shape[0])
    _L().orc_spmv(A.shape[0], A.indptr.astype(np.int64).ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                  A.indices.astype(np.int32).ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                  _dp(np.ascontiguousarray(A.data)), _dp(x), _dp(y))
    return y


def apply_matfree(P: Problem, x: np.ndarray, mass: bool = True, stiff: bool = True):
    """(M x, S x) for x of shape [..., mz, my, mx] by the element-loop bilinear form."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    lead = x.shape[:-3]
    xf = x.reshape(-1, P.ndof)
    yM = np.zeros_like(xf) if mass else None
    yS = np.zeros_like(xf) if stiff else None
    for b in range(xf.shape[0]):
        xb = np.ascontiguousarray(xf[b])
        om = np.zeros(P.ndof) if mass else None
        os_ = np.zeros(P.ndof) if stiff else None
        if _L().orc_apply_matfree(*P._args(), _dp(xb), _dp(om), _dp(os_)):
            raise ValueError("oracle apply failed")
        if mass:
            yM[b] = om
        if stiff:
            yS[b] = os_
    shp = lead + tuple(x.shape[-3:])
    return (yM.reshape(shp) if mass else None, yS.reshape(shp) if stiff else None)


def apply_rows(P: Problem, x: np.ndarray, rows: np.ndarray, mass: bool = True, stiff: bool = True):
    """(M x)[rows], (S x)[rows] for ONE vector x (kept-DoF linear row indices)."""
    xb = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    assert xb.size == P.ndof
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    yM = np.zeros(rows.size) if mass else None
    yS = np.zeros(rows.size) if stiff else None
    if _L().orc_apply_rows(*P._args(), _dp(xb), rows.size, rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                           _dp(yM), _dp(yS)):
        raise ValueError("oracle apply_rows failed")
    return yM, yS


# ----------------------------------------------------------------------------------- KKT
def kkt_apply(applyM, applyS, applyST, X: np.ndarray, tau: float, beta: float) -> np.ndarray:
    """Eq. (KKTSystem) PAPER.md:313-319 applied to X = [y, u, lam], each [n_t, N].

    Written as the paper's gradient rows, k = 1..n_t, with
    y_0 = 0 and lambda_{n_t+1} = 0 (reading G9: tau kept as in
    PAPER.md:291,298,308):
      r_y[k]   = tau M y_k - M lam_{k+1} + M lam_k + tau K^T lam_k
      r_u[k]   = tau beta M u_k - tau M lam_k
      r_lam[k] = M y_k - M y_{k-1} + tau K y_k - tau M u_k
    PAPER.md:306 writes the y-row as the row vector lambda_k (M + tau K), i.e. (M + tau K)^T
    lambda_k, and Eq. (KKTSystem) puts calK^T in the first block row: K^T, not K (the two
    differ when q_kl != q_lk, which the paper allows: every q_kl is approximated on its own,
    PAPER.md:202-206).  M is symmetric by Eq. (massMatrix).
    applyM / applyS / applyST map one [N] vector to M v / K v / K^T v (oracle routes)."""
    y, u, lam = X[0], X[1], X[2]
    nt = y.shape[0]
    My = [applyM(y[k]) for k in range(nt)]
    Mu = [applyM(u[k]) for k in range(nt)]
    Ml = [applyM(lam[k]) for k in range(nt)]
    Sy = [applyS(y[k]) for k in range(nt)]
    STl = [applyST(lam[k]) for k in range(nt)]
    out = np.zeros_like(X)
    for k in range(nt):
        Ml_next = Ml[k + 1] if k + 1 < nt else 0.0
        My_prev = My[k - 1] if k >= 1 else 0.0
        out[0, k] = tau * My[k] - Ml_next + Ml[k] + tau * STl[k]
        out[1, k] = tau * beta * Mu[k] - tau * Ml[k]
        out[2, k] = My[k] - My_prev + tau * Sy[k] - tau * Mu[k]
    return out


def kkt_apply_csr(M, S, X: np.ndarray, tau: float, beta: float) -> np.ndarray:
    """kkt_apply with the CSR routes: M v, S v and S^T v (the transpose of the assembled CSR
    matrix, scipy.sparse, then the same naive SpMV)."""
    shp = X.shape
    Xf = X.reshape(3, shp[1], -1)
    ST = S.T.tocsr()
    out = kkt_apply(lambda v: spmv(M, v), lambda v: spmv(S, v), lambda v: spmv(ST, v), Xf, tau, beta)
    return out.reshape(shp)


def transpose_problem(P: Problem) -> Problem:
    """The problem whose stiffness matrix is K^T: every block q_kl replaced by q_lk.
    By Eq. (stiffnessMatrix), (K^T)_ij = K_ji = sum_kl int q_kl d_l beta_j
    d_k beta_i = sum_kl int q_lk d_l beta_i d_k beta_j, i.e. the same definition with Q^T.
    The mass part is unchanged (M is symmetric)."""
    qs = P.q_terms
    qT = None if qs is None else [qs[l * 3 + k] for k in range(3) for l in range(3)]
    w3 = None
    if P.weights3d is not None:
        w3 = np.array(P.weights3d, copy=True)
        for k in range(3):
            for l in range(3):
                w3[1 + k * 3 + l] = P.weights3d[1 + l * 3 + k]
    return Problem(knots=P.knots, p=P.p, nq=P.nq, mass_terms=P.mass_terms, q_terms=qT, dirichlet=P.dirichlet,
                   weights3d=w3)


def kkt_rows(P: Problem, X: np.ndarray, tau: float, beta: float, steps: Sequence[int],
             rows: np.ndarray) -> np.ndarray:
    """Sampled KKT outputs: out[blk, j, i] for time steps `steps` (0-based) and spatial
    rows `rows`, via the same three paper rows with row-restricted applies (K^T v from the
    transposed problem, transpose_problem)."""
    nt = X.shape[1]
    Xf = X.reshape(3, nt, -1)
    res = np.zeros((3, len(steps), len(rows)))
    PT = transpose_problem(P)

    def M_(v):
        return apply_rows(P, v, rows, mass=True, stiff=False)[0]

    def S_(v):
        return apply_rows(P, v, rows, mass=False, stiff=True)[1]

    def ST_(v):
        return apply_rows(PT, v, rows, mass=False, stiff=True)[1]

    for j, k in enumerate(steps):
        y, u, lam = Xf[0], Xf[1], Xf[2]
        My = M_(y[k]); Mu = M_(u[k]); Ml = M_(lam[k])
        Ml_next = M_(lam[k + 1]) if k + 1 < nt else 0.0
        My_prev = M_(y[k - 1]) if k >= 1 else 0.0
        Sy = S_(y[k]); STl = ST_(lam[k])
        res[0, j] = tau * My - Ml_next + Ml + tau * STl
        res[1, j] = tau * beta * Mu - tau * Ml
        res[2, j] = My - My_prev + tau * Sy - tau * Mu
    return res


def kkt_dense(M, S, n_t: int, tau: float, beta: float) -> np.ndarray:
    """Dense KKT matrix of Eq. (KKTSystem) PAPER.md:313-319:
        [[tau calM, 0, calK^T], [0, tau beta calM, -tau calM], [calK, -tau calM, 0]]
    with calM = I_{n_t} (x) M and calK = I_{n_t} (x) tau S + C (x) M, C = 1 on the diagonal and
    -1 on the first subdiagonal.  Block order (y, u, lambda), each block
    time-major [n_t][N] like the GPU layout.  Small sizes only."""
    Md = M.toarray() if hasattr(M, "toarray") else np.asarray(M)
    Sd = S.toarray() if hasattr(S, "toarray") else np.asarray(S)
    I = np.eye(n_t)
    C = np.eye(n_t) - np.eye(n_t, k=-1)
    calM = np.kron(I, Md)
    calK = np.kron(I, tau * Sd) + np.kron(C, Md)
    Z = np.zeros_like(calM)
    return np.block([[tau * calM, Z, calK.T], [Z, tau * beta * calM, -tau * calM], [calK, -tau * calM, Z]])


def minres(matvec, b: np.ndarray, x0: Optional[np.ndarray] = None, maxit: int = 1000, rtol: float = 1e-8,
           precond=None):
    """Preconditioned MINRES for symmetric A and SPD P (Paige & Saunders 1975), Elman, Silvester
    & Wathen, Algorithm 2.4, written out step by step (P = I when precond is None):

        v_0 = 0, w_0 = w_1 = 0, v_1 = b - A x_0, z_1 = P^{-1} v_1, gamma_1 = sqrt(z_1' v_1),
        gamma_0 = 1, eta = gamma_1, s_0 = s_1 = 0, c_0 = c_1 = 1;  for j = 1, 2, ...
          z_j = z_j / gamma_j;  delta_j = (A z_j)' z_j
          v_{j+1} = A z_j - (delta_j / gamma_j) v_j - (gamma_j / gamma_{j-1}) v_{j-1}
          z_{j+1} = P^{-1} v_{j+1};  gamma_{j+1} = sqrt(z_{j+1}' v_{j+1})
          a0 = c_j delta_j - c_{j-1} s_j gamma_j;  a1 = sqrt(a0^2 + gamma_{j+1}^2)
          a2 = s_j delta_j + c_{j-1} c_j gamma_j;  a3 = s_{j-1} gamma_j
          c_{j+1} = a0 / a1;  s_{j+1} = gamma_{j+1} / a1
          w_{j+1} = (z_j - a3 w_{j-1} - a2 w_j) / a1;  x_j = x_{j-1} + c_{j+1} eta w_{j+1}
          eta = -s_{j+1} eta          (|eta| = |b - A x_j| in the P^{-1} norm)

    Stops when |eta| <= rtol gamma_1 or after maxit iterations.  Returns (x, iters, |eta| /
    gamma_1, gamma_1).  Vectors are flat float64; matvec / precond map flat vectors."""
    Pinv = (lambda v: v.copy()) if precond is None else precond
    b = np.asarray(b, dtype=np.float64).ravel()
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64).ravel()
    v = b - matvec(x) if x0 is not None else b.copy()
    z = Pinv(v)
    gamma = float(np.sqrt(max(z @ v, 0.0)))
    gamma_prev = 1.0
    res0 = gamma
    v_prev = np.zeros_like(b)
    w_prev = np.zeros_like(b)
    w = np.zeros_like(b)
    eta = gamma
    c_prev = c = 1.0
    s_prev = s = 0.0
    z = z / gamma if gamma > 0 else z * 0.0
    it = 0
    while it < maxit and abs(eta) > rtol * res0:
        Az = matvec(z)
        delta = float(Az @ z)
        v_next = Az - (delta / gamma) * v - (gamma / gamma_prev) * v_prev
        z_next = Pinv(v_next)
        gamma_next = float(np.sqrt(max(z_next @ v_next, 0.0)))
        a0 = c * delta - c_prev * s * gamma
        a1 = float(np.sqrt(a0 * a0 + gamma_next * gamma_next))
        a2 = s * delta + c_prev * c * gamma
        a3 = s_prev * gamma
        c_next = a0 / a1 if a1 > 0 else 1.0
        s_next = gamma_next / a1 if a1 > 0 else 0.0
        w_next = (z - a3 * w_prev - a2 * w) / a1 if a1 > 0 else np.zeros_like(b)
        x = x + (c_next * eta) * w_next
        eta = -s_next * eta
        v_prev, v = v, v_next
        z = z_next / gamma_next if gamma_next > 0 else z_next * 0.0
        w_prev, w = w, w_next
        c_prev, c = c, c_next
        s_prev, s = s, s_next
        gamma_prev, gamma = gamma, gamma_next
        it += 1
    return x, it, (abs(eta) / res0 if res0 > 0 else 0.0), res0


def kkt_prec_dense(P: "Problem", M, S, n_t: int, tau: float, beta: float, exact: bool = False):
    """The block-diagonal KKT preconditioner of DESIGN.md §11 as a dense matrix (small sizes):

        P = blkdiag(tau I (x) Mh,  tau beta I (x) Mh,  Sh),
        Sh = (1/tau) G (I (x) Mh)^{-1} G',   G = I (x) (tau Sh0) + C (x) Mh + g I (x) Mh,
        g = tau / sqrt(beta),  Mh = mbar M0,  Sh0 = sbar S0,

    M0 = M0z (x) M0y (x) M0x and S0 = K0z(x)M0y(x)M0x + M0z(x)K0y(x)M0x + M0z(x)M0y(x)K0x from
    the unit-weight univariate Grams (gram_1d with amp = 0, Eq. (massMatrix1D) PAPER.md:192-196;
    patterns (0,0) and (1,1)), Dirichlet-sliced like the problem; mbar = v1' M v1 / v1' M0 v1 and
    sbar = v1' S v1 / v1' S0 v1 for v1 = e1z (x) e1y (x) e1x, e1d the eigenvector of the smallest
    positive eigenvalue of K0d v = lam M0d v (scipy.linalg.eigh).  exact=True uses M, S themselves
    (Mh = M, Sh0 = S: the ideal matching preconditioner).  Returns (P, mbar, sbar, lam per dir)."""
    import scipy.linalg as sla
    M0d, K0d, e1, lams = [], [], [], []
    for d in range(3):
        kn, p = P.knots[d], P.p[d]
        G0 = gram_1d(kn, p, P.nq, 0.0, 1.0, 0.0, 0, 0)
        G1 = gram_1d(kn, p, P.nq, 0.0, 1.0, 0.0, 1, 1)
        if P.dirichlet:
            G0, G1 = G0[1:-1, 1:-1], G1[1:-1, 1:-1]
        lam, V = sla.eigh(G1, G0)
        M0d.append(G0)
        K0d.append(G1)
        # smoothest mode with a positive eigenvalue: without Dirichlet the constant lies in the
        # kernel of K0d (sbar would be 0/0 there); DESIGN.md §2 (reading R2-1)
        pos = np.where(lam > 1e-8 * lam.max())[0]
        e1.append(V[:, int(pos[np.argmin(lam[pos])])])
        lams.append(lam)
    kron3 = lambda a, b, c: np.kron(c, np.kron(b, a))  # x fastest: (z) (x) (y) (x) (x)
    M0 = kron3(M0d[0], M0d[1], M0d[2])
    S0 = kron3(K0d[0], M0d[1], M0d[2]) + kron3(M0d[0], K0d[1], M0d[2]) + kron3(M0d[0], M0d[1], K0d[2])
    v1 = kron3(e1[0][:, None], e1[1][:, None], e1[2][:, None]).ravel()
    Md = M.toarray() if hasattr(M, "toarray") else np.asarray(M)
    Sd = S.toarray() if hasattr(S, "toarray") else np.asarray(S)
    mbar = (v1 @ Md @ v1) / (v1 @ M0 @ v1)
    sbar = (v1 @ Sd @ v1) / (v1 @ S0 @ v1)
    Mh, Sh0 = (Md, Sd) if exact else (mbar * M0, sbar * S0)
    g = tau / np.sqrt(beta)
    I = np.eye(n_t)
    C = np.eye(n_t) - np.eye(n_t, k=-1)
    G = np.kron(I, tau * Sh0) + np.kron(C, Mh) + g * np.kron(I, Mh)
    calMh = np.kron(I, Mh)
    Sh = (G @ np.linalg.solve(calMh, G.T)) / tau
    Z = np.zeros_like(calMh)
    Pm = np.block([[tau * calMh, Z, Z], [Z, tau * beta * calMh, Z], [Z, Z, Sh]])
    return Pm, mbar, sbar, lams


# ----------------------------------------------------------------------------- NEXT-2 (weights)
def greville(knots, p: int) -> np.ndarray:
    """Greville abscissae xi*_i = (t_{i+1} + ... + t_{i+p}) / p (the interpolation points)."""
    t = np.asarray(knots, dtype=np.float64)
    n = len(t) - p - 1
    return np.array([t[i + 1:i + p + 1].sum() / p for i in range(n)])


def collocation(knots, p: int, pts) -> np.ndarray:
    """B[i, j] = beta_j(pts_i) from the full Cox-de Boor triangle (basis_all)."""
    t = np.asarray(knots, dtype=np.float64)
    n = len(t) - p - 1
    return np.array([basis_all(t, p, float(x))[0][:n] for x in pts])


def tt_svd(S: np.ndarray, eps: float):
    """TT-SVD (Oseledets 2011) of a 3-way tensor S[z, y, x] (slowest first), truncating each
    unfolding to the smallest rank whose discarded singular values have squared sum
    <= (eps |S|_F / sqrt(2))^2.  Returns cores (G1 [nz, R1], G2 [R1, ny, R2], G3 [R2, nx])."""
    nz, ny, nx = S.shape
    d2 = (eps * np.linalg.norm(S)) ** 2 / 2.0

    def rank(sv):
        r = len(sv)
        tail = 0.0
        while r > 1 and tail + sv[r - 1] ** 2 <= d2:
            tail += sv[r - 1] ** 2
            r -= 1
        return r

    U, sv, Vt = np.linalg.svd(S.reshape(nz, ny * nx), full_matrices=False)
    R1 = rank(sv)
    G1 = U[:, :R1]
    C = (sv[:R1, None] * Vt[:R1]).reshape(R1 * ny, nx)
    U, sv, Vt = np.linalg.svd(C, full_matrices=False)
    R2 = rank(sv)
    G2 = U[:, :R2].reshape(R1, ny, R2)
    G3 = sv[:R2, None] * Vt[:R2]
    return G1, G2, G3


def weight_lowrank(nodes, tilde_knots, tilde_p, samples: np.ndarray, eps: float):
    """Eqs. (TTranks) PAPER.md:243-246 and (weightEquationSolve) PAPER.md:256-262: the TT
    cores of the samples, each factor vector solved against the univariate collocation matrix
    at the Greville points, the R1 R2 canonical terms evaluated at `nodes` (per direction x, y,
    z).  Returns tabs [x, y, z], each [R, len(nodes_d)], and the TT ranks."""
    G1, G2, G3 = tt_svd(np.asarray(samples, dtype=np.float64), eps)
    R1, R2 = G1.shape[1], G3.shape[0]
    B = [collocation(tilde_knots[d], tilde_p[d], greville(tilde_knots[d], tilde_p[d])) for d in range(3)]
    E = [collocation(tilde_knots[d], tilde_p[d], nodes[d]) for d in range(3)]
    tabs = [np.zeros((R1 * R2, len(nodes[d]))) for d in range(3)]
    for r1 in range(R1):
        for r2 in range(R2):
            r = r1 * R2 + r2
            for d, f in ((2, G1[:, r1]), (1, G2[r1, :, r2]), (0, G3[r2, :])):
                tabs[d][r] = E[d] @ np.linalg.solve(B[d], f)
    return tabs, (R1, R2)


# ------------------------------------------------------------------ TT vectors (NEXT-3)
# Plain definitions for checking the library's TT entry points; 3D, cores in
# the paper's order (slowest direction first): gz [mz, R1], gy [R1, my, R2], gx [R2, mx].
def tt_full(gz: np.ndarray, gy: np.ndarray, gx: np.ndarray) -> np.ndarray:
    """Eq. (tt): v(iz, iy, ix) = sum_{a,b} gz[iz, a] gy[a, iy, b] gx[b, ix]."""
    return np.einsum("za,ayb,bx->zyx", gz, gy, gx)


def tt_frame(gz: np.ndarray, gy: np.ndarray, gx: np.ndarray, site: int) -> np.ndarray:
    """Frame matrix F_{!=d} of Eq. (frame), dense, rows (iz, iy, ix), columns
    (r_{d-1}, j_d, r_d) row-major; site 0 = x, 1 = y, 2 = z (d = 3, 2, 1 in the paper)."""
    mz, R1 = gz.shape
    _, my, R2 = gy.shape
    mx = gx.shape[1]
    if site == 1:   # F[(iz,iy,ix),(a,jy,b)] = gz[iz,a] delta(iy,jy) gx[b,ix]
        F = np.einsum("za,yj,bx->zyxajb", gz, np.eye(my), gx)
        return F.reshape(mz * my * mx, R1 * my * R2)
    if site == 2:   # F[(iz,iy,ix),(jz,a)] = delta(iz,jz) sum_b gy[a,iy,b] gx[b,ix]
        right = np.einsum("ayb,bx->ayx", gy, gx)
        F = np.einsum("zj,ayx->zyxja", np.eye(mz), right)
        return F.reshape(mz * my * mx, mz * R1)
    # site 0: F[(iz,iy,ix),(b,jx)] = sum_a gz[iz,a] gy[a,iy,b] delta(ix,jx)
    left = np.einsum("za,ayb->zyb", gz, gy)
    F = np.einsum("zyb,xj->zyxbj", left, np.eye(mx))
    return F.reshape(mz * my * mx, R2 * mx)


def tt_project(A, gz, gy, gx, site: int) -> np.ndarray:
    """The projected matrix F_{!=d}^T A F_{!=d} of Eq. (KKT_red), A dense or
    sparse over the row-major (z, y, x) DoFs."""
    F = tt_frame(gz, gy, gx, site)
    return F.T @ (A @ F)
