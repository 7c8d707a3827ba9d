"""B200-native low-rank IgA operator library (arXiv:1811.06797 hot path) — Python binding.

Thin ctypes marshalling over the C ABI in ``include/iga_lr.h`` (``libigalr.so`` built in-tree
by ``_build.py``).  Every step of the path runs in the library's CUDA kernels; PyTorch is used
only for device memory (``tensor.data_ptr()``) and streams (``torch.cuda.Stream``).  There is
no CPU fallback: if the shared library is missing this module raises ImportError, and every
ABI failure raises ``IgaError`` with the library's message.

Names follow the paper: ``mass`` = M (Eq. (massFinal)), ``stiff`` = K/S
(Eq. (stiffnessFinal)), ``kkt_apply`` = Eq. (KKTSystem) PAPER.md:313-319.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libigalr.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        "libigalr.so not found in %s — build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(no CPU fallback exists)" % _HERE)

_lib = ctypes.CDLL(LIB_PATH)

IGA_OK, IGA_EINVAL, IGA_ENOMEM, IGA_ECUDA, IGA_EUNSUPPORTED, IGA_ESTATE = range(6)
IGA_DIRICHLET = 0x1
PATHS = {"auto": 0x0, "unfused": 0x10, "fused": 0x20, "fused_v1": 0x40}
STATUS_NAMES = {0: "IGA_OK", 1: "IGA_EINVAL", 2: "IGA_ENOMEM", 3: "IGA_ECUDA", 4: "IGA_EUNSUPPORTED",
                5: "IGA_ESTATE"}

ABI_SYMBOLS = ["iga_quad_nodes", "iga_lr_assemble_factors", "iga_lr_destroy", "iga_lr_apply", "iga_lr_apply2",
               "iga_kkt_apply", "iga_lr_apply_host", "iga_kkt_apply_host", "iga_lr_info", "iga_lr_export_factor",
               "iga_last_error", "iga_version", "iga_kkt_minres", "iga_kkt_prec_create", "iga_kkt_prec_destroy",
               "iga_kkt_prec_apply", "iga_kkt_prec_info", "iga_greville", "iga_weight_lowrank",
               "iga_weight_lowrank_sep", "iga_weight_lowrank_free", "iga_lr_terms", "iga_tt_kron_apply",
               "iga_tt_interfaces", "iga_tt_local_apply"]
MINRES_X0 = 0x100


class _Knobs(ctypes.Structure):
    """iga_test_knobs (include/iga_lr_testing.h): test-only kernel-selection overrides."""
    _fields_ = [("force_generic", ctypes.c_int32), ("qx", ctypes.c_int32), ("minlen", ctypes.c_int32),
                ("no_yres", ctypes.c_int32), ("no_tma", ctypes.c_int32), ("vpack", ctypes.c_int32)]


class IgaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status


class _Dir(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int32), ("n", ctypes.c_int32), ("knots", ctypes.POINTER(ctypes.c_double))]


class _Space(ctypes.Structure):
    _fields_ = [("dir", _Dir * 3), ("nq", ctypes.c_int32)]


class _Sep(ctypes.Structure):
    _fields_ = [("R", ctypes.c_int32), ("coef", ctypes.POINTER(ctypes.c_double)),
                ("tab", ctypes.POINTER(ctypes.c_double) * 3)]


class _Info(ctypes.Structure):
    _fields_ = [("dims", ctypes.c_int64 * 3), ("p", ctypes.c_int32 * 3), ("nq", ctypes.c_int32),
                ("n_factors", ctypes.c_int32 * 3), ("n_rounds", ctypes.c_int32), ("n_xprod", ctypes.c_int32),
                ("n_yprod", ctypes.c_int32), ("n_zprod", ctypes.c_int32), ("has_mass", ctypes.c_int32),
                ("has_stiff", ctypes.c_int32), ("fused_ok", ctypes.c_int32), ("fused2_ok", ctypes.c_int32), ("plan_flops_per_vec", ctypes.c_double),
                ("min_bytes_per_vec", ctypes.c_double), ("plan_flops_mass", ctypes.c_double),
                ("plan_flops_stiff", ctypes.c_double), ("canon_mass", ctypes.c_int32),
                ("canon_stiff", ctypes.c_int32), ("stiff_symmetric", ctypes.c_int32),
                ("f2_rounds_stiff", ctypes.c_int32)]


class MinresInfo(ctypes.Structure):
    """iga_minres_info: iterations, convergence flag, |r|/|r_0| and |r_0| of iga_kkt_minres."""
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32), ("relres", ctypes.c_double),
                ("res0", ctypes.c_double)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_lib.iga_last_error.restype = ctypes.c_char_p
_lib.iga_version.restype = ctypes.c_char_p
_lib.iga_quad_nodes.argtypes = [ctypes.POINTER(_Space), ctypes.c_int32, _D, ctypes.POINTER(ctypes.c_int64)]
_lib.iga_lr_assemble_factors.argtypes = [ctypes.POINTER(_Space), ctypes.POINTER(_Sep),
                                         ctypes.POINTER(ctypes.POINTER(_Sep)), ctypes.c_uint32, _P,
                                         ctypes.POINTER(_P)]
_lib.iga_lr_destroy.argtypes = [_P]
_lib.iga_lr_destroy.restype = None
_lib.iga_lr_apply.argtypes = [_P, _P, _P, _P, ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_uint32, _P]
_lib.iga_lr_apply2.argtypes = [_P, _P, _P, _P, ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_uint32,
                               _P]
_lib.iga_kkt_apply.argtypes = [_P, ctypes.c_int32, ctypes.c_double, ctypes.c_double, _P, _P, ctypes.c_uint32, _P]
_lib.iga_lr_apply_host.argtypes = [_P, _P, _P, _P, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                   ctypes.c_uint32, _P]
_lib.iga_kkt_apply_host.argtypes = [_P, ctypes.c_int32, ctypes.c_double, ctypes.c_double, _P, _P, ctypes.c_uint32,
                                    _P]
_lib.iga_lr_info.argtypes = [_P, ctypes.POINTER(_Info)]
_lib.iga_kkt_minres.argtypes = [_P, _P, ctypes.c_int32, ctypes.c_double, ctypes.c_double, _P, _P, ctypes.c_double,
                                ctypes.c_int32, ctypes.c_uint32, _P, ctypes.POINTER(MinresInfo)]
_lib.iga_kkt_prec_create.argtypes = [_P, ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_uint32, _P,
                                     ctypes.POINTER(_P)]
_lib.iga_kkt_prec_destroy.argtypes = [_P]
_lib.iga_kkt_prec_destroy.restype = None
_lib.iga_kkt_prec_apply.argtypes = [_P, _P, _P, _P]
_lib.iga_kkt_prec_info.argtypes = [_P, _D, _D, _D]
_lib.iga_greville.argtypes = [ctypes.POINTER(_Dir), _D]
_lib.iga_weight_lowrank.argtypes = [ctypes.POINTER(_Space), ctypes.POINTER(_Dir), _D, ctypes.c_double, ctypes.c_int32,
                                    ctypes.POINTER(_P)]
_lib.iga_weight_lowrank_sep.argtypes = [_P, ctypes.POINTER(_Sep), ctypes.POINTER(ctypes.c_int32),
                                        ctypes.POINTER(ctypes.c_double)]
_lib.iga_weight_lowrank_free.argtypes = [_P]
_lib.iga_weight_lowrank_free.restype = None
_I32P = ctypes.POINTER(ctypes.c_int32)
_lib.iga_lr_terms.argtypes = [_P, ctypes.c_int32, _I32P, _I32P, _D]
_lib.iga_tt_kron_apply.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P]
_lib.iga_tt_interfaces.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P,
                                   _P, _P, _P]
_lib.iga_tt_local_apply.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P,
                                    _P, _P]
_lib.iga_lr_test_knobs.argtypes = [_P, ctypes.POINTER(_Knobs)]
_lib.iga_lr_test_tile.argtypes = [_P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                  ctypes.POINTER(ctypes.c_int32)]
_lib.iga_lr_export_factor.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, _D, ctypes.POINTER(ctypes.c_int32),
                                      ctypes.POINTER(ctypes.c_int32)]


def lib() -> ctypes.CDLL:
    return _lib


def version() -> str:
    return _lib.iga_version().decode()


def _check(rc: int):
    if rc != IGA_OK:
        raise IgaError(rc, _lib.iga_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _space(knots: Sequence[np.ndarray], p: Sequence[int], nq: int):
    ks = [np.ascontiguousarray(k, dtype=np.float64) for k in knots]
    sp = _Space()
    for d in range(3):
        sp.dir[d].p = int(p[d])
        sp.dir[d].n = int(len(ks[d]) - int(p[d]) - 1)
        sp.dir[d].knots = _dptr(ks[d])
    sp.nq = int(nq)
    return sp, ks


def quad_nodes(knots: Sequence[np.ndarray], p: Sequence[int], nq: int = 0) -> List[np.ndarray]:
    """Quadrature nodes of each direction (iga_quad_nodes): where weight tables are sampled."""
    sp, keep = _space(knots, p, nq)
    out = []
    for d in range(3):
        cnt = ctypes.c_int64(0)
        _check(_lib.iga_quad_nodes(ctypes.byref(sp), d, None, ctypes.byref(cnt)))
        buf = np.zeros(cnt.value)
        _check(_lib.iga_quad_nodes(ctypes.byref(sp), d, _dptr(buf), ctypes.byref(cnt)))
        out.append(buf)
    return out


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _tensor_ptr(t, name: str, numel: Optional[int] = None, device: Optional[int] = None) -> int:
    """data_ptr of a contiguous float64 CUDA tensor holding at least `numel` elements (the extent
    the library will touch) on CUDA device `device`; ValueError otherwise (an undersized buffer
    would be written out of bounds by the kernels)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("%s must be a torch.Tensor" % name)
    if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
        raise ValueError("%s must be a contiguous float64 CUDA tensor" % name)
    if numel is not None and t.numel() < numel:
        raise ValueError("%s has %d elements, the call touches %d" % (name, t.numel(), numel))
    if device is not None and t.device.index != device:
        raise ValueError("%s is on cuda:%s, the op on cuda:%d" % (name, t.device.index, device))
    return t.data_ptr()


def _host_buf(a: Optional[np.ndarray], name: str, numel: int):
    if a is None:
        return None
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("%s must be a C-contiguous float64 numpy array" % name)
    if a.size < numel:
        raise ValueError("%s has %d elements, the call touches %d" % (name, a.size, numel))
    return a.ctypes.data


def greville(knots: np.ndarray, p: int) -> np.ndarray:
    """Greville abscissae of one univariate space (iga_greville)."""
    k = np.ascontiguousarray(knots, dtype=np.float64)
    d = _Dir()
    d.p, d.n, d.knots = int(p), int(len(k) - p - 1), _dptr(k)
    out = np.zeros(d.n)
    _check(_lib.iga_greville(ctypes.byref(d), _dptr(out)))
    return out


def weight_lowrank(target_knots: Sequence[np.ndarray], target_p: Sequence[int], tilde_knots: Sequence[np.ndarray],
                   tilde_p: Sequence[int], samples: np.ndarray, eps: float = 1e-10, max_terms: int = 64,
                   nq: int = 0):
    """Rank-R separable weight from samples at the Greville points of S~ (iga_weight_lowrank,
    NEXT-2).  samples: [n~z, n~y, n~x].  Returns (SepWeight tabulated at the target's
    quadrature nodes, (R1, R2) TT ranks, relative TT truncation error of the samples)."""
    sp, keep = _space(target_knots, target_p, nq)
    tk = [np.ascontiguousarray(k, dtype=np.float64) for k in tilde_knots]
    td = (_Dir * 3)()
    for d in range(3):
        td[d].p, td[d].n, td[d].knots = int(tilde_p[d]), int(len(tk[d]) - int(tilde_p[d]) - 1), _dptr(tk[d])
    smp = np.ascontiguousarray(samples, dtype=np.float64)
    if smp.shape != (td[2].n, td[1].n, td[0].n):
        raise ValueError("samples must be [n~z, n~y, n~x]")
    h = _P()
    _check(_lib.iga_weight_lowrank(ctypes.byref(sp), td, _dptr(smp), float(eps), int(max_terms), ctypes.byref(h)))
    try:
        sep = _Sep()
        ranks = (ctypes.c_int32 * 2)()
        err = ctypes.c_double()
        _check(_lib.iga_weight_lowrank_sep(h, ctypes.byref(sep), ranks, ctypes.byref(err)))
        nodes = quad_nodes(target_knots, target_p, nq)
        R = int(sep.R)
        tabs = [np.ctypeslib.as_array(sep.tab[d], shape=(R * len(nodes[d]),)).reshape(R, len(nodes[d])).copy()
                for d in range(3)]
        coef = np.ctypeslib.as_array(sep.coef, shape=(R,)).copy()
        return SepWeight(coef, tabs), (int(ranks[0]), int(ranks[1])), float(err.value)
    finally:
        _lib.iga_weight_lowrank_free(h)


class SepWeight:
    """Rank-R separable weight tabulated at the quadrature nodes (iga_sep):
    f(x,y,z) = sum_r coef[r] tab[0][r](x) tab[1][r](y) tab[2][r](z)."""

    def __init__(self, coef: Optional[np.ndarray], tabs: Sequence[np.ndarray]):
        self.tabs = [np.ascontiguousarray(t, dtype=np.float64) for t in tabs]
        self.R = int(self.tabs[0].shape[0])
        self.coef = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)

    def _c(self) -> _Sep:
        s = _Sep()
        s.R = self.R
        s.coef = _dptr(self.coef) if self.coef is not None else ctypes.POINTER(ctypes.c_double)()
        for d in range(3):
            s.tab[d] = _dptr(self.tabs[d])
        return s


class LowRankOperator:
    """Mass and stiffness operators in low-rank Kronecker form on one GPU (iga_lr_op)."""

    def __init__(self, knots: Sequence[np.ndarray], p: Sequence[int], omega: Optional[SepWeight],
                 q: Optional[Sequence[Optional[SepWeight]]], nq: int = 0, dirichlet: bool = False, stream=None):
        self._h = None
        sp, keep = _space(knots, p, nq)
        om = omega._c() if omega is not None else None
        qarr = None
        keep_q = []
        if q is not None:
            assert len(q) == 9
            qarr = (ctypes.POINTER(_Sep) * 9)()
            for b in range(9):
                if q[b] is not None:
                    s = q[b]._c()
                    keep_q.append(s)
                    qarr[b] = ctypes.pointer(s)
        h = _P()
        _check(_lib.iga_lr_assemble_factors(ctypes.byref(sp), ctypes.byref(om) if om is not None else None,
                                            qarr, IGA_DIRICHLET if dirichlet else 0, _stream_handle(stream),
                                            ctypes.byref(h)))
        self._h = h
        self.info = self._info()
        self.dims = tuple(int(v) for v in self.info.dims)  # (mx, my, mz)
        import torch
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.iga_lr_destroy(self._h)
            self._h = None

    def _info(self) -> _Info:
        inf = _Info()
        _check(_lib.iga_lr_info(self._h, ctypes.byref(inf)))
        return inf

    @property
    def ndof(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def info_dict(self) -> dict:
        i = self.info
        return {"dims": list(i.dims), "p": list(i.p), "nq": i.nq, "n_factors": list(i.n_factors),
                "n_rounds": i.n_rounds, "n_xprod": i.n_xprod, "n_yprod": i.n_yprod, "n_zprod": i.n_zprod,
                "has_mass": bool(i.has_mass), "has_stiff": bool(i.has_stiff), "fused_ok": bool(i.fused_ok), "fused2_ok": bool(i.fused2_ok),
                "plan_flops_per_vec": i.plan_flops_per_vec, "min_bytes_per_vec": i.min_bytes_per_vec,
                "plan_flops_mass": i.plan_flops_mass, "plan_flops_stiff": i.plan_flops_stiff,
                "canon_mass": bool(i.canon_mass), "canon_stiff": bool(i.canon_stiff),
                "stiff_symmetric": bool(i.stiff_symmetric), "f2_rounds_stiff": int(i.f2_rounds_stiff)}

    def _test_knobs(self, force_generic: bool = False, qx: int = 0, minlen: int = 0, no_yres: bool = False,
                    no_tma: bool = False, vpack: int = 0):
        """TEST-ONLY: override this op's kernel selection (iga_lr_test_knobs); all defaults
        restore the product's own choices."""
        k = _Knobs(int(bool(force_generic)), int(qx), int(minlen), int(bool(no_yres)), int(bool(no_tma)),
                   int(vpack))
        _check(_lib.iga_lr_test_knobs(self._h, ctypes.byref(k)))
        self.info = self._info()

    def _test_tile(self, batch: int) -> Tuple[int, int, int]:
        """TEST-ONLY: the canonical tile (qx, lw, vp) for a launch over `batch` vectors."""
        q, lw, vp = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.iga_lr_test_tile(self._h, int(batch), ctypes.byref(q), ctypes.byref(lw), ctypes.byref(vp)))
        return q.value, lw.value, vp.value

    def export_factor(self, d: int, fid: int) -> Tuple[np.ndarray, int, int]:
        m = self.dims[d]
        bw = 2 * self.info.p[d] + 1
        band = np.zeros((m, bw))
        pat = ctypes.c_int32(0)
        tab = ctypes.c_int32(0)
        _check(_lib.iga_lr_export_factor(self._h, d, fid, _dptr(band), ctypes.byref(pat), ctypes.byref(tab)))
        return band, pat.value, tab.value

    # ------------------------------------------------------------------ TT (NEXT-3)
    def terms(self, part: int) -> Tuple[np.ndarray, np.ndarray]:
        """The op's Kronecker terms of `part` (0 mass, 1 stiffness): fid [T, 3] (x, y, z factor
        ids, see export_factor) and coef [T] (iga_lr_terms)."""
        T = ctypes.c_int32(0)
        _check(_lib.iga_lr_terms(self._h, int(part), ctypes.byref(T), None, None))
        fid = np.zeros((T.value, 3), dtype=np.int32)
        coef = np.zeros(T.value)
        _check(_lib.iga_lr_terms(self._h, int(part), ctypes.byref(T), fid.ctypes.data_as(_I32P), _dptr(coef)))
        return fid, coef

    def tt_kron_apply(self, part: int, gz, gy, gx, wz, wy, wx, stream=None):
        """A v for a TT vector v with device cores gz [mz, R1], gy [R1, my, R2], gx [R2, mx]:
        per-term cores wz [T, mz, R1] (coefficient folded in), wy [T, R1, my, R2], wx [T, R2, mx]
        (iga_tt_kron_apply)."""
        R1, R2 = int(gy.shape[0]), int(gy.shape[2])
        mx, my, mz = self.dims
        T = len(self.terms(part)[1])
        _check(_lib.iga_tt_kron_apply(self._h, int(part), R1, R2, self._t(gz, "gz", mz * R1),
                                      self._t(gy, "gy", R1 * my * R2), self._t(gx, "gx", R2 * mx),
                                      self._t(wz, "wz", T * mz * R1), self._t(wy, "wy", T * R1 * my * R2),
                                      self._t(wx, "wx", T * R2 * mx), _stream_handle(stream)))

    def tt_interfaces(self, part: int, site: int, gz, gy, gx, L, R, stream=None):
        """Frame interfaces of `site` (0 x, 1 y, 2 z) for every term: L [T, Rl, Rl], R [T, Rr, Rr]
        (iga_tt_interfaces)."""
        R1, R2 = int(gy.shape[0]), int(gy.shape[2])
        mx, my, mz = self.dims
        T = len(self.terms(part)[1])
        Rl = (1, R1, R2)[2 - int(site)] if int(site) in (0, 1, 2) else 1
        Rr = (R1, R2, 1)[2 - int(site)] if int(site) in (0, 1, 2) else 1
        _check(_lib.iga_tt_interfaces(self._h, int(part), int(site), R1, R2, self._t(gz, "gz", mz * R1),
                                      self._t(gy, "gy", R1 * my * R2), self._t(gx, "gx", R2 * mx),
                                      self._t(L, "L", T * Rl * Rl), self._t(R, "R", T * Rr * Rr),
                                      _stream_handle(stream)))

    def tt_local_apply(self, part: int, site: int, L, R, x, y, stream=None):
        """y = (sum_t c_t L_t (x) A_t^(site) (x) R_t) x for local cores x, y [Rl, m_site, Rr]
        (iga_tt_local_apply)."""
        Rl, Rr = int(x.shape[0]), int(x.shape[2])
        T = len(self.terms(part)[1])
        m = self.dims[int(site)] if int(site) in (0, 1, 2) else 0
        _check(_lib.iga_tt_local_apply(self._h, int(part), int(site), Rl, Rr, self._t(L, "L", T * Rl * Rl),
                                       self._t(R, "R", T * Rr * Rr), self._t(x, "x", Rl * m * Rr),
                                       self._t(y, "y", Rl * m * Rr), _stream_handle(stream)))

    # ------------------------------------------------------------------ device applies
    def _batch(self, ref, batch: Optional[int]) -> int:
        if batch is not None:
            return int(batch)
        if ref.numel() % self.ndof:
            raise ValueError("tensor of %d elements is not a batch of %d-DoF vectors" % (ref.numel(), self.ndof))
        return ref.numel() // self.ndof

    def _t(self, t, name, numel):
        return _tensor_ptr(t, name, numel, self.device) if t is not None else None

    def apply(self, x, y_mass=None, y_stiff=None, alpha: float = 1.0, gamma: float = 1.0, path: str = "auto",
              stream=None, batch: Optional[int] = None):
        """y_mass = alpha M x, y_stiff = gamma S x on device tensors [batch, nz, ny, nx]."""
        b = self._batch(x, batch)
        n = b * self.ndof
        _check(_lib.iga_lr_apply(self._h, self._t(x, "x", n), self._t(y_mass, "y_mass", n),
                                 self._t(y_stiff, "y_stiff", n), float(alpha), float(gamma), int(b), PATHS[path],
                                 _stream_handle(stream)))

    def apply2(self, x_mass, x_stiff, out, alpha: float = 1.0, gamma: float = 1.0, path: str = "auto",
               stream=None, batch: Optional[int] = None):
        ref = x_mass if x_mass is not None else x_stiff
        b = self._batch(ref, batch)
        n = b * self.ndof
        _check(_lib.iga_lr_apply2(self._h, self._t(x_mass, "x_mass", n), self._t(x_stiff, "x_stiff", n),
                                  self._t(out, "out", n), float(alpha), float(gamma), int(b), PATHS[path],
                                  _stream_handle(stream)))

    def kkt_apply(self, X, out, n_t: int, tau: float, beta: float, path: str = "auto", stream=None):
        """out = KKT(tau, beta, n_t) X for device tensors [3, n_t, nz, ny, nx] (Eq. (KKTSystem))."""
        n = 3 * int(n_t) * self.ndof
        _check(_lib.iga_kkt_apply(self._h, int(n_t), float(tau), float(beta), self._t(X, "X", n),
                                  self._t(out, "out", n), PATHS[path], _stream_handle(stream)))

    def kkt_minres(self, rhs, x, n_t: int, tau: float, beta: float, rtol: float = 1e-8, maxit: int = 1000,
                   x0: bool = False, prec: "Optional[KKTPreconditioner]" = None, path: str = "auto",
                   stream=None) -> MinresInfo:
        """MINRES solve of KKT(tau, beta, n_t) x = rhs (device tensors [3, n_t, nz, ny, nx]);
        x holds the initial guess when x0 is True; prec: a KKTPreconditioner built for the same
        (n_t, tau, beta) or None.  Returns the iga_minres_info record."""
        info = MinresInfo()
        flags = PATHS[path] | (MINRES_X0 if x0 else 0)
        n = 3 * int(n_t) * self.ndof
        _check(_lib.iga_kkt_minres(self._h, prec._h if prec is not None else None, int(n_t), float(tau), float(beta),
                                   self._t(rhs, "rhs", n), self._t(x, "x", n), float(rtol), int(maxit), flags,
                                   _stream_handle(stream), ctypes.byref(info)))
        return info

    def kkt_preconditioner(self, n_t: int, tau: float, beta: float, path: str = "auto",
                           stream=None) -> "KKTPreconditioner":
        return KKTPreconditioner(self, n_t, tau, beta, path, stream)

    # ------------------------------------------------------------------ host (end-to-end) applies
    def apply_host(self, x: np.ndarray, y_mass: Optional[np.ndarray], y_stiff: Optional[np.ndarray],
                   alpha: float = 1.0, gamma: float = 1.0, path: str = "auto", stream=None):
        if not isinstance(x, np.ndarray) or x.size % self.ndof or x.size == 0:
            raise ValueError("x must hold a whole batch of %d-DoF vectors" % self.ndof)
        n = x.size
        b = n // self.ndof
        _check(_lib.iga_lr_apply_host(self._h, _host_buf(x, "x", n), _host_buf(y_mass, "y_mass", n),
                                      _host_buf(y_stiff, "y_stiff", n), float(alpha), float(gamma), int(b),
                                      PATHS[path], _stream_handle(stream)))

    def kkt_apply_host(self, X: np.ndarray, out: np.ndarray, n_t: int, tau: float, beta: float,
                       path: str = "auto", stream=None):
        n = 3 * int(n_t) * self.ndof
        _check(_lib.iga_kkt_apply_host(self._h, int(n_t), float(tau), float(beta), _host_buf(X, "X", n),
                                       _host_buf(out, "out", n), PATHS[path], _stream_handle(stream)))


class KKTPreconditioner:
    """Block-diagonal KKT preconditioner (iga_kkt_prec_*): blkdiag(tau Mh, tau beta Mh, Sh) with
    Kronecker fast-diagonalisation solves (include/iga_lr.h)."""

    def __init__(self, op: "LowRankOperator", n_t: int, tau: float, beta: float, path: str = "auto", stream=None):
        h = _P()
        _check(_lib.iga_kkt_prec_create(op._h, int(n_t), float(tau), float(beta), PATHS[path],
                                        _stream_handle(stream), ctypes.byref(h)))
        self._h = h.value
        self._op = op  # keeps the op (and its device) alive
        self.n_t, self.tau, self.beta = int(n_t), float(tau), float(beta)
        self.dims = op.dims

    def apply(self, r, out, stream=None):
        """out = P^{-1} r for device tensors [3, n_t, nz, ny, nx]."""
        n = 3 * self.n_t * self.dims[0] * self.dims[1] * self.dims[2]
        dev = self._op.device
        _check(_lib.iga_kkt_prec_apply(self._h, _tensor_ptr(r, "r", n, dev), _tensor_ptr(out, "out", n, dev),
                                       _stream_handle(stream)))

    def info(self):
        mb, sb = ctypes.c_double(), ctypes.c_double()
        lam = np.empty(sum(self.dims), dtype=np.float64)
        _check(_lib.iga_kkt_prec_info(self._h, ctypes.byref(mb), ctypes.byref(sb),
                                      lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        nx, ny, nz = self.dims
        return mb.value, sb.value, (lam[:nx], lam[nx:nx + ny], lam[nx + ny:])

    def close(self):
        if getattr(self, "_h", None):
            _lib.iga_kkt_prec_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
