"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the GPU
path (``paper_1811_06797_b200``).  It holds no arithmetic of the method (no
quadrature, no basis functions, no operator application): only the problem
*definition* — knot vectors, the closed-form separable weight functions and the
random draws — exactly as DESIGN.md §3 ("input recipe") states them.

Readings (listed again in DESIGN.md):
  G6  stiffness weight Q(x) = sum_r v_r(x) A_r, A_r seeded SPD 3x3.
  G7  each univariate weight factor is 1 + 0.5 sin(k pi t + phi), k in {1..4},
      phi in [0, 2 pi), one independent (k, phi) per (operator, r, direction).
  G8  numpy Generator(PCG64(181106797 + config_index)); draw order: mass (r, d:
      k then phi), stiffness (r, d: k then phi), A_r (diagonal, then upper
      off-diagonal row-major), then the input vectors (standard normal, C order).
  G15 uniform open knots, interior knot i/(n-p) computed directly.

A weight "term" is a row of 10 doubles
    [coef, amp_x, k_x, phi_x, amp_y, k_y, phi_y, amp_z, k_z, phi_z]
meaning coef * prod_{d in x,y,z} (1 + amp_d sin(k_d pi t_d + phi_d)).
Directions are ordered x (fastest, contiguous), y, z (slowest); arrays are
C-ordered [..., z, y, x].
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np

SEED_BASE = 181106797
TERM_WIDTH = 10


@dataclasses.dataclass(frozen=True)
class Config:
    index: int            # 1-based, as in BASELINE.json "configs"
    name: str
    n: int                # basis functions per direction
    p: int                # spline degree
    R: int                # separable rank of omega and of every q_kl
    batch: int            # number of input vectors (apply) / 1 for KKT
    constant_weight: bool = False  # config 1: w == 1, Q == I
    dirichlet: bool = False
    n_t: int = 0          # KKT time steps (0 => plain mass+stiffness apply)
    tau: float = 0.0
    beta: float = 0.0

    @property
    def kkt(self) -> bool:
        return self.n_t > 0

    @property
    def dims(self):
        """DoF extents (nx, ny, nz) after optional Dirichlet elimination."""
        m = self.n - 2 if self.dirichlet else self.n
        return (m, m, m)

    @property
    def ndof(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz


CONFIGS: Dict[str, Config] = {
    "c1": Config(1, "c1_unit_cube_p2_n8", n=8, p=2, R=1, batch=4, constant_weight=True),
    "c2": Config(2, "c2_p3_n64_R4", n=64, p=3, R=4, batch=1),
    "c3": Config(3, "c3_p3_n128_R8_B8", n=128, p=3, R=8, batch=8),
    "c4": Config(4, "c4_kkt_p3_n48_R4_nt64", n=48, p=3, R=4, batch=1, dirichlet=True,
                 n_t=64, tau=1.0 / 64.0, beta=1e-4),
    "c5": Config(5, "c5_p4_n256_R6", n=256, p=4, R=6, batch=1),
}


def scaled(cfg: Config, n: int, batch: Optional[int] = None, n_t: Optional[int] = None) -> Config:
    """Same weight recipe / degree / rank at another mesh size (parity-test cases)."""
    return dataclasses.replace(cfg, n=n, batch=cfg.batch if batch is None else batch,
                               n_t=cfg.n_t if n_t is None else n_t)


def uniform_open_knots(n: int, p: int) -> np.ndarray:
    """Open uniform knot vector of Eq. (knotVector), G15."""
    if n < p + 1:
        raise ValueError("need n >= p+1")
    ne = n - p
    inner = [i / ne for i in range(1, ne)]
    return np.array([0.0] * (p + 1) + inner + [1.0] * (p + 1), dtype=np.float64)


def weight_factor(t, amp: float, k: float, phi: float):
    """Closed-form univariate weight factor 1 + amp*sin(k*pi*t + phi) (G7)."""
    return 1.0 + amp * np.sin(k * math.pi * np.asarray(t, dtype=np.float64) + phi)


@dataclasses.dataclass
class Weights:
    """Separable weights of one configuration.

    mass:  [R, 10] terms of omega.
    v:     [R, 3, 3] (amp, k, phi) per direction of the stiffness factors v_r.
    A:     [R, 3, 3] symmetric coefficient matrices A_r  (Q = sum_r v_r A_r).
    """
    mass: np.ndarray
    v: np.ndarray
    A: np.ndarray

    def q_block_terms(self) -> List[np.ndarray]:
        """The 9 blocks q_kl (k = row-major index over x,y,z) as term arrays.

        Reading A of G6: every block shares the same factor tables v_r and
        carries coef (A_r)_kl.  Blocks whose coefficients are all zero are
        returned as empty arrays (absent block)."""
        R = self.v.shape[0]
        out = []
        for k in range(3):
            for l in range(3):
                rows = []
                for r in range(R):
                    c = float(self.A[r, k, l])
                    if c == 0.0:
                        continue
                    rows.append([c] + list(self.v[r].reshape(-1)))
                out.append(np.array(rows, dtype=np.float64).reshape(-1, TERM_WIDTH))
        return out


def _rng(cfg: Config) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + cfg.index))


def draw_weights(cfg: Config, rng: Optional[np.random.Generator] = None) -> Weights:
    """Draw the seeded weights of ``cfg`` (G6-G8).  Consumes rng in G8 order."""
    R = cfg.R
    if cfg.constant_weight:
        mass = np.zeros((R, TERM_WIDTH))
        mass[:, 0] = 1.0 / R
        mass[:, 2::3] = 1.0  # k (unused, amp = 0)
        v = np.zeros((R, 3, 3))
        v[:, :, 1] = 1.0
        A = np.zeros((R, 3, 3))
        for r in range(R):
            A[r] = np.eye(3) / R
        return Weights(mass=mass, v=v, A=A)
    if rng is None:
        rng = _rng(cfg)
    mass = np.zeros((R, TERM_WIDTH))
    for r in range(R):
        mass[r, 0] = 1.0
        for d in range(3):
            kk = int(rng.integers(1, 5))
            ph = float(rng.uniform(0.0, 2.0 * math.pi))
            mass[r, 1 + 3 * d:4 + 3 * d] = (0.5, kk, ph)
    v = np.zeros((R, 3, 3))
    for r in range(R):
        for d in range(3):
            kk = int(rng.integers(1, 5))
            ph = float(rng.uniform(0.0, 2.0 * math.pi))
            v[r, d] = (0.5, kk, ph)
    A = np.zeros((R, 3, 3))
    for r in range(R):
        for d in range(3):
            A[r, d, d] = rng.uniform(1.0, 2.0)
        for k in range(3):
            for l in range(k + 1, 3):
                val = rng.uniform(-0.4, 0.4)
                A[r, k, l] = val
                A[r, l, k] = val
    return Weights(mass=mass, v=v, A=A)


def draw_problem(cfg: Config):
    """(knots[3], weights, x) for ``cfg`` with the G8 draw order.

    x has shape [batch, nz, ny, nx] (apply) or [3, n_t, nz, ny, nx] (KKT,
    blocks y, u, lambda), interior extents when cfg.dirichlet."""
    rng = _rng(cfg)
    w = draw_weights(cfg, rng)
    nx, ny, nz = cfg.dims
    if cfg.kkt:
        x = rng.standard_normal((3, cfg.n_t, nz, ny, nx))
    else:
        x = rng.standard_normal((cfg.batch, nz, ny, nx))
    knots = [uniform_open_knots(cfg.n, cfg.p) for _ in range(3)]
    return knots, w, x


def tabulate(terms: np.ndarray, nodes: List[np.ndarray]) -> List[np.ndarray]:
    """Tabulate each term's univariate factors at given per-direction points.

    Returns tab[d] of shape [nterms, len(nodes[d])]; the term's coef is NOT
    folded in.  This is evaluation of the input definition only."""
    tabs = []
    for d in range(3):
        t = np.empty((terms.shape[0], len(nodes[d])))
        for r in range(terms.shape[0]):
            amp, k, ph = terms[r, 1 + 3 * d:4 + 3 * d]
            t[r] = weight_factor(nodes[d], amp, k, ph)
        tabs.append(t)
    return tabs
