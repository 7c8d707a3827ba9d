"""Analytic geometries for the weight-from-geometry workloads (NEXT-2 / NEXT-4).

Problem definitions only, like the rest of ``synth``: a map G from the parameter cube [0,1]^3
to the physical domain and the two weight fields the paper derives from it (PAPER.md:120-143,
Eqs. (massMatrix)/(stiffnessMatrix) after the change of variables):

    omega(x) = |det grad G(x)|,        Q(x) = omega(x) (grad G(x))^{-1} (grad G(x))^{-T}.

No basis functions, quadrature or low-rank arithmetic lives here.  Point sets (Greville points,
quadrature nodes) are passed in by the caller.

The quarter annulus extruded in z is the paper's rank-1 domain:
    G(s, t, u) = (r(s) cos(pi t / 2), r(s) sin(pi t / 2), h u),  r(s) = r0 + (r1 - r0) s.
Then grad G = R(t) diag(r1 - r0, r(s) pi / 2, h) with a rotation R(t), so
    omega = (r1 - r0) (pi / 2) r(s) h,
    Q = diag(omega / (r1 - r0)^2, omega / (r(s) pi / 2)^2, omega / h^2),
each a function of s alone times constants (TT rank 1).  omega is degree 1 in s; Q_22 is
proportional to 1 / r(s), not a polynomial, so its spline interpolation is inexact.
"""
from __future__ import annotations

import math
from typing import Sequence, Tuple

import numpy as np


class QuarterAnnulus:
    """Extruded quarter annulus: radii r0 < r1, height h."""

    def __init__(self, r0: float = 1.0, r1: float = 2.0, h: float = 0.5):
        self.r0, self.r1, self.h = float(r0), float(r1), float(h)

    @property
    def volume(self) -> float:
        return (math.pi / 4.0) * (self.r1 ** 2 - self.r0 ** 2) * self.h

    def fields(self, x: np.ndarray, y: np.ndarray, z: np.ndarray) -> np.ndarray:
        """omega and the 9 entries of Q on the tensor grid of the 1D point sets x (s, fastest),
        y (t), z (u): array [10, len(z), len(y), len(x)], index 0 = omega, 1 + k*3 + l = Q_kl."""
        s = np.asarray(x, dtype=np.float64)[None, None, :]
        r = self.r0 + (self.r1 - self.r0) * s
        shape = (len(z), len(y), len(x))
        om = np.broadcast_to((self.r1 - self.r0) * (math.pi / 2.0) * r * self.h, shape)
        out = np.zeros((10,) + shape)
        out[0] = om
        out[1 + 0] = om / (self.r1 - self.r0) ** 2
        out[1 + 4] = om / (r * math.pi / 2.0) ** 2
        out[1 + 8] = om / self.h ** 2
        return out


def grid_samples(geom, pts: Sequence[np.ndarray]) -> np.ndarray:
    """The geometry's 10 weight fields on the tensor grid of pts = (x, y, z) point sets."""
    return geom.fields(pts[0], pts[1], pts[2])


def refinement_knots(p: int, spans: int) -> np.ndarray:
    """Open uniform knot vector of degree p with `spans` equal spans (the paper's h-refinement
    inserts 4 knots per knot span per level: spans 1, 5, 25, ...)."""
    inner = [i / spans for i in range(1, spans)]
    return np.array([0.0] * (p + 1) + inner + [1.0] * (p + 1))
