"""Operators for the BASELINE.json workloads (used by bench.py, smoke() and the GPU tests).

Builds a ``LowRankOperator`` from a ``synth`` configuration: uniform open knots, the seeded
separable weights tabulated at the library's own quadrature nodes (``iga_quad_nodes``), and
reading A of G6 for the stiffness blocks (q_kl = sum_r (A_r)_kl v_r, all nine blocks sharing
the v_r tables).  ``synth`` holds only the input definition; everything the
method computes happens in libigalr.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

import synth
from . import LowRankOperator, SepWeight, quad_nodes


def build_operator(cfg: synth.Config, weights: synth.Weights, n: Optional[int] = None, nq: int = 0,
                   mass: bool = True, stiff: bool = True, dirichlet: Optional[bool] = None,
                   knots=None, stream=None) -> LowRankOperator:
    nn = cfg.n if n is None else n
    if knots is None:
        knots = [synth.uniform_open_knots(nn, cfg.p) for _ in range(3)]
    p = [cfg.p] * 3
    nodes = quad_nodes(knots, p, nq)
    omega = None
    if mass:
        omega = SepWeight(weights.mass[:, 0], synth.tabulate(weights.mass, nodes))
    q = None
    if stiff:
        R = weights.v.shape[0]
        vterms = np.zeros((R, synth.TERM_WIDTH))
        vterms[:, 0] = 1.0
        vterms[:, 1:] = weights.v.reshape(R, 9)
        vt = synth.tabulate(vterms, nodes)
        q = []
        for k in range(3):
            for l in range(3):
                c = weights.A[:, k, l]
                q.append(SepWeight(c, vt) if np.any(c != 0.0) else None)
    return LowRankOperator(knots, p, omega, q, nq=nq, dirichlet=cfg.dirichlet if dirichlet is None else dirichlet,
                           stream=stream)
