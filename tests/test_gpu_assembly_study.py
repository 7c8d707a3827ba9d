"""NEXT-4: the paper's assembly study on the extruded quarter annulus.

The low-rank route (geometry weights sampled at Greville points of a degree-(2p+1) space,
TT-SVD + collocation, GPU univariate factors) against the oracle's full 3D quadrature assembly
with the exact geometry weights, 5-point Gauss rule in both.  What the mathematics fixes:

  * omega = |det grad G| is linear in s and every Q entry is a function of s alone: TT ranks 1;
  * omega (and q11, q33, multiples of omega) lie in the interpolation space, so M~ = M and the
    (1,1), (3,3) stiffness blocks are exact to rounding;
  * q22 ~ 1/r(s) is interpolated with error O(h^(2p+2)): diff_S is small and falls with h.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def study():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import study_assembly
    from synth.geometry import QuarterAnnulus
    levels = [int(v) for v in os.environ.get("IGALR_STUDY_LEVELS", "1,5").split(",")]
    p = int(os.environ.get("IGALR_STUDY_P", "2"))
    res = [study_assembly.level(p, s, QuarterAnnulus()) for s in levels]
    out = os.environ.get("IGALR_STUDY_OUT")
    if out:
        print(study_assembly.write(res, out, p))
    return res


def test_ranks_are_one(study):
    for r in study:
        assert r["ranks"]["omega"] == (1, 1)
        for k in ("q11", "q22", "q33"):
            assert r["ranks"][k] == (1, 1), (k, r["ranks"][k])


def test_mass_exact_stiffness_close(study):
    for r in study:
        assert r["probe_err"] <= 1e-13
        assert r["diff_M"] <= 1e-13, r
        assert r["diff_S"] <= 1e-3, r
    d = [r["diff_S"] for r in study]
    assert all(b < a for a, b in zip(d, d[1:])), d  # refinement reduces the interpolation error


def test_storage_advantage_grows(study):
    s = [r["storage_ratio"] for r in study]
    assert all(b > a for a, b in zip(s, s[1:])), s
