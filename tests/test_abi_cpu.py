"""CPU checks of the C ABI boundary (no GPU): the library loads, exports every symbol that
include/iga_lr.h declares, and its host-only logic (quadrature nodes, validation) behaves."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def igalr():
    from paper_1811_06797_b200 import _build
    _build.build()
    import paper_1811_06797_b200 as m
    return m


def _declared_symbols(header="iga_lr.h"):
    hdr = open(os.path.join(ROOT, "include", header)).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(iga_[a-z0-9_]+)\s*\(", hdr)))


def test_header_symbols_exported(igalr):
    lib = ctypes.CDLL(igalr.LIB_PATH)
    names = _declared_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), "missing export " + n
    assert set(names) == set(igalr.ABI_SYMBOLS)


def test_testing_header_symbols_exported(igalr):
    """include/iga_lr_testing.h (test-only kernel-selection knobs) is exported too, and the
    product binding no longer takes its library path from the environment."""
    lib = ctypes.CDLL(igalr.LIB_PATH)
    names = _declared_symbols("iga_lr_testing.h")
    assert names == ["iga_lr_test_knobs", "iga_lr_test_tile"]
    for n in names:
        assert hasattr(lib, n), "missing export " + n
    assert igalr.LIB_PATH == os.path.join(ROOT, "paper_1811_06797_b200", "libigalr.so")
    src = open(os.path.join(ROOT, "paper_1811_06797_b200", "__init__.py")).read()
    assert "environ" not in src
    # and no kernel-selection environment variable is read anywhere in the library sources
    csrc = os.path.join(ROOT, "paper_1811_06797_b200", "csrc")
    for f in os.listdir(csrc):
        assert "getenv" not in open(os.path.join(csrc, f)).read(), f


def test_version_and_last_error(igalr):
    assert "sm_100a" in igalr.version()
    assert igalr.lib().iga_last_error() == b""


def test_quad_nodes_match_oracle(igalr):
    """Host Gauss rule of the library vs the oracle's (independent implementations)."""
    import oracle
    import synth
    for p, n, nq in [(1, 5, 2), (2, 8, 3), (3, 20, 4), (4, 30, 5), (3, 9, 7)]:
        kn = synth.uniform_open_knots(n, p)
        mine = igalr.quad_nodes([kn] * 3, [p] * 3, nq)
        ref = oracle.quad_nodes(kn, p, nq)
        for d in range(3):
            assert mine[d].shape == ref.shape
            assert np.abs(mine[d] - ref).max() < 4e-16


def test_quad_nodes_nonuniform_repeated(igalr):
    import oracle
    kn = np.array([0, 0, 0, 0.2, 0.5, 0.5, 0.7, 1, 1, 1.0])
    p = 2
    mine = igalr.quad_nodes([kn] * 3, [p] * 3, 0)
    ref = oracle.quad_nodes(kn, p, p + 1)
    assert mine[0].size == 4 * 3  # 4 nonempty spans
    assert np.abs(mine[0] - ref).max() < 4e-16


@pytest.mark.parametrize("bad,code", [
    (dict(knots=[0, 0.1, 0.5, 1, 1]), 1),          # not open
    (dict(knots=[0, 0, 0.6, 0.5, 1, 1]), 1),       # decreasing
    (dict(knots=[0, 0, 1.5, 1, 1]), 1),            # outside [0, 1]
    (dict(p=0, knots=[0, 0.5, 1]), 1),             # p < 1
    (dict(p=9, knots=[0] * 10 + [1] * 10), 4),      # unsupported degree
    (dict(knots=[0, 0, 0, 0.5, 0.5, 0.5, 1, 1, 1], p=2), 1),  # interior multiplicity > p
])
def test_invalid_knots_rejected(igalr, bad, code):
    p = bad.get("p", 1)
    kn = np.array(bad["knots"], dtype=float)
    with pytest.raises(igalr.IgaError) as ei:
        igalr.quad_nodes([kn] * 3, [p] * 3, 0)
    assert ei.value.status == code


def test_nq_out_of_range(igalr):
    import synth
    kn = synth.uniform_open_knots(6, 2)
    with pytest.raises(igalr.IgaError) as ei:
        igalr.quad_nodes([kn] * 3, [2] * 3, 40)
    assert ei.value.status == igalr.IGA_EUNSUPPORTED


def test_product_does_not_import_oracle():
    """The product package never imports the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_1811_06797_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
    osrc = open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert "paper_1811_06797_b200" not in re.sub(r'""".*?"""', "", osrc, flags=re.S)
