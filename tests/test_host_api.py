"""Host-side mirror API (no GPU): geometry, orders and error behaviour match
the reference (grid.py, taskgen.py) and its golden vectors; the C ABI
library loads and exports every symbol include/cellsched_b200.h declares."""

from __future__ import annotations

import os
import re
import warnings

import pytest

import paper_1401_4441_b200 as P
from paper_1401_4441_b200 import _lib, grid, taskgen
from conftest import ROOT


def test_canonical_stencil_and_orders(golden):
    for dim in (2, 3):
        assert [list(o) for o in grid.canonical_half_stencil(dim).offsets] == golden["canonical_stencil"][str(dim)]
    assert [list(o) for o in taskgen.naive_order().offsets] == golden["orders"]["2"]["naive"]
    assert [list(o) for o in taskgen.bad_order().offsets] == golden["orders"]["2"]["bad"]
    assert [list(o) for o in taskgen.opt_order().offsets] == golden["orders"]["2"]["opt"]
    for d in (1, 2, 14):
        assert [list(o) for o in taskgen.order_with_displacement(3, d).offsets] == golden["orders"]["3"][f"delta{d}"]
    for dim in (2, 3):
        for k, v in golden["displacement"][str(dim)].items():
            order = taskgen.StencilOrder(tuple(tuple(o) for o in golden["orders"][str(dim)][k]))
            assert taskgen.displacement(order) == v


def test_intra_first_orders():
    orders = list(taskgen.intra_first_orders(2))
    assert len(orders) == 24 and len(set(orders)) == 24


def test_gridspec_errors_and_warnings():
    with pytest.raises(ValueError):
        grid.GridSpec((4,))
    with pytest.raises(ValueError):
        grid.GridSpec((4, 0))
    with pytest.warns(UserWarning):
        grid.GridSpec((2, 4))
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        grid.GridSpec((2, 4), periodic=False)
    g = grid.GridSpec((4, 5, 6))
    for c in g.cells():
        assert g.index(g.coords(c)) == c
    assert g.coords(1) == (1, 0, 0)  # x-fastest
    with pytest.raises(ValueError):
        g.coords(120)
    with pytest.raises(ValueError):
        grid.neighbor(0, (2, 0, 0), g)
    with pytest.raises(ValueError):
        grid.neighbor(0, (1, 0), g)
    assert grid.neighbor(0, (-1, 0, 0), g) == 3
    assert grid.neighbor(0, (-1, 0), grid.GridSpec((4, 4), periodic=False)) is None


def test_colors_match_golden(golden):
    for case in golden["cases"]:
        g = grid.GridSpec(tuple(case["extents"]), periodic=case["periodic"])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            assert [grid.color(c, g) for c in g.cells()] == case["colors"]


def test_stencil_validation():
    with pytest.raises(ValueError):
        grid.Stencil(((0, 0), (1, 0), (-1, 0), (0, 1), (1, 1)))
    with pytest.raises(ValueError):
        grid.Stencil(((1, 0),))
    with pytest.raises(ValueError):
        taskgen.StencilOrder(((0, 0), (1, 0)))
    # any valid half-stencil is accepted (taskgen.py:79-83)
    taskgen.StencilOrder(((0, 0),) + grid.FIGURE_HALF_STENCIL_2D)


def test_generate_dispatch_errors():
    with pytest.raises(ValueError):
        taskgen.generate("bogus", grid.GridSpec((4, 4)))
    with pytest.raises(ValueError):
        taskgen.generate_basic(grid.GridSpec((4, 4)), taskgen.StencilOrder.canonical(3))


def test_scalar_payload_helpers(golden):
    # antisymmetry and the golden charges/pair values through the exact-int mirror
    a, b = 12345, -987654
    g1, g2 = P.pair_contribution(a, b, (1, -1, 0))
    assert g1 == -g2
    assert P.pair_contribution(b, a, (-1, 1, 0))[0] == -g1


def _header_symbols():
    path = os.path.join(ROOT, "include", "cellsched_b200.h")
    text = open(path).read()
    return sorted(set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", text)))


def test_abi_exports_every_header_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.EXPORTS)
    assert lib.cs_abi_version() == 1


def test_abi_host_only_calls():
    import ctypes as C

    lib = _lib.load()
    g = grid.GridSpec((4, 4, 4))._cs_grid()
    assert lib.cs_stream_count(C.byref(g), _lib.STREAM_LOOPEX, None, 0, 2) == 896
    g2 = grid.GridSpec((5, 4), periodic=False)._cs_grid()
    order = (C.c_int8 * 10)(*[v for o in taskgen.naive_order().offsets for v in o])
    ref = sum(1 for _ in range(1))  # noqa
    n = lib.cs_stream_count(C.byref(g2), _lib.STREAM_BASIC, order, 5, 2)
    # 20 intra + (0,-1): 5*3 + (1,-1): 4*3 + (1,0): 4*4 + (1,1): 4*3
    assert n == 20 + 15 + 12 + 16 + 12
