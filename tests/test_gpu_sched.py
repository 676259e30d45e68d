"""K4 on the device vs the reference's golden streams, edges and depths
(bit-exact), through the C ABI."""

from __future__ import annotations

import warnings

import numpy as np
import pytest

import paper_1401_4441_b200 as P
from paper_1401_4441_b200 import schedule, taskgen
from conftest import case_id

pytestmark = pytest.mark.gpu


def _order(golden, dim, name):
    return taskgen.StencilOrder(tuple(tuple(o) for o in golden["orders"][str(dim)][name]))


def _grid(case):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return P.GridSpec(tuple(case["extents"]), periodic=case["periodic"])


def test_streams_edges_depths_match_reference(golden, cuda):
    for case in golden["cases"]:
        g = _grid(case)
        for name, ref in case["streams"].items():
            if name == "loopex":
                s = schedule.device_stream(g, "loopex")
            else:
                s = schedule.device_stream(g, "basic", _order(golden, g.dim, name.split(":")[1]))
            assert s.home.cpu().tolist() == ref["home"], (case_id(case), name)
            assert s.nbr.cpu().tolist() == ref["nbr"], (case_id(case), name)
            assert s.entry.cpu().tolist() == ref["entry"], (case_id(case), name)
            eu, ev = s.edge_arrays()
            assert eu.cpu().tolist() == ref["edges_u"], (case_id(case), name)
            assert ev.cpu().tolist() == ref["edges_v"], (case_id(case), name)
            assert s.depth() == ref["depth"], (case_id(case), name)
            if "levels" in ref:
                assert s.levels()[0].cpu().tolist() == ref["levels"]
            # both depth methods agree where both apply
            if name.startswith("basic"):
                assert s.levels("relax")[1] == ref["depth"]


def test_mirror_api_objects(golden, cuda):
    g = P.GridSpec((4, 4, 4))
    tasks = P.generate_loopex(g)
    assert len(tasks) == 896 and [t.id for t in tasks] == list(range(896))
    assert tasks[0].offset is None and tasks[0].kind == "intra"
    assert all(len(t.resources) == 2 for t in tasks if t.kind == "inter")
    graph = P.detect_dependencies(tasks)
    assert graph.edge_count == 1664 and P.critical_path(graph) == 27
    graph = P.detect_dependencies(P.generate_basic(g, P.StencilOrder.canonical(3)))
    assert P.critical_path(graph) == 692
    assert P.critical_path(P.TaskGraph([], ())) == 0
    with pytest.warns(UserWarning):
        P.generate_loopex(P.GridSpec((5, 5, 5)))


def test_depth_at_config_grids(golden, cuda):
    for rec in golden["depths"]:
        s = schedule.device_stream(P.GridSpec(tuple(rec["extents"])), rec["strategy"])
        assert s.ntasks == rec["tasks"]
        assert s.edges()[2] == rec["edges"]
        assert s.depth() == rec["depth"], rec


def test_large_depths(golden_large, cuda):
    for rec in golden_large:
        ext = tuple(rec["extents"])
        strat = rec["strategy"]
        if strat == "stride3":
            s = schedule.device_stream(P.GridSpec(ext), "loopex", stride=3)
        else:
            s = schedule.device_stream(P.GridSpec(ext), strat)
        assert s.ntasks == rec["tasks"]
        assert s.edges()[2] == rec["edges"]
        assert s.depth() == rec["depth"], rec


def test_edges_match_oracle_random_orders(oracle, cuda):
    rng = np.random.default_rng(7)
    base = P.StencilOrder.canonical(3)
    for ext, per in (((6, 4, 8), True), ((5, 3, 4), False), ((4, 4, 4), True)):
        inter = list(base.offsets[1:])
        rng.shuffle(inter)
        order = P.StencilOrder(tuple(inter[:4]) + (base.offsets[0],) + tuple(inter[4:]))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g = P.GridSpec(ext, periodic=per)
        s = schedule.device_stream(g, "basic", order)
        h, nb, e = oracle.stream_basic(ext, per, np.array(order.offsets, np.int8))
        assert np.array_equal(s.home.cpu().numpy(), h)
        eu, ev = oracle.detect_edges_stream(h, nb)
        deu, dev = s.edge_arrays()
        assert np.array_equal(deu.cpu().numpy(), eu) and np.array_equal(dev.cpu().numpy(), ev)
        assert s.depth() == oracle.critical_path(len(h), eu, ev)


def test_plane_ring_depth_matches_relaxation(cuda):
    """The shared-memory plane-ring DP (periodic cell-grouped streams) gives the
    same per-task levels as edge relaxation, incl. plane 0 parked and restored
    (>= 5 planes), 2D grids and orders with the intra task inside."""
    import torch

    rng = np.random.default_rng(11)
    for ext in ((6, 4, 8), (5, 3, 7), (3, 3, 3), (4, 4, 5), (7, 9), (3, 11), (8, 6, 12)):
        base = P.canonical_half_stencil(len(ext)).offsets
        inter = list(base[1:])
        rng.shuffle(inter)
        k = int(rng.integers(0, len(inter) + 1))
        order = P.StencilOrder(tuple(inter[:k]) + (base[0],) + tuple(inter[k:]))
        g = P.GridSpec(ext)
        s = schedule.device_stream(g, "basic", order)
        lc, dc = s.levels("chain")
        lr, dr = s.levels("relax")
        assert dc == dr, ext
        assert torch.equal(lc, lr), ext
