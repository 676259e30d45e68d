"""Device list scheduling (schedsim.py:63-163) and the device-generated
buffered stream against golden values from the unmodified reference
(tests/golden/make_golden_sim.py): makespans, per-task start steps and
workers, realized nested graphs and spawn logs -- all exact."""

from __future__ import annotations

import hashlib
import json
import os
import warnings

import numpy as np
import pytest

from paper_1401_4441_b200 import analytics, depgraph, schedsim, taskgen
from paper_1401_4441_b200.grid import GridSpec

pytestmark = pytest.mark.gpu
SIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_sim.json")


@pytest.fixture(scope="module")
def sim():
    with open(SIM) as f:
        return json.load(f)


def _grid(r):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return GridSpec(tuple(r["extents"]), periodic=r["periodic"])


def _stream(g, name):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if name == "loopex":
            return taskgen.generate_loopex(g)
        order = {"basic/canonical": taskgen.StencilOrder.canonical(g.dim),
                 "basic/opt": taskgen.opt_order()}.get(name)
        if order is None:
            order = taskgen.order_with_displacement(3, int(name.split("delta")[1]))
        return taskgen.generate_basic(g, order)


def _workers(res, n):
    st, wk = [-1] * n, [-1] * n
    for w, lane in enumerate(res.timeline):
        for t, tid in lane:
            st[tid], wk[tid] = t, w
    return st, wk


def test_simulate_static(sim, cuda):
    graphs = {}
    for r in sim["static"]:
        key = (tuple(r["extents"]), r["periodic"], r["stream"])
        if key not in graphs:
            graphs[key] = depgraph.detect_dependencies(_stream(_grid(r), r["stream"]))
        graph = graphs[key]
        assert graph.task_count == r["tasks"]
        res = schedsim.simulate(graph, schedsim.SimConfig(r["workers"]))
        assert res.makespan == r["makespan"], (key, r["workers"])
        assert res.speedup == pytest.approx(r["speedup"], rel=1e-15)
        if "start" in r:
            st, wk = _workers(res, graph.task_count)
            assert st == r["start"] and wk == r["worker"], (key, r["workers"])
        if r["workers"] >= graph.task_count:  # W = infinity: makespan = critical path
            assert res.makespan == depgraph.critical_path(graph)


def test_simulate_nested(sim, cuda):
    for r in sim["nested"]:
        g = _grid(r)
        plan = taskgen.NestedPlan(g)
        res = schedsim.simulate_dynamic(plan, schedsim.SimConfig(r["workers"]))
        key = (tuple(r["extents"]), r["periodic"], r["workers"])
        assert (res.makespan, res.graph.task_count) == (r["makespan"], r["tasks"]), key
        if "home" not in r:
            continue
        assert [t.home for t in res.graph.tasks] == r["home"], key
        assert [plan.chain_position(t) for t in res.graph.tasks] == r["entry"], key
        assert [-1 if s.parent is None else s.parent for s in res.spawn_log] == r["parent"], key
        assert [list(e) for e in res.graph.edges] == r["edges"], key
        st, wk = _workers(res, res.graph.task_count)
        assert st == r["start"] and wk == r["worker"], key
        if r["unlimited"] and g.cell_count <= 128:
            # the log replays into the same graph (depgraph.py:130-157)
            assert depgraph.detect_dependencies_dynamic(plan, res.spawn_log).edges == res.graph.edges


def test_speedup_curves_and_eq2(cuda):
    """30x10x10, W = 8/16 -- basic delta=1 7.983 / 13.457 against
    Eq. 2 (capped), loop-exchange and nested 8 / 16 / 31.988."""
    g = GridSpec((30, 10, 10))
    graph = depgraph.detect_dependencies(taskgen.generate_basic(g, taskgen.order_with_displacement(3, 1)))
    curve = dict(schedsim.speedup_curve(graph, [8, 16]))
    assert round(curve[8].speedup, 3) == 7.983 and round(curve[16].speedup, 3) == 13.457
    m = analytics.AnalyticModel(1, g.cell_count, 14)
    assert analytics.compare(m, curve[16], workers=16).passed
    lx = dict(schedsim.speedup_curve(depgraph.detect_dependencies(taskgen.generate_loopex(g)), [8, 32]))
    assert lx[8].speedup == 8.0 and round(lx[32].speedup, 3) == 31.988
    ne = schedsim.simulate_dynamic(taskgen.NestedPlan(g), schedsim.SimConfig(32))
    assert round(ne.speedup, 3) == 31.988
    inf = schedsim.simulate_dynamic(taskgen.NestedPlan(GridSpec((4, 4, 4))),
                                    schedsim.unlimited_workers(taskgen.NestedPlan(GridSpec((4, 4, 4)))))
    assert inf.makespan == 49


def test_simulate_errors(cuda):
    with pytest.raises(ValueError):
        schedsim.SimConfig(0)
    with pytest.raises(ValueError):
        schedsim.simulate(depgraph.TaskGraph([], ()), schedsim.SimConfig(2))
    # a cycle (only reachable through simulate_edges, TaskGraph rejects it) stalls
    with pytest.raises(RuntimeError, match="cycle"):
        schedsim.simulate_edges(3, [0, 2, 1], [1, 1, 2], 4)


def _buffered_hash(tasks):
    rows = []
    for t in tasks:
        rows.append([t.id, t.kind, t.home, list(t.offset) if t.offset is not None else None,
                     sorted(list(r) for r in t.resources), sorted(list(r) for r in t.reads)])
    return hashlib.sha256(json.dumps(rows, separators=(",", ":")).encode()).hexdigest()


def test_buffered_stream_device(sim, cuda):
    for r in sim["buffered"]:
        tasks = taskgen.generate_buffered(_grid(r))
        assert len(tasks) == r["tasks"] and _buffered_hash(tasks) == r["hash"], r["extents"]
