"""Closed forms (analytics.py:44-137), NestedPlan's host API (taskgen.py:279-325)
and export_dot against golden values from the unmodified reference
(tests/golden/make_golden_sim.py).  CPU only."""

from __future__ import annotations

import json
import os
from fractions import Fraction

import pytest

from paper_1401_4441_b200 import analytics as A
from paper_1401_4441_b200 import depgraph, taskgen
from paper_1401_4441_b200.grid import GridSpec

SIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_sim.json")


@pytest.fixture(scope="module")
def sim():
    with open(SIM) as f:
        return json.load(f)


def F(p):
    return Fraction(p[0], p[1])


def test_closed_forms(sim):
    a = sim["analytics"]
    for r in a["stencil"]:
        m = A.AnalyticModel(r["delta"], r["k"], r["n"])
        assert A.speedup_stencil(m) == F(r["speedup_stencil"])
        assert A.speedup_max(r["delta"], r["n"]) == F(r["speedup_max"])
        for w, v in r["capped"].items():
            assert A.speedup_capped(m, int(w)) == F(v)
    for r in a["pipeline"]:
        assert A.speedup_pipeline(r["n"], r["k"]) == F(r["value"])
    # the paper's headline values
    assert A.speedup_max(2, 14) == 7 and A.speedup_max(1, 5) == 5 and A.speedup_max(4, 5) == Fraction(5, 4)
    with pytest.raises(ValueError):
        A.AnalyticModel(0, 10, 14)
    with pytest.raises(ValueError):
        A.AnalyticModel(15, 10, 14)
    with pytest.raises(ValueError):
        A.AnalyticModel(1, 0, 14)
    with pytest.raises(ValueError):
        A.speedup_pipeline(0, 3)


def test_sweeps(sim):
    a = sim["analytics"]
    got = A.permutation_sweep(2)
    assert [[list(o) for o in e.order.offsets] for e in got] == [r["offsets"] for r in a["sweep2"]]
    assert [e.delta for e in got] == [r["delta"] for r in a["sweep2"]]
    assert [e.s_max for e in got] == [F(r["s_max"]) for r in a["sweep2"]]
    sw = A.sampled_permutation_sweep(3, count=200, seed=7)
    ref = a["sweep3_seed7_count200"]
    assert [e.delta for e in sw] == ref["deltas"]
    assert [[list(o) for o in e.order.offsets] for e in sw[:5]] == ref["first_orders"]
    assert {str(k): v for k, v in A.delta_histogram(sw).items()} == ref["histogram"]
    with pytest.raises(ValueError):
        A.permutation_sweep(3)


def test_compare_report(sim):
    class M:
        def __init__(self, s):
            self.speedup = s

    for r in sim["analytics"]["compare"]:
        rep = A.compare(A.AnalyticModel(1, 3000, 14), M(r["measured"]), workers=r["workers"])
        assert rep.predicted == pytest.approx(r["predicted"], rel=1e-15)
        assert rep.rel_error == pytest.approx(r["rel_error"], rel=1e-12)
        assert rep.passed == r["passed"]


def test_nested_plan_host_api(sim):
    """successor() reproduces every spawn of the reference's realized plans."""
    for r in sim["nested"]:
        if "home" not in r:
            continue
        g = GridSpec(tuple(r["extents"]), periodic=r["periodic"])
        plan = taskgen.NestedPlan(g)
        init = plan.initial_tasks()
        assert [t.home for t in init] == list(range(g.cell_count))
        offs = plan.order.offsets
        tasks = []
        for tid, (h, e, par) in enumerate(zip(r["home"], r["entry"], r["parent"])):
            if par < 0:
                t = init[tid]
            else:
                t = plan.successor(tasks[par], tid)
                assert t is not None and t.home == h and plan.chain_position(t) == e
                assert t.offset == offs[e]
            tasks.append(t)
        # chain ends: no task of the log spawns past the last entry
        spawned = set(p for p in r["parent"] if p >= 0)
        for t in tasks:
            if t.id not in spawned:
                assert plan.successor(t, len(tasks)) is None
    with pytest.raises(ValueError):
        taskgen.NestedPlan(GridSpec((4, 4, 4)), taskgen.order_with_displacement(3, 1))
    with pytest.raises(ValueError):
        taskgen.NestedPlan(GridSpec((4, 4)), taskgen.StencilOrder.canonical(3))
    assert isinstance(taskgen.generate("nested", GridSpec((4, 4, 4))), taskgen.NestedPlan)


def test_export_dot():
    T = taskgen.Task
    tasks = [T(0, "intra", 0, None, frozenset()), T(1, "inter", 0, (1, 0), frozenset()),
             T(2, "inter", 1, (0, 1), frozenset()), T(3, "reduce", 2, None, frozenset())]
    g = depgraph.TaskGraph(tasks, ((0, 1), (0, 2), (1, 2), (2, 3), (0, 3)))
    full = depgraph.export_dot(g)
    assert full.splitlines()[:3] == ["digraph tasks {", "  rankdir=TB;", '  t0 [label="0 intra c0"];']
    assert '  t1 [label="1 inter c0 (1,0)"];' in full and full.endswith("}\n")
    assert [l for l in full.splitlines() if "->" in l] == [
        "  t0 -> t1;", "  t0 -> t2;", "  t0 -> t3;", "  t1 -> t2;", "  t2 -> t3;"]
    red = depgraph.export_dot(g, transitive_reduction=True)
    assert [l for l in red.splitlines() if "->" in l] == ["  t0 -> t1;", "  t1 -> t2;", "  t2 -> t3;"]


def test_spawn_contract_violations():
    """detect_dependencies_dynamic rejects tampered logs (test_depgraph.py:200-212)."""
    g = GridSpec((4, 4, 4))
    plan = taskgen.NestedPlan(g)
    init = plan.initial_tasks()
    child = plan.successor(init[0], len(init))
    log = [depgraph.SpawnRecord(t, None) for t in init] + [depgraph.SpawnRecord(child, 0)]
    bad = log[:-1] + [depgraph.SpawnRecord(child, 0, parent_completed=False)]
    with pytest.raises(RuntimeError, match="before parent"):
        depgraph.detect_dependencies_dynamic(plan, bad)
    bad = log[:-1] + [depgraph.SpawnRecord(child, 5)]
    with pytest.raises(RuntimeError, match="different cell"):
        depgraph.detect_dependencies_dynamic(plan, bad)
    other = taskgen.Task(len(init), "intra", 0, None, child.resources)
    bad = log[:-1] + [depgraph.SpawnRecord(other, 0)]
    with pytest.raises(RuntimeError, match="advance"):
        depgraph.detect_dependencies_dynamic(plan, bad)
