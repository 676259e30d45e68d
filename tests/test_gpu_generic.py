"""Generic task lists on the device: the reference's own depgraph unit cases
(test_depgraph.py:37-90 semantics), the buffered strategy (read-only reduce
inputs) and plain lists of the standard streams, all against golden values."""

from __future__ import annotations

import warnings

import pytest

import paper_1401_4441_b200 as P
from paper_1401_4441_b200 import depgraph, taskgen
from paper_1401_4441_b200.taskgen import Task
from conftest import case_id

pytestmark = pytest.mark.gpu


def mk(i, reads=(), writes=()):
    return Task(i, "t", None, None, frozenset(writes), frozenset(reads))


def test_vector_example(golden, cuda):
    vec = [mk(0, writes={"a"}), mk(1, writes={"b"}), mk(2, writes={"c"}),
           mk(3, reads={"b"}, writes={"c"}), mk(4, reads={"a", "b"}, writes={"d"}),
           mk(5, reads={"c", "d"}, writes={"s"})]
    g = depgraph.detect_dependencies(vec)
    assert [list(e) for e in g.edges] == golden["vector_example"]["edges"]
    assert depgraph.critical_path(g) == golden["vector_example"]["depth"] == 3
    assert g.roots() == [0, 1, 2] and g.sinks() == [5]


def test_small_rules(cuda):
    assert depgraph.detect_dependencies([mk(0, writes={"x"}), mk(1, writes={"y"})]).edges == ()
    chain = depgraph.detect_dependencies([mk(i, writes={"r"}) for i in range(6)])
    assert set(chain.edges) == {(i, i + 1) for i in range(5)}
    assert depgraph.critical_path(chain) == 6
    dup = depgraph.detect_dependencies([mk(0, writes={"a", "b"}), mk(1, writes={"a", "b"})])
    assert dup.edges == ((0, 1),)
    with pytest.raises(ValueError):
        depgraph.detect_dependencies([mk(0, writes={"a"}), mk(2, writes={"b"})])
    # inout wins: a task reading and writing r depends on the last writer only once
    g = depgraph.detect_dependencies([mk(0, writes={"r"}), mk(1, reads={"r"}, writes={"r"})])
    assert g.edges == ((0, 1),)
    # many readers then a writer: the writer waits for every reader
    g = depgraph.detect_dependencies([mk(0, writes={"r"})] + [mk(i, reads={"r"}) for i in range(1, 5)]
                                     + [mk(5, writes={"r"})])
    assert set(g.edges) == {(0, i) for i in range(1, 5)} | {(i, 5) for i in range(1, 5)}
    assert depgraph.critical_path(g) == 3


def test_buffered_streams_and_payload(golden, cuda):
    for case in golden["cases"]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g = P.GridSpec(tuple(case["extents"]), periodic=case["periodic"])
        tasks = taskgen.generate_buffered(g)
        graph = depgraph.detect_dependencies(tasks)
        ref = case["buffered"]
        assert (len(tasks), graph.edge_count) == (ref["tasks"], ref["edges"]), case_id(case)
        assert depgraph.critical_path(graph) == ref["depth"], case_id(case)
        for seed, pl in list(case["payload"].items())[:2]:
            acc = P.execute_with_payload("buffered", g, int(seed))
            assert [acc[c] for c in g.cells()] == pl["oracle"], (case_id(case), seed)


def test_generic_matches_closed_form_on_plain_lists(golden, cuda):
    for case in golden["cases"][:8]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g = P.GridSpec(tuple(case["extents"]), periodic=case["periodic"])
            tasks = list(P.generate_loopex(g))  # plain list: no device stream attached
        ref = case["streams"]["loopex"]
        graph = depgraph.detect_dependencies(tasks)
        assert [u for u, _ in graph.edges] == ref["edges_u"] and [v for _, v in graph.edges] == ref["edges_v"]
        assert depgraph.critical_path(graph) == ref["depth"]
        assert depgraph.levels(graph) == ref["levels"]
        acc = P.apply_tasks(tasks, g, 42)
        assert [acc[c] for c in g.cells()] == case["payload"]["42"]["oracle"]


def test_non_forward_edge_rejected(cuda):
    with pytest.raises(ValueError):
        depgraph.TaskGraph([mk(0), mk(1)], ((1, 0),))


def test_dag_runtime_matches_reference(golden, cuda):
    """dependency-driven execution (ready queue, no levels) of the
    basic, loop-exchange and buffered streams gives the reference accumulators
    with zero write conflicts (executor.verify_execution's contract)."""
    from paper_1401_4441_b200.generic import execute_dag

    for case in golden["cases"][:8]:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g = P.GridSpec(tuple(case["extents"]), periodic=case["periodic"])
            streams = {"basic": list(P.generate_basic(g, P.StencilOrder.canonical(g.dim))),
                       "loopex": list(P.generate_loopex(g)),
                       "buffered": taskgen.generate_buffered(g)}
        for name, tasks in streams.items():
            for seed, pl in list(case["payload"].items())[:1]:
                acc, conflicts = execute_dag(tasks, g, int(seed))
                assert conflicts == 0, (case_id(case), name)
                assert [acc[c] for c in g.cells()] == pl["oracle"], (case_id(case), name, seed)


def test_dag_runtime_detects_missing_dependencies(cuda):
    """Without its edges every task of a 6^3 loop-exchange stream is ready at
    once: the device race detector must report write conflicts."""
    from paper_1401_4441_b200.generic import execute_dag

    g = P.GridSpec((6, 6, 6))
    tasks = list(P.generate_loopex(g))
    _, conflicts = execute_dag(tasks, g, 7, edges=())
    assert conflicts > 0
