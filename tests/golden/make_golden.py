"""Generate golden vectors by importing the UNMODIFIED reference package.

Run in the build container only (the reference is absent on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json.  Every value comes from calling
the reference's own public API (cellsched.grid / taskgen / depgraph /
payload); nothing here re-implements it.  Streams are stored as flat
(home, nbr, entry) arrays, nbr = -1 for intra tasks and entry indexing the
order (basic) or the canonical stencil (loopex).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from cellsched import depgraph, grid as rgrid, payload, taskgen  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")


def stream_arrays(tasks, entries, g):
    home, nbr, entry = [], [], []
    zero = rgrid.zero_offset(g.dim)
    for t in tasks:
        home.append(t.home)
        if t.kind == taskgen.INTRA:
            nbr.append(-1)
            entry.append(entries.index(zero))
        else:
            nbr.append(rgrid.neighbor(t.home, t.offset, g))
            entry.append(entries.index(t.offset))
    return home, nbr, entry


def acc_array(acc, g):
    return [int(acc[c]) for c in g.cells()]


def sha(arr):
    return hashlib.sha256(np.asarray(arr, dtype=np.int64).tobytes()).hexdigest()


def orders_for(dim):
    out = {"canonical": taskgen.StencilOrder.canonical(dim)}
    if dim == 2:
        out.update(naive=taskgen.naive_order(), bad=taskgen.bad_order(), opt=taskgen.opt_order())
    else:
        out.update(
            delta1=taskgen.order_with_displacement(3, 1),
            delta2=taskgen.order_with_displacement(3, 2),
            delta14=taskgen.order_with_displacement(3, 14),
        )
    return out


def main():
    warnings.simplefilter("ignore")
    gold = {"generator": "cellsched (reference) via tests/golden/make_golden.py", "cases": []}
    gold["canonical_stencil"] = {
        str(d): [list(o) for o in rgrid.canonical_half_stencil(d).offsets] for d in (2, 3)
    }
    gold["orders"] = {
        str(d): {k: [list(o) for o in v.offsets] for k, v in orders_for(d).items()} for d in (2, 3)
    }
    gold["displacement"] = {
        str(d): {k: taskgen.displacement(v) for k, v in orders_for(d).items()} for d in (2, 3)
    }

    small = [
        ((4, 4), True), ((5, 5), True), ((6, 4), True), ((4, 6), True), ((3, 3), True),
        ((6, 1), False), ((5, 4), False),
        ((4, 4, 4), True), ((6, 6, 6), True), ((4, 4, 6), True), ((6, 4, 8), True),
        ((5, 5, 5), True), ((3, 4, 4), True), ((4, 3, 5), False),
    ]
    for ext, periodic in small:
        g = rgrid.GridSpec(ext, periodic=periodic)
        case = {"extents": list(ext), "periodic": periodic, "streams": {}}
        stencil = list(rgrid.canonical_half_stencil(g.dim).offsets)
        for name, order in orders_for(g.dim).items():
            tasks = taskgen.generate_basic(g, order)
            graph = depgraph.detect_dependencies(tasks)
            h, nb, e = stream_arrays(tasks, list(order.offsets), g)
            case["streams"]["basic:" + name] = {
                "home": h, "nbr": nb, "entry": e,
                "edges_u": [u for u, _ in graph.edges], "edges_v": [v for _, v in graph.edges],
                "depth": depgraph.critical_path(graph),
            }
        tasks = taskgen.generate_loopex(g)
        graph = depgraph.detect_dependencies(tasks)
        h, nb, e = stream_arrays(tasks, stencil, g)
        lvl = [1] * graph.task_count
        for v in range(graph.task_count):
            for u in graph.preds[v]:
                lvl[v] = max(lvl[v], lvl[u] + 1)
        case["streams"]["loopex"] = {
            "home": h, "nbr": nb, "entry": e,
            "edges_u": [u for u, _ in graph.edges], "edges_v": [v for _, v in graph.edges],
            "depth": depgraph.critical_path(graph), "levels": lvl,
        }
        # buffered stream: exercises read-only resources in detection
        btasks = taskgen.generate_buffered(g)
        bgraph = depgraph.detect_dependencies(btasks)
        case["buffered"] = {"tasks": len(btasks), "edges": bgraph.edge_count,
                            "depth": depgraph.critical_path(bgraph)}
        case["colors"] = [rgrid.color(c, g) for c in g.cells()]
        case["payload"] = {}
        for seed in (0, 1, 42, 2**40 + 7, -3):
            ref = payload.reference_oracle(g, seed)
            case["payload"][str(seed)] = {
                "charges": payload.charges(g, seed),
                "oracle": acc_array(ref, g),
                "loopex": acc_array(payload.execute_with_payload("loopex", g, seed), g),
                "basic": acc_array(payload.execute_with_payload("basic", g, seed), g),
            }
        gold["cases"].append(case)
        print("case", ext, periodic, flush=True)

    # 100-seed payload hashes on 4^3, 6^3, 8^3
    gold["payload_hashes"] = {}
    for ext in ((4, 4, 4), (6, 6, 6), (8, 8, 8)):
        g = rgrid.GridSpec(ext)
        gold["payload_hashes"]["x".join(map(str, ext))] = [
            sha(acc_array(payload.reference_oracle(g, seed), g)) for seed in range(100)
        ]
        print("hashes", ext, flush=True)

    # the reference's own Fig. 1/2 vector example (test_depgraph.py:37-66)
    def mk(i, reads=(), writes=()):
        return taskgen.Task(i, "t", None, None, frozenset(writes), frozenset(reads))

    vec = [
        mk(0, writes={"a"}), mk(1, writes={"b"}), mk(2, writes={"c"}),
        mk(3, reads={"b"}, writes={"c"}), mk(4, reads={"a", "b"}, writes={"d"}),
        mk(5, reads={"c", "d"}, writes={"s"}),
    ]
    vg = depgraph.detect_dependencies(vec)
    gold["vector_example"] = {"edges": [list(e) for e in vg.edges], "depth": depgraph.critical_path(vg)}

    # depth / edge counts at larger grids (serialization depth at configs)
    gold["depths"] = []
    for ext in ((8, 8, 8), (16, 16, 16), (32, 32, 32)):
        g = rgrid.GridSpec(ext)
        for strat in ("basic", "loopex"):
            t0 = time.time()
            tasks = taskgen.generate(strat, g)
            graph = depgraph.detect_dependencies(tasks)
            d = depgraph.critical_path(graph)
            gold["depths"].append({"extents": list(ext), "strategy": strat, "tasks": len(tasks),
                                   "edges": graph.edge_count, "depth": d,
                                   "edges_sha": sha([x for e in graph.edges for x in e]),
                                   "seconds": round(time.time() - t0, 2)})
            print("depth", ext, strat, d, flush=True)
            del tasks, graph

    with open(OUT, "w") as f:
        json.dump(gold, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
