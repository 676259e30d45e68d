"""Golden vectors for the worker-pool model and the closed forms, taken from
the UNMODIFIED reference package (schedsim.py, analytics.py, taskgen.py
NestedPlan, depgraph.py dynamic detection).

Run in the build container only (the reference is absent on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_sim.py

Writes tests/golden/reference_sim.json:
  * simulate(detect_dependencies(stream), SimConfig(W)) for basic (canonical,
    delta=1, delta=14) and loopex streams -- makespan and, for small graphs,
    the per-task start time and worker (from SimResult.timeline);
  * simulate_dynamic(NestedPlan(grid, order), SimConfig(W)) -- makespan, the
    realized tasks (home, chain entry), edges, spawn-log parents and start
    times;
  * speedup_stencil / speedup_max / speedup_pipeline / speedup_capped as
    exact fractions, permutation_sweep(2) and sampled_permutation_sweep(3).
Nothing here re-implements the reference.
"""

from __future__ import annotations

import json
import os
import sys
import warnings

sys.path.insert(0, "/root/reference/pkg/src")
from cellsched import analytics, depgraph, schedsim, taskgen  # noqa: E402
from cellsched.grid import GridSpec, zero_offset  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_sim.json")


def starts(res, n):
    st, wk = [-1] * n, [-1] * n
    for w, lane in enumerate(res.timeline):
        for t, tid in lane:
            st[tid], wk[tid] = t, w
    return st, wk


def buffered_hash(tasks):
    """sha256 over a canonical text form of a buffered stream."""
    import hashlib

    rows = []
    for t in tasks:
        rows.append([t.id, t.kind, t.home, list(t.offset) if t.offset is not None else None,
                     sorted(list(r) for r in t.resources), sorted(list(r) for r in t.reads)])
    return hashlib.sha256(json.dumps(rows, separators=(",", ":")).encode()).hexdigest()


def frac(f):
    return [f.numerator, f.denominator]


def main():
    warnings.simplefilter("ignore")
    out = {"static": [], "nested": [], "analytics": {}}
    grids = [((4, 4, 4), True), ((6, 4, 8), True), ((30, 10, 10), True), ((5, 5), True),
             ((4, 6), False), ((3, 4, 5), False), ((5, 5, 5), True)]
    for ext, per in grids:
        g = GridSpec(ext, periodic=per)
        dim = g.dim
        streams = {"basic/canonical": taskgen.generate_basic(g, taskgen.StencilOrder.canonical(dim))}
        if dim == 3:
            streams["basic/delta1"] = taskgen.generate_basic(g, taskgen.order_with_displacement(3, 1))
            streams["basic/delta14"] = taskgen.generate_basic(g, taskgen.order_with_displacement(3, 14))
        else:
            streams["basic/opt"] = taskgen.generate_basic(g, taskgen.opt_order())
        streams["loopex"] = taskgen.generate_loopex(g)
        for name, tasks in streams.items():
            graph = depgraph.detect_dependencies(tasks)
            n = graph.task_count
            for W in (1, 3, 8, 16, 32, n):
                res = schedsim.simulate(graph, schedsim.SimConfig(W))
                rec = {"extents": list(ext), "periodic": per, "stream": name, "workers": W,
                       "tasks": n, "makespan": res.makespan, "speedup": res.speedup}
                if n <= 4000:
                    rec["start"], rec["worker"] = starts(res, n)
                out["static"].append(rec)
        for oname, order in (("canonical", None),
                             ("delta1", taskgen.order_with_displacement(dim, 1) if dim == 3 else None)):
            if oname == "delta1" and dim != 3:
                continue
            try:
                plan = taskgen.NestedPlan(g, order)
            except ValueError:
                continue  # the delta=1 order does not start with intra: rejected
            W_inf = schedsim.unlimited_workers(plan).workers
            for W in (1, 8, 16, 32, W_inf):
                res = schedsim.simulate_dynamic(plan, schedsim.SimConfig(W))
                gr = res.graph
                rec = {"extents": list(ext), "periodic": per, "order": oname, "workers": W,
                       "unlimited": W == W_inf, "tasks": gr.task_count, "makespan": res.makespan,
                       "speedup": res.speedup}
                if gr.task_count <= 4000:
                    z = zero_offset(dim)
                    rec["home"] = [t.home for t in gr.tasks]
                    rec["entry"] = [plan.order.offsets.index(t.offset if t.offset is not None else z)
                                    for t in gr.tasks]
                    rec["parent"] = [r.parent if r.parent is not None else -1 for r in res.spawn_log]
                    rec["edges"] = [list(e) for e in gr.edges]
                    rec["start"], rec["worker"] = starts(res, gr.task_count)
                    # the dynamic detector replays the log into the same graph
                    assert depgraph.detect_dependencies_dynamic(plan, res.spawn_log).edges == gr.edges
                out["nested"].append(rec)
    # the buffered stream, task by task (kind, home, offset, resources, reads)
    out["buffered"] = []
    for ext, per in (((4, 4, 4), True), ((4, 6), False), ((3, 4, 5), False), ((5, 5), True)):
        g = GridSpec(ext, periodic=per)
        tasks = taskgen.generate_buffered(g)
        out["buffered"].append({"extents": list(ext), "periodic": per, "hash": buffered_hash(tasks),
                                "tasks": len(tasks)})
    a = out["analytics"]
    a["stencil"] = []
    for delta, k, n in ((1, 100, 5), (4, 2500, 5), (10, 64, 14), (14, 3000, 14), (1, 3000, 14),
                        (5, 1, 5), (2, 7, 14)):
        m = analytics.AnalyticModel(delta, k, n)
        a["stencil"].append({"delta": delta, "k": k, "n": n,
                             "speedup_stencil": frac(analytics.speedup_stencil(m)),
                             "speedup_max": frac(analytics.speedup_max(delta, n)),
                             "capped": {str(w): frac(analytics.speedup_capped(m, w)) for w in (1, 8, 32)}})
    a["pipeline"] = [{"n": n, "k": k, "value": frac(analytics.speedup_pipeline(n, k))}
                     for n, k in ((100, 5), (3000, 14), (1, 1), (7, 3))]
    a["sweep2"] = [{"offsets": [list(o) for o in e.order.offsets], "delta": e.delta,
                    "s_max": frac(e.s_max)} for e in analytics.permutation_sweep(2)]
    sw3 = analytics.sampled_permutation_sweep(3, count=200, seed=7)
    a["sweep3_seed7_count200"] = {"deltas": [e.delta for e in sw3],
                                  "first_orders": [[list(o) for o in e.order.offsets] for e in sw3[:5]],
                                  "histogram": {str(k): v for k, v in analytics.delta_histogram(sw3).items()}}
    # compare() against simulated speedups (the reference's Eq. 2 check)
    g = GridSpec((30, 10, 10))
    order = taskgen.order_with_displacement(3, 1)
    graph = depgraph.detect_dependencies(taskgen.generate_basic(g, order))
    a["compare"] = []
    for W in (8, 16):
        res = schedsim.simulate(graph, schedsim.SimConfig(W))
        rep = analytics.compare(analytics.AnalyticModel(1, g.cell_count, 14), res, workers=W)
        a["compare"].append({"workers": W, "predicted": rep.predicted, "measured": rep.measured,
                             "rel_error": rep.rel_error, "passed": rep.passed})
    with open(OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
