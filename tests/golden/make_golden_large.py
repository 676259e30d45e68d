"""Serialization depths on the BASELINE config grids, computed with the
UNMODIFIED reference (build container only; minutes and ~10 GB RAM).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py

The 3x3x3 colour order is not a reference function: it is generate_loopex's
loop nest (taskgen.py:202-234) with colour = sum_k (coord_k mod 3) 3^k,
built here from the reference's own Task / neighbor / accumulator and fed
to the reference's detect_dependencies + critical_path.
"""
import json, os, sys, time, warnings
sys.path.insert(0, "/root/reference/pkg/src")
from cellsched import depgraph, grid as rgrid, taskgen  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_depths_large.json")


def loopex_stride(g, s):
    stencil = rgrid.canonical_half_stencil(g.dim)
    zero = rgrid.zero_offset(g.dim)
    groups = [[] for _ in range(s ** g.dim)]
    for cell in g.cells():
        c = g.coords(cell)
        groups[sum((v % s) * s ** k for k, v in enumerate(c))].append(cell)
    tasks = []
    for off in stencil.offsets:
        for cells in groups:
            for cell in cells:
                if off == zero:
                    tasks.append(taskgen.Task(len(tasks), taskgen.INTRA, cell, None,
                                              frozenset((taskgen.accumulator(cell),))))
                else:
                    nbr = rgrid.neighbor(cell, off, g)
                    tasks.append(taskgen.Task(len(tasks), taskgen.INTER, cell, off,
                                              frozenset((taskgen.accumulator(cell), taskgen.accumulator(nbr)))))
    return tasks


def main():
    warnings.simplefilter("ignore")
    out = []
    jobs = [((64, 64, 64), "basic"), ((64, 64, 64), "loopex"), ((64, 64, 192), "basic"),
            ((64, 64, 192), "loopex"), ((64, 64, 192), "stride3"), ((4, 4, 4), "stride3"),
            ((6, 6, 6), "stride3"), ((32, 32, 32), "stride3")]
    for ext, strat in jobs:
        g = rgrid.GridSpec(ext)
        t0 = time.time()
        tasks = loopex_stride(g, 3) if strat == "stride3" else taskgen.generate(strat, g)
        graph = depgraph.detect_dependencies(tasks)
        d = depgraph.critical_path(graph)
        rec = {"extents": list(ext), "strategy": strat, "tasks": len(tasks),
               "edges": graph.edge_count, "depth": d, "seconds": round(time.time() - t0, 1)}
        print(rec, flush=True)
        out.append(rec)
        del tasks, graph
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
