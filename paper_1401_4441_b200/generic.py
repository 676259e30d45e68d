"""Arbitrary task lists on the device (K4/K5 generic paths).

Task lists that do not come from this package's stream generator (hand-built
graphs, the buffered strategy with read-only reduce inputs, ...) are interned
on the host -- resources become dense integer ids, accesses are listed in
stream order with a task's reads before its writes (reads of a resource the
task also writes are dropped: "inout wins", depgraph.py:32-33) -- and the
dependency rule, the longest path and the payload replay run on the device.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _torch():
    import torch

    return torch


def _intern(tasks):
    ids: dict = {}
    tptr = [0]
    acc_task, acc_res, acc_w = [], [], []
    for t in tasks:
        for r in t.reads:
            if r in t.resources:
                continue
            acc_task.append(t.id)
            acc_res.append(ids.setdefault(r, len(ids)))
            acc_w.append(0)
        for r in t.resources:
            acc_task.append(t.id)
            acc_res.append(ids.setdefault(r, len(ids)))
            acc_w.append(1)
        tptr.append(len(acc_task))
    return ids, np.asarray(tptr, np.int64), np.asarray(acc_task, np.int32), \
        np.asarray(acc_res, np.int32), np.asarray(acc_w, np.uint8)


def detect_edges_generic(tasks):
    """Edges (eu, ev) of detect_dependencies for any task list, computed on the
    device with the full _DependenceState rule (depgraph.py:28-49)."""
    torch = _torch()
    _lib.require_cuda()
    ids, tptr, at, ar, aw = _intern(tasks)
    nt, na = len(tasks), len(at)
    dev = "cuda"
    g = lambda a: torch.from_numpy(a).to(dev) if len(a) else torch.zeros(1, dtype=torch.from_numpy(a).dtype, device=dev)
    d_tptr, d_at, d_ar, d_aw = g(tptr), g(at), g(ar), g(aw)
    npm = 2 * na + 1
    L = _lib.load()
    wsb = L.cs_detect_ws_bytes(nt, na, npm)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    ne = C.c_int64()
    s = _lib.stream_handle()
    _lib.call("cs_detect_generic", nt, na, max(len(ids), 1), _lib.ptr(d_tptr), _lib.ptr(d_at),
              _lib.ptr(d_ar), _lib.ptr(d_aw), npm, C.byref(ne), _lib.ptr(ws), wsb, s)
    eu = torch.empty(max(ne.value, 1), dtype=torch.int64, device=dev)
    ev = torch.empty_like(eu)
    _lib.call("cs_detect_generic_emit", nt, na, _lib.ptr(d_tptr), npm, _lib.ptr(eu), _lib.ptr(ev),
              _lib.ptr(ws), wsb, s)
    return eu[: ne.value].cpu().numpy(), ev[: ne.value].cpu().numpy()


def longest_path_device(ntasks, edges, return_levels=False):
    """critical_path (depgraph.py:160-174) of a forward edge list."""
    torch = _torch()
    _lib.require_cuda()
    if ntasks == 0:
        return (0, []) if return_levels else 0
    e = np.asarray(list(edges), np.int64).reshape(-1, 2)
    order = np.lexsort((e[:, 0], e[:, 1])) if len(e) else np.zeros(0, np.int64)
    e = e[order]
    dev = "cuda"
    eu = torch.from_numpy(np.ascontiguousarray(e[:, 0])).to(dev) if len(e) else torch.zeros(1, dtype=torch.int64, device=dev)
    ev = torch.from_numpy(np.ascontiguousarray(e[:, 1])).to(dev) if len(e) else torch.zeros(1, dtype=torch.int64, device=dev)
    lv = torch.empty(ntasks, dtype=torch.int32, device=dev)
    wsb = _lib.load().cs_longest_path_ws_bytes(ntasks)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    depth = C.c_int64()
    st = _lib.load().cs_longest_path(ntasks, len(e), _lib.ptr(eu), _lib.ptr(ev), _lib.ptr(lv),
                                     C.byref(depth), _lib.ptr(ws), wsb, _lib.stream_handle())
    if st == _lib.CS_ECYCLE:
        raise RuntimeError(_lib.load().cs_last_error().decode())
    _lib.check(st, "cs_longest_path")
    if return_levels:
        return depth.value, lv.cpu().tolist()
    return depth.value


def _payload_arrays(tasks, grid):
    """Per-task payload descriptors of apply_tasks (payload.py:84-119) with
    resources interned to dense accumulator ids."""
    from .grid import neighbor
    from .taskgen import INTER, INTRA, REDUCE, accumulator

    ids, tptr, at, ar, aw = _intern(tasks)
    nt = len(tasks)
    kind = np.zeros(nt, np.int8)
    home = np.zeros(nt, np.int32)
    nbr = np.zeros(nt, np.int32)
    w0 = np.zeros(nt, np.int32)
    w1 = np.zeros(nt, np.int32)
    off = np.zeros((nt, 3), np.int8)
    rptr = [0]
    rres = []
    for t in tasks:
        i = t.id
        home[i] = t.home
        if t.kind == INTRA:
            kind[i] = 0
            w0[i] = ids[next(iter(t.resources))]
        elif t.kind == INTER:
            kind[i] = 1
            nb = neighbor(t.home, t.offset, grid)
            nbr[i] = nb
            off[i, : grid.dim] = t.offset
            rs = list(t.resources)
            if len(rs) == 1:  # self-neighbour: both terms hit one accumulator
                w0[i] = w1[i] = ids[rs[0]]
            else:
                first = [r for r in rs if r == accumulator(t.home) or (r[0] == "buf" and r[2] == "out")]
                w0[i] = ids[first[0]]
                w1[i] = ids[[r for r in rs if r is not first[0] and r != first[0]][0]]
        elif t.kind == REDUCE:
            kind[i] = 2
            w0[i] = ids[next(iter(t.resources))]
            rres += [ids[r] for r in t.reads]
        else:
            raise ValueError(f"task {t.id} has non-payload kind {t.kind!r}")
        rptr.append(len(rres))
    return ids, [kind, home, nbr, w0, w1, off.ravel(), np.asarray(rptr, np.int64), np.asarray(rres, np.int32)]




def _dev(a, dtype):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda") if len(a) else torch.zeros(1, dtype=dtype, device="cuda")


def _result(grid, ids, val):
    from .taskgen import accumulator

    vals = val.cpu().tolist()
    return {c: (vals[ids[accumulator(c)]] if accumulator(c) in ids else 0) for c in grid.cells()}


def apply_tasks_generic(tasks, grid, seed):
    """apply_tasks (payload.py:84-119) for any accumulator / buffered stream,
    executed level by level on the device."""
    torch = _torch()
    from .payload import _signed64, charges_device

    _lib.require_cuda()
    tasks = list(tasks)
    ids, arrs = _payload_arrays(tasks, grid)
    nt = len(tasks)
    from .depgraph import detect_dependencies

    graph = detect_dependencies(tasks)
    depth, levels = longest_path_device(nt, graph.edges, return_levels=True)
    dts = [torch.int8, torch.int32, torch.int32, torch.int32, torch.int32, torch.int8, torch.int64, torch.int32]
    args = [_dev(a, dt) for a, dt in zip(arrs, dts)]
    q = charges_device(grid, _signed64(seed))
    nres = max(len(ids), 1)
    val = torch.zeros(nres, dtype=torch.int64, device="cuda")
    lv = torch.tensor(levels, dtype=torch.int32, device="cuda")
    wsb = _lib.load().cs_payload_generic_ws_bytes(nt, depth)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    _lib.call("cs_payload_generic", nt, grid.dim, *(_lib.ptr(a) for a in args), _lib.ptr(q),
              _lib.ptr(lv), depth, nres, _lib.ptr(val), _lib.ptr(ws), wsb, _lib.stream_handle())
    return _result(grid, ids, val)


def execute_dag(tasks, grid, seed, race_check: bool = True, edges=None):
    """run any task graph on the device in dependency order (ready
    queue + indegree counters, no levels) with the apply_tasks payload.
    Returns (accumulators by cell, write conflicts observed); with the
    reference's dependency rule the conflicts are 0 and the accumulators equal
    reference_oracle's -- executor.verify_execution's contract (executor.py:357-377)."""
    torch = _torch()
    from .payload import _signed64, charges_device

    _lib.require_cuda()
    tasks = list(tasks)
    nt = len(tasks)
    ids, arrs = _payload_arrays(tasks, grid)
    if edges is None:
        eu, ev = detect_edges_generic(tasks)
    else:  # caller-supplied dependencies (tests: a wrong graph must show conflicts)
        e = np.asarray(list(edges), np.int64).reshape(-1, 2)
        eu, ev = e[:, 0], e[:, 1]
    order = np.argsort(eu, kind="stable")
    eu, ev = eu[order].astype(np.int64), ev[order].astype(np.int64)
    sptr = np.zeros(nt + 1, np.int64)
    np.cumsum(np.bincount(eu, minlength=nt), out=sptr[1:])
    dts = [torch.int8, torch.int32, torch.int32, torch.int32, torch.int32, torch.int8, torch.int64, torch.int32]
    args = [_dev(a, dt) for a, dt in zip(arrs, dts)]
    q = charges_device(grid, _signed64(seed))
    nres = max(len(ids), 1)
    val = torch.zeros(nres, dtype=torch.int64, device="cuda")
    d_sptr, d_succ, d_ev = _dev(sptr, torch.int64), _dev(ev, torch.int64), _dev(ev, torch.int64)
    conflicts = torch.zeros(1, dtype=torch.int64, device="cuda")
    wsb = _lib.load().cs_dag_ws_bytes(nt, nres)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    st = _lib.load().cs_dag_execute(nt, grid.dim, *(_lib.ptr(a) for a in args), _lib.ptr(q), len(ev),
                                    _lib.ptr(d_sptr), _lib.ptr(d_succ), _lib.ptr(d_ev), nres,
                                    _lib.ptr(val), 1 if race_check else 0, _lib.ptr(conflicts),
                                    _lib.ptr(ws), wsb, _lib.stream_handle())
    if st == _lib.CS_ECYCLE:
        raise RuntimeError(_lib.load().cs_last_error().decode())
    _lib.check(st, "cs_dag_execute")
    return _result(grid, ids, val), int(conflicts.item())
