"""The reference's worker-pool model, run on the device.

Mirrors `cellsched.schedsim` (schedsim.py:18-185): `SimConfig`, `SimResult`,
`simulate`, `simulate_dynamic`, `speedup_curve`, `unlimited_workers`, with
the same semantics -- unit task durations, W workers, and at every time step
the ready tasks handed out in ascending id order (schedsim.py:75-87); nested
plans spawn each cell's next chain entry when its predecessor finishes, the
dependency rule applied at spawn time (schedsim.py:93-163).

The schedules themselves run in one persistent CTA (`cs_simulate_static`,
`cs_simulate_nested`, csrc/cs_listsched.cuh).  The device returns per-task
start steps; a task's worker is its rank among the tasks of its step, which
is exactly the batch position the reference pops it into.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .depgraph import SpawnRecord, TaskGraph
from .taskgen import INTER, INTRA, NestedPlan, Task, accumulator


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class SimConfig:
    """Worker count; every task takes one time unit (schedsim.py:18-26)."""

    workers: int

    def __post_init__(self) -> None:
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")


@dataclass
class SimResult:
    """One simulated schedule (schedsim.py:29-60).  timeline[w] lists
    (start_time, task_id) per worker; speedup = serial_time / makespan."""

    makespan: int
    serial_time: int
    workers: int
    timeline: list = field(repr=False)
    graph: TaskGraph | None = field(repr=False, default=None)
    spawn_log: list | None = field(repr=False, default=None)
    start: object = field(repr=False, default=None)  # numpy int32 start step per task

    @property
    def speedup(self) -> float:
        return self.serial_time / self.makespan

    @property
    def utilization(self) -> float:
        return self.serial_time / (self.workers * self.makespan)

    def execution_order(self) -> list[int]:
        """Task ids by (start time, worker): the replay order of a payload."""
        st = np.asarray(self.start)
        return np.lexsort((np.arange(len(st)), st)).tolist()


def _timeline(start: np.ndarray, workers: int) -> list:
    """Worker lanes from start steps: within a step, ids ascend with the
    worker index (the batch is popped from a min-heap)."""
    n = len(start)
    order = np.lexsort((np.arange(n), start))
    st_sorted = start[order]
    first = np.searchsorted(st_sorted, st_sorted, side="left")
    rank = np.arange(n) - first
    lanes: list[list[tuple[int, int]]] = [[] for _ in range(workers)]
    for tid, t, w in zip(order.tolist(), st_sorted.tolist(), rank.tolist()):
        lanes[w].append((t, tid))
    return lanes


def _csr(n: int, eu: np.ndarray, ev: np.ndarray):
    order = np.argsort(eu, kind="stable")
    succ = ev[order].astype(np.int32)
    sptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(eu, minlength=n), out=sptr[1:])
    return sptr, succ


def simulate_edges(ntasks: int, eu, ev, workers: int):
    """Device list schedule of a forward edge list: (start[] numpy, makespan)."""
    torch = _torch()
    _lib.require_cuda()
    if ntasks == 0:
        raise ValueError("cannot simulate an empty graph")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    eu = np.asarray(eu, np.int64)
    ev = np.asarray(ev, np.int64)
    sptr, succ = _csr(ntasks, eu, ev)
    dev = "cuda"
    d_sptr = torch.from_numpy(sptr).to(dev)
    d_succ = torch.from_numpy(succ if len(succ) else np.zeros(1, np.int32)).to(dev)
    start = torch.empty(ntasks, dtype=torch.int32, device=dev)
    wsb = _lib.load().cs_listsched_ws_bytes(ntasks)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    mk = C.c_int64()
    maxdeg = int(np.bincount(ev, minlength=1).max()) if len(ev) else 0
    st = _lib.load().cs_simulate_static(ntasks, len(succ), _lib.ptr(d_sptr), _lib.ptr(d_succ),
                                         int(workers), maxdeg, _lib.ptr(start), C.byref(mk),
                                         _lib.ptr(ws), wsb, _lib.stream_handle())
    if st == _lib.CS_ECYCLE:
        raise RuntimeError(_lib.load().cs_last_error().decode())
    _lib.check(st, "cs_simulate_static")
    return start.cpu().numpy(), int(mk.value)


def simulate(graph: TaskGraph, cfg: SimConfig) -> SimResult:
    """Greedy work-conserving schedule of a static task graph (schedsim.py:63-90)."""
    n = graph.task_count
    if n == 0:
        raise ValueError("cannot simulate an empty graph")
    e = np.asarray(graph.edges, np.int64).reshape(-1, 2)
    start, makespan = simulate_edges(n, e[:, 0], e[:, 1], cfg.workers)
    return SimResult(makespan=makespan, serial_time=n, workers=cfg.workers,
                     timeline=_timeline(start, cfg.workers), start=start)


def _order_array(plan: NestedPlan):
    dim = plan.grid.dim
    arr = (C.c_int8 * (plan.order.n * dim))()
    for e, off in enumerate(plan.order.offsets):
        for k in range(dim):
            arr[e * dim + k] = int(off[k])
    return arr


def nested_device(plan: NestedPlan, workers: int):
    """Run simulate_dynamic's schedule on the device; returns numpy arrays
    (home, entry, parent, pred_a, pred_b, start) over the realized tasks and
    the makespan."""
    torch = _torch()
    _lib.require_cuda()
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    g = plan.grid._cs_grid()
    cap = plan.grid.cell_count * plan.order.n
    dev = "cuda"
    i32 = lambda: torch.empty(cap, dtype=torch.int32, device=dev)
    home, parent, pa, pb, start = i32(), i32(), i32(), i32(), i32()
    entry = torch.empty(cap, dtype=torch.int16, device=dev)
    wsb = _lib.load().cs_nested_ws_bytes(C.byref(g), plan.order.n)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    nt, mk = C.c_int64(), C.c_int64()
    st = _lib.load().cs_simulate_nested(C.byref(g), _order_array(plan), plan.order.n, int(workers),
                                         _lib.ptr(home), _lib.ptr(entry), _lib.ptr(parent),
                                         _lib.ptr(pa), _lib.ptr(pb), _lib.ptr(start), cap,
                                         C.byref(nt), C.byref(mk), _lib.ptr(ws), wsb,
                                         _lib.stream_handle())
    if st == _lib.CS_ECYCLE:
        raise RuntimeError(_lib.load().cs_last_error().decode())
    _lib.check(st, "cs_simulate_nested")
    k = int(nt.value)
    out = {name: t[:k].cpu().numpy() for name, t in (("home", home), ("entry", entry), ("parent", parent),
                                                      ("pred_a", pa), ("pred_b", pb), ("start", start))}
    return out, int(mk.value)


def simulate_dynamic(plan: NestedPlan, cfg: SimConfig) -> SimResult:
    """Schedule a nested plan with spawning (schedsim.py:93-163).  The result
    carries the realized graph and the spawn log, as in the reference."""
    from .grid import neighbor

    arr, makespan = nested_device(plan, cfg.workers)
    grid, offs = plan.grid, plan.order.offsets
    tasks, log = [], []
    for tid, (h, e, par) in enumerate(zip(arr["home"].tolist(), arr["entry"].tolist(),
                                          arr["parent"].tolist())):
        off = offs[e]
        if e == 0:
            t = Task(tid, INTRA, h, None, frozenset((accumulator(h),)))
        else:
            nb = neighbor(h, off, grid)
            t = Task(tid, INTER, h, off, frozenset((accumulator(h), accumulator(nb))))
        tasks.append(t)
        log.append(SpawnRecord(t, None if par < 0 else par, True))
    edges = []
    for v, (a, b) in enumerate(zip(arr["pred_a"].tolist(), arr["pred_b"].tolist())):
        for p in (a, b):
            if p >= 0:
                edges.append((p, v))
    graph = TaskGraph(tasks, tuple(edges))
    return SimResult(makespan=makespan, serial_time=len(tasks), workers=cfg.workers,
                     timeline=_timeline(arr["start"], cfg.workers), graph=graph, spawn_log=log,
                     start=arr["start"])


def speedup_curve(subject, workers: list[int]) -> list:
    """One simulation per worker count (schedsim.py:166-176)."""
    run = simulate_dynamic if isinstance(subject, NestedPlan) else simulate
    return [(w, run(subject, SimConfig(w))) for w in workers]


def unlimited_workers(subject) -> SimConfig:
    """A worker count that is never the bottleneck (schedsim.py:179-185)."""
    if isinstance(subject, NestedPlan):
        n = subject.grid.cell_count * subject.order.n
    else:
        n = subject.task_count
    return SimConfig(max(1, n))
