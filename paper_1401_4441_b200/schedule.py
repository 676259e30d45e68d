"""Device-resident task streams, dependency edges and serialization depth (K4).

The array form of the reference's stream / graph API: a stream is three
device arrays (home, nbr, entry) in creation order, edges are (pred_a,
pred_b) per task, and the serialization depth (`critical_path`,
depgraph.py:160-174) is computed on the device.  `to_tasks()` /
`to_graph()` materialise the reference's Python objects for small grids.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import GridSpec, Offset, canonical_half_stencil, zero_offset

_STRATS = {"basic": _lib.STREAM_BASIC, "loopex": _lib.STREAM_LOOPEX}


def _torch():
    import torch

    return torch


def _order_array(order_offsets, dim):
    arr = (C.c_int8 * (len(order_offsets) * dim))()
    for e, off in enumerate(order_offsets):
        for k in range(dim):
            arr[e * dim + k] = int(off[k])
    return arr


@dataclass
class DeviceStream:
    """A task stream held as device arrays."""

    grid: GridSpec
    strategy: str
    stride: int
    entries: tuple[Offset, ...]  # what entry[t] indexes
    home: object  # torch.int32 [ntasks]
    nbr: object  # torch.int32 [ntasks], -1 for intra
    entry: object  # torch.int16 [ntasks]
    _edges: tuple | None = field(default=None, repr=False)
    _levels: tuple | None = field(default=None, repr=False)

    @property
    def ntasks(self) -> int:
        return int(self.home.numel())

    def _args(self):
        g = self.grid._cs_grid()
        order = _order_array(self.entries, self.grid.dim)
        return g, order

    # ---------------------------------------------------------------- edges
    def edges(self):
        """(pred_a, pred_b, edge_count): each task's <= 2 predecessors,
        pred_a < pred_b, -1 = none (detect_dependencies, depgraph.py:102-117)."""
        if self._edges is None:
            torch = _torch()
            g, order = self._args()
            n = len(self.entries)
            strat = _STRATS[self.strategy]
            pa = torch.empty(self.ntasks, dtype=torch.int32, device=self.home.device)
            pb = torch.empty_like(pa)
            wsb = _lib.load().cs_edges_ws_bytes(C.byref(g), n, self.ntasks)
            ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=self.home.device)
            ne = C.c_int64()
            _lib.call("cs_stream_edges", C.byref(g), strat, order, n, self.stride,
                      _lib.ptr(self.home), _lib.ptr(self.nbr), self.ntasks, _lib.ptr(pa),
                      _lib.ptr(pb), C.byref(ne), _lib.ptr(ws), wsb, _lib.stream_handle())
            self._edges = (pa, pb, int(ne.value))
        return self._edges

    def edge_arrays(self):
        """(eu, ev) int64 device arrays sorted by (succ, pred)."""
        torch = _torch()
        pa, pb, ne = self.edges()
        eu = torch.empty(max(ne, 1), dtype=torch.int64, device=self.home.device)
        ev = torch.empty_like(eu)
        g, _ = self._args()
        wsb = _lib.load().cs_edges_ws_bytes(C.byref(g), len(self.entries), self.ntasks)
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=self.home.device)
        _lib.call("cs_edges_compact", self.ntasks, _lib.ptr(pa), _lib.ptr(pb), _lib.ptr(eu),
                  _lib.ptr(ev), _lib.ptr(ws), wsb, _lib.stream_handle())
        return eu[:ne], ev[:ne]

    # ---------------------------------------------------------------- depth
    def levels(self, method: str = "auto"):
        """(level[t], depth): longest path ending at t, and the serialization
        depth (critical_path, depgraph.py:160-174)."""
        if self._levels is None or method != "auto":
            torch = _torch()
            pa, pb, _ = self.edges()
            g, _ = self._args()
            lv = torch.empty(self.ntasks, dtype=torch.int32, device=self.home.device)
            wsb = _lib.load().cs_depth_ws_bytes(self.grid.cell_count + self.ntasks)
            ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=self.home.device)
            depth = C.c_int64()
            m = {"relax": 0, "chain": 1, "auto": 2}[method]
            _lib.call("cs_stream_depth", C.byref(g), _STRATS[self.strategy], len(self.entries),
                      self.ntasks, _lib.ptr(self.home), _lib.ptr(self.nbr), _lib.ptr(pa),
                      _lib.ptr(pb), _lib.ptr(lv), m, C.byref(depth), _lib.ptr(ws), wsb,
                      _lib.stream_handle())
            res = (lv, int(depth.value))
            if method != "auto":
                return res
            self._levels = res
        return self._levels

    def depth(self) -> int:
        return self.levels()[1]

    # -------------------------------------------------------- materialising
    def to_tasks(self):
        """Reference-style list[Task] (taskgen.py:51-66); small grids only."""
        from .taskgen import INTER, INTRA, Task, TaskList, accumulator

        home = self.home.cpu().numpy()
        nbr = self.nbr.cpu().numpy()
        entry = self.entry.cpu().numpy()
        out = TaskList()
        for t in range(self.ntasks):
            h, nb = int(home[t]), int(nbr[t])
            if nb < 0:
                out.append(Task(t, INTRA, h, None, frozenset((accumulator(h),))))
            else:
                off = self.entries[int(entry[t])]
                out.append(Task(t, INTER, h, off, frozenset((accumulator(h), accumulator(nb)))))
        out.device_stream = self
        return out


def device_stream(grid: GridSpec, strategy: str = "loopex", order=None, stride: int = 2,
                  device=None) -> DeviceStream:
    """Generate a stream on the device.  strategy 'basic' (generate_basic,
    taskgen.py:180-199; order defaults to canonical) or 'loopex'
    (generate_loopex, taskgen.py:202-234; `stride` > 2 is the stride-k
    colour generalisation used for the 3x3x3 colour order)."""
    torch = _torch()
    _lib.require_cuda()
    if strategy not in _STRATS:
        raise ValueError(f"device streams support {tuple(_STRATS)}, got {strategy!r}")
    dim = grid.dim
    if strategy == "basic":
        from .taskgen import StencilOrder

        order = order if order is not None else StencilOrder.canonical(dim)
        if order.dim != dim:
            raise ValueError(f"order is {order.dim}D but grid is {dim}D")
        entries = tuple(order.offsets)
    else:
        entries = tuple(canonical_half_stencil(dim).offsets)
    g = grid._cs_grid()
    oarr = _order_array(entries, dim)
    strat = _STRATS[strategy]
    nt = _lib.load().cs_stream_count(C.byref(g), strat, oarr, len(entries), stride)
    if nt < 0:
        _lib.check(_lib.CS_EINVAL, "cs_stream_count")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    home = torch.empty(max(nt, 1), dtype=torch.int32, device=dev)[:nt]
    nbr = torch.empty(max(nt, 1), dtype=torch.int32, device=dev)[:nt]
    entry = torch.empty(max(nt, 1), dtype=torch.int16, device=dev)[:nt]
    wsb = _lib.load().cs_stream_ws_bytes(C.byref(g), len(entries))
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    _lib.call("cs_stream_generate", C.byref(g), strat, oarr, len(entries), stride,
              _lib.ptr(home), _lib.ptr(nbr), _lib.ptr(entry), nt, _lib.ptr(ws), wsb,
              _lib.stream_handle())
    return DeviceStream(grid, strategy, stride, entries, home, nbr, entry)


def serialization_depth(grid: GridSpec, strategy: str = "basic", order=None, stride: int = 2) -> int:
    """critical_path(detect_dependencies(generate(strategy, grid, order)))
    computed entirely on the device."""
    return device_stream(grid, strategy, order, stride).depth()


def degree_of_serialization(grid: GridSpec, strategy: str = "basic", order=None,
                            stride: int = 2) -> float:
    """S = tasks / depth (PAPER Eq. 1; = SimResult.speedup at W = inf)."""
    s = device_stream(grid, strategy, order, stride)
    return s.ntasks / s.depth()
