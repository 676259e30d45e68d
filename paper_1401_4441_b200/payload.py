"""Integer interaction payload, mirroring `cellsched.payload` (K5).

Bit-exact device restatement of /root/reference/pkg/src/cellsched/payload.py:
splitmix64 charges (:58-61), intra term (:64-66), antisymmetric pair term
(:69-81), task replay (apply_tasks, :84-119), strategy dispatch
(execute_with_payload, :122-144) and the direct oracle (reference_oracle,
:152-174).  The scalar helpers below are exact Python integers (one value
each); every per-grid computation runs on the device.
"""

from __future__ import annotations

import ctypes as C

from . import _lib
from .grid import GridSpec, Offset, negate

_MASK64 = (1 << 64) - 1
_PAIR_KEY = 0xA0761D6478BD642F
_INTRA_KEY = 0x2545F4914F6CDD1D


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def _center32(x: int) -> int:
    return (x & 0xFFFFFFFF) - (1 << 31)


def _code(offset: Offset) -> int:
    return sum((c + 1) * 3**k for k, c in enumerate(offset))


def intra_contribution(charge: int) -> int:
    return _center32(_splitmix64(_INTRA_KEY ^ (charge & _MASK64)))


def _mix(a: int, b: int, offset: Offset) -> int:
    h = _splitmix64(_PAIR_KEY ^ (a & _MASK64))
    h = _splitmix64(h ^ (b & _MASK64))
    return _splitmix64(h ^ _code(offset)) & 0x7FFFFFFF


def pair_contribution(charge_a: int, charge_b: int, offset: Offset) -> tuple[int, int]:
    g = _mix(charge_a, charge_b, offset) - _mix(charge_b, charge_a, negate(offset))
    return g, -g


# ------------------------------------------------------------------ device --
def _torch():
    import torch

    return torch


def charges_device(grid: GridSpec, seed: int):
    torch = _torch()
    _lib.require_cuda()
    q = torch.empty(grid.cell_count, dtype=torch.int64, device="cuda")
    g = grid._cs_grid()
    _lib.call("cs_payload_charges", C.byref(g), _signed64(int(seed)),
              _lib.ptr(q), _lib.stream_handle())
    return q


def charges(grid: GridSpec, seed: int) -> list[int]:
    return charges_device(grid, _signed64(seed)).cpu().tolist()


def _signed64(seed: int) -> int:
    s = seed & _MASK64
    return s - (1 << 64) if s >= (1 << 63) else s


def _acc_dict(acc, grid):
    vals = acc.cpu().tolist()
    return {c: vals[c] for c in grid.cells()}


def reference_oracle_device(grid: GridSpec, seed: int):
    torch = _torch()
    q = charges_device(grid, _signed64(seed))
    acc = torch.empty_like(q)
    g = grid._cs_grid()
    _lib.call("cs_payload_direct", C.byref(g), 0, _lib.ptr(q), _lib.ptr(acc), _lib.stream_handle())
    return acc


def reference_oracle(grid: GridSpec, seed: int) -> dict[int, int]:
    """Direct full-neighbourhood sum, no task machinery (payload.py:152-174)."""
    return _acc_dict(reference_oracle_device(grid, seed), grid)


def apply_stream_device(stream, seed: int):
    """apply_tasks over a DeviceStream: executed level by level along its own
    dependency levels (tasks of one level are write-disjoint), no atomics."""
    torch = _torch()
    grid = stream.grid
    q = charges_device(grid, _signed64(seed))
    acc = torch.empty_like(q)
    lv, depth = stream.levels()
    g = grid._cs_grid()
    from .schedule import _order_array

    offs = _order_array(stream.entries, grid.dim)
    wsb = _lib.load().cs_payload_levels_ws_bytes(stream.ntasks, depth)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    _lib.call("cs_payload_levels", C.byref(g), _lib.ptr(q), stream.ntasks, _lib.ptr(stream.home),
              _lib.ptr(stream.nbr), _lib.ptr(stream.entry), offs, len(stream.entries),
              _lib.ptr(lv), depth, _lib.ptr(acc), _lib.ptr(ws), wsb, _lib.stream_handle())
    return acc


def apply_tasks(tasks, grid: GridSpec, seed: int) -> dict[int, int]:
    """Apply each task's contribution once (payload.py:84-119)."""
    ds = getattr(tasks, "device_stream", None)
    if ds is None:
        from .generic import apply_tasks_generic

        return apply_tasks_generic(tasks, grid, seed)
    return _acc_dict(apply_stream_device(ds, seed), grid)


def execute_with_payload(strategy: str, grid: GridSpec, seed: int, order=None,
                         workers: int | None = None) -> dict[int, int]:
    """Run a strategy's stream and return the accumulators (payload.py:122-144).

    The device executes the stream level by level (the W = infinity schedule);
    integer addition commutes, so the result equals any W's replay order."""
    from .taskgen import generate

    if strategy in ("basic", "loopex"):
        from .schedule import device_stream

        if strategy == "basic":
            from .taskgen import StencilOrder

            order = order if order is not None else StencilOrder.canonical(grid.dim)
            if order.dim != grid.dim:
                raise ValueError(f"order is {order.dim}D but grid is {grid.dim}D")
        return _acc_dict(apply_stream_device(device_stream(grid, strategy, order), seed), grid)
    return apply_tasks(generate(strategy, grid, order), grid, seed)


def colour_pass_payload(grid: GridSpec, seed: int, schedule: str = "block", block=(2, 2, 2),
                        race_check: bool = True):
    """The integer payload under the LJ kernel's colour-pass schedule
    ('loopex' = 27 passes, 'block' = 8 block passes); raises on a detected
    same-pass writer conflict.  Returns the accumulators as a device tensor."""
    torch = _torch()
    q = charges_device(grid, _signed64(seed))
    acc = torch.empty_like(q)
    g = grid._cs_grid()
    blk = (C.c_int32 * 3)(*block)
    wsb = _lib.load().cs_payload_colour_ws_bytes(C.byref(g))
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    sched = {"loopex": _lib.SCHED_LOOPEX, "block": _lib.SCHED_BLOCK}[schedule]
    _lib.call("cs_payload_colour", C.byref(g), sched, blk, _lib.ptr(q), _lib.ptr(acc),
              int(race_check), _lib.ptr(ws), wsb, _lib.stream_handle())
    return acc


def conservation_defect(acc: dict[int, int], grid: GridSpec, seed: int) -> int:
    """Sum of accumulators minus the intra terms (payload.py:177-181)."""
    q = charges(grid, seed)
    return sum(acc.values()) - sum(intra_contribution(q[c]) for c in grid.cells())
