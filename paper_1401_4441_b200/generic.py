"""Generic (non-accumulator) task lists on the device.

Arbitrary resources and read-only inputs (e.g. the buffered strategy's
reduce tasks, or hand-built graphs) are interned to dense integer ids on the
host and resolved by device kernels implementing _DependenceState.add
(depgraph.py:28-49).
"""

from __future__ import annotations


def detect_edges_generic(tasks):
    raise NotImplementedError("generic device dependency detection is not built yet")


def longest_path_device(ntasks, edges, return_levels=False):
    raise NotImplementedError("generic device longest path is not built yet")


def apply_tasks_generic(tasks, grid, seed):
    raise NotImplementedError("generic device payload replay is not built yet")
