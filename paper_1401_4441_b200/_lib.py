"""ctypes binding of the C ABI in include/cellsched_b200.h.

This is the whole host<->device boundary: plain pointers, sizes and a
cudaStream_t.  torch is used only to own device memory and streams.  There is
no CPU fallback: if the shared library is missing or no CUDA device is
present, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os

from ._build import LIB

CS_OK = 0
CS_EINVAL = -1
CS_ECAPACITY = -2
CS_ECONFLICT = -3
CS_ERANGE = -4
CS_ECYCLE = -5

STREAM_BASIC, STREAM_LOOPEX = 0, 1
SCHED_LOOPEX, SCHED_BLOCK, SCHED_SHELL, SCHED_BUFFERED, SCHED_DATAFLOW = 0, 1, 2, 3, 4


class CsGrid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("ext", C.c_int32 * 3), ("periodic", C.c_int32 * 3)]


class CsBox(C.Structure):
    _fields_ = [
        ("nc", C.c_int32 * 3),
        ("gnc", C.c_int32 * 3),
        ("x0", C.c_int32),
        ("owned_x", C.c_int32),
        ("periodic", C.c_int32 * 3),
        ("block", C.c_int32 * 3),
        ("L", C.c_double * 3),
        ("inv", C.c_double * 3),
    ]


class CsLJ(C.Structure):
    _fields_ = [("eps", C.c_double), ("sigma", C.c_double), ("rc", C.c_double), ("mass", C.c_double)]


class CellschedError(RuntimeError):
    """Raised when a device call fails (the reference raises RuntimeError on
    contract violations, depgraph.py:139-154)."""


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double
_SZ = C.c_size_t

_SIGS = {
    "cs_abi_version": (C.c_int, []),
    "cs_last_error": (C.c_char_p, []),
    "cs_device_synchronize": (C.c_int, []),
    "cs_stream_count": (_I64, [_P, C.c_int, _P, C.c_int, C.c_int]),
    "cs_stream_ws_bytes": (_SZ, [_P, C.c_int]),
    "cs_stream_generate": (C.c_int, [_P, C.c_int, _P, C.c_int, C.c_int, _P, _P, _P, _I64, _P, _SZ, _P]),
    "cs_edges_ws_bytes": (_SZ, [_P, C.c_int, _I64]),
    "cs_stream_edges": (C.c_int, [_P, C.c_int, _P, C.c_int, C.c_int, _P, _P, _I64, _P, _P, _P, _P, _SZ, _P]),
    "cs_edges_compact": (C.c_int, [_I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "cs_depth_ws_bytes": (_SZ, [_I64]),
    "cs_stream_depth": (C.c_int, [_P, C.c_int, C.c_int, _I64, _P, _P, _P, _P, _P, C.c_int, _P, _P, _SZ, _P]),
    "cs_payload_charges": (C.c_int, [_P, _I64, _P, _P]),
    "cs_payload_direct": (C.c_int, [_P, _I64, _P, _P, _P]),
    "cs_payload_levels_ws_bytes": (_SZ, [_I64, _I64]),
    "cs_payload_levels": (C.c_int, [_P, _P, _I64, _P, _P, _P, _P, C.c_int, _P, _I64, _P, _P, _SZ, _P]),
    "cs_payload_colour": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, _P, _SZ, _P]),
    "cs_payload_colour_ws_bytes": (_SZ, [_P]),
    "cs_init_fcc": (C.c_int, [_P, _P, _P, _D, _I64, _P, _P, _P, _P, _P]),
    "cs_reduce_ws_bytes": (_SZ, [_I64]),
    "cs_init_velocities": (C.c_int, [_I64, _D, _D, _I64, _P, _P, _P, _P, _SZ, _P]),
    "cs_bin_ws_bytes": (_SZ, [_I64, _P]),
    "cs_build_cells": (C.c_int, [_I64, _P] + [_P] * 18 + [_P, _SZ, _P]),
    "cs_bin_errors": (C.c_int, [_I64, _P, _P, _SZ, _P, _P]),
    "cs_memset_async": (C.c_int, [_P, C.c_int, _SZ, _P]),
    "cs_copy_async": (C.c_int, [_P, _P, _SZ, _P]),
    "cs_accumulate_i64": (C.c_int, [_P, _P, _P]),
    "cs_force_ws_bytes": (_SZ, [_P, C.c_int, _I64]),
    "cs_lj_forces": (C.c_int, [_P, _P, C.c_int, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "cs_vv_kick_predict": (C.c_int, [_I64, _D, _D, C.c_int] + [_P] * 12 + [_D, _P, _P]),
    "cs_vv_kick": (C.c_int, [_I64, _D, _P, _P, _P, _P, _P, _P, _P]),
    "cs_vv_kick_drift": (C.c_int, [_I64, _D, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "cs_kinetic": (C.c_int, [_I64, _D, _P, _P, _P, _P, _P, _SZ, _P]),
    "cs_sum3": (C.c_int, [_I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "cs_verlet_list_bytes": (_SZ, [_P]),
    "cs_verlet_build": (C.c_int, [_P, _P, _D, _P, _P, _P, _P, _P, _SZ, _P, _P, _P, _I64, _P, _P]),
    "cs_lj_forces_verlet": (C.c_int, [_P, _P, C.c_int, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "cs_wrap_positions": (C.c_int, [_I64, _P, _P, _P, _P, _P]),
    "cs_vv_kick_drift_track": (C.c_int, [_I64, _D, _D] + [_P] * 12 + [_D, _P, _P]),
    "cs_copy7": (C.c_int, [_I64] + [_P] * 15),
    "cs_capture_if_begin": (C.c_int, [_P, _P, _P, _P]),
    "cs_capture_if_end": (C.c_int, [_P]),
    "cs_pack_plane": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _D, _P, _P]),
    "cs_add_plane_forces": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _P, _P]),
    "cs_probe_dfma": (C.c_int, [C.c_int, C.c_int, _P, _P]),
    "cs_detect_ws_bytes": (_SZ, [_I64, _I64, _I64]),
    "cs_detect_generic": (C.c_int, [_I64, _I64, _I64, _P, _P, _P, _P, _I64, _P, _P, _SZ, _P]),
    "cs_detect_generic_emit": (C.c_int, [_I64, _I64, _P, _I64, _P, _P, _P, _SZ, _P]),
    "cs_longest_path_ws_bytes": (_SZ, [_I64]),
    "cs_longest_path": (C.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "cs_payload_generic_ws_bytes": (_SZ, [_I64, _I64]),
    "cs_payload_generic": (C.c_int, [_I64, C.c_int] + [_P] * 10 + [_I64, _I64, _P, _P, _SZ, _P]),
    "cs_dag_ws_bytes": (_SZ, [_I64, _I64]),
    "cs_dag_execute": (C.c_int, [_I64, C.c_int] + [_P] * 9 + [_I64, _P, _P, _P, _I64, _P, C.c_int, _P, _P, _SZ, _P]),
    "cs_listsched_ws_bytes": (_SZ, [_I64]),
    "cs_simulate_static": (C.c_int, [_I64, _I64, _P, _P, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "cs_nested_ws_bytes": (_SZ, [_P, C.c_int]),
    "cs_simulate_nested": (C.c_int, [_P, _P, C.c_int, _I64] + [_P] * 6 + [_I64, _P, _P, _P, _SZ, _P]),
    "cs_slab_ws_bytes": (_SZ, [_I64]),
    "cs_slab_split": (C.c_int, [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _I64, _P, _P, _SZ, _P]),
    "cs_unpack7": (C.c_int, [_I64, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "cs_plane_counts": (C.c_int, [_P, C.c_int, _P, _P, _P, _P]),
    "cs_ghost_ws_bytes": (_SZ, [_P]),
    "cs_pack_range": (C.c_int, [_I64, _I64, _P, _P, _P, _D, _P, _P]),
    "cs_add_range_forces": (C.c_int, [_I64, _I64, _P, _P, _P, _P, _P]),
    "cs_set_ghost_plane": (C.c_int, [_P, _I64, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
}

EXPORTS = tuple(_SIGS)

_lib = None


def load(path: str | None = None):
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        # (CELLSCHED_B200_LIB: load a differently built copy, for kernel experiments)
        p = path or os.environ.get("CELLSCHED_B200_LIB") or LIB
        if not os.path.exists(p):
            raise ImportError(
                f"{p} not found: build it with `python -m paper_1401_4441_b200._build` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(p)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int, what: str = "") -> None:
    if status == CS_OK:
        return
    msg = load().cs_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == CS_EINVAL:
        raise ValueError(text)
    raise CellschedError(f"{text} (status {status})")


def call(name: str, *args):
    """Invoke an int-returning entry point and raise on failure."""
    st = getattr(load(), name)(*args)
    check(st, name)
    return st


def ptr(t) -> C.c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())


def hptr(obj) -> C.c_void_p:
    """Host pointer of a ctypes object / array."""
    return C.cast(C.pointer(obj), C.c_void_p) if not isinstance(obj, C.Array) else C.cast(obj, C.c_void_p)


def stream_handle(stream=None) -> C.c_void_p:
    """cudaStream_t of `stream` or of torch's current stream on the current
    device (raw-handle fast path: this sits in front of every kernel launch)."""
    import torch

    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return C.c_void_p(raw(torch._C._cuda_getDevice()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise CellschedError("no CUDA device: the B200 path has no CPU fallback")
    load()
