"""ctypes wrapper for the CPU oracle (oracle/libcs_oracle.so).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Importable only
from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.  See
cs_oracle.c for what each function restates (reference file:line) and for
the parity-pinning status (schedule/payload pinned to reference golden
vectors; LJ parity unpinned w.r.t. the reference, which has no LJ code).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcs_oracle.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_P = C.c_void_p

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.o_neighbor.restype = C.c_int64
        L.o_neighbor.argtypes = [C.c_int64, _i8p, _i32p, _i32p, C.c_int]
        L.o_color.restype = C.c_int
        L.o_color.argtypes = [C.c_int64, _i32p, C.c_int, C.c_int]
        L.o_canonical_stencil.restype = C.c_int
        L.o_canonical_stencil.argtypes = [C.c_int, _i8p]
        L.o_stream_basic.restype = C.c_int64
        L.o_stream_basic.argtypes = [_i32p, _i32p, C.c_int, _i8p, C.c_int, _P, _P, _P]
        L.o_stream_loopex.restype = C.c_int64
        L.o_stream_loopex.argtypes = [_i32p, _i32p, C.c_int, C.c_int, _P, _P, _P]
        L.o_detect_edges.restype = C.c_int64
        L.o_detect_edges.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _i64p, _i64p, _P, _P]
        L.o_critical_path.restype = C.c_int64
        L.o_critical_path.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _P]
        L.o_splitmix64.restype = C.c_uint64
        L.o_splitmix64.argtypes = [C.c_uint64]
        L.o_charges.argtypes = [_i32p, C.c_int, C.c_int64, _i64p]
        L.o_payload_reference.argtypes = [_i32p, _i32p, C.c_int, C.c_int64, _i64p]
        L.o_payload_apply.argtypes = [_i32p, _i32p, C.c_int, C.c_int64, C.c_int64, _i32p, _i32p,
                                      _i16p, _i8p, _i64p]
        L.o_fcc_positions.argtypes = [_i32p, _f64p, _f64p, C.c_double, C.c_int64, _f64p, _f64p, _f64p]
        L.o_velocities.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_int64, _f64p, _f64p, _f64p]
        L.o_bin.argtypes = [C.c_int64, _f64p, _f64p, _f64p, _P, _i32p, _f64p, _i32p, _i32p, _i32p]
        L.o_lj_direct.argtypes = [_i32p, _i32p, _f64p, _f64p, _i32p, _f64p, _f64p, _f64p,
                                  _f64p, _f64p, _f64p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.o_lj_tasks.argtypes = [_i32p, _i32p, _f64p, _f64p, _i32p, _f64p, _f64p, _f64p, C.c_int64,
                                 _i32p, _i32p, _i16p, _i8p, _f64p, _f64p, _f64p,
                                 C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.o_lj_brute.argtypes = [C.c_int64, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p,
                                 C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.o_lj_loopex_threads.argtypes = [_i32p, _f64p, _f64p, _i32p, _f64p, _f64p, _f64p, _f64p,
                                          _f64p, _f64p, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_int64)]
        L.o_kick.argtypes = [C.c_int64, C.c_double, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p]
        L.o_drift.argtypes = [C.c_int64, C.c_double, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p]
        L.o_kinetic.restype = C.c_double
        L.o_kinetic.argtypes = [C.c_int64, C.c_double, _f64p, _f64p, _f64p]
        L.o_md_run.argtypes = [C.c_int64, _i32p, _f64p, _f64p, C.c_double, C.c_double, C.c_int,
                               C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _i32p,
                               _f64p, _f64p, _f64p, _i32p, _f64p, _f64p]
        L.o_md_steps.argtypes = [C.c_int64, _i32p, _f64p, _f64p, C.c_double, C.c_double, C.c_int,
                                 C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _i32p,
                                 _f64p, _f64p, _f64p, _i32p, _f64p, _f64p, _i64p]
        L.o_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _ext(extents):
    e = np.zeros(3, np.int32)
    e[: len(extents)] = extents
    return e


def _per(periodic, dim):
    if isinstance(periodic, (bool, int, np.bool_)):
        periodic = [bool(periodic)] * dim
    p = np.zeros(3, np.int32)
    p[:dim] = [int(x) for x in periodic]
    return p


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------- schedule --
def canonical_stencil(dim):
    out = np.zeros(27 * 3, np.int8)
    n = lib().o_canonical_stencil(dim, out)
    return out[: n * dim].reshape(n, dim).copy()


def stream_basic(extents, periodic, order):
    dim = len(extents)
    order = np.ascontiguousarray(np.asarray(order, np.int8).reshape(-1, dim))
    e, p = _ext(extents), _per(periodic, dim)
    n = lib().o_stream_basic(e, p, dim, order.ravel(), len(order), None, None, None)
    h, nb, en = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int16)
    lib().o_stream_basic(e, p, dim, order.ravel(), len(order), _ptr(h), _ptr(nb), _ptr(en))
    return h, nb, en


def stream_loopex(extents, periodic=True, stride=2):
    dim = len(extents)
    e, p = _ext(extents), _per(periodic, dim)
    n = lib().o_stream_loopex(e, p, dim, stride, None, None, None)
    h, nb, en = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int16)
    lib().o_stream_loopex(e, p, dim, stride, _ptr(h), _ptr(nb), _ptr(en))
    return h, nb, en


def detect_edges_csr(ntasks, nres, wptr, wres, rptr, rres):
    a = [np.ascontiguousarray(x, np.int64) for x in (wptr, wres, rptr, rres)]
    ne = lib().o_detect_edges(ntasks, nres, *a, None, None)
    eu, ev = np.zeros(ne, np.int64), np.zeros(ne, np.int64)
    lib().o_detect_edges(ntasks, nres, *a, _ptr(eu), _ptr(ev))
    return eu, ev


def detect_edges_stream(home, nbr):
    """inout accumulator stream -> edges (each task writes acc(home), acc(nbr))."""
    n = len(home)
    home = np.asarray(home, np.int64)
    nbr = np.asarray(nbr, np.int64)
    two = (nbr >= 0) & (nbr != home)
    cnt = 1 + two.astype(np.int64)
    wptr = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=wptr[1:])
    wres = np.zeros(wptr[-1], np.int64)
    wres[wptr[:-1]] = home
    wres[wptr[:-1][two] + 1] = nbr[two]
    nres = int(max(home.max(initial=-1), nbr.max(initial=-1)) + 1)
    zero = np.zeros(n + 1, np.int64)
    return detect_edges_csr(n, nres, wptr, wres, zero, np.zeros(0, np.int64))


def critical_path(ntasks, eu, ev, levels=False):
    eu = np.ascontiguousarray(eu, np.int64)
    ev = np.ascontiguousarray(ev, np.int64)
    lv = np.zeros(max(ntasks, 1), np.int64)
    d = lib().o_critical_path(ntasks, len(eu), eu, ev, _ptr(lv))
    return (d, lv[:ntasks]) if levels else d


# ---------------------------------------------------------------- payload --
def charges(extents, seed):
    e = _ext(extents)
    q = np.zeros(int(np.prod(extents)), np.int64)
    lib().o_charges(e, len(extents), int(seed), q)
    return q


def payload_reference(extents, periodic, seed):
    dim = len(extents)
    acc = np.zeros(int(np.prod(extents)), np.int64)
    lib().o_payload_reference(_ext(extents), _per(periodic, dim), dim, int(seed), acc)
    return acc


def payload_apply(extents, periodic, seed, home, nbr, entry, offsets):
    dim = len(extents)
    acc = np.zeros(int(np.prod(extents)), np.int64)
    offs = np.ascontiguousarray(np.asarray(offsets, np.int8).reshape(-1, dim)).ravel()
    lib().o_payload_apply(_ext(extents), _per(periodic, dim), dim, int(seed), len(home),
                          np.ascontiguousarray(home, np.int32), np.ascontiguousarray(nbr, np.int32),
                          np.ascontiguousarray(entry, np.int16), offs, acc)
    return acc


# --------------------------------------------------------------------- LJ --
def fcc_positions(nuc, a, L, jitter, seed):
    n = 4 * int(np.prod(nuc))
    x, y, z = (np.zeros(n) for _ in range(3))
    lib().o_fcc_positions(np.asarray(nuc, np.int32), np.asarray(a, np.float64),
                          np.asarray(L, np.float64), float(jitter), int(seed), x, y, z)
    return x, y, z


def velocities(n, T, mass, seed):
    vx, vy, vz = (np.zeros(n) for _ in range(3))
    lib().o_velocities(n, float(T), float(mass), int(seed), vx, vy, vz)
    return vx, vy, vz


def bin_cells(x, y, z, ids, nc, inv):
    n = len(x)
    nc = np.asarray(nc, np.int32)
    cell_of = np.zeros(n, np.int32)
    start = np.zeros(int(np.prod(nc)) + 1, np.int32)
    order = np.zeros(n, np.int32)
    idp = None if ids is None else _ptr(np.ascontiguousarray(ids, np.int32))
    lib().o_bin(n, x, y, z, idp, nc, np.asarray(inv, np.float64), cell_of, start, order)
    return cell_of, start, order


def _prm(eps, sigma, rc):
    return np.array([eps, sigma, rc], np.float64)


def lj_direct(nc, L, start, x, y, z, eps=1.0, sigma=1.0, rc=2.5, periodic=(1, 1, 1)):
    n = len(x)
    f = [np.zeros(n) for _ in range(3)]
    pe, npair = C.c_double(), C.c_int64()
    lib().o_lj_direct(np.asarray(nc, np.int32), np.asarray(periodic, np.int32),
                      np.asarray(L, np.float64), _prm(eps, sigma, rc),
                      np.ascontiguousarray(start, np.int32), x, y, z, *f, C.byref(pe), C.byref(npair))
    return np.stack(f, 1), pe.value, npair.value


def lj_tasks(nc, L, start, x, y, z, home, nbr, entry, offsets, eps=1.0, sigma=1.0, rc=2.5,
             periodic=(1, 1, 1)):
    n = len(x)
    f = [np.zeros(n) for _ in range(3)]
    pe, npair = C.c_double(), C.c_int64()
    offs = np.ascontiguousarray(np.asarray(offsets, np.int8).reshape(-1, 3)).ravel()
    lib().o_lj_tasks(np.asarray(nc, np.int32), np.asarray(periodic, np.int32),
                     np.asarray(L, np.float64), _prm(eps, sigma, rc),
                     np.ascontiguousarray(start, np.int32), x, y, z, len(home),
                     np.ascontiguousarray(home, np.int32), np.ascontiguousarray(nbr, np.int32),
                     np.ascontiguousarray(entry, np.int16), offs, *f, C.byref(pe), C.byref(npair))
    return np.stack(f, 1), pe.value, npair.value


def lj_brute(L, x, y, z, eps=1.0, sigma=1.0, rc=2.5):
    n = len(x)
    f = [np.zeros(n) for _ in range(3)]
    pe, npair = C.c_double(), C.c_int64()
    lib().o_lj_brute(n, np.asarray(L, np.float64), _prm(eps, sigma, rc), x, y, z, *f,
                     C.byref(pe), C.byref(npair))
    return np.stack(f, 1), pe.value, npair.value


def lj_loopex_threads(nc, L, start, x, y, z, nthreads=0, eps=1.0, sigma=1.0, rc=2.5):
    n = len(x)
    f = [np.zeros(n) for _ in range(3)]
    pe, npair = C.c_double(), C.c_int64()
    lib().o_lj_loopex_threads(np.asarray(nc, np.int32), np.asarray(L, np.float64),
                              _prm(eps, sigma, rc), np.ascontiguousarray(start, np.int32),
                              x, y, z, *f, int(nthreads), C.byref(pe), C.byref(npair))
    return np.stack(f, 1), pe.value, npair.value


def md_run(x, y, z, vx, vy, vz, ids, nc, L, nsteps, dt=0.005, mass=1.0, eps=1.0, sigma=1.0,
           rc=2.5, mode=0, nthreads=0):
    """Returns dict with cell-sorted x, v, id, f, cell_start and pe/ke per step."""
    n = len(x)
    arrs = [np.array(a, np.float64, copy=True) for a in (x, y, z, vx, vy, vz)]
    ids = np.array(ids, np.int32, copy=True)
    f = [np.zeros(n) for _ in range(3)]
    start = np.zeros(int(np.prod(nc)) + 1, np.int32)
    pe, ke = np.zeros(nsteps + 1), np.zeros(nsteps + 1)
    lib().o_md_run(n, np.asarray(nc, np.int32), np.asarray(L, np.float64), _prm(eps, sigma, rc),
                   mass, dt, nsteps, mode, nthreads, *arrs, ids, *f, start, pe, ke)
    return {"x": np.stack(arrs[:3], 1), "v": np.stack(arrs[3:], 1), "id": ids,
            "f": np.stack(f, 1), "cell_start": start, "pe": pe, "ke": ke}


class CpuMD:
    """Cell-sorted host state advanced by o_md_steps (CPU baseline)."""

    def __init__(self, x, y, z, vx, vy, vz, ids, nc, L, dt=0.005, mass=1.0, eps=1.0, sigma=1.0,
                 rc=2.5, nthreads=0):
        r = md_run(x, y, z, vx, vy, vz, ids, nc, L, 0, dt, mass, eps, sigma, rc, mode=1,
                   nthreads=nthreads)
        self.n = len(x)
        self.nc = np.asarray(nc, np.int32)
        self.L = np.asarray(L, np.float64)
        self.prm = _prm(eps, sigma, rc)
        self.dt, self.mass, self.nthreads = dt, mass, nthreads
        self.a = [np.ascontiguousarray(r["x"][:, k]) for k in range(3)]
        self.a += [np.ascontiguousarray(r["v"][:, k]) for k in range(3)]
        self.id = r["id"]
        self.f = [np.ascontiguousarray(r["f"][:, k]) for k in range(3)]
        self.start = r["cell_start"]

    def steps(self, k):
        pe, ke, npairs = np.zeros(k), np.zeros(k), np.zeros(k, np.int64)
        lib().o_md_steps(self.n, self.nc, self.L, self.prm, self.mass, self.dt, k, self.nthreads,
                         *self.a, self.id, *self.f, self.start, pe, ke, npairs)
        return pe, ke, npairs


def max_threads():
    return lib().o_max_threads()
