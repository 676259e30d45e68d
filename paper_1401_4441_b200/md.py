"""Lennard-Jones link-cell molecular dynamics on the B200 (K1, K2, K3, K6).

The reference has no particle code; this module
extends its idiom at the payload plug-in point (payload.py:84-174): frozen
dataclasses for parameters and geometry, x-fastest cell ids from
`grid.GridSpec`, ValueError on bad input.  A step is

    kick + drift + wrap (K3) -> cell list as a stable counting sort (K1)
    -> fp64 LJ half-shell forces with Newton-3 reaction writes under a
       conflict-free colour-pass schedule (K2) -> kick (K3) [-> energies, K6]

all on one CUDA stream, capturable in a CUDA graph.  Particles live in
cell-sorted SoA fp64 arrays (x, y, z, vx, vy, vz, fx, fy, fz) plus int32 ids,
ping-ponged between two buffers by the rebinning gather.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

from . import _lib
from .grid import GridSpec

SCHEDULES = {"loopex": _lib.SCHED_LOOPEX, "block": _lib.SCHED_BLOCK, "shell": _lib.SCHED_SHELL,
             "buffered": _lib.SCHED_BUFFERED,
             # the shell colour order as a dataflow: one persistent launch, each
             # block waits only for its lower-colour neighbour blocks
             "dataflow": _lib.SCHED_DATAFLOW,
             # Verlet lists on cells of edge >= rc + skin, under the
             # same block structures
             "verlet": _lib.SCHED_BUFFERED, "verlet_shell": _lib.SCHED_SHELL,
             "verlet_dataflow": _lib.SCHED_DATAFLOW}
VERLET_SCHEDULES = ("verlet", "verlet_shell", "verlet_dataflow")


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class LJParams:
    """U(r) = 4 eps [(sigma/r)^12 - (sigma/r)^6] for r < rc, unshifted."""

    epsilon: float = 1.0
    sigma: float = 1.0
    rc: float = 2.5
    mass: float = 1.0

    def __post_init__(self) -> None:
        if self.epsilon <= 0 or self.sigma <= 0 or self.rc <= 0 or self.mass <= 0:
            raise ValueError("LJ parameters must be positive")


@dataclass(frozen=True)
class LJBox:
    """Periodic orthorhombic box split into cells of edge >= rc."""

    lengths: tuple[float, float, float]
    cells: tuple[int, int, int]

    def __post_init__(self) -> None:
        object.__setattr__(self, "lengths", tuple(float(v) for v in self.lengths))
        object.__setattr__(self, "cells", tuple(int(v) for v in self.cells))
        if len(self.lengths) != 3 or len(self.cells) != 3:
            raise ValueError("LJ boxes are 3D")
        if min(self.cells) < 3:
            raise ValueError(f"link cells need >= 3 cells per axis, got {self.cells}")

    @classmethod
    def for_cutoff(cls, lengths, rc: float) -> "LJBox":
        cells = tuple(int(math.floor(L / rc)) for L in lengths)
        return cls(tuple(lengths), cells)

    @property
    def grid(self) -> GridSpec:
        return GridSpec(self.cells)

    @property
    def cell_edge(self) -> tuple[float, ...]:
        return tuple(L / n for L, n in zip(self.lengths, self.cells))

    @property
    def inv(self) -> tuple[float, ...]:
        # binning factor, computed once on the host and shared with the oracle
        return tuple(float(n) / L for L, n in zip(self.lengths, self.cells))

    @property
    def cell_count(self) -> int:
        return self.cells[0] * self.cells[1] * self.cells[2]


def fcc_box(n_unit_cells, density: float, rc: float = 2.5):
    """Box holding n^3 FCC unit cells (4 sites each) at `density`; returns
    (box, unit-cell edges)."""
    nuc = tuple(int(v) for v in (n_unit_cells if hasattr(n_unit_cells, "__len__") else (n_unit_cells,) * 3))
    a = (4.0 / density) ** (1.0 / 3.0)
    lengths = tuple(n * a for n in nuc)
    return LJBox.for_cutoff(lengths, rc), nuc, (a, a, a)


def liquid_vapour_positions(cells=(64, 64, 192), edge: float = 2.5, rho_liquid: float = 0.8,
                            rho_vapour: float = 0.02, rmin: float = 0.9, seed: int = 42):
    """BASELINE configs[4] (cfg5): a periodic box of cells x edge; the middle
    third along z holds an FCC liquid, the rest a uniform-random vapour with
    no pair closer than rmin.  Host set-up (numpy + scipy's periodic KD-tree),
    deterministic in `seed`.  Returns (lengths, xyz[n, 3]); liquid first.

    The liquid is a cubic FCC lattice that tiles x and y exactly, with the
    number of unit cells closest to rho_liquid (cfg5: 94 per 160 sigma, density
    0.811), filling 94 unit cells of the middle third along z.  Vapour
    candidates are drawn in batches; one closer than rmin to the liquid, to an
    accepted vapour particle or to an earlier candidate of its batch is
    redrawn (a deterministic batch form of rejection sampling)."""
    import numpy as np
    from scipy.spatial import cKDTree

    L = np.asarray(cells, np.float64) * edge
    if abs(L[0] - L[1]) > 1e-12:
        raise ValueError("the liquid lattice needs equal x and y extents")
    a0 = (4.0 / rho_liquid) ** (1.0 / 3.0)
    nx = max(1, int(round(L[0] / a0)))
    a = L[0] / nx
    nz = max(1, min(int(round(L[2] / 3.0 / a)), int(L[2] // a)))
    z0 = (L[2] - nz * a) / 2.0
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(nx), np.arange(nz), indexing="ij")
    basis = np.array([[0, 0, 0], [0, 0.5, 0.5], [0.5, 0, 0.5], [0.5, 0.5, 0]])
    cell = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], 1).astype(np.float64)
    liquid = ((cell[:, None, :] + basis[None, :, :] + 0.25) * a).reshape(-1, 3)
    liquid[:, 2] += z0
    vap_h = L[2] - nz * a
    nv = int(round(rho_vapour * L[0] * L[1] * vap_h))
    rng = np.random.default_rng(seed)
    tree_l = cKDTree(liquid, boxsize=L)
    vap = np.zeros((0, 3))
    while len(vap) < nv:
        cand = rng.random((nv - len(vap), 3)) * np.array([L[0], L[1], vap_h])
        cand[:, 2] = np.where(cand[:, 2] < z0, cand[:, 2], cand[:, 2] + nz * a)
        cand = np.mod(cand, L)
        ok = tree_l.query(cand, distance_upper_bound=rmin)[0] >= rmin
        if len(vap):
            ok &= cKDTree(vap, boxsize=L).query(cand, distance_upper_bound=rmin)[0] >= rmin
        bad = set()
        for i, j in sorted(cKDTree(cand, boxsize=L).query_pairs(rmin)):
            if i not in bad:
                bad.add(j)
        if bad:
            ok[sorted(bad)] = False
        vap = np.concatenate([vap, cand[ok]])
    return tuple(float(v) for v in L), np.concatenate([liquid, vap])


def verlet_box(lengths, rc: float, skin: float):
    """Cells for the Verlet schedules: edge >= rc + skin, a multiple of 4 per
    axis (the 2x2x2 block colouring), at least 4.  A box too small for 4
    cells of rc + skin (cfg1: L = 10.08, rc + 0.35 = 2.85) keeps 4 cells and
    narrows the skin to the widest the cells allow (cfg1: L/4 - rc = 0.0194),
    with a UserWarning -- the list is then rebuilt every few steps.  Returns
    (box, skin)."""
    import warnings

    fit = [int(math.floor(L / (rc + skin))) for L in lengths]
    box = LJBox(tuple(lengths), tuple(max(4, c - c % 4) for c in fit))
    edge = min(box.cell_edge)
    if edge < (rc + skin) * (1 - 1e-12):
        if edge <= rc:
            raise ValueError(f"box {box.lengths} is too small for 4 cells of edge > rc = {rc}")
        narrowed = edge - rc
        warnings.warn(f"4 cells of edge {edge:.6g} cannot hold rc + skin = {rc + skin:.6g}; "
                      f"using skin {narrowed:.6g}", stacklevel=3)
        skin = narrowed
    return box, skin


def choose_block(cells, density_per_cell: float = 13.5, cap: int = 2048):
    """Largest block (By, Bz >= 2) whose 2x2x2 colour passes still fill the
    GPU (>= 296 CTAs per pass) and whose footprint fits the staging cap."""
    best = None
    for shape in ((2, 2, 2), (2, 2, 4), (2, 4, 4), (4, 4, 4)):
        if any(c % (2 * b) for c, b in zip(cells, shape)):
            continue
        foot = (shape[0] + 1) * (shape[1] + 2) * (shape[2] + 2)
        if foot * density_per_cell * 1.3 > cap:
            continue
        per_pass = (cells[0] * cells[1] * cells[2]) // (8 * shape[0] * shape[1] * shape[2])
        if best is None or per_pass >= 296:
            best = shape
    return best


class LJSystem:
    """Particles + cell list + workspaces on one GPU (single periodic domain)."""

    def __init__(self, box: LJBox, n: int, params: LJParams = LJParams(), schedule: str = "block",
                 block=None, device=None, skin: float = 0.3):
        torch = _torch()
        _lib.require_cuda()
        if schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {tuple(SCHEDULES)}")
        self.verlet = schedule in VERLET_SCHEDULES
        self.skin = float(skin) if self.verlet else 0.0
        if self.skin < 0:
            raise ValueError("skin must be >= 0")
        for e in box.cell_edge:
            if e < (params.rc + self.skin) * (1 - 1e-12):
                raise ValueError(f"cell edge {e} below cutoff {params.rc}"
                                 + (f" + skin {self.skin}" if self.verlet else ""))
        self.box, self.params, self.n = box, params, int(n)
        self.schedule = schedule
        even = all(c % 2 == 0 for c in box.cells)
        if schedule in ("shell", "buffered", "dataflow") or self.verlet:
            self.block = tuple(block) if block is not None else (2, 2, 2)
        elif schedule == "block":
            self.block = tuple(block) if block is not None else choose_block(box.cells)
            if self.block is None:
                raise ValueError(f"no valid block shape for cells {box.cells}; use schedule='loopex'")
        else:
            if not even:
                raise ValueError("loop-exchange colour passes need even periodic extents")
            self.block = tuple(block) if block is not None else (2, 2, 2)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        d, f64, i32 = self.device, torch.float64, torch.int32
        self._buf = [
            {k: torch.zeros(max(self.n, 1), dtype=f64, device=d) for k in ("x", "y", "z", "vx", "vy", "vz", "fx", "fy", "fz")}
            for _ in range(2)
        ]
        for b in self._buf:
            b["id"] = torch.zeros(max(self.n, 1), dtype=i32, device=d)
        self.cur = 0
        self.cell_start = torch.zeros(box.cell_count + 1, dtype=i32, device=d)
        self._cbox = self._make_cbox()
        self._clj = _lib.CsLJ(params.epsilon, params.sigma, params.rc, params.mass)
        L = _lib.load()
        wsb = max(L.cs_bin_ws_bytes(self.n, C.byref(self._cbox)),
                  L.cs_force_ws_bytes(C.byref(self._cbox), SCHEDULES[schedule], self.n),
                  L.cs_reduce_ws_bytes(self.n))
        self._wsb = int(wsb)
        self._ws = torch.empty(self._wsb, dtype=torch.uint8, device=d)
        # step results in one device block, read back with one copy (readout)
        self._out = torch.zeros(80, dtype=torch.uint8, device=d)
        self.scal = self._out[0:64].view(f64)  # [0]=PE [1]=KE
        self.npairs = self._out[64:72].view(torch.int64)
        self.status = self._out[72:76].view(torch.int32)  # kernel capacity flags
        self._out_host = torch.empty(80, dtype=torch.uint8).pin_memory()
        self.dt = 0.005
        self.nstep = 0  # VV steps taken (eager or replayed); kept in checkpoints
        self.seed = None
        self._graphs = {}
        self._capturing = False
        if self.verlet:
            nb = int(L.cs_verlet_list_bytes(C.byref(self._cbox)))
            self.vlist = torch.zeros(nb, dtype=torch.uint8, device=d)
            self.xref = [torch.zeros(max(self.n, 1), dtype=f64, device=d) for _ in range(3)]
            self.vflag = torch.zeros(1, dtype=i32, device=d)  # displacement > skin/2
            self.graph_builds = torch.zeros(1, dtype=i32, device=d)  # rebuilds taken inside graphs
            self.list_builds = 0  # host-side count (eager steps and explicit rebuilds)

    # ----------------------------------------------------------- plumbing
    def _make_cbox(self):
        b = _lib.CsBox()
        for k in range(3):
            b.nc[k] = b.gnc[k] = self.box.cells[k]
            b.periodic[k] = 1
            b.block[k] = self.block[k]
            b.L[k] = self.box.lengths[k]
            b.inv[k] = self.box.inv[k]
        b.x0 = 0
        b.owned_x = self.box.cells[0]
        return b

    def _s(self):
        return _lib.stream_handle()

    def _a(self, name, which=None):
        return self._buf[self.cur if which is None else which][name]

    @property
    def x(self):
        return self._a("x")

    @property
    def y(self):
        return self._a("y")

    @property
    def z(self):
        return self._a("z")

    # ------------------------------------------------------------- set up
    @classmethod
    def fcc(cls, n_unit_cells=6, density: float = 0.8442, temperature: float = 0.722,
            jitter: float = 0.05, seed: int = 42, params: LJParams = LJParams(),
            schedule: str = "block", block=None, dt: float = 0.005, skin: float = 0.3):
        """FCC lattice + seeded uniform jitter + Gaussian velocities at T
        (momentum removed, 3N-3 dof), then cell list + initial forces.
        Verlet schedules bin on cells of edge >= rc + skin."""
        verlet = schedule in VERLET_SCHEDULES
        box, nuc, a = fcc_box(n_unit_cells, density, params.rc + (skin if verlet else 0.0))
        if verlet:
            box, skin = verlet_box(box.lengths, params.rc, skin)
        n = 4 * nuc[0] * nuc[1] * nuc[2]
        s = cls(box, n, params, schedule, block, skin=skin)
        s.dt = dt
        s.seed_fcc(nuc, a, temperature, jitter, seed)
        return s

    @classmethod
    def liquid_vapour(cls, cells=(64, 64, 192), edge: float = 2.5, temperature: float = 0.85,
                      seed: int = 42, params: LJParams = LJParams(), schedule: str = "buffered",
                      block=None, dt: float = 0.005, skin: float = 0.3, **kw):
        """cfg5 (BASELINE configs[4]): liquid slab + vapour (liquid_vapour_positions),
        Gaussian velocities at T on the device.  Link-cell schedules bin on the
        given cells (edge = rc for cfg5); Verlet schedules on cells of edge
        >= rc + skin (multiples of 4)."""
        L, xyz = liquid_vapour_positions(cells, edge, seed=seed, **kw)
        verlet = schedule in VERLET_SCHEDULES
        box = LJBox(L, cells)
        if verlet:
            box, skin = verlet_box(L, params.rc, skin)
        s = cls(box, len(xyz), params, schedule, block, skin=skin)
        s.dt = dt
        s.seed_positions(xyz, temperature, seed)
        return s

    def seed_positions(self, xyz, temperature, seed):
        """Host positions (ids = row order) + device Gaussian velocities at T."""
        torch = _torch()
        self.seed = int(seed)
        b = self._buf[self.cur]
        for k, col in zip(("x", "y", "z"), range(3)):
            b[k][: self.n].copy_(torch.as_tensor(xyz[:, col], dtype=torch.float64))
        b["id"][: self.n].copy_(torch.arange(self.n, dtype=torch.int32))
        _lib.call("cs_init_velocities", self.n, float(temperature), self.params.mass, int(seed),
                  _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]), _lib.ptr(self._ws),
                  self._wsb, self._s())
        self.initial = {k: b[k].clone() for k in ("x", "y", "z", "vx", "vy", "vz", "id")}
        self.rebuild()

    def seed_fcc(self, nuc, a, temperature, jitter, seed):
        self.seed = int(seed)
        src = self.cur
        b = self._buf[src]
        nu = (C.c_int32 * 3)(*nuc)
        aa = (C.c_double * 3)(*a)
        LL = (C.c_double * 3)(*self.box.lengths)
        _lib.call("cs_init_fcc", nu, aa, LL, float(jitter), int(seed), _lib.ptr(b["x"]),
                  _lib.ptr(b["y"]), _lib.ptr(b["z"]), _lib.ptr(b["id"]), self._s())
        _lib.call("cs_init_velocities", self.n, float(temperature), self.params.mass, int(seed),
                  _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]), _lib.ptr(self._ws),
                  self._wsb, self._s())
        self.initial = {k: b[k].clone() for k in ("x", "y", "z", "vx", "vy", "vz", "id")}
        self.rebuild()

    def load_host(self, x, y, z, vx, vy, vz, ids):
        """Copy host arrays in (any order), rebuild cells and forces."""
        torch = _torch()
        b = self._buf[self.cur]
        # (non-blocking: pinned host sources overlap; pageable ones copy synchronously)
        for k, arr in zip(("x", "y", "z", "vx", "vy", "vz"), (x, y, z, vx, vy, vz)):
            b[k][: self.n].copy_(torch.as_tensor(arr, dtype=torch.float64), non_blocking=True)
        b["id"][: self.n].copy_(torch.as_tensor(ids, dtype=torch.int32), non_blocking=True)
        if not self.verlet:  # (the Verlet rebuild wraps first itself)
            _lib.call("cs_wrap_positions", self.n, C.byref(self._cbox), _lib.ptr(b["x"]), _lib.ptr(b["y"]),
                      _lib.ptr(b["z"]), self._s())
        self.rebuild()

    def rebuild(self, energy: bool = True):
        if self.verlet:
            self._rebuild_list()
        else:
            self.build_cells()
        self.compute_forces(energy=energy)

    def _rebuild_list(self):
        """Verlet mode: wrap, rebin in place, rebuild the round tables and
        remember the positions for the displacement check."""
        b = self._buf[self.cur]
        _lib.call("cs_wrap_positions", self.n, C.byref(self._cbox), _lib.ptr(b["x"]), _lib.ptr(b["y"]),
                  _lib.ptr(b["z"]), self._s())
        self.build_cells()
        b = self._buf[self.cur]
        _lib.call("cs_verlet_build", C.byref(self._cbox), C.byref(self._clj), self.skin,
                  _lib.ptr(self.cell_start), _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]),
                  _lib.ptr(self.vlist), self.vlist.numel(), *(_lib.ptr(t) for t in self.xref),
                  self.n, _lib.ptr(self.status), self._s())
        if not self._capturing:
            self.list_builds += 1

    # ------------------------------------------------------------- kernels
    def build_cells(self):
        """K1: stable counting sort into the other buffer, then swap."""
        a, b = self._buf[self.cur], self._buf[1 - self.cur]
        _lib.call("cs_build_cells", self.n, C.byref(self._cbox), _lib.ptr(a["x"]), _lib.ptr(a["y"]),
                  _lib.ptr(a["z"]), _lib.ptr(a["vx"]), _lib.ptr(a["vy"]), _lib.ptr(a["vz"]),
                  _lib.ptr(a["id"]), _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]),
                  _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]), _lib.ptr(b["id"]),
                  _lib.ptr(b["fx"]), _lib.ptr(b["fy"]), _lib.ptr(b["fz"]), _lib.ptr(self.cell_start),
                  _lib.ptr(self._ws), self._wsb, self._s())
        if self.verlet:  # in place: the rebuild may sit inside a conditional graph node
            ks = ("x", "y", "z", "vx", "vy", "vz", "id")
            _lib.call("cs_copy7", self.n, *(_lib.ptr(b[k]) for k in ks), *(_lib.ptr(a[k]) for k in ks),
                      self._s())
        else:
            self.cur = 1 - self.cur

    def compute_forces(self, energy: bool = False, count_pairs: bool = True):
        """K2 (forces must be zero on entry; build_cells zeroes them)."""
        b = self._buf[self.cur]
        if energy:
            _lib.call("cs_memset_async", _lib.ptr(self.scal), 0, 8, self._s())
        if count_pairs:
            _lib.call("cs_memset_async", _lib.ptr(self.npairs), 0, 8, self._s())
        if self.verlet:
            _lib.call("cs_lj_forces_verlet", C.byref(self._cbox), C.byref(self._clj),
                      SCHEDULES[self.schedule], self.n, _lib.ptr(self.cell_start), _lib.ptr(self.vlist),
                      _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]), _lib.ptr(b["fx"]),
                      _lib.ptr(b["fy"]), _lib.ptr(b["fz"]), _lib.ptr(self.scal) if energy else None,
                      _lib.ptr(self.npairs) if count_pairs else None, _lib.ptr(self.status),
                      _lib.ptr(self._ws), self._wsb, self._s())
            return
        _lib.call("cs_lj_forces", C.byref(self._cbox), C.byref(self._clj), SCHEDULES[self.schedule],
                  self.n, _lib.ptr(self.cell_start), _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]),
                  _lib.ptr(b["fx"]), _lib.ptr(b["fy"]), _lib.ptr(b["fz"]),
                  _lib.ptr(self.scal) if energy else None,
                  _lib.ptr(self.npairs) if count_pairs else None, _lib.ptr(self.status),
                  _lib.ptr(self._ws), self._wsb, self._s())

    def kinetic(self):
        b = self._buf[self.cur]
        _lib.call("cs_kinetic", self.n, self.params.mass, _lib.ptr(b["vx"]), _lib.ptr(b["vy"]),
                  _lib.ptr(b["vz"]), _lib.ptr(self.scal[1:]), _lib.ptr(self._ws), self._wsb, self._s())

    def _pre_verlet(self):
        """Verlet mode: kick + drift (no wrap) with the displacement check, then
        the list rebuild if any particle moved more than skin/2 -- decided on
        the host when eager, by a conditional graph node when captured."""
        torch = _torch()
        hdtm = 0.5 * self.dt / self.params.mass
        b = self._buf[self.cur]
        _lib.call("cs_vv_kick_drift_track", self.n, hdtm, self.dt, _lib.ptr(b["fx"]), _lib.ptr(b["fy"]),
                  _lib.ptr(b["fz"]), _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]),
                  _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]), *(_lib.ptr(t) for t in self.xref),
                  0.5 * self.skin, _lib.ptr(self.vflag), self._s())
        if self._capturing:
            side = self._side
            _lib.call("cs_capture_if_begin", self._s(), side.cuda_stream, _lib.ptr(self.vflag),
                      _lib.ptr(self.graph_builds))
            with torch.cuda.stream(side):
                self._rebuild_list()
            _lib.call("cs_capture_if_end", side.cuda_stream)
        elif int(self.vflag.item()):
            _lib.call("cs_memset_async", _lib.ptr(self.vflag), 0, 4, self._s())
            self._rebuild_list()

    def step(self, energy: bool = False):
        """One velocity-Verlet step (K3 kick+drift, K1, K2, K3 kick)."""
        if not self._capturing:
            self.nstep += 1
        hdtm = 0.5 * self.dt / self.params.mass
        if self.verlet:
            self._pre_verlet()
            self.compute_forces(energy=energy)
            b = self._buf[self.cur]
            _lib.call("cs_vv_kick", self.n, hdtm, _lib.ptr(b["fx"]), _lib.ptr(b["fy"]), _lib.ptr(b["fz"]),
                      _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]), self._s())
            if energy:
                self.kinetic()
            return
        b = self._buf[self.cur]
        _lib.call("cs_vv_kick_drift", self.n, hdtm, self.dt, C.byref(self._cbox), _lib.ptr(b["fx"]),
                  _lib.ptr(b["fy"]), _lib.ptr(b["fz"]), _lib.ptr(b["vx"]), _lib.ptr(b["vy"]),
                  _lib.ptr(b["vz"]), _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]), self._s())
        self.build_cells()
        self.compute_forces(energy=energy)
        b = self._buf[self.cur]
        _lib.call("cs_vv_kick", self.n, hdtm, _lib.ptr(b["fx"]), _lib.ptr(b["fy"]), _lib.ptr(b["fz"]),
                  _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]), self._s())
        if energy:
            self.kinetic()

    # ---------------------------------------------------------- CUDA graph
    def _graph(self, key, fn):
        """Capture fn() once per (key, buffer parity) and replay it.  Capture
        only records work, so it does not advance the state; the Python-side
        buffer parity after the call is remembered with the graph."""
        torch = _torch()
        gkey = (key, self.cur)
        if gkey not in self._graphs:
            start = self.cur
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(device=self.device)
            self._side = torch.cuda.Stream(device=self.device)
            s.wait_stream(torch.cuda.current_stream())
            self._capturing = True
            try:
                with torch.cuda.stream(s):
                    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
                        fn()
            finally:
                self._capturing = False
            torch.cuda.current_stream().wait_stream(s)
            self._graphs[gkey] = (g, self.cur)
            self.cur = start
        g, after = self._graphs[gkey]
        g.replay()
        self.cur = after

    def graph_step(self, energy: bool = False):
        """One VV step replayed from a CUDA graph (one graph per parity)."""
        self._graph(("step", energy), lambda: self.step(energy))
        self.nstep += 1

    def graph_phases(self):
        """The step as three graphs (kick+drift+rebin | forces | kick), so a
        caller can put timing events between the phases."""
        hdtm = 0.5 * self.dt / self.params.mass

        def pre():
            if self.verlet:
                self._pre_verlet()
                return
            b = self._buf[self.cur]
            _lib.call("cs_vv_kick_drift", self.n, hdtm, self.dt, C.byref(self._cbox),
                      _lib.ptr(b["fx"]), _lib.ptr(b["fy"]), _lib.ptr(b["fz"]), _lib.ptr(b["vx"]),
                      _lib.ptr(b["vy"]), _lib.ptr(b["vz"]), _lib.ptr(b["x"]), _lib.ptr(b["y"]),
                      _lib.ptr(b["z"]), self._s())
            self.build_cells()

        def post():
            b = self._buf[self.cur]
            _lib.call("cs_vv_kick", self.n, hdtm, _lib.ptr(b["fx"]), _lib.ptr(b["fy"]),
                      _lib.ptr(b["fz"]), _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]),
                      self._s())

        return (lambda: self._graph("pre", pre),
                lambda: self._graph("force", lambda: self.compute_forces(energy=False)),
                lambda: self._graph("post", post))

    def launches_per_step(self, energy: bool = False) -> int:
        """Kernels this package launches per step (memsets excluded)."""
        build = 1 + 3 + 1 + 1  # count, scan x3, scatter, sort-gather
        # force kernels: buffered = block sizes, scan x3, force, gather; shell =
        # 8 colour passes; dataflow = 1 persistent launch; + pair/energy reduce x2
        per = {"loopex": 27, "block": 8, "shell": 8, "buffered": 6, "dataflow": 1,
               "verlet": 2, "verlet_shell": 8, "verlet_dataflow": 1}  # verlet: layout cached at build
        direct = self.schedule not in ("loopex", "block")  # pair counts via atomics in the kernel
        force = per[self.schedule] + (2 if (energy or not direct) else 0)
        if self.verlet:  # kick_drift_track, set_cond (rebuilds run inside the graph's IF node)
            return 2 + force + 1 + (3 if energy else 0)
        return 1 + build + force + 1 + (3 if energy else 0)

    REBUILD_LAUNCHES = 16  # wrap, rebin (count, scan x3, scatter, sort-gather), copy-back,
    #                        round tables (main + crowded-cell pass), reference copy, block
    #                        sizes, scan x3, block tables

    def candidate_pairs_dev(self):
        """Half-shell candidate pairs C of the current cell list as a device
        scalar (no synchronisation): the C of the 8 C + 20 P convention of
        SURVEY 8(d) for the link-cell schedules."""
        torch = _torch()
        from .grid import canonical_half_stencil

        cnt = (self.cell_start[1:] - self.cell_start[:-1]).long().view(*self.box.cells[::-1])
        c = (cnt * (cnt - 1) // 2).sum()
        for ox, oy, oz in canonical_half_stencil(3).inter_offsets:
            c = c + (cnt * torch.roll(cnt, shifts=(-oz, -oy, -ox), dims=(0, 1, 2))).sum()
        return c

    def candidate_pairs(self) -> int:
        return int(self.candidate_pairs_dev())

    def rc_grid_candidates_dev(self):
        """C of SURVEY 8(d)'s fixed convention: half-shell candidates on cells of
        edge >= rc (floor(L / rc) per axis), counted from the current positions
        on the device -- the same algorithmic work whatever the schedule."""
        torch = _torch()
        from .grid import canonical_half_stencil

        b = self._buf[self.cur]
        n = self.n
        nc = [int(math.floor(L / self.params.rc)) for L in self.box.lengths]
        idx = None
        for k, key in enumerate(("x", "y", "z")):
            L = self.box.lengths[k]
            c = torch.floor(torch.remainder(b[key][:n], L) * (nc[k] / L)).long().clamp_(0, nc[k] - 1)
            idx = c if idx is None else idx + c * int(math.prod(nc[:k]))
        cnt = torch.bincount(idx, minlength=int(math.prod(nc))).view(nc[2], nc[1], nc[0])
        c = (cnt * (cnt - 1) // 2).sum()
        for ox, oy, oz in canonical_half_stencil(3).inter_offsets:
            c = c + (cnt * torch.roll(cnt, shifts=(-oz, -oy, -ox), dims=(0, 1, 2))).sum()
        return c

    def list_pairs_dev(self):
        """Verlet mode: pairs held in the current round tables, as a device
        scalar (each is distance-tested every step)."""
        torch = _torch()
        nc = self.box.cell_count
        sl = lambda b: (b + 255) // 256 * 256  # cs_ws_slice, layout of vl_view
        o2 = sl(4 * nc) + sl(96 * nc)
        nr = self.vlist[: 4 * nc].view(torch.int32).long()
        desc = self.vlist[o2: o2 + 2 * 64 * 32 * nc].view(torch.int16).view(nc, 64, 32)
        live = torch.arange(64, device=self.device)[None, :] < nr[:, None]
        return ((desc != 0x0F00) & live[:, :, None]).sum()  # VL_IDLE

    def list_pairs(self) -> int:
        return int(self.list_pairs_dev())

    def list_rounds(self):
        """Verlet mode: (rounds per cell as a host array, lane use)."""
        torch = _torch()
        nc = self.box.cell_count
        nr = self.vlist[: 4 * nc].view(torch.int32).cpu().numpy()
        rounds = nr
        return rounds, self.list_pairs() / (32.0 * max(int(rounds.sum()), 1))

    def _state_tensors(self):
        out = []
        for b in self._buf:
            out += [b[k] for k in ("x", "y", "z", "vx", "vy", "vz", "fx", "fy", "fz", "id")]
        return out + [self.cell_start, self.scal, self.npairs]

    def run(self, nsteps: int, energy_every: int = 0, graph: bool = True):
        """Advance nsteps; returns [(step, pe, ke)] at the energy steps."""
        out = []
        for k in range(1, nsteps + 1):
            en = energy_every > 0 and k % energy_every == 0
            (self.graph_step if graph else self.step)(energy=en)
            if en:
                pe, ke = self.energies()
                out.append((k, pe, ke))
        return out

    # --------------------------------------------------- checkpoint/resume
    _STATE = ("x", "y", "z", "vx", "vy", "vz", "fx", "fy", "fz", "id")

    def checkpoint(self, path) -> None:
        """npz of the full step state: positions, velocities, forces and ids in
        cell order, the cell list, step counter, seed, box, parameters and
        schedule; Verlet systems also store the reference positions, the
        round tables and the displacement flag, so `restore` continues
        bit-identically (no list rebuild at load)."""
        import numpy as np

        torch = _torch()
        torch.cuda.current_stream().synchronize()
        b = self._buf[self.cur]
        n = self.n
        d = {k: b[k][:n].cpu().numpy() for k in self._STATE}
        d.update(cell_start=self.cell_start.cpu().numpy(), nstep=self.nstep,
                 seed=-1 if self.seed is None else self.seed, lengths=np.asarray(self.box.lengths),
                 cells=np.asarray(self.box.cells), block=np.asarray(self.block), dt=self.dt,
                 skin=self.skin, schedule=self.schedule,
                 params=np.asarray([self.params.epsilon, self.params.sigma, self.params.rc, self.params.mass]))
        if self.verlet:
            d.update(xref=np.stack([t[:n].cpu().numpy() for t in self.xref]), vlist=self.vlist.cpu().numpy(),
                     vflag=self.vflag.cpu().numpy(), graph_builds=self.graph_builds.cpu().numpy(),
                     list_builds=self.list_builds)
        np.savez(path, **d)

    @classmethod
    def restore(cls, path, device=None) -> "LJSystem":
        """A system continuing exactly from `checkpoint(path)`."""
        import numpy as np

        torch = _torch()
        z = np.load(path)
        eps, sig, rc, mass = (float(v) for v in z["params"])
        box = LJBox(tuple(float(v) for v in z["lengths"]), tuple(int(v) for v in z["cells"]))
        n = int(len(z["x"]))
        s = cls(box, n, LJParams(eps, sig, rc, mass), str(z["schedule"]),
                tuple(int(v) for v in z["block"]), device=device, skin=float(z["skin"]))
        s.dt = float(z["dt"])
        s.nstep = int(z["nstep"])
        s.seed = None if int(z["seed"]) < 0 else int(z["seed"])
        b = s._buf[s.cur]
        for k in cls._STATE:
            b[k][:n].copy_(torch.from_numpy(z[k]))
        s.cell_start.copy_(torch.from_numpy(z["cell_start"]))
        if s.verlet:
            for t, a in zip(s.xref, z["xref"]):
                t[:n].copy_(torch.from_numpy(a))
            s.vlist.copy_(torch.from_numpy(z["vlist"]))
            s.vflag.copy_(torch.from_numpy(z["vflag"]))
            s.graph_builds.copy_(torch.from_numpy(z["graph_builds"]))
            s.list_builds = int(z["list_builds"])
        s.initial = {k: b[k].clone() for k in ("x", "y", "z", "vx", "vy", "vz", "id")}
        return s

    # -------------------------------------------------------------- output
    def bin_errors(self) -> int:
        """1 if the last cell-list build clamped a particle outside the box
        into an edge cell (cs_bin_errors; synchronises)."""
        flag = C.c_int(0)
        _lib.call("cs_bin_errors", self.n, C.byref(self._cbox), _lib.ptr(self._ws), self._wsb,
                  C.byref(flag), self._s())
        return int(flag.value)

    def check_status(self):
        """Raise if a kernel reported a capacity overflow (buffered schedule)."""
        st = int(self.status.item())
        if st & 1:
            raise _lib.CellschedError(
                "buffered force schedule: a block exceeded its shared-memory capacity; "
                "use schedule='shell' (in-place fallback) for this density")
        if st & 2:
            raise _lib.CellschedError("Verlet list: a cell holds more than 64 particles; "
                                      "use a link-cell schedule for this density")
        if st & 4:
            raise _lib.CellschedError("Verlet list: a home cell needs more than 64 rounds; "
                                      "reduce the skin")

    def readout(self):
        """(PE, KE, pairs) of the last step with one device->host copy and one
        synchronisation (raises on a kernel capacity flag)."""
        import numpy as np

        torch = _torch()
        self._out_host.copy_(self._out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        raw = self._out_host.numpy()
        if int(raw[72:76].view(np.int32)[0]):
            self.check_status()
        e = raw[0:16].view(np.float64)
        return float(e[0]), float(e[1]), int(raw[64:72].view(np.int64)[0])

    def energies(self):
        """(PE, KE) of the last energy evaluation (synchronises)."""
        v = self.scal.cpu().tolist()
        self.check_status()
        return v[0], v[1]

    def pair_count(self) -> int:
        self.check_status()
        return int(self.npairs.item())

    def snapshot(self):
        """Host copies in cell-sorted order: x, v, f as (n, 3), ids, cell_start."""
        torch = _torch()
        b = self._buf[self.cur]
        n = self.n
        st = lambda ks: torch.stack([b[k][:n] for k in ks], 1).cpu().numpy()
        return {"x": st(("x", "y", "z")), "v": st(("vx", "vy", "vz")), "f": st(("fx", "fy", "fz")),
                "id": b["id"][:n].cpu().numpy(), "cell_start": self.cell_start.cpu().numpy()}


# reference-style functional entry points ------------------------------------
def build_cell_list(system: LJSystem) -> None:
    system.build_cells()


def lj_forces(system: LJSystem, energy: bool = True):
    """Zero the forces, evaluate them; returns (PE, pairs within rc)."""
    for k in ("fx", "fy", "fz"):
        _lib.call("cs_memset_async", _lib.ptr(system._a(k)), 0, 8 * system.n, system._s())
    system.compute_forces(energy=energy)
    return system.energies()[0], system.pair_count()


def vv_step(system: LJSystem, energy: bool = False) -> None:
    system.step(energy=energy)
