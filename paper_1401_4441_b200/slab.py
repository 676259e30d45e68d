"""x-slab decomposition of the LJ link-cell step over ranks.

Rank r owns cell planes [x0, x1) of the periodic box.  All 13 half-shell
offsets have o_x in {0, +1} (grid.py:26-33, canonical_half_stencil), so a rank
needs exactly ONE ghost plane: the first owned plane of rank r+1 (periodic
ring).  One force evaluation per step exchanges

    positions of plane x0 -> rank r-1      (ghost positions, +L across the seam)
    reaction forces on the ghost plane -> rank r+1   (added to its plane x0)

plus particle migration after the drift.  The rank-local schedule keeps the
same conflict-free colour passes on the local grid (x open, ghost plane last;
SURVEY A.5).  `SlabStep` holds the protocol (order of operations, routing,
the +L shift); an engine does the local work: `CudaSlabEngine` (C ABI kernels,
the product) or a CPU engine in the tests.  Messages go through
`NeighbourExchanger` (torch.distributed point-to-point: NCCL on GPUs, gloo on
CPU).  Energies are summed with one all-reduce.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class SlabLayout:
    """Which x-planes a rank owns (contiguous block partition)."""

    nx: int
    world: int
    rank: int

    def __post_init__(self) -> None:
        if not (0 <= self.rank < self.world):
            raise ValueError("rank out of range")
        if self.nx < self.world:
            raise ValueError(f"{self.nx} cell planes cannot be split over {self.world} ranks")

    def planes(self, r: int | None = None) -> tuple[int, int]:
        r = self.rank if r is None else r
        return (r * self.nx) // self.world, ((r + 1) * self.nx) // self.world

    @property
    def x0(self) -> int:
        return self.planes()[0]

    @property
    def owned(self) -> int:
        a, b = self.planes()
        return b - a

    @property
    def left(self) -> int:
        return (self.rank - 1) % self.world

    @property
    def right(self) -> int:
        return (self.rank + 1) % self.world

    def owner(self, plane: int) -> int:
        plane %= self.nx
        for r in range(self.world):
            a, b = self.planes(r)
            if a <= plane < b:
                return r
        raise AssertionError


class NeighbourExchanger:
    """Variable-size exchange with the left and right ranks of the ring.

    `exchange(to_left, to_right) -> (from_left, from_right)`: sizes first, then
    payloads, as one batch of point-to-point ops.  Leftward messages use tag
    1, rightward tag 2, so world size 2 (left == right) is unambiguous."""

    def __init__(self, layout: SlabLayout, group=None):
        self.layout, self.group = layout, group

    def exchange(self, to_left, to_right):
        torch = _torch()
        L = self.layout
        if L.world == 1:
            return to_right, to_left  # the ring closes on itself
        import torch.distributed as dist

        dev = to_left.device
        n_send = [torch.tensor([to_left.numel()], dtype=torch.int64, device=dev),
                  torch.tensor([to_right.numel()], dtype=torch.int64, device=dev)]
        n_recv = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2)]
        self._run([(n_send[0], L.left, 1, True), (n_send[1], L.right, 2, True),
                   (n_recv[0], L.right, 1, False), (n_recv[1], L.left, 2, False)])
        from_right = torch.empty(int(n_recv[0].item()), dtype=to_left.dtype, device=dev)
        from_left = torch.empty(int(n_recv[1].item()), dtype=to_left.dtype, device=dev)
        # empty payloads are skipped on both sides (the sizes are known to both)
        self._run([op for op in ((to_left, L.left, 1, True), (to_right, L.right, 2, True),
                                 (from_right, L.right, 1, False), (from_left, L.left, 2, False))
                   if op[0].numel() > 0])
        return from_left, from_right

    def exchange_fixed(self, to_left, to_right, n_from_left, n_from_right):
        """Same as exchange() when both sides already know the sizes (a Verlet
        slab between rebuilds): payloads only, no size round trip."""
        torch = _torch()
        L = self.layout
        if L.world == 1:
            return to_right, to_left
        dev = to_left.device
        from_right = torch.empty(n_from_right, dtype=to_left.dtype, device=dev)
        from_left = torch.empty(n_from_left, dtype=to_left.dtype, device=dev)
        self._run([op for op in ((to_left, L.left, 1, True), (to_right, L.right, 2, True),
                                 (from_right, L.right, 1, False), (from_left, L.left, 2, False))
                   if op[0].numel() > 0])
        return from_left, from_right

    def _run(self, ops):
        import torch.distributed as dist

        if not ops:
            return
        backend = dist.get_backend(self.group)
        if backend == "nccl":
            p2p = [dist.P2POp(dist.isend if send else dist.irecv, t, peer, self.group, tag)
                   for t, peer, tag, send in ops]
            for w in dist.batch_isend_irecv(p2p):
                w.wait()
        else:
            works = []
            for t, peer, tag, send in ops:
                fn = dist.isend if send else dist.irecv
                works.append(fn(t, peer, group=self.group, tag=tag))
            for w in works:
                w.wait()

    def allreduce_max_int(self, value: int) -> int:
        """Global OR / max of a small integer (the Verlet rebuild decision)."""
        torch = _torch()
        if self.layout.world == 1:
            return int(value)
        import torch.distributed as dist

        t = torch.tensor([int(value)], dtype=torch.int64)
        if dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def allreduce_sum(self, values):
        torch = _torch()
        t = torch.tensor(values, dtype=torch.float64)
        if self.layout.world > 1:
            import torch.distributed as dist

            if dist.get_backend(self.group) == "nccl":
                t = t.cuda()
            dist.all_reduce(t, group=self.group)
        return t.cpu().tolist()


class SlabStep:
    """The per-rank protocol of one velocity-Verlet step (and of the initial
    force evaluation), independent of where the local work runs."""

    def __init__(self, engine, exchanger: NeighbourExchanger):
        self.e, self.x = engine, exchanger
        # Verlet engines migrate and rebin only at list rebuilds, which every
        # rank takes in the same step (global OR of the displacement flags);
        # in between, the ghost plane keeps its particles and order
        self.verlet = bool(getattr(engine, "verlet", False))
        self.rebuilds = 0
        self._kd_ahead = False

    def migrate(self):
        stay, to_left, to_right = self.e.split()
        from_left, from_right = self.x.exchange(to_left, to_right)
        self.e.assemble(stay, from_left, from_right)

    def forces(self, energy: bool, rebuild: bool = True):
        L = self.x.layout
        fixed = self.verlet and not rebuild  # same ghost particles, same order, same sizes
        counts, xyz = self.e.pack_first_plane(xshift=self.e.box_length_x if L.rank == 0 else 0.0,
                                              cached=fixed)
        # positions of my first plane go left; the right rank's first plane is my ghost
        if fixed:
            _, g_xyz_r = self.x.exchange_fixed(xyz, xyz[:0], 0, 3 * self.e.n_ghost)
            self.e.update_ghosts(g_xyz_r)
        else:
            g_counts_l, g_counts_r = self.x.exchange(counts, counts[:0])
            g_xyz_l, g_xyz_r = self.x.exchange(xyz, xyz[:0])
            self._g_counts = g_counts_r
            self._n_first = xyz.numel() // 3
            self.e.set_ghosts(g_counts_r, g_xyz_r)
        if self.verlet and rebuild:
            self.e.build_list()
        pe, npairs = self.e.forces(energy, sync=not fixed or energy)
        # reactions on my ghost plane go back to its owner (the right rank)
        fg = self.e.pack_ghost_forces()
        if fixed:
            f_from_left, _ = self.x.exchange_fixed(fg[:0], fg, 3 * self._n_first, 0)
        else:
            f_from_left, _ = self.x.exchange(fg[:0], fg)
        self.e.add_first_plane_forces(f_from_left)
        return pe, npairs

    def _rebuild(self):
        if self.verlet:
            self.e.wrap()
        self.migrate()
        self.e.build_cells()
        self.rebuilds += 1

    def start(self, energy=True):
        self._rebuild()
        pe, npairs = self.forces(energy, rebuild=True)
        if self.verlet:
            self._decide(kick=False)
        return self._energies(pe, npairs, energy)

    def _decide(self, kick: bool, lookahead: bool = False):
        """Verlet: the post-kick fused with the exact prediction of the next
        kick-drift's displacement flag, and the global rebuild decision for
        the next step (one all-reduce) -- taken at the end of this step, so
        the next one starts without waiting for its own flag."""
        self.e.kick_predict(kick)
        if lookahead:
            self.e.kick_drift(track=False)
            self._kd_ahead = True
        self._next_rebuild = self.x.allreduce_max_int(self.e.take_flag()) > 0

    def step(self, energy: bool = False, reduce: bool = True, lookahead: bool = False):
        """One VV step.  reduce=False (non-energy steps) skips the global sums:
        pair counts stay in the engine's device accumulator (pairs_total).

        lookahead=True (Verlet, non-energy steps): the NEXT step's kick-drift
        -- which does not depend on the rebuild decision -- is launched before
        this step waits for that decision, so the device is not idle while
        the host takes it.  The state then stands half a step ahead until the
        next step() call: use it only inside a run of steps (not on the last
        one, and not when the state is read in between)."""
        if self.verlet:
            if self._kd_ahead:
                self._kd_ahead = False  # launched by the previous step
            else:
                self.e.kick_drift(track=False)
            rebuild = self._next_rebuild
        else:
            self.e.kick_drift()
            rebuild = True
        if rebuild:
            self._rebuild()
        pe, npairs = self.forces(energy, rebuild=rebuild)
        if self.verlet:
            self._decide(kick=True, lookahead=lookahead and not energy)
        else:
            self.e.kick()
        if not reduce and not energy:
            return None
        return self._energies(pe, npairs, energy)

    def pairs_total(self) -> int:
        """Pairs accumulated on the device over all force evaluations, summed
        over ranks (one synchronisation)."""
        tot = self.x.allreduce_sum([float(self.e.pairs_acc.item())])
        return int(tot[0])

    def _energies(self, pe, npairs, energy):
        ke = self.e.kinetic() if energy else 0.0
        tot = self.x.allreduce_sum([pe, ke, float(npairs), float(self.e.n_owned)])
        return {"pe": tot[0], "ke": tot[1], "pairs": int(tot[2]), "n": int(tot[3])}


class CudaSlabEngine:
    """Rank-local state and C ABI kernels for one x-slab on one GPU."""

    def __init__(self, box, layout: SlabLayout, params, schedule="buffered", block=(2, 2, 2),
                 capacity: int | None = None, dt: float = 0.005, device=None, skin: float = 0.3):
        torch = _torch()
        _lib.require_cuda()
        from .md import SCHEDULES, VERLET_SCHEDULES

        self.box, self.layout, self.params, self.dt = box, layout, params, dt
        self.schedule = schedule
        self.verlet = schedule in VERLET_SCHEDULES
        self.skin = float(skin) if self.verlet else 0.0
        if self.verlet and min(box.cell_edge) < (params.rc + self.skin) * (1 - 1e-12):
            raise ValueError("Verlet slabs need cells of edge >= rc + skin")
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        nx, ny, nz = box.cells
        owned = layout.owned
        self.box_length_x = box.lengths[0]
        b = _lib.CsBox()
        b.nc[0], b.nc[1], b.nc[2] = owned + 1, ny, nz
        b.gnc[0], b.gnc[1], b.gnc[2] = nx, ny, nz
        b.x0 = layout.x0
        b.owned_x = owned
        b.periodic[0], b.periodic[1], b.periodic[2] = 0, 1, 1
        for k in range(3):
            b.block[k] = block[k]
            b.L[k] = box.lengths[k]
            b.inv[k] = box.inv[k]
        self.cbox = b
        self.sched = SCHEDULES[schedule]
        self.clj = _lib.CsLJ(params.epsilon, params.sigma, params.rc, params.mass)
        self.cap = int(capacity) if capacity else 0
        self.n_owned = 0
        self.n_ghost = 0
        self.ncells_local = (owned + 1) * ny * nz
        self.plane_cells = ny * nz

    # -- allocation (capacity in particles, owned + ghost) --------------------
    def _alloc(self, cap):
        torch = _torch()
        d, f64 = self.device, torch.float64
        self.cap = cap
        mk = lambda: {k: torch.zeros(cap, dtype=f64, device=d) for k in
                      ("x", "y", "z", "vx", "vy", "vz", "fx", "fy", "fz")}
        self.A, self.B = mk(), mk()
        self.A["id"] = torch.zeros(cap, dtype=torch.int32, device=d)
        self.B["id"] = torch.zeros(cap, dtype=torch.int32, device=d)
        self.cell_start = torch.zeros(self.ncells_local + 1, dtype=torch.int32, device=d)
        self.mcap = max(1024, cap // 8)
        self.P_stay = torch.zeros(7 * cap, dtype=f64, device=d)
        self.P_l = torch.zeros(7 * self.mcap, dtype=f64, device=d)
        self.P_r = torch.zeros(7 * self.mcap, dtype=f64, device=d)
        L = _lib.load()
        wsb = max(L.cs_bin_ws_bytes(cap, C.byref(self.cbox)),
                  L.cs_force_ws_bytes(C.byref(self.cbox), self.sched, cap),
                  L.cs_reduce_ws_bytes(cap), L.cs_slab_ws_bytes(cap),
                  L.cs_ghost_ws_bytes(C.byref(self.cbox)))
        self.wsb = int(wsb)
        self.ws = torch.empty(self.wsb, dtype=torch.uint8, device=d)
        self.scal = torch.zeros(8, dtype=f64, device=d)
        self.npairs = torch.zeros(1, dtype=torch.int64, device=d)
        self.pairs_acc = torch.zeros(1, dtype=torch.int64, device=d)
        self.status = torch.zeros(1, dtype=torch.int32, device=d)
        self.counts = torch.zeros(self.plane_cells, dtype=torch.int32, device=d)
        if self.verlet:
            self.vlist = torch.zeros(int(L.cs_verlet_list_bytes(C.byref(self.cbox))), dtype=torch.uint8, device=d)
            self.xref = [torch.zeros(cap, dtype=f64, device=d) for _ in range(3)]
            self.vflag = torch.zeros(1, dtype=torch.int32, device=d)
            self.vflag_scratch = torch.zeros(1, dtype=torch.int32, device=d)

    def _s(self):
        return _lib.stream_handle()

    def load_global(self, x, y, z, vx, vy, vz, ids, global_n: int | None = None):
        """Take this rank's particles out of device arrays holding the global
        state or any superset of this rank's particles (same classification
        kernel as the migration; the others are dropped).  global_n: the
        total particle count when the arrays hold a subset (sizes the
        buffers)."""
        torch = _torch()
        n = int(x.numel())
        if not hasattr(self, "A"):
            tot = int(global_n) if global_n else n
            self._alloc(self.cap or int(tot / self.layout.world * 1.3) + 4 * self.plane_cells * 32 + 4096)
        big = torch.zeros(7 * n, dtype=torch.float64, device=self.device)
        scratch = torch.zeros(7 * n, dtype=torch.float64, device=self.device)
        ws = torch.empty(_lib.load().cs_slab_ws_bytes(n), dtype=torch.uint8, device=self.device)
        cnt = (C.c_int64 * 3)()
        _lib.call("cs_slab_split", n, C.byref(self.cbox), _lib.ptr(x), _lib.ptr(y), _lib.ptr(z),
                  _lib.ptr(vx), _lib.ptr(vy), _lib.ptr(vz), _lib.ptr(ids), _lib.ptr(big), n,
                  _lib.ptr(scratch), _lib.ptr(scratch), n, cnt, _lib.ptr(ws), ws.numel(), self._s())
        m = cnt[0]
        if m > self.cap:
            raise _lib.CellschedError("slab capacity too small for the initial load")
        a = self.A
        _lib.call("cs_unpack7", m, _lib.ptr(big), n, _lib.ptr(a["x"]), _lib.ptr(a["y"]), _lib.ptr(a["z"]),
                  _lib.ptr(a["vx"]), _lib.ptr(a["vy"]), _lib.ptr(a["vz"]), _lib.ptr(a["id"]), self._s())
        self.n_owned = m

    # -- protocol hooks --------------------------------------------------------
    def kick_drift(self, track: bool = True):
        """track=False (Verlet, the decision came from kick_predict): the
        flag goes to a scratch word and is never read."""
        a = self.A
        hdtm = 0.5 * self.dt / self.params.mass
        if self.verlet:  # no wrap between rebuilds; flag particles past skin/2
            flag = self.vflag if track else self.vflag_scratch
            _lib.call("cs_vv_kick_drift_track", self.n_owned, hdtm, self.dt, _lib.ptr(a["fx"]),
                      _lib.ptr(a["fy"]), _lib.ptr(a["fz"]), _lib.ptr(a["vx"]), _lib.ptr(a["vy"]),
                      _lib.ptr(a["vz"]), _lib.ptr(a["x"]), _lib.ptr(a["y"]), _lib.ptr(a["z"]),
                      *(_lib.ptr(t) for t in self.xref), 0.5 * self.skin, _lib.ptr(flag), self._s())
            return
        _lib.call("cs_vv_kick_drift", self.n_owned, hdtm, self.dt, C.byref(self.cbox),
                  _lib.ptr(a["fx"]), _lib.ptr(a["fy"]), _lib.ptr(a["fz"]), _lib.ptr(a["vx"]),
                  _lib.ptr(a["vy"]), _lib.ptr(a["vz"]), _lib.ptr(a["x"]), _lib.ptr(a["y"]),
                  _lib.ptr(a["z"]), self._s())

    def take_flag(self) -> int:
        """Verlet mode: this rank's displacement flag (cleared)."""
        v = int(self.vflag.item())
        _lib.call("cs_memset_async", _lib.ptr(self.vflag), 0, 4, self._s())
        return v

    def wrap(self):
        a = self.A
        _lib.call("cs_wrap_positions", self.n_owned, C.byref(self.cbox), _lib.ptr(a["x"]), _lib.ptr(a["y"]),
                  _lib.ptr(a["z"]), self._s())

    def build_list(self):
        """Round tables over the local grid (owned planes + the ghost plane)."""
        a = self.A
        _lib.call("cs_verlet_build", C.byref(self.cbox), C.byref(self.clj), self.skin,
                  _lib.ptr(self.cell_start), _lib.ptr(a["x"]), _lib.ptr(a["y"]), _lib.ptr(a["z"]),
                  _lib.ptr(self.vlist), self.vlist.numel(), *(_lib.ptr(t) for t in self.xref),
                  self.n_owned, _lib.ptr(self.status), self._s())

    def kick_predict(self, kick: bool = True):
        """Verlet: post-kick (optional) + this rank's flag for the next step."""
        a = self.A
        hdtm = 0.5 * self.dt / self.params.mass
        _lib.call("cs_vv_kick_predict", self.n_owned, hdtm, self.dt, int(kick), _lib.ptr(a["fx"]),
                  _lib.ptr(a["fy"]), _lib.ptr(a["fz"]), _lib.ptr(a["vx"]), _lib.ptr(a["vy"]),
                  _lib.ptr(a["vz"]), _lib.ptr(a["x"]), _lib.ptr(a["y"]), _lib.ptr(a["z"]),
                  *(_lib.ptr(t) for t in self.xref), 0.5 * self.skin, _lib.ptr(self.vflag), self._s())

    def kick(self):
        a = self.A
        hdtm = 0.5 * self.dt / self.params.mass
        _lib.call("cs_vv_kick", self.n_owned, hdtm, _lib.ptr(a["fx"]), _lib.ptr(a["fy"]),
                  _lib.ptr(a["fz"]), _lib.ptr(a["vx"]), _lib.ptr(a["vy"]), _lib.ptr(a["vz"]), self._s())

    def split(self):
        a = self.A
        cnt = (C.c_int64 * 3)()
        _lib.call("cs_slab_split", self.n_owned, C.byref(self.cbox), _lib.ptr(a["x"]), _lib.ptr(a["y"]),
                  _lib.ptr(a["z"]), _lib.ptr(a["vx"]), _lib.ptr(a["vy"]), _lib.ptr(a["vz"]),
                  _lib.ptr(a["id"]), _lib.ptr(self.P_stay), self.cap, _lib.ptr(self.P_l),
                  _lib.ptr(self.P_r), self.mcap, cnt, _lib.ptr(self.ws), self.wsb, self._s())
        self._nstay = cnt[0]
        pack = lambda P, m, stride: P.view(7, stride)[:, :m].reshape(-1)
        return ((self.P_stay, cnt[0], self.cap), pack(self.P_l, cnt[1], self.mcap),
                pack(self.P_r, cnt[2], self.mcap))

    def assemble(self, stay, from_left, from_right):
        P, m, stride = stay
        b = self.B
        off = 0
        for src, cnt, st in ((P, m, stride), (from_left, from_left.numel() // 7, from_left.numel() // 7),
                             (from_right, from_right.numel() // 7, from_right.numel() // 7)):
            if cnt == 0:
                continue
            if off + cnt > self.cap:
                raise _lib.CellschedError("slab capacity exceeded by migration")
            sl = {k: b[k][off:] for k in ("x", "y", "z", "vx", "vy", "vz", "id")}
            _lib.call("cs_unpack7", cnt, _lib.ptr(src), st, *(_lib.ptr(sl[k]) for k in
                      ("x", "y", "z", "vx", "vy", "vz", "id")), self._s())
            off += cnt
        self.n_owned = off
        self.A, self.B = self.B, self.A  # owned particles now live in A (unsorted)

    def build_cells(self):
        a, b = self.A, self.B
        _lib.call("cs_build_cells", self.n_owned, C.byref(self.cbox), _lib.ptr(a["x"]), _lib.ptr(a["y"]),
                  _lib.ptr(a["z"]), _lib.ptr(a["vx"]), _lib.ptr(a["vy"]), _lib.ptr(a["vz"]),
                  _lib.ptr(a["id"]), _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]),
                  _lib.ptr(b["vx"]), _lib.ptr(b["vy"]), _lib.ptr(b["vz"]), _lib.ptr(b["id"]),
                  _lib.ptr(b["fx"]), _lib.ptr(b["fy"]), _lib.ptr(b["fz"]), _lib.ptr(self.cell_start),
                  _lib.ptr(self.ws), self.wsb, self._s())
        self.A, self.B = self.B, self.A

    def pack_first_plane(self, xshift, cached: bool = False):
        torch = _torch()
        if cached:  # Verlet between rebuilds: same cells, same particle range
            lo, hi = self._first_range
        else:
            rng = (C.c_int64 * 2)()
            _lib.call("cs_plane_counts", C.byref(self.cbox), 0, _lib.ptr(self.cell_start),
                      _lib.ptr(self.counts), rng, self._s())
            lo, hi = self._first_range = (rng[0], rng[1])
        out = torch.empty(3 * (hi - lo), dtype=torch.float64, device=self.device)
        a = self.A
        _lib.call("cs_pack_range", lo, hi, _lib.ptr(a["x"]), _lib.ptr(a["y"]), _lib.ptr(a["z"]),
                  float(xshift), _lib.ptr(out), self._s())
        return (None if cached else self.counts.to(torch.float64)), out

    def set_ghosts(self, counts, xyz):
        torch = _torch()
        m = xyz.numel() // 3
        if self.n_owned + m > self.cap:
            raise _lib.CellschedError("slab capacity exceeded by the ghost plane")
        c32 = counts.to(torch.int32).to(self.device)
        a = self.A
        _lib.call("cs_set_ghost_plane", C.byref(self.cbox), self.n_owned, _lib.ptr(c32),
                  _lib.ptr(xyz.to(self.device)), m, _lib.ptr(self.cell_start), _lib.ptr(a["x"]),
                  _lib.ptr(a["y"]), _lib.ptr(a["z"]), _lib.ptr(a["fx"]), _lib.ptr(a["fy"]),
                  _lib.ptr(a["fz"]), _lib.ptr(self.ws), self.wsb, self._s())
        self.n_ghost = m

    def update_ghosts(self, xyz):
        """Verlet, between rebuilds: same ghost particles in the same slots --
        overwrite their positions only (no cell-list work, no host sync)."""
        m, o, a = self.n_ghost, self.n_owned, self.A
        src = xyz.view(3, m)
        for k, key in enumerate(("x", "y", "z")):
            _lib.call("cs_copy_async", _lib.ptr(a[key][o:o + m]), _lib.ptr(src[k]), 8 * m, self._s())

    def forces(self, energy, sync: bool = True):
        """Local forces.  sync=False (Verlet, between rebuilds, no energy): no
        host reads; pairs go to the device accumulator only."""
        a = self.A
        _lib.call("cs_memset_async", _lib.ptr(self.scal), 0, 8, self._s())
        _lib.call("cs_memset_async", _lib.ptr(self.npairs), 0, 8, self._s())
        if self.verlet:
            _lib.call("cs_lj_forces_verlet", C.byref(self.cbox), C.byref(self.clj), self.sched,
                      self.n_owned + self.n_ghost, _lib.ptr(self.cell_start), _lib.ptr(self.vlist),
                      _lib.ptr(a["x"]), _lib.ptr(a["y"]), _lib.ptr(a["z"]), _lib.ptr(a["fx"]),
                      _lib.ptr(a["fy"]), _lib.ptr(a["fz"]), _lib.ptr(self.scal) if energy else None,
                      _lib.ptr(self.npairs), _lib.ptr(self.status), _lib.ptr(self.ws), self.wsb, self._s())
            _lib.call("cs_accumulate_i64", _lib.ptr(self.pairs_acc), _lib.ptr(self.npairs), self._s())
            if not sync:
                return 0.0, 0
            if int(self.status.item()):
                raise _lib.CellschedError("Verlet slab: kernel capacity flag %d" % int(self.status.item()))
            return float(self.scal[0].item()) if energy else 0.0, int(self.npairs.item())
        _lib.call("cs_lj_forces", C.byref(self.cbox), C.byref(self.clj), self.sched,
                  self.n_owned + self.n_ghost, _lib.ptr(self.cell_start), _lib.ptr(a["x"]),
                  _lib.ptr(a["y"]), _lib.ptr(a["z"]), _lib.ptr(a["fx"]), _lib.ptr(a["fy"]),
                  _lib.ptr(a["fz"]), _lib.ptr(self.scal) if energy else None, _lib.ptr(self.npairs),
                  _lib.ptr(self.status), _lib.ptr(self.ws), self.wsb, self._s())
        _lib.call("cs_accumulate_i64", _lib.ptr(self.pairs_acc), _lib.ptr(self.npairs), self._s())
        if int(self.status.item()):
            raise _lib.CellschedError("force kernel capacity overflow (use schedule='shell')")
        return float(self.scal[0].item()) if energy else 0.0, int(self.npairs.item())

    def pack_ghost_forces(self):
        """Ghost-plane forces (the ghost plane is the array tail [n_owned, n_owned + n_ghost))."""
        torch = _torch()
        out = torch.empty(3 * self.n_ghost, dtype=torch.float64, device=self.device)
        a = self.A
        _lib.call("cs_pack_range", self.n_owned, self.n_owned + self.n_ghost, _lib.ptr(a["fx"]),
                  _lib.ptr(a["fy"]), _lib.ptr(a["fz"]), 0.0, _lib.ptr(out), self._s())
        return out

    def add_first_plane_forces(self, f):
        a = self.A
        lo, hi = self._first_range  # set by pack_first_plane in the same force evaluation
        _lib.call("cs_add_range_forces", lo, hi, _lib.ptr(f.to(self.device)), _lib.ptr(a["fx"]),
                  _lib.ptr(a["fy"]), _lib.ptr(a["fz"]), self._s())

    def kinetic(self):
        a = self.A
        _lib.call("cs_kinetic", self.n_owned, self.params.mass, _lib.ptr(a["vx"]), _lib.ptr(a["vy"]),
                  _lib.ptr(a["vz"]), _lib.ptr(self.scal[1:]), _lib.ptr(self.ws), self.wsb, self._s())
        return float(self.scal[1].item())

    def owned_arrays(self):
        """Host copies of the owned particles (cell-sorted): ids, x (n,3), f (n,3)."""
        torch = _torch()
        a, n = self.A, self.n_owned
        return {"id": a["id"][:n].cpu().numpy(),
                "x": torch.stack([a[k][:n] for k in ("x", "y", "z")], 1).cpu().numpy(),
                "v": torch.stack([a[k][:n] for k in ("vx", "vy", "vz")], 1).cpu().numpy(),
                "f": torch.stack([a[k][:n] for k in ("fx", "fy", "fz")], 1).cpu().numpy()}
