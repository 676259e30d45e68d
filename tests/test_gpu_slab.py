"""CUDA x-slab engine on one GPU: a 1-rank ring (ghost = own first plane +L)
and 2-3 virtual ranks in one process (threads + an in-process exchanger; no
kernel ever waits on another), checked against the single-domain oracle."""

from __future__ import annotations

import threading

import numpy as np
import pytest

from paper_1401_4441_b200 import md, slab

pytestmark = pytest.mark.gpu
RHO = 0.8442


class ThreadRingExchanger(slab.NeighbourExchanger):
    """In-process stand-in for torch.distributed: ranks are threads."""

    def __init__(self, layout, hub):
        super().__init__(layout)
        self.hub = hub

    def exchange(self, to_left, to_right):
        L, hub = self.layout, self.hub
        hub["box"][(L.rank, "L")] = to_left.clone()
        hub["box"][(L.rank, "R")] = to_right.clone()
        hub["bar"].wait()
        from_left = hub["box"][(L.left, "R")]
        from_right = hub["box"][(L.right, "L")]
        hub["bar"].wait()
        return from_left, from_right

    def exchange_fixed(self, to_left, to_right, n_from_left, n_from_right):
        return self.exchange(to_left, to_right)

    def allreduce_sum(self, values):
        L, hub = self.layout, self.hub
        hub["box"][(L.rank, "sum")] = list(values)
        hub["bar"].wait()
        tot = [sum(hub["box"][(r, "sum")][k] for r in range(L.world)) for k in range(len(values))]
        hub["bar"].wait()
        return tot


def _run(world, nuc, steps, schedule, oracle, cuda):
    torch = cuda
    box, nucs, a = md.fcc_box(nuc, RHO)
    ref_sys = md.LJSystem.fcc(nuc, schedule="loopex" if all(c % 2 == 0 for c in box.cells) else "block")
    ini = ref_sys.initial
    n = ref_sys.n
    hub = {"box": {}, "bar": threading.Barrier(world)}
    results, errors = {}, []

    def rank_main(r):
        try:
            lay = slab.SlabLayout(box.cells[0], world, r)
            eng = slab.CudaSlabEngine(box, lay, md.LJParams(), schedule=schedule)
            eng.load_global(*(ini[k][:n] for k in ("x", "y", "z", "vx", "vy", "vz", "id")))
            ex = ThreadRingExchanger(lay, hub) if world > 1 else slab.NeighbourExchanger(lay)
            st = slab.SlabStep(eng, ex)
            out = [st.start(energy=True)]
            f0 = eng.owned_arrays()
            for _ in range(steps):
                out.append(st.step(energy=True))
            torch.cuda.synchronize()
            results[r] = (out, f0, eng.owned_arrays())
        except Exception as exc:  # surface in the main thread
            errors.append(exc)
            hub["bar"].abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    hx = {k: ini[k][:n].cpu().numpy() for k in ini}
    ref = oracle.md_run(hx["x"], hx["y"], hx["z"], hx["vx"], hx["vy"], hx["vz"], hx["id"],
                        list(box.cells), list(box.lengths), steps)
    ref0 = oracle.md_run(hx["x"], hx["y"], hx["z"], hx["vx"], hx["vy"], hx["vz"], hx["id"],
                         list(box.cells), list(box.lengths), 0)
    ids = np.concatenate([results[r][1]["id"] for r in range(world)])
    f = np.concatenate([results[r][1]["f"] for r in range(world)])
    assert sorted(ids.tolist()) == list(range(n))
    fref = np.empty((n, 3))
    fref[ref0["id"]] = ref0["f"]
    frms = np.sqrt((fref ** 2).sum(1).mean())
    err = np.linalg.norm(f - fref[ids], axis=1) / np.maximum(np.linalg.norm(fref[ids], axis=1), frms)
    assert err.max() < 1e-10, err.max()
    e = np.array([o["pe"] + o["ke"] for o in results[0][0]])
    eref = ref["pe"] + ref["ke"]
    assert np.abs(e - eref).max() / abs(eref[0]) < 1e-12
    assert results[0][0][-1]["n"] == n


@pytest.mark.parametrize("schedule", ["loopex", "buffered", "shell"])
def test_slab_one_rank_ring(oracle, cuda, schedule):
    _run(1, 6, 4, schedule, oracle, cuda)


@pytest.mark.parametrize("world,schedule", [(2, "buffered"), (2, "loopex"), (3, "shell")])
def test_slab_virtual_ranks(oracle, cuda, world, schedule):
    _run(world, 12, 4, schedule, oracle, cuda)


def _run_verlet(world, nuc, steps, skin, oracle, cuda):
    """Verlet slabs: cells of edge >= rc + skin, list rebuilds (with migration)
    taken by every rank together, ghost plane refreshed in place between them."""
    torch = cuda
    box0, nucs, a = md.fcc_box(nuc, RHO)
    cells = md.LJBox.for_cutoff(box0.lengths, 2.5 + skin).cells
    box = md.LJBox(box0.lengths, (cells[0],) + tuple(c - c % 4 for c in cells[1:]))
    ref_sys = md.LJSystem.fcc(nuc, schedule="verlet", skin=skin)  # the seeded initial state
    ini = ref_sys.initial
    n = ref_sys.n
    hub = {"box": {}, "bar": threading.Barrier(world)}
    results, errors = {}, []

    class Ring(ThreadRingExchanger):
        def allreduce_max_int(self, value):
            L, hub = self.layout, self.hub
            hub["box"][(L.rank, "max")] = int(value)
            hub["bar"].wait()
            m = max(hub["box"][(r, "max")] for r in range(L.world))
            hub["bar"].wait()
            return m

    def rank_main(r):
        try:
            lay = slab.SlabLayout(box.cells[0], world, r)
            eng = slab.CudaSlabEngine(box, lay, md.LJParams(), schedule="verlet", skin=skin)
            eng.load_global(*(ini[k][:n] for k in ("x", "y", "z", "vx", "vy", "vz", "id")))
            ex = Ring(lay, hub) if world > 1 else slab.NeighbourExchanger(lay)
            st = slab.SlabStep(eng, ex)
            out = [st.start(energy=True)]
            f0 = eng.owned_arrays()
            for _ in range(steps):
                out.append(st.step(energy=True))
            torch.cuda.synchronize()
            results[r] = (out, f0, st.rebuilds)
        except Exception as exc:
            errors.append(exc)
            hub["bar"].abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    hx = {k: ini[k][:n].cpu().numpy() for k in ini}
    ref = oracle.md_run(hx["x"], hx["y"], hx["z"], hx["vx"], hx["vy"], hx["vz"], hx["id"],
                        list(box.cells), list(box.lengths), steps)
    ref0 = oracle.md_run(hx["x"], hx["y"], hx["z"], hx["vx"], hx["vy"], hx["vz"], hx["id"],
                         list(box.cells), list(box.lengths), 0)
    ids = np.concatenate([results[r][1]["id"] for r in range(world)])
    f = np.concatenate([results[r][1]["f"] for r in range(world)])
    assert sorted(ids.tolist()) == list(range(n))
    fref = np.empty((n, 3))
    fref[ref0["id"]] = ref0["f"]
    frms = np.sqrt((fref ** 2).sum(1).mean())
    err = np.linalg.norm(f - fref[ids], axis=1) / np.maximum(np.linalg.norm(fref[ids], axis=1), frms)
    assert err.max() < 1e-10, err.max()
    e = np.array([o["pe"] + o["ke"] for o in results[0][0]])
    eref = ref["pe"] + ref["ke"]
    assert np.abs(e - eref).max() / abs(eref[0]) < 1e-12
    assert results[0][0][-1]["n"] == n
    assert results[0][2] >= 2  # the initial build + at least one rebuild with migration


@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_verlet(oracle, cuda, world):
    _run_verlet(world, 14, 10, 0.12, oracle, cuda)


def test_slab_lookahead_is_bit_identical(cuda):
    """SlabStep(lookahead=True) launches the next kick-drift before the
    rebuild decision; over a run with rebuilds the result is bit for bit the
    plain stepping's."""
    import torch
    from paper_1401_4441_b200 import md, slab

    g = md.LJSystem.fcc(14, schedule="verlet", skin=0.12)  # the global initial state (10,976 particles)
    box, n = g.box, g.n
    ini = {k: v[:n] for k, v in g.initial.items()}
    c = md.LJBox.for_cutoff(box.lengths, 2.5 + 0.12).cells  # 8^3 Verlet cells, ~21 particles each
    vbox = md.LJBox(box.lengths, (c[0] - c[0] % 2,) + tuple(v - v % 4 for v in c[1:]))
    out = []
    for la in (False, True):
        lay = slab.SlabLayout(vbox.cells[0], 1, 0)
        eng = slab.CudaSlabEngine(vbox, lay, md.LJParams(), schedule="verlet", skin=0.12)
        eng.load_global(*(ini[k] for k in ("x", "y", "z", "vx", "vy", "vz", "id")))
        st = slab.SlabStep(eng, slab.NeighbourExchanger(lay))
        st.start(energy=True)
        nsteps = 25
        for k in range(nsteps):
            st.step(energy=False, reduce=False, lookahead=la and k < nsteps - 1)
        torch.cuda.synchronize()
        out.append((st.rebuilds, eng.owned_arrays()))
    assert out[0][0] == out[1][0] and out[0][0] >= 2
    for key in ("id", "x", "v", "f"):
        assert (out[0][1][key] == out[1][1][key]).all(), key
