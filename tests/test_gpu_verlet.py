"""Verlet-list forces on the device vs the CPU oracle.

The Verlet schedules bin on cells of edge >= rc + skin, build per-cell round
tables from the cell list, and re-test every listed pair exactly (r^2 < rc^2),
so forces match the link-cell path and the oracle within the same tolerances
(per-particle force rel. err <= 1e-10, energy rel. err <= 1e-12 after 10
steps); positions are only wrapped at list rebuilds.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_1401_4441_b200 import md

pytestmark = pytest.mark.gpu

FORCE_TOL = 1e-10
ENERGY_TOL = 1e-12


def force_err(f, ref):
    frms = np.sqrt((ref ** 2).sum(1).mean())
    return (np.linalg.norm(f - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), frms)).max()


def by_id(snap, key):
    o = np.argsort(snap["id"])
    return snap[key][o]


def wrapped_diff(a, b, L):
    d = a - b
    return np.abs(d - np.asarray(L) * np.rint(d / np.asarray(L))).max()


@pytest.mark.parametrize("sched", ["verlet", "verlet_shell", "verlet_dataflow"])
def test_verlet_forces_vs_oracle(oracle, cuda, sched):
    s = md.LJSystem.fcc(14, schedule=sched, skin=0.3)
    assert s.box.cells == (8, 8, 8) and s.n == 10976
    snap = s.snapshot()
    x = snap["x"]
    f, pe, npair = oracle.lj_direct(list(s.box.cells), list(s.box.lengths), snap["cell_start"],
                                    np.ascontiguousarray(x[:, 0]), np.ascontiguousarray(x[:, 1]),
                                    np.ascontiguousarray(x[:, 2]), rc=2.5)
    assert force_err(snap["f"], f) < FORCE_TOL
    assert abs(s.energies()[0] - pe) / abs(pe) < ENERGY_TOL
    assert s.pair_count() == npair


@pytest.mark.parametrize("sched", ["verlet", "verlet_shell", "verlet_dataflow"])
def test_verlet_trajectory_with_rebuilds(oracle, cuda, sched):
    """10 steps with a small skin (several list rebuilds) against the
    oracle's link-cell trajectory from the same initial state."""
    s = md.LJSystem.fcc(14, schedule=sched, skin=0.12)
    ini = {k: v.cpu().numpy()[: s.n] for k, v in s.initial.items()}
    s.kinetic()
    e_dev = [sum(s.energies())]
    for _ in range(10):
        s.step(energy=True)
        e_dev.append(sum(s.energies()))
    assert s.list_builds >= 3
    ref = oracle.md_run(ini["x"], ini["y"], ini["z"], ini["vx"], ini["vy"], ini["vz"], ini["id"],
                        list(s.box.cells), list(s.box.lengths), 10)
    e_ref = ref["pe"] + ref["ke"]
    rel = np.abs(np.array(e_dev) - e_ref) / abs(e_ref[0])
    assert rel.max() <= ENERGY_TOL, rel
    snap = s.snapshot()
    o = np.argsort(ref["id"])
    assert wrapped_diff(by_id(snap, "x"), ref["x"][o], s.box.lengths) < 1e-11
    assert force_err(by_id(snap, "f"), ref["f"][o]) < 1e-9


def test_verlet_graph_matches_eager(cuda):
    """The CUDA graph with the conditional rebuild node replays the eager
    host-decided steps bit for bit, rebuilds included."""
    a = md.LJSystem.fcc(14, schedule="verlet", skin=0.12)
    b = md.LJSystem.fcc(14, schedule="verlet", skin=0.12)
    for _ in range(12):
        a.step()
        b.graph_step()
    assert a.list_builds >= 3
    sa, sb = a.snapshot(), b.snapshot()
    for k in ("x", "v", "f", "id", "cell_start"):
        assert np.array_equal(sa[k], sb[k]), k


def test_verlet_cfg2_matches_link_cell(cuda):
    """cfg2 (442,368 particles): Verlet forces (28^3 cells, skin 0.3) agree
    with the link-cell buffered kernel (32^3 cells) pair for pair."""
    v = md.LJSystem.fcc(48, schedule="verlet", skin=0.3)
    c = md.LJSystem.fcc(48, schedule="buffered")
    assert v.box.cells == (28, 28, 28)
    assert v.pair_count() == c.pair_count()
    fv, fc = by_id(v.snapshot(), "f"), by_id(c.snapshot(), "f")
    assert force_err(fv, fc) < FORCE_TOL
    assert abs(v.energies()[0] - c.energies()[0]) / abs(c.energies()[0]) < ENERGY_TOL
    # colour passes and their dataflow execution add in the same order
    vs = md.LJSystem.fcc(48, schedule="verlet_shell", skin=0.3)
    vd = md.LJSystem.fcc(48, schedule="verlet_dataflow", skin=0.3)
    assert np.array_equal(vs.snapshot()["f"], vd.snapshot()["f"])
    # deterministic round tables: a second build gives bit-identical forces
    v2 = md.LJSystem.fcc(48, schedule="verlet", skin=0.3)
    assert np.array_equal(v2.snapshot()["f"], v.snapshot()["f"])


def test_verlet_needs_wide_cells(cuda):
    box, nuc, a = md.fcc_box(14, 0.8442)  # cells of edge >= rc only
    with pytest.raises(ValueError):
        md.LJSystem(box, 4 * 14 ** 3, schedule="verlet", skin=0.3)


def test_verlet_crowded_cells_second_pass(oracle, cuda):
    """Home cells of 33-64 particles take the builder's second pass (two
    particles per lane): a dense-liquid-like fluctuation -- 14 particles added
    to one cell of an FCC system (21 per cell), no two closer than 0.75 --
    gives forces and pair count that still match the oracle."""
    rng = np.random.default_rng(5)
    base = md.LJSystem.fcc(14, schedule="verlet", skin=0.3)  # 8^3 cells of edge 2.94
    snap0 = base.snapshot()
    pts = snap0["x"] % np.asarray(base.box.lengths)
    edge = base.box.lengths[0] / base.box.cells[0]
    extra = []
    while len(extra) < 14:
        c = 0.1 + rng.random(3) * (edge - 0.2)
        allp = np.concatenate([pts, np.array(extra).reshape(-1, 3)])
        if np.min(np.linalg.norm(allp - c, axis=1)) >= 0.75:
            extra.append(c)
    pts = np.concatenate([pts, np.array(extra)])
    n = len(pts)
    s = md.LJSystem(base.box, n, schedule="verlet", skin=0.3)
    z = np.zeros(n)
    s.load_host(pts[:, 0], pts[:, 1], pts[:, 2], z, z, z, np.arange(n))
    snap = s.snapshot()
    assert 32 < np.diff(snap["cell_start"]).max() <= 64
    x = snap["x"]
    f, pe, npair = oracle.lj_direct(list(s.box.cells), list(s.box.lengths), snap["cell_start"],
                                    np.ascontiguousarray(x[:, 0]), np.ascontiguousarray(x[:, 1]),
                                    np.ascontiguousarray(x[:, 2]), rc=2.5)
    assert s.pair_count() == npair  # (also raises on a capacity flag)
    frms = np.sqrt((f ** 2).sum(1).mean())
    err = (np.linalg.norm(snap["f"] - f, axis=1) / np.maximum(np.linalg.norm(f, axis=1), frms)).max()
    assert err < 1e-10
    assert abs(s.energies()[0] - pe) / abs(pe) < 1e-12


def test_verlet_crowded_cell_is_reported(cuda):
    """A home cell with more than 64 particles cannot be laid out on a warp's
    lanes: the build flags it and the system raises instead of returning
    partial forces."""
    rng = np.random.default_rng(5)
    box = md.LJBox((24.0, 24.0, 24.0), (8, 8, 8))
    n = 3000
    pts = rng.random((n, 3)) * 24.0
    pts[:70] = 0.2 + rng.random((70, 3)) * 2.5  # 70 particles in one cell
    s = md.LJSystem(box, n, schedule="verlet", skin=0.3)
    z = np.zeros(n)
    s.load_host(pts[:, 0], pts[:, 1], pts[:, 2], z, z, z, np.arange(n))
    with pytest.raises(Exception, match="more than 64 particles"):
        s.energies()
