"""Oracle parity of the BENCHMARKED path at BASELINE's full sizes.

The bench's default schedule is `verlet` (round tables on cells of edge >=
rc + skin, skin 0.35, buffered block schedule).  These tests run exactly that
path on cfg1 (the north star's tolerance config), full cfg2, cfg3, cfg4 and
full cfg5 and compare it with the CPU oracle (oracle/cs_oracle.c, the
reference_oracle pattern of payload.py:152-174, OpenMP over cells):

* cell lists (cell_start + id order) bit-exact, at the start and at list
  rebuilds inside a trajectory;
* pair counts exact;
* per-particle force rel. err <= 1e-10 with the F_rms floor, PE <= 1e-12;
* total energy per step <= 1e-12 (relative) for the first 10 steps of a
  cfg2 trajectory that spans >= 5 list rebuilds; the drift to 100 steps is
  reported (chaotic growth of round-off) and bounded at 1e-10.

Summation orders differ (device: per-round lane sums and fixed-order block
merges; oracle: sequential per particle), which is what the tolerances cover.
"""

from __future__ import annotations

import warnings

import numpy as np
import pytest

from paper_1401_4441_b200 import md

pytestmark = pytest.mark.gpu

FORCE_TOL = 1e-10
ENERGY_TOL = 1e-12
SKIN = 0.35


def force_err(f, ref):
    frms = np.sqrt((ref ** 2).sum(1).mean())
    return (np.linalg.norm(f - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), frms)).max()


def check_cell_list(oracle, s, snap):
    """The device cell list equals the oracle's stable counting sort of the
    same positions (fed in id order)."""
    o = np.argsort(snap["id"])
    x = np.ascontiguousarray(snap["x"][o])
    _, start, order = oracle.bin_cells(np.ascontiguousarray(x[:, 0]), np.ascontiguousarray(x[:, 1]),
                                       np.ascontiguousarray(x[:, 2]), snap["id"][o], list(s.box.cells),
                                       list(s.box.inv))
    assert np.array_equal(start, snap["cell_start"])
    assert np.array_equal(snap["id"][o][order], snap["id"])


def check_forces(oracle, s, snap=None):
    snap = snap or s.snapshot()
    x = snap["x"]
    f, pe, npair = oracle.lj_direct(list(s.box.cells), list(s.box.lengths), snap["cell_start"],
                                    np.ascontiguousarray(x[:, 0]), np.ascontiguousarray(x[:, 1]),
                                    np.ascontiguousarray(x[:, 2]), rc=s.params.rc)
    err = force_err(snap["f"], f)
    pe_dev = s.energies()[0]
    assert err <= FORCE_TOL, err
    assert abs(pe_dev - pe) / abs(pe) <= ENERGY_TOL, (pe_dev, pe)
    assert s.pair_count() == npair
    return err, npair


def test_cfg1_verlet_path(oracle, cuda):
    """cfg1 (864 particles, 4^3 cells) on the benchmarked Verlet path: the
    skin narrows to L/4 - rc (4 cells is the minimum), one force evaluation
    plus 10 VV steps against the oracle."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s = md.LJSystem.fcc(6, schedule="verlet", skin=SKIN)
    assert s.box.cells == (4, 4, 4) and s.n == 864 and 0 < s.skin < 0.02
    check_cell_list(oracle, s, s.snapshot())
    check_forces(oracle, s)
    ini = {k: v.cpu().numpy()[: s.n] for k, v in s.initial.items()}
    s.kinetic()
    e_dev = [sum(s.energies())]
    for _ in range(10):
        s.graph_step(energy=True)
        e_dev.append(sum(s.energies()))
    ref = oracle.md_run(ini["x"], ini["y"], ini["z"], ini["vx"], ini["vy"], ini["vz"], ini["id"],
                        [4, 4, 4], list(s.box.lengths), 10)
    e_ref = ref["pe"] + ref["ke"]
    assert (np.abs(np.array(e_dev) - e_ref) / abs(e_ref[0])).max() <= ENERGY_TOL
    assert int(s.graph_builds.item()) >= 2  # the narrow skin forces rebuilds


def test_cfg2_bench_path_forces(oracle, cuda):
    """Full cfg2 (442,368 particles), the bench system: cell list, pairs,
    forces, PE."""
    s = md.LJSystem.fcc(48, schedule="verlet", skin=SKIN)
    assert s.box.cells == (28, 28, 28) and s.n == 442368
    snap = s.snapshot()
    check_cell_list(oracle, s, snap)
    check_forces(oracle, s, snap)


def test_cfg2_trajectory_100_steps(oracle, cuda):
    """100 graph-replayed VV steps of the bench system (list rebuilds inside
    the graph, >= 5 of them) against the oracle's trajectory from the same
    initial state; cell lists checked at every rebuild."""
    s = md.LJSystem.fcc(48, schedule="verlet", skin=SKIN)
    ini = {k: v.cpu().numpy()[: s.n] for k, v in s.initial.items()}
    s.kinetic()
    e_dev = [sum(s.energies())]
    builds, checked = int(s.graph_builds.item()), 0
    for _ in range(100):
        s.graph_step(energy=True)
        e_dev.append(sum(s.energies()))
        nb = int(s.graph_builds.item())
        if nb != builds:  # a rebuild happened in this step: its cell list is current
            check_cell_list(oracle, s, s.snapshot())
            builds, checked = nb, checked + 1
    assert checked >= 5, checked
    ref = oracle.md_run(ini["x"], ini["y"], ini["z"], ini["vx"], ini["vy"], ini["vz"], ini["id"],
                        list(s.box.cells), list(s.box.lengths), 100)
    e_ref = ref["pe"] + ref["ke"]
    rel = np.abs(np.array(e_dev) - e_ref) / abs(e_ref[0])
    print(f"cfg2 energy rel err: first 10 steps {rel[:11].max():.2e}, 100 steps {rel.max():.2e}, "
          f"{checked} rebuilds checked")
    assert rel[:11].max() <= ENERGY_TOL
    assert rel.max() <= 1e-10
    snap = s.snapshot()
    o, r = np.argsort(snap["id"]), np.argsort(ref["id"])
    d = snap["x"][o] - ref["x"][r]
    L = np.asarray(s.box.lengths)
    assert np.abs(d - L * np.rint(d / L)).max() < 1e-9


def test_cfg3_forces(oracle, cuda):
    """cfg3 (96^3 FCC = 3,538,944 particles; Verlet cells 56^3)."""
    s = md.LJSystem.fcc(96, schedule="verlet", skin=SKIN)
    assert s.n == 3538944 and s.box.cells == (56, 56, 56)
    snap = s.snapshot()
    check_cell_list(oracle, s, snap)
    check_forces(oracle, s, snap)


def test_cfg5_forces_and_steps(oracle, cuda):
    """Full cfg5 (liquid-vapour slab on the 64x64x192 box of edge 2.5;
    Verlet cells 56x56x168): forces at t = 0, then 20 VV steps whose energy
    follows the oracle's trajectory."""
    s = md.LJSystem.liquid_vapour(schedule="verlet", skin=SKIN, seed=42)
    assert s.box.lengths == (160.0, 160.0, 480.0) and s.n > 3_000_000
    snap = s.snapshot()
    check_cell_list(oracle, s, snap)
    check_forces(oracle, s, snap)
    ini = {k: v.cpu().numpy()[: s.n] for k, v in s.initial.items()}
    s.kinetic()
    e_dev = [sum(s.energies())]
    for _ in range(20):
        s.graph_step(energy=True)
        e_dev.append(sum(s.energies()))
    ref = oracle.md_run(ini["x"], ini["y"], ini["z"], ini["vx"], ini["vy"], ini["vz"], ini["id"],
                        list(s.box.cells), list(s.box.lengths), 20)
    e_ref = ref["pe"] + ref["ke"]
    assert (np.abs(np.array(e_dev) - e_ref) / abs(e_ref[0])).max() <= ENERGY_TOL


@pytest.mark.slow
def test_cfg4_forces(oracle, cuda):
    """cfg4 (192^3 FCC = 28,311,552 particles; Verlet cells 112^3)."""
    s = md.LJSystem.fcc(192, schedule="verlet", skin=SKIN)
    assert s.n == 28311552 and s.box.cells == (112, 112, 112)
    snap = s.snapshot()
    check_cell_list(oracle, s, snap)
    check_forces(oracle, s, snap)
