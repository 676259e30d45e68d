"""cfg5 (BASELINE configs[4]): liquid slab + vapour, load-imbalance stress.

A scaled-down box (24 x 24 x 72 cells of edge 2.5: 171,500 liquid + 2,880
vapour particles) against the CPU oracle: forces, energy, pair count, and
10 steps, under the link-cell schedules and the Verlet schedule.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_1401_4441_b200 import md

pytestmark = pytest.mark.gpu

CELLS = (24, 24, 72)


def force_err(f, ref):
    frms = np.sqrt((ref ** 2).sum(1).mean())
    return (np.linalg.norm(f - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), frms)).max()


def by_id(snap, key):
    return snap[key][np.argsort(snap["id"])]


@pytest.mark.parametrize("sched", ["buffered", "dataflow", "verlet", "verlet_shell", "verlet_dataflow"])
def test_cfg5_small_forces(oracle, cuda, sched):
    s = md.LJSystem.liquid_vapour(CELLS, schedule=sched, skin=0.3)
    snap = s.snapshot()
    counts = np.diff(snap["cell_start"])
    assert counts.max() >= 10 and (counts <= 1).sum() > 0.3 * counts.size  # liquid vs vapour cells
    x = snap["x"]
    f, pe, npair = oracle.lj_direct(list(s.box.cells), list(s.box.lengths), snap["cell_start"],
                                    np.ascontiguousarray(x[:, 0]), np.ascontiguousarray(x[:, 1]),
                                    np.ascontiguousarray(x[:, 2]), rc=2.5)
    assert force_err(snap["f"], f) < 1e-10
    assert abs(s.energies()[0] - pe) / abs(pe) < 1e-12
    assert s.pair_count() == npair


def test_cfg5_small_trajectory(oracle, cuda):
    s = md.LJSystem.liquid_vapour(CELLS, schedule="verlet", skin=0.3)
    ini = {k: v.cpu().numpy()[: s.n] for k, v in s.initial.items()}
    s.kinetic()
    e_dev = [sum(s.energies())]
    for _ in range(10):
        s.step(energy=True)
        e_dev.append(sum(s.energies()))
    ref = oracle.md_run(ini["x"], ini["y"], ini["z"], ini["vx"], ini["vy"], ini["vz"], ini["id"],
                        list(CELLS), list(s.box.lengths), 10)
    e_ref = ref["pe"] + ref["ke"]
    assert (np.abs(np.array(e_dev) - e_ref) / abs(e_ref[0])).max() <= 1e-12
    o = np.argsort(ref["id"])
    assert force_err(by_id(s.snapshot(), "f"), ref["f"][o]) < 1e-9
