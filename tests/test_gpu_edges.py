"""Edge cases of the LJ path against the O(N^2) minimum-image oracle: empty
and single-particle systems, pairs at exactly rc (excluded, r^2 < rc^2 is
strict) and at the force zero 2^(1/6), pairs across every periodic face,
positions at 0, -0.0 and just below L -- for the link-cell and the Verlet
schedules."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1401_4441_b200 import md

pytestmark = pytest.mark.gpu
SCHEDS = ["buffered", "shell", "dataflow", "loopex", "verlet", "verlet_dataflow"]


def system(sched, xyz, L=20.16):
    kw = {"skin": 0.3} if sched.startswith("verlet") else {}
    if sched.startswith("verlet"):
        box, skin = md.verlet_box((L, L, L), 2.5, kw["skin"])
        kw["skin"] = skin
    else:
        box = md.LJBox.for_cutoff((L, L, L), 2.5)
    n = len(xyz)
    s = md.LJSystem(box, n, schedule=sched, **kw)
    z = np.zeros(n)
    s.load_host(xyz[:, 0] if n else z, xyz[:, 1] if n else z, xyz[:, 2] if n else z, z, z, z,
                np.arange(n, dtype=np.int32))
    return s


def check(oracle, s, xyz):
    n = len(xyz)
    snap = s.snapshot()
    pe_dev = s.energies()[0]
    if n < 2:
        assert pe_dev == 0.0 and s.pair_count() == 0 and np.all(snap["f"] == 0)
        return
    L = np.asarray(s.box.lengths)
    f, pe, npair = oracle.lj_brute(L, *(np.ascontiguousarray(xyz[:, k] % L[k]) for k in range(3)))
    o = np.argsort(snap["id"])
    assert s.pair_count() == npair
    fd = snap["f"][o]
    scale = max(np.abs(f).max(), 1.0)
    assert np.abs(fd - f).max() <= 1e-12 * scale
    assert abs(pe_dev - pe) <= 1e-12 * max(abs(pe), 1.0)


@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("n", [0, 1])
def test_empty_and_single(oracle, cuda, sched, n):
    xyz = np.array([[1.0, 2.0, 3.0]])[:n]
    check(oracle, system(sched, xyz), xyz)


@pytest.mark.parametrize("sched", SCHEDS)
def test_cutoff_and_force_zero_across_faces(oracle, cuda, sched):
    L = 20.16
    r0 = 2.0 ** (1.0 / 6.0)
    pts = [
        [0.0, 5.0, 5.0], [L - 2.5 + 1e-9, 5.0, 5.0],      # just outside rc across the x face
        [10.0, 0.0, 10.0], [10.0, L - 2.4, 10.0],          # inside rc across the y face
        [15.0, 15.0, -0.0], [15.0, 15.0, L - r0],          # exactly at the force zero across z
        [5.0, 15.0, 15.0], [5.0 + 2.5, 15.0, 15.0],        # exactly rc: excluded
        [L - 1e-12, L - 1e-12, L - 1e-12], [0.5, 0.5, 0.5],  # corner images
    ]
    xyz = np.array(pts)
    check(oracle, system(sched, xyz, L), xyz)
