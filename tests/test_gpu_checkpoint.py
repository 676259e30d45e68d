"""npz checkpoint / resume (SURVEY section 5 auxiliaries): a restored system
continues bit-identically -- link-cell and Verlet schedules, eager and
graph-replayed steps, list rebuilds after the restore included."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1401_4441_b200 import md

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("sched,graph", [("buffered", False), ("verlet", True), ("verlet_dataflow", False)])
def test_checkpoint_resume_bit_identical(cuda, tmp_path, sched, graph):
    kw = {"skin": 0.12} if sched.startswith("verlet") else {}
    a = md.LJSystem.fcc(14 if sched.startswith("verlet") else 12, schedule=sched, seed=7, **kw)
    stepper = (lambda s: s.graph_step()) if graph else (lambda s: s.step())
    for _ in range(5):
        stepper(a)
    a.checkpoint(tmp_path / "ck.npz")
    b = md.LJSystem.restore(tmp_path / "ck.npz")
    assert (b.nstep, b.seed, b.schedule, b.box) == (5, 7, sched, a.box)
    for _ in range(12):
        stepper(a)
        stepper(b)
    if sched.startswith("verlet"):
        assert a.list_builds + int(a.graph_builds.item()) > 1  # rebuilds happened after the restore
    sa, sb = a.snapshot(), b.snapshot()
    for k in ("x", "v", "f", "id", "cell_start"):
        assert np.array_equal(sa[k], sb[k]), k
    a.kinetic(), b.kinetic()
    assert a.energies()[1] == b.energies()[1]
