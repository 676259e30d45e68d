"""Host-side LJ set-up logic (no GPU): cfg5 liquid-vapour generator, boxes."""

from __future__ import annotations

import numpy as np
import pytest
from scipy.spatial import cKDTree

from paper_1401_4441_b200 import md


def test_liquid_vapour_small():
    L, xyz = md.liquid_vapour_positions((8, 8, 24), seed=3)
    assert L == (20.0, 20.0, 60.0)
    assert xyz.dtype == np.float64 and xyz.shape[1] == 3
    assert (xyz >= 0).all() and (xyz < np.array(L)).all()
    # liquid: FCC tiling x and y exactly, in the middle third along z
    nx = round(20.0 / (4 / 0.8) ** (1 / 3))
    nl = 4 * nx * nx * round(20.0 / (20.0 / nx))
    liq, vap = xyz[:nl], xyz[nl:]
    assert liq[:, 2].min() > 19.0 and liq[:, 2].max() < 41.0
    assert len(vap) == round(0.02 * 20 * 20 * (60 - 20))
    assert ((vap[:, 2] < 20.0) | (vap[:, 2] >= 40.0)).all()
    # no pair closer than 0.9 sigma (periodic)
    d = cKDTree(xyz, boxsize=L).query(xyz, k=2)[0][:, 1]
    assert d.min() >= 0.9
    # deterministic in the seed
    _, again = md.liquid_vapour_positions((8, 8, 24), seed=3)
    assert np.array_equal(again, xyz)
    _, other = md.liquid_vapour_positions((8, 8, 24), seed=4)
    assert not np.array_equal(other[nl:], vap)


def test_liquid_vapour_rejects_non_square():
    with pytest.raises(ValueError):
        md.liquid_vapour_positions((8, 12, 24))


def test_boxes():
    box, nuc, a = md.fcc_box(48, 0.8442)
    assert box.cells == (32, 32, 32) and nuc == (48, 48, 48)
    assert abs(box.lengths[0] - 48 * (4 / 0.8442) ** (1 / 3)) < 1e-12
    wide = md.LJBox.for_cutoff(box.lengths, 2.5 + 0.35)
    assert wide.cells == (28, 28, 28) and min(wide.cell_edge) >= 2.85
    with pytest.raises(ValueError):
        md.LJBox((10.0, 10.0, 10.0), (2, 4, 4))
    with pytest.raises(ValueError):
        md.LJParams(rc=-1.0)
