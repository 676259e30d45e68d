"""C-ABI guards from the round-1 review: odd periodic extents under the
loop-exchange passes are rejected (not raced), unwrapped host positions are
wrapped before binning and the range flag is readable, and per-device set-up
(stencil table, kernel attributes) is repeated on a second GPU."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1401_4441_b200 import _lib, md

pytestmark = pytest.mark.gpu


def test_loopex_rejects_odd_periodic_extent(cuda):
    """A direct C-ABI caller with an odd periodic extent gets EINVAL (the
    check runs before any launch, so the buffers are never touched)."""
    s = md.LJSystem.fcc(6, schedule="loopex")
    odd = _lib.CsBox()
    C.memmove(C.byref(odd), C.byref(s._cbox), C.sizeof(odd))
    odd.nc[1] = odd.gnc[1] = 3
    odd.L[1] = 3 * 2.6
    odd.inv[1] = 3 / odd.L[1]
    b = s._buf[s.cur]
    with pytest.raises(ValueError, match="even periodic extents"):
        _lib.call("cs_lj_forces", C.byref(odd), C.byref(s._clj), _lib.SCHED_LOOPEX, s.n,
                  _lib.ptr(s.cell_start), _lib.ptr(b["x"]), _lib.ptr(b["y"]), _lib.ptr(b["z"]),
                  _lib.ptr(b["fx"]), _lib.ptr(b["fy"]), _lib.ptr(b["fz"]), None, None,
                  _lib.ptr(s.status), _lib.ptr(s._ws), s._wsb, s._s())


@pytest.mark.parametrize("sched", ["buffered", "loopex"])
def test_unwrapped_positions_are_wrapped(cuda, sched):
    """load_host with positions shifted by whole box lengths gives the same
    cell list and forces as the wrapped positions, and no range flag."""
    ref = md.LJSystem.fcc(6, schedule=sched)
    ini = {k: v.cpu().numpy()[: ref.n] for k, v in ref.initial.items()}
    L = np.asarray(ref.box.lengths)
    shift = np.random.default_rng(1).integers(-2, 3, size=(ref.n, 3)) * L
    s = md.LJSystem(ref.box, ref.n, schedule=sched)
    s.load_host(ini["x"] + shift[:, 0], ini["y"] + shift[:, 1], ini["z"] + shift[:, 2],
                ini["vx"], ini["vy"], ini["vz"], ini["id"])
    assert s.bin_errors() == 0
    a, b = s.snapshot(), ref.snapshot()
    assert (a["x"] >= 0).all() and (a["x"] < L).all()
    oa, ob = np.argsort(a["id"]), np.argsort(b["id"])
    d = a["x"][oa] - b["x"][ob]
    assert np.abs(d - L * np.rint(d / L)).max() < 1e-12
    fa, fb = a["f"][oa], b["f"][ob]
    frms = np.sqrt((fb ** 2).sum(1).mean())
    assert (np.linalg.norm(fa - fb, axis=1) / np.maximum(np.linalg.norm(fb, axis=1), frms)).max() < 1e-10


def test_second_device(cuda):
    """Per-device set-up: the same system on cuda:1 after cuda:0 gives the
    same forces (the stencil table and kernel attributes are per device)."""
    if cuda.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    out = []
    for d in (0, 1):
        with cuda.cuda.device(d):
            s = md.LJSystem.fcc(14, schedule="verlet", skin=0.3)
            out.append(s.snapshot()["f"])
    assert np.array_equal(out[0], out[1])
