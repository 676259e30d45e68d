"""Pin the LJ part of the oracle (no reference LJ exists -- parity unpinned
w.r.t. the reference): known answers, Newton 3, brute-force agreement, and
agreement of the direct / task-replay / threaded colour-pass restatements
over the reference's own task streams."""

from __future__ import annotations

import numpy as np
import pytest

RHO, T0 = 0.8442, 0.722


def cfg1(oracle, seed=42):
    a = (4 / RHO) ** (1 / 3)
    L = 6 * a
    x, y, z = oracle.fcc_positions([6] * 3, [a] * 3, [L] * 3, 0.05, seed)
    return x, y, z, L


def test_known_answers(oracle):
    L = [20.0] * 3
    for r, U, F in ((2 ** (1 / 6), -1.0, 0.0), (1.0, 0.0, 24.0), (2.5, 0.0, 0.0)):
        x = np.array([5.0, 5.0 + r])
        y = np.array([5.0, 5.0])
        z = y.copy()
        f, pe, n = oracle.lj_brute(L, x, y, z)
        if r == 2.5:  # r == rc is outside the strict cutoff
            assert n == 0 and pe == 0.0
            continue
        assert n == 1
        assert pe == pytest.approx(U, abs=1e-14)
        assert f[0, 0] == pytest.approx(-F, abs=1e-12)
        assert np.array_equal(f[0], -f[1])  # Newton 3, exactly


def test_direct_tasks_brute_threads_agree(oracle):
    x, y, z, L = cfg1(oracle)
    nc = [4, 4, 4]
    _, start, order = oracle.bin_cells(x, y, z, None, nc, [4 / L] * 3)
    xs, ys, zs = x[order], y[order], z[order]
    fd, ped, npd = oracle.lj_direct(nc, [L] * 3, start, xs, ys, zs)
    st = oracle.canonical_stencil(3)
    fl, pel, npl = oracle.lj_tasks(nc, [L] * 3, start, xs, ys, zs, *oracle.stream_loopex(nc), st)
    h, nb, e = oracle.stream_basic(nc, True, st)
    fb, peb, npb = oracle.lj_tasks(nc, [L] * 3, start, xs, ys, zs, h, nb, e, st)
    fx, pex, npx = oracle.lj_brute([L] * 3, xs, ys, zs)
    ft, pet, npt = oracle.lj_loopex_threads(nc, [L] * 3, start, xs, ys, zs, 4)
    frms = np.sqrt((fd ** 2).sum(1).mean())
    for f, pe, npair in ((fl, pel, npl), (fb, peb, npb), (fx, pex, npx), (ft, pet, npt)):
        assert npair == npd
        assert abs(pe - ped) / abs(ped) < 1e-13
        err = np.linalg.norm(f - fd, axis=1) / np.maximum(np.linalg.norm(fd, axis=1), frms)
        assert err.max() < 1e-12
    assert np.abs(fd.sum(0)).max() < 1e-10 * frms * len(x)
    assert 23000 < npd < 24500  # ~27.6 pairs per particle at rho 0.8442


def test_cell_list_canonical_order(oracle):
    x, y, z, L = cfg1(oracle)
    ids = np.arange(len(x), dtype=np.int32)
    perm = np.random.default_rng(0).permutation(len(x))
    c1, s1, o1 = oracle.bin_cells(x, y, z, ids, [4] * 3, [4 / L] * 3)
    c2, s2, o2 = oracle.bin_cells(x[perm], y[perm], z[perm], ids[perm], [4] * 3, [4 / L] * 3)
    assert np.array_equal(s1, s2)
    assert np.array_equal(ids[o1], ids[perm][o2])  # (cell, id) order is history free


def test_velocities_and_trajectory(oracle):
    x, y, z, L = cfg1(oracle)
    n = len(x)
    vx, vy, vz = oracle.velocities(n, T0, 1.0, 42)
    assert abs(vx.sum()) < 1e-12 and abs(vy.sum()) < 1e-12
    ke = 0.5 * (vx @ vx + vy @ vy + vz @ vz)
    assert ke / (1.5 * (n - 1)) == pytest.approx(T0, rel=1e-14)
    r0 = oracle.md_run(x, y, z, vx, vy, vz, np.arange(n), [4] * 3, [L] * 3, 10, mode=0)
    r1 = oracle.md_run(x, y, z, vx, vy, vz, np.arange(n), [4] * 3, [L] * 3, 10, mode=1, nthreads=4)
    e0, e1 = r0["pe"] + r0["ke"], r1["pe"] + r1["ke"]
    assert np.abs(e1 - e0).max() / abs(e0[0]) < 1e-12
    # unshifted cutoff: small jumps, but bounded drift over 10 steps
    assert abs(e0[-1] - e0[0]) / abs(e0[0]) < 1e-3
