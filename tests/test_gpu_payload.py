"""K5: the reference's integer payload on the device, bit-exact vs the
reference's golden accumulators -- directly, replayed along stream levels,
and under the LJ kernel's colour-pass schedules with the race detector on."""

from __future__ import annotations

import hashlib
import warnings

import numpy as np
import pytest

import paper_1401_4441_b200 as P
from paper_1401_4441_b200 import payload
from conftest import case_id

pytestmark = pytest.mark.gpu


def _grid(case):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return P.GridSpec(tuple(case["extents"]), periodic=case["periodic"])


def test_payload_matches_reference(golden, cuda):
    for case in golden["cases"]:
        g = _grid(case)
        for seed, ref in case["payload"].items():
            seed = int(seed)
            assert P.charges(g, seed) == ref["charges"], case_id(case)
            want = ref["oracle"]
            assert payload.reference_oracle_device(g, seed).cpu().tolist() == want
            for strat in ("loopex", "basic"):
                got = P.execute_with_payload(strat, g, seed)
                assert [got[c] for c in g.cells()] == ref[strat], (case_id(case), strat)


def test_payload_100_seeds(golden, cuda):
    for key, hashes in golden["payload_hashes"].items():
        g = P.GridSpec(tuple(int(v) for v in key.split("x")))
        for seed, ref in enumerate(hashes):
            acc = payload.reference_oracle_device(g, seed).cpu().numpy().astype(np.int64)
            assert hashlib.sha256(acc.tobytes()).hexdigest() == ref, (key, seed)


@pytest.mark.parametrize("ext", [(4, 4, 4), (8, 8, 8), (6, 4, 8), (16, 16, 16), (32, 32, 32)])
@pytest.mark.parametrize("sched,block", [("loopex", (2, 2, 2)), ("block", (2, 2, 2)),
                                         ("block", (1, 2, 2)), ("block", (2, 2, 4))])
def test_colour_passes_race_free_and_exact(ext, sched, block, cuda):
    if any(e % (2 * b) for e, b in zip(ext, block)):
        pytest.skip("block does not tile the grid")
    g = P.GridSpec(ext)
    for seed in (0, 42):
        want = payload.reference_oracle_device(g, seed)
        got = payload.colour_pass_payload(g, seed, sched, block, race_check=True)
        assert cuda.equal(got, want), (ext, sched, block, seed)


def test_race_detector_fires_on_invalid_schedule(cuda):
    # 2x2x2 whole-shell colouring is NOT conflict-free;
    # block (2,1,2) violates By >= 2 and must be rejected up front
    g = P.GridSpec((8, 8, 8))
    with pytest.raises(ValueError):
        payload.colour_pass_payload(g, 1, "block", (2, 1, 2))
    # odd extents break the loop-exchange parity classes: conflicts detected
    g = P.GridSpec((5, 6, 6))
    with pytest.raises(Exception):
        payload.colour_pass_payload(g, 1, "loopex", (2, 2, 2), race_check=True)
