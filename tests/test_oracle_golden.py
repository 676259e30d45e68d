"""Pin the CPU oracle to the reference's own outputs (golden vectors generated
by importing the unmodified reference, tests/golden/make_golden.py)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import case_id


def _orders(golden, dim):
    return {k: np.array(v, np.int8) for k, v in golden["orders"][str(dim)].items()}


def test_canonical_stencil(golden, oracle):
    for dim in (2, 3):
        st = oracle.canonical_stencil(dim)
        assert st.tolist() == golden["canonical_stencil"][str(dim)]


def test_streams_edges_depths(golden, oracle):
    for case in golden["cases"]:
        ext, per = case["extents"], case["periodic"]
        dim = len(ext)
        orders = _orders(golden, dim)
        for name, ref in case["streams"].items():
            if name == "loopex":
                h, nb, e = oracle.stream_loopex(ext, per)
            else:
                h, nb, e = oracle.stream_basic(ext, per, orders[name.split(":")[1]])
            assert h.tolist() == ref["home"], (case_id(case), name)
            assert nb.tolist() == ref["nbr"], (case_id(case), name)
            assert e.tolist() == ref["entry"], (case_id(case), name)
            eu, ev = oracle.detect_edges_stream(h, nb)
            assert eu.tolist() == ref["edges_u"] and ev.tolist() == ref["edges_v"], (case_id(case), name)
            d, lv = oracle.critical_path(len(h), eu, ev, levels=True)
            assert d == ref["depth"], (case_id(case), name)
            if "levels" in ref:
                assert lv.tolist() == ref["levels"]


def test_colors(golden, oracle):
    import ctypes as C

    for case in golden["cases"]:
        ext = case["extents"]
        e = oracle._ext(ext)
        got = [oracle.lib().o_color(c, e, len(ext), 2) for c in range(int(np.prod(ext)))]
        assert got == case["colors"]


def test_payload(golden, oracle):
    for case in golden["cases"]:
        ext, per = case["extents"], case["periodic"]
        st = oracle.canonical_stencil(len(ext))
        h, nb, e = oracle.stream_loopex(ext, per)
        for seed, ref in case["payload"].items():
            seed = int(seed)
            assert oracle.charges(ext, seed).tolist() == ref["charges"]
            acc = oracle.payload_reference(ext, per, seed)
            assert acc.tolist() == ref["oracle"], (case_id(case), seed)
            assert oracle.payload_apply(ext, per, seed, h, nb, e, st).tolist() == ref["loopex"]


def test_payload_100_seed_hashes(golden, oracle):
    for key, hashes in golden["payload_hashes"].items():
        ext = [int(v) for v in key.split("x")]
        for seed, ref in enumerate(hashes):
            acc = oracle.payload_reference(ext, True, seed)
            assert hashlib.sha256(acc.astype(np.int64).tobytes()).hexdigest() == ref, (key, seed)


def test_vector_example_with_reads(golden, oracle):
    # test_depgraph.py:37-66 Fig. 1/2 program: writes a,b,c; reads b writes c;
    # reads a,b writes d; reads c,d writes s   (resources a..s -> 0..5)
    w = [[0], [1], [2], [2], [3], [4]]
    r = [[], [], [], [1], [0, 1], [2, 3]]
    wptr = np.cumsum([0] + [len(x) for x in w])
    rptr = np.cumsum([0] + [len(x) for x in r])
    eu, ev = oracle.detect_edges_csr(6, 5, wptr, sum(w, []), rptr, sum(r, []))
    assert [list(p) for p in zip(eu.tolist(), ev.tolist())] == golden["vector_example"]["edges"]
    assert oracle.critical_path(6, eu, ev) == golden["vector_example"]["depth"]


def test_large_grid_depths(golden, oracle):
    for rec in golden["depths"]:
        ext = rec["extents"]
        if np.prod(ext) > 5000:
            continue  # the 32^3 values are checked on the device
        if rec["strategy"] == "loopex":
            h, nb, _ = oracle.stream_loopex(ext, True)
        else:
            h, nb, _ = oracle.stream_basic(ext, True, oracle.canonical_stencil(3))
        eu, ev = oracle.detect_edges_stream(h, nb)
        assert len(h) == rec["tasks"] and len(eu) == rec["edges"]
        assert oracle.critical_path(len(h), eu, ev) == rec["depth"]
