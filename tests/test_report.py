"""The 15-column CSV schema (report.py:16-115 of the reference) and device rows."""

from __future__ import annotations

import csv

import pytest

from paper_1401_4441_b200 import report
from paper_1401_4441_b200.grid import GridSpec
from paper_1401_4441_b200.taskgen import StencilOrder, naive_order, opt_order


def test_columns_and_rows(tmp_path):
    assert report.CSV_COLUMNS == ("kind", "strategy", "dim", "ex", "ey", "ez", "order", "delta",
                                  "workers", "tasks", "makespan", "speedup", "utilization",
                                  "duration_ns", "seed")
    row = report.make_row("simulated", "basic", grid=GridSpec((4, 4)), order="canonical", delta=2,
                          workers=4, tasks=100, makespan=30, speedup=10 / 3, utilization=0.5)
    assert row == ["simulated", "basic", "2", "4", "4", "1", "canonical", "2", "4", "100", "30",
                   "3.333333", "0.500000", "", ""]
    row3 = report.make_row("executed", "loopex", grid=GridSpec((4, 6, 8)), duration_ns=12, seed=7)
    assert row3[:6] == ["executed", "loopex", "3", "4", "6", "8"] and row3[-2:] == ["12", "7"]
    p = report.write_csv(tmp_path / "sub" / "rows.csv", [row, row3])
    with open(p) as f:
        got = list(csv.reader(f))
    assert got[0] == list(report.CSV_COLUMNS) and got[1] == row and got[2] == row3
    acc = report.write_accumulators(tmp_path / "acc.csv", {3: -5, 1: 2})
    assert acc.read_text().splitlines() == ["cell,accumulator", "1,2", "3,-5"]


def test_order_labels():
    assert report.order_label(None) == ""
    assert report.order_label(StencilOrder.canonical(3)) == "canonical"
    assert report.order_label(naive_order()) == "naive"
    assert report.order_label(opt_order()) == "opt"
    o = StencilOrder(((0, 0), (0, 1), (1, -1), (1, 0), (1, 1)))
    assert report.encode_order(o) == "0:0;0:1;1:-1;1:0;1:1"


@pytest.mark.gpu
def test_device_depth_rows(cuda):
    g = GridSpec((4, 4, 4))
    basic = report.device_depth_row("basic", g)
    loopex = report.device_depth_row("loopex", g)
    cols = report.CSV_COLUMNS
    assert basic[cols.index("makespan")] == "692" and loopex[cols.index("makespan")] == "27"
    assert basic[cols.index("tasks")] == loopex[cols.index("tasks")] == str(14 * 64)
    assert basic[cols.index("kind")] == "device" and int(loopex[cols.index("duration_ns")]) > 0


def test_simulated_row_and_row_records(tmp_path):
    class Res:  # the SimResult fields simulated_row reads
        workers, serial_time, makespan = 8, 42000, 5261
        speedup = 42000 / 5261
        utilization = 42000 / (8 * 5261)

    g = GridSpec((30, 10, 10))
    row = report.simulated_row(Res(), "basic", g, order=StencilOrder.canonical(3), delta=10)
    cols = report.CSV_COLUMNS
    assert row[cols.index("kind")] == "simulated" and row[cols.index("order")] == "canonical"
    assert row[cols.index("makespan")] == "5261" and row[cols.index("speedup")] == "7.983273"
    assert row[cols.index("utilization")] == "0.997909" and row[cols.index("ez")] == "10"
    rec = report.Row("device", "loopex", 3, 4, 4, 4, tasks=896, makespan=27)
    p = report.write_csv(tmp_path / "r.csv", [rec, row])
    lines = p.read_text().splitlines()
    assert lines[1] == "device,loopex,3,4,4,4,,,,896,27,,,," and len(lines) == 3
