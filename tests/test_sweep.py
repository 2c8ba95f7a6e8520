"""Sweep harness (sweep.py) against the reference's file schema and cell
rules (pkg/src/proxtomo/bench.py:22-262): pure host logic here, one tiny
GPU sweep at the end."""

import csv
import math
import os

import numpy as np
import pytest

from paper_2602_09527_b200 import sweep as S
from paper_2602_09527_b200.metrics import StoppingRule
from paper_2602_09527_b200.solvers import RunRecord


def test_labels_and_names():
    assert S.algorithm_label("fista", 0.5) == "fista"
    assert S.algorithm_label("ista", 1.0) == "ista"
    assert S.algorithm_label("ista", 0.2) == "proxskip"
    assert S.algorithm_label("saga", 1.0) == "proxsaga"
    assert S.algorithm_label("svrg", 0.1) == "proxsvrg-skip"
    assert S.cell_name("svrg", 10, 0.1, 20, 3) == "proxsvrg-skip_N10_p0.1_inner20_seed3"


def test_grid_cells():
    g = S.SweepGrid(("fista", "ista", "saga"), n_subsets=(5, 10), probabilities=(1.0, 0.2),
                    inner_iterations=(10,), seeds=(0, 1))
    cells = g.cells()
    # fista: once per (inner, seed); ista: per p; saga: per (N, p)
    assert cells[:2] == [("fista", 1, 1.0, 10, 0), ("fista", 1, 1.0, 10, 1)]
    assert ("ista", 1, 0.2, 10, 0) in cells
    assert sum(c[0] == "saga" for c in cells) == 2 * 2 * 2
    assert len(cells) == 2 + 4 + 8
    with pytest.raises(ValueError):
        S.SweepGrid(("pdhg",))
    with pytest.raises(ValueError):
        S.SweepGrid(("saga",), seeds=())


def test_stopping_rule_validation():
    StoppingRule(tolerance=1e-3, max_data_passes=10)
    with pytest.raises(ValueError):
        StoppingRule(tolerance=1e-3)
    with pytest.raises(ValueError):
        StoppingRule(max_data_passes=math.inf, time_budget=None)
    with pytest.raises(ValueError):
        StoppingRule(max_data_passes=0)


def _record(rows):
    r = RunRecord()
    for k, (passes, wall, rel, prox) in enumerate(rows):
        r.rows.append((passes, wall, rel, None, None, prox, None))
        r.iterations.append(10 * k)
    return r


def test_summary_and_speedups(tmp_path):
    fast = _record([(1.0, 0.0, 0.5, 0), (2.0, 1.0, 0.05, 3), (3.0, 2.0, 0.01, 5)])
    slow = _record([(1.0, 0.0, 0.5, 0), (2.0, 2.0, 0.2, 10), (3.0, 4.0, 0.04, 20)])
    never = _record([(1.0, 0.0, 0.5, 0), (2.0, 1.0, 0.3, 1)])
    rows = [S.summarise(("svrg", 10, 1.0, 10, 0), slow, False, 0.1),
            S.summarise(("svrg", 10, 0.2, 10, 0), fast, False, 0.1),
            S.summarise(("svrg", 10, 0.1, 10, 0), never, True, 0.1)]
    assert rows[0]["reached"] and rows[0]["time_to_tol"] == 4.0
    assert rows[0]["iterations_to_tol"] == 20 and rows[0]["passes_to_tol"] == 3.0
    assert rows[1]["time_to_tol"] == 1.0 and rows[1]["prox_calls"] == 5
    assert not rows[2]["reached"] and rows[2]["time_to_tol"] is None and rows[2]["diverged"]
    sp = S.compute_speedups(rows)
    assert [p["probability"] for p in sp] == [0.2, 0.1]
    assert sp[0]["speedup"] == 4.0 and sp[1]["speedup"] is None
    S.write_summary_csv(tmp_path / "summary.csv", rows)
    S.write_speedups_csv(tmp_path / "speedups.csv", sp)
    with open(tmp_path / "summary.csv") as fh:
        lines = list(csv.reader(fh))
    assert tuple(lines[0]) == S.SUMMARY_COLUMNS
    assert lines[1][:7] == ["proxsvrg", "svrg", "10", "1.0", "10", "0", "1"]
    assert lines[3][7] == "--" and lines[3][-1] == "1"
    with open(tmp_path / "speedups.csv") as fh:
        lines = list(csv.reader(fh))
    assert tuple(lines[0]) == S.SPEEDUP_COLUMNS
    assert lines[1][-1] == "4.0" and lines[2][-1] == "--"


def test_export_curve(tmp_path):
    r = _record([(1.0, 0.0, 0.5, 0), (2.0, 1.0, float("nan"), 3), (3.0, 2.0, 0.01, 5)])
    S.export_curve(r, tmp_path / "c.txt")
    text = (tmp_path / "c.txt").read_text().splitlines()
    assert text == ["# wall_seconds rel_err", "0.0 0.5", "2.0 0.01"]


@pytest.mark.gpu
def test_gpu_sweep_writes_reference_schema(tmp_path):
    from paper_2602_09527_b200 import (ParallelGeometry, Projector, TomoProblem, TvProxConfig,
                                       problems)
    g = ParallelGeometry.uniform(20, 31)
    proj = Projector(g, 24, 24)
    x_true = problems.ellipse_phantom(24, 4, 0)
    b = proj.forward(x_true).double().cpu().numpy()
    problem = TomoProblem(proj, b, tv=TvProxConfig(alpha=1e-3, inner_iterations=5))
    grid = S.SweepGrid(("fista", "svrg", "saga"), n_subsets=(4,), probabilities=(1.0, 0.5))
    rows = S.run_sweep(grid, problem, x_true, tmp_path, StoppingRule(tolerance=0.5,
                                                                      max_data_passes=6))
    assert len(rows) == 1 + 2 + 2
    names = sorted(os.listdir(tmp_path))
    assert "summary.csv" in names and "speedups.csv" in names
    assert "proxsvrg-skip_N4_p0.5_inner10_seed0.csv" in names
    for row in rows:
        assert row["reached"], row
        assert 0 < row["final_rel_err"] < 0.5
    with open(tmp_path / "proxsaga_N4_p1_inner10_seed0.csv") as fh:
        head = fh.readline().strip().split(",")
    from paper_2602_09527_b200.solvers import RUN_COLUMNS
    assert tuple(head) == tuple(RUN_COLUMNS)
