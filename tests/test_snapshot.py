"""snapshot CSV and metrics I/O."""
import os

import numpy as np
import pytest

from paper_2103_02903_b200 import build_config, finest_cells, initial_finest
from paper_2103_02903_b200.abi import StepStats
from paper_2103_02903_b200.snapshot import (MetricsWriter, conserved_rows, moments, occupation_rates,
                                            read_snapshot, write_snapshot)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cells_c1_J6_s5.csv")


def _oracle(cid, J, steps):
    from oracle import pyoracle
    sc, rc = build_config(cid, J)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(cid, sc, rc))
    o.commit()
    o.step(steps)
    o.scheme, o.cfg = sc, rc  # the writer's solver interface
    return sc, rc, o


def test_conserved_rows():
    for cid, rows in [(1, [0]), (2, [0, 3, 6]), (3, [0]), (4, [0, 4, 8, 12]), (5, [0, 1, 2])]:
        sc, _ = build_config(cid, 0)
        assert conserved_rows(sc) == rows, cid


def test_snapshot_golden_byte_identical(tmp_path):
    _, _, o = _oracle(1, 6, 5)
    p = write_snapshot(o, 5, str(tmp_path))
    assert os.path.basename(p) == "cells_5.csv"
    assert open(p, "rb").read() == open(GOLDEN, "rb").read()


@pytest.mark.parametrize("cid,J,steps", [(1, 7, 20), (5, 5, 6)])
def test_snapshot_round_trip(tmp_path, cid, J, steps):
    sc, rc, o = _oracle(cid, J, steps)
    p = write_snapshot(o, steps, str(tmp_path))
    back, hdr = read_snapshot(p)
    assert hdr[0] == "level" and hdr[-len(conserved_rows(sc)):] == [f"m{h}" for h in conserved_rows(sc)]
    for lv in range(rc.j_min, rc.j_max + 1):
        idx, f = o.read_leaves(lv)
        if idx.shape[0] == 0:
            assert lv not in back
            continue
        bi, bm = back[lv]
        assert np.array_equal(bi, idx)
        assert np.array_equal(bm, moments(sc, f, conserved_rows(sc)))  # 17 digits: exact reload


def test_snapshot_full_mesh_row_count(tmp_path):
    sc, rc, o = _oracle(1, 6, 0)
    p = write_snapshot(o, 0, str(tmp_path))
    with open(p) as fh:
        assert sum(1 for _ in fh) - 1 == o.n_finest


def test_metrics_writer_and_rates(tmp_path):
    sc, rc = build_config(5, 5)
    st = StepStats()
    st.levels = rc.j_max - rc.j_min + 1
    nx, ny = rc.base_cells[0] << (rc.j_max - rc.j_min), rc.base_cells[1] << (rc.j_max - rc.j_min)
    st.leaves[st.levels - 1] = nx * ny  # full finest mesh
    full_tree = sum((rc.base_cells[0] << k) * (rc.base_cells[1] << k) for k in range(st.levels))
    st.internal[0] = full_tree - nx * ny
    assert occupation_rates(rc, 2, st) == (1.0, 1.0)
    w = MetricsWriter(str(tmp_path), rc, 2)
    w.append(1, st)
    st.leaves[st.levels - 1] = nx * ny // 4
    w.append(2, st, E=1.5e-3)
    w.close()
    lines = open(os.path.join(str(tmp_path), "metrics.csv")).read().splitlines()
    assert lines[0] == ",".join(MetricsWriter.COLUMNS)
    assert lines[1].split(",")[3] == "1" and lines[2].split(",")[3] == "0.25"
    assert lines[2].split(",")[-1] == format(1.5e-3, ".17g")
    # append-only: a second writer adds lines without a new header
    w2 = MetricsWriter(str(tmp_path), rc, 2)
    w2.append(3, st)
    w2.close()
    assert len(open(os.path.join(str(tmp_path), "metrics.csv")).read().splitlines()) == 4


@pytest.mark.gpu
def test_gpu_snapshot_matches_golden(tmp_path):
    from paper_2103_02903_b200 import Solver
    sc, rc = build_config(1, 6)
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(1, sc, rc))
    s.commit()
    s.step(5)
    p = write_snapshot(s, 5, str(tmp_path))
    assert open(p, "rb").read() == open(GOLDEN, "rb").read()
