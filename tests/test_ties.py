"""Near-threshold tie logging (BASELINE north_star: meshes may differ from the CPU run
only where a detail lies within 1e-12 relative of its threshold, and every such case
is logged; thresholds inclusive).

Crafted datum: config 3 (D2Q4, periodic) at J_bar = 5 on the full finest mesh, all
populations 0 except population 0 of one finest cell, which is delta.  The projected
parent is delta/4 and its stencil neighbours are 0, so the prediction of the cell is
delta/4 and its detail 3 delta / 4 (siblings -delta/4): the group metric is exactly
3 delta / 4.  With delta = 4 and epsilon = 3 the metric equals eps_J exactly, and one
level up the projected value delta/4 gives metric 3/4 = eps_{J-1} = 2^-2 * 3, and so
on: one exact tie per level l = J_min+1 .. J_bar, all in step 1.
"""
import numpy as np
import pytest

from paper_2103_02903_b200 import build_config, finest_cells

CELL = (13, 9)


def crafted(delta, eps=3.0, J=5):
    sc, rc = build_config(3, J, eps)
    idx = finest_cells(sc, rc)
    f = np.zeros((sc.q, idx.shape[0]))
    ny = int(rc.base_cells[1]) << (J - rc.j_min)
    f[0, CELL[0] * ny + CELL[1]] = delta
    return sc, rc, idx, f


def expected_ties(rc, delta=4.0, eps=3.0):
    out = []
    for l in range(rc.j_min + 1, rc.j_max + 1):
        sh = rc.j_max - l + 1
        thr = np.ldexp(eps, 2 * (l - rc.j_max))
        out.append((1, l, CELL[0] >> sh, CELL[1] >> sh, 0, 0, thr, thr))
    return out


def run_oracle(sc, rc, idx, f, steps=1):
    from oracle import pyoracle
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, idx, f)
    o.commit()
    o.step(steps)
    return o


def test_oracle_exact_ties_logged_and_kept():
    sc, rc, idx, f = crafted(4.0)
    o = run_oracle(sc, rc, idx, f)
    ties = o.tie_log()
    assert ties == expected_ties(rc)
    # inclusive threshold: the finest group holding the cell is kept (its 4 siblings are leaves)
    li, _ = o.read_leaves(rc.j_max)
    sib = {(2 * (CELL[0] // 2) + a, 2 * (CELL[1] // 2) + b) for a in (0, 1) for b in (0, 1)}
    assert sib <= {tuple(r) for r in li}
    assert o.tie_log(reset=True) and o.tie_log() == []
    o.close()


@pytest.mark.parametrize("rel,logged", [(5e-13, True), (-5e-13, True), (1e-11, False), (-1e-11, False)])
def test_oracle_tie_window(rel, logged):
    """A metric within 1e-12 relative of eps_J is logged, one further away is not."""
    delta = 4.0 * (1.0 + rel)
    sc, rc, idx, f = crafted(delta)
    o = run_oracle(sc, rc, idx, f)
    fin = [t for t in o.tie_log() if t[1] == rc.j_max]
    assert bool(fin) == logged
    if logged:
        assert fin[0][6] == 0.75 * delta and fin[0][7] == 3.0
    o.close()


@pytest.mark.gpu
@pytest.mark.parametrize("delta", [4.0, 4.0 * (1 + 5e-13), 4.0 * (1 - 5e-13), 4.0 * (1 + 1e-11)])
def test_gpu_tie_log_matches_oracle(delta):
    from paper_2103_02903_b200 import Solver
    from parity_util import compare
    sc, rc, idx, f = crafted(delta)
    g = Solver(sc, rc)
    g.load_leaves(rc.j_max, idx, f)
    g.commit()
    o = run_oracle(sc, rc, idx, f, steps=0)
    for _ in range(3):
        g.step(1)
        o.step(1)
        compare(g, o, rc, "crafted tie")
    assert g.tie_log() == o.tie_log()
    if delta == 4.0:
        assert g.tie_log()[: rc.j_max - rc.j_min] == expected_ties(rc)
    g.tie_log(reset=True)
    assert g.tie_log() == []
    g.close()
    o.close()


@pytest.mark.gpu
@pytest.mark.parametrize("cid,J,steps", [(1, 8, 64), (4, 6, 20), (5, 7, 40)])
def test_gpu_tie_log_matches_oracle_configs(cid, J, steps):
    """On the BASELINE data the logs agree too (typically both empty)."""
    from parity_util import make_pair, compare
    sc, rc, g, o = make_pair(cid, J)
    for _ in range(steps // 8):
        g.step(8)
        o.step(8)
        compare(g, o, rc, f"config {cid}")
    assert g.tie_log() == o.tie_log()
    g.close()
    o.close()
