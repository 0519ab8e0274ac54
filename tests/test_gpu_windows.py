"""Parity where the bench measures (-m gpu): config 5 at its BASELINE size (levels
2..12, 8192 x 4096 finest) in snapshot-restart windows, and configs 2 and 4 at their
BASELINE J_bar up to their common blow-up step.

Restart windows ("dump the GPU state at step n, load it into the
oracle, run k steps on both, compare"): the GPU runs from the seeded initial datum to
step n; every level is read back through the C-ABI (mrlbm_read_leaves, CellIndex
order) and loaded into the oracle (and into a second GPU context); then all three
step k times and are compared bit for bit after every step.  n covers the driver's
bench window (steps 5..24 after W = 5), the settled mesh (step 200) and the developing
flow (step 3000), which is most of the 50 000-step BASELINE run.
"""
import numpy as np
import pytest

from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
from parity_util import make_pair, compare

pytestmark = pytest.mark.gpu


def snapshot(s, rc):
    return {lv: s.read_leaves(lv) for lv in range(rc.j_min, rc.j_max + 1)}


def load(obj, snap):
    for lv, (idx, f) in snap.items():
        if idx.shape[0]:
            obj.load_leaves(lv, idx, f)
    obj.commit()


def compare_gpu(a, b, rc, tag):
    for lv in range(rc.j_min, rc.j_max + 1):
        ai, af = a.read_leaves(lv)
        bi, bf = b.read_leaves(lv)
        assert np.array_equal(ai, bi), f"{tag}: leaf set differs at level {lv}"
        assert np.array_equal(af.view(np.uint64), bf.view(np.uint64)), f"{tag}: fields differ at level {lv}"


@pytest.mark.parametrize("restart,steps", [(5, 3), (24, 3), (200, 5), (3000, 5)])
def test_restart_window_config5_full_size(restart, steps):
    from oracle import pyoracle
    sc, rc = build_config(5)
    assert rc.j_max == 12
    g = Solver(sc, rc)
    g.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc))
    g.commit()
    g.step(restart)
    snap = snapshot(g, rc)
    o = pyoracle.Oracle(sc, rc)
    load(o, snap)
    g2 = Solver(sc, rc)
    load(g2, snap)
    del snap
    for k in range(steps):
        g.step(1)
        o.step(1)
        g2.step(1)
        rel, bitwise, total = compare(g, o, rc, f"config 5 J=12 restart {restart} step +{k + 1}")
        assert rel <= 1e-12 and bitwise, f"restart {restart} step +{k + 1}: rel {rel}"
        compare_gpu(g, g2, rc, f"GPU restart {restart} step +{k + 1}")
    assert g.tie_log() == o.tie_log()
    print(f"config 5 J=12 restart at step {restart}: {steps} steps bit-exact, {total} leaves")
    g.close()
    g2.close()
    o.close()


@pytest.mark.parametrize("cid,J", [(2, 14), (4, 11)])
def test_baseline_size_until_common_blowup(cid, J):
    """Configs 2 and 4 at their BASELINE J_bar, compared after every step until both
    sides report the non-finite state (status 3) at the same step (the
    configurations are unstable as specified)."""
    sc, rc, g, o = make_pair(cid, J)
    assert rc.j_max == J
    for k in range(400):
        eg = eo = None
        try:
            g.step(1)
        except FloatingPointError as e:
            eg = e
        try:
            o.step(1)
        except FloatingPointError as e:
            eo = e
        assert (eg is None) == (eo is None), f"config {cid} J={J}: blow-up at different steps ({k + 1})"
        if eg is not None:
            print(f"config {cid} J={J}: both sides report status 3 at step {k + 1}")
            break
        rel, bitwise, total = compare(g, o, rc, f"config {cid} J={J} step {k + 1}")
        assert rel <= 1e-12 and bitwise
    else:
        pytest.fail("no blow-up within 400 steps")
    g.close()
    o.close()
