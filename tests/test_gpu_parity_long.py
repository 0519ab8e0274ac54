"""Longer / larger GPU-vs-oracle parity runs and full-size invariants (-m gpu).

Sizes are chosen so the oracle finishes in seconds to a minute; full-size
config 5 (8192 x 4096) is checked through size-independent properties.
"""
import numpy as np
import pytest

from parity_util import make_pair, compare

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid,J,eps,steps,every", [
    (1, 10, -1.0, 2048, 64),   # config 1 at its full BASELINE size, the whole run to T = 2
    (3, 9, -1.0, 24, 4),       # config 3 at full size (512 x 512) up to its CFL blow-up window
    (3, 9, 0.0, 24, 4),        # the BASELINE uniform-mesh run (epsilon = 0) at level 9
    (4, 8, -1.0, 40, 5),       # config 4 at J_bar = 8 (256^2) before its blow-up (~47 steps)
    (5, 8, -1.0, 120, 20),     # config 5 at J_bar = 8 (512 x 256)
])
def test_parity_long(cid, J, eps, steps, every):
    sc, rc, gpu, ora = make_pair(cid, J, eps)
    done, worst = 0, 0.0
    while done < steps:
        n = min(every, steps - done)
        gpu.step(n)
        ora.step(n)
        done += n
        rel, bitwise, total = compare(gpu, ora, rc, f"config {cid} J={J} step {done}")
        assert rel <= 1e-12
        worst = max(worst, rel)
    print(f"config {cid} J={J} eps={eps}: {steps} steps, worst rel {worst:.3e}")
    gpu.close()
    ora.close()


def test_full_size_config5_invariants():
    """Config 5 at BASELINE size (levels 2..12, 8192 x 4096): leaves tile the domain
    exactly, fields stay finite, and the mesh adapts."""
    from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
    sc, rc = build_config(5)
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc))
    s.commit()
    area = 8 * 4 * 2.0 ** (-2 * rc.j_min)  # domain area in cell units of level j_min... = 2 x 1
    for k in range(6):
        st = s.step(5)
        cover = sum(st.leaves[i] * 2.0 ** (-2 * (rc.j_min + i)) for i in range(st.levels))
        assert cover == pytest.approx(2.0, abs=0) and cover == 2.0
    assert sum(st.leaves[i] for i in range(st.levels)) < 8192 * 4096
    idx, f = s.read_leaves(rc.j_max)
    assert np.isfinite(f).all()
    s.close()
    assert area == 2.0


def test_parity_full_size_config5():
    """The bench configuration itself (config 5, levels 2..12, 8192 x 4096 finest,
    33.5 M initial leaves): two adaptive steps, GPU vs oracle, bit-exact on every level."""
    sc, rc, gpu, ora = make_pair(5, 12)
    for k in range(2):
        gpu.step(1)
        ora.step(1)
        rel, bitwise, total = compare(gpu, ora, rc, f"config 5 J=12 step {k}")
        assert rel <= 1e-12 and bitwise
    print(f"config 5 J=12: 2 steps bit-exact, {total} leaves")
    gpu.close()
    ora.close()


@pytest.mark.gpu
def test_uniform_mode_config3_baseline_size_vs_numpy():
    """BASELINE config 3 "plus a uniform-mesh run (epsilon=0) at level 9": the GPU step in
    uniform mode on the full 512 x 512 mesh against the independent numpy uniform LBM
    (tests/uniform_ref.py), per step <= 1e-12 (north_star: "The same check runs in uniform-mesh
    mode (epsilon=0)").  Both start each step from the same state, so the growth
    of the (a, b) = (1, 1) instability does not enter."""
    import numpy as np
    from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
    from uniform_ref import UniformLBM
    sc, rc = build_config(3, 9, 0.0)
    f0 = initial_finest(3, sc, rc)
    g = Solver(sc, rc)
    g.load_leaves(rc.j_max, finest_cells(sc, rc), f0)
    g.commit()
    ref = UniformLBM(sc, rc, f0)
    worst = 0.0
    for k in range(24):
        ref.f = g.read_leaves(rc.j_max)[1].reshape(ref.f.shape).copy()
        g.step(1)
        ref.step()
        for lv in range(rc.j_min, rc.j_max):
            assert g.level_count(lv) == 0, "epsilon = 0 must keep the full finest mesh"
        _, f = g.read_leaves(rc.j_max)
        scale = max(1.0, float(np.abs(ref.soa()).max()))
        err = float(np.abs(f - ref.soa()).max()) / scale
        assert err <= 1e-12, f"step {k}: {err}"
        worst = max(worst, err)
    g.close()
    print(f"config 3 uniform mode at J=9: worst per-step difference {worst:.2e}")
