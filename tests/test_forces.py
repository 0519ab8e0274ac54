"""Config-5 integral diagnostics: obstacle force, C_D / C_L,
Strouhal number.

CPU tests: the C-ABI drag/lift and Strouhal host functions against a numpy
restatement and SPEC's known answers (pure sinusoid -> St within one bin,
constant series -> no dominant peak, affine invariance), and the oracle's force
accumulation (rest state -> zero force, symmetric unperturbed flow -> zero lift).
GPU tests: the device force history equals the oracle's step by step.
"""
import numpy as np
import pytest

from paper_2103_02903_b200 import build_config, drag_lift, strouhal


def np_strouhal(cl, dt, u0, L, skip=0):
    """numpy restatement of mrlbm_strouhal: detrend, Hann window, DFT, argmax bin >= 1."""
    y = np.asarray(cl, dtype=np.float64)[skip:]
    n = y.size
    t = np.arange(n, dtype=np.float64)
    b, a = np.polyfit(t, y, 1)
    r = y - (a + b * t)
    w = r * (0.5 - 0.5 * np.cos(2 * np.pi * t / (n - 1)))
    p = np.abs(np.fft.rfft(w)) ** 2
    k = 1 + int(np.argmax(p[1: n // 2 + 1]))
    return L * (k / (n * dt)) / u0, 1.0 / (n * dt)


def test_drag_lift_formula():
    cd, cl = drag_lift(3.0, -1.5, 1.0, 0.05, 0.125)
    assert cd == pytest.approx(2 * 3.0 / (0.05 ** 2 * 0.125), rel=1e-15)
    assert cl == pytest.approx(2 * -1.5 / (0.05 ** 2 * 0.125), rel=1e-15)
    assert drag_lift(0.0, 0.0, 1.0, 0.05, 0.125) == (0.0, 0.0)
    with pytest.raises(ValueError):
        drag_lift(1.0, 1.0, 1.0, 0.0, 0.125)


@pytest.mark.parametrize("f", [0.7, 1.3, 2.25])
def test_strouhal_sinusoid(f):
    dt, u0, L = 0.01, 0.05, 0.125
    t = np.arange(4000) * dt
    cl = np.sin(2 * np.pi * f * t) + 0.3 + 0.01 * t   # offset and drift are detrended away
    st, df = strouhal(cl, dt, u0, L, skip=200)
    assert abs(st - L * f / u0) <= L * df / u0 + 1e-12   # within one frequency bin
    st_np, df_np = np_strouhal(cl, dt, u0, L, skip=200)
    assert st == pytest.approx(st_np, rel=1e-12) and df == pytest.approx(df_np, rel=1e-15)


def test_strouhal_flat_raises():
    with pytest.raises(FloatingPointError):
        strouhal(np.full(512, 0.42), 0.01, 0.05, 0.125)
    with pytest.raises(FloatingPointError):
        strouhal(0.5 + 0.002 * np.arange(512), 0.01, 0.05, 0.125)   # a pure trend is flat too
    with pytest.raises(ValueError):
        strouhal(np.zeros(4), 0.01, 0.05, 0.125)


def test_strouhal_affine_invariance():
    rng = np.random.default_rng(7)
    t = np.arange(3000) * 0.02
    cl = np.sin(2 * np.pi * 0.9 * t) + 0.05 * rng.standard_normal(t.size)
    st0, _ = strouhal(cl, 0.02, 0.05, 0.125)
    st1, _ = strouhal(-7.5 * cl + 3.0, 0.02, 0.05, 0.125)
    assert st0 == st1


def _oracle(cid, J, f0=None):
    from oracle import pyoracle
    from paper_2103_02903_b200 import finest_cells, initial_finest
    sc, rc = build_config(cid, J)
    idx = finest_cells(sc, rc)
    if f0 is None:
        f0 = initial_finest(cid, sc, rc)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, idx, f0)
    o.commit()
    return sc, rc, o


def _rest_state(sc, rc):
    from paper_2103_02903_b200 import finest_cells
    n = finest_cells(sc, rc).shape[0]
    feq = np.array([rc.obstacle_feq[h] for h in range(sc.q)])
    return np.repeat(feq[:, None], n, axis=1)


def test_oracle_force_rest_state_is_zero():
    """Fluid at rest, far from the moving walls for one step -> no momentum at the disc."""
    sc, rc = build_config(5, 6)
    sc, rc, o = _oracle(5, 6, _rest_state(sc, rc))
    o.set_force_tracking(True)
    o.step(1)
    fx, fy = o.force_history()
    assert fx.shape == (1,) and fx[0] == 0.0 and fy[0] == 0.0
    o.close()


def test_oracle_force_symmetric_flow_has_no_lift():
    """Unperturbed inflow past the disc is mirror-symmetric about y = 0.5 -> C_L ~ 0
    (SPEC.md:473), while the drag is positive once the inflow reaches the disc."""
    sc, rc = build_config(5, 6)
    sc, rc, o = _oracle(5, 6, _rest_state(sc, rc))
    o.set_force_tracking(True)
    o.step(60)
    fx, fy = o.force_history()
    assert fx.shape == (60,)
    assert fx[-1] > 0.0
    assert np.max(np.abs(fy)) <= 1e-9 * np.max(np.abs(fx))
    o.close()


def test_oracle_force_tracking_needs_obstacle():
    sc, rc, o = _oracle(1, 6)
    with pytest.raises(ValueError):
        o.set_force_tracking(True)
    o.close()


@pytest.mark.gpu
def test_gpu_force_history_matches_oracle():
    """Device force per step vs the oracle (different but fixed summation orders:
    within 1e-12 of the magnitude of the force terms)."""
    from parity_util import make_pair, compare
    sc, rc, gpu, ora = make_pair(5, 7)
    gpu.set_force_tracking(64)
    ora.set_force_tracking(True)
    for k in range(25):
        gpu.step(1)
        ora.step(1)
    rel, _, _ = compare(gpu, ora, rc, "config 5 J=7")
    assert rel <= 1e-12
    gx, gy = gpu.force_history()
    ox, oy = ora.force_history()
    assert gx.shape == ox.shape == (25,)
    scale = max(np.max(np.abs(ox)), np.max(np.abs(oy)))
    assert scale > 0.0
    assert np.max(np.abs(gx - ox)) <= 1e-12 * scale
    assert np.max(np.abs(gy - oy)) <= 1e-12 * scale
    cd, cl = drag_lift(gx[-1], gy[-1], 1.0, 0.05, 2 * rc.obstacle_radius)
    assert np.isfinite(cd) and np.isfinite(cl)
    gpu.close()
    ora.close()


@pytest.mark.gpu
def test_gpu_force_tracking_off_and_errors():
    from paper_2103_02903_b200 import Solver, finest_cells, initial_finest
    sc, rc = build_config(1, 6)
    s = Solver(sc, rc)
    with pytest.raises(ValueError):
        s.set_force_tracking(8)
    s.close()
    sc, rc = build_config(5, 6)
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc))
    s.commit()
    s.set_force_tracking(2)
    s.step(3)
    with pytest.raises(Exception):
        s.force_history()          # 3 steps > capacity 2 -> status 5
    s.set_force_tracking(0)
    with pytest.raises(Exception):
        s.force_history()          # tracking off -> status 6
    s.step(1)
    s.close()
