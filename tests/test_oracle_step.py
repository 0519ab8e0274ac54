"""CPU tests of the oracle step (the parity checker): equivalence at epsilon=0
with an independent uniform solver, conservation, mesh invariants, golden pins."""
import os

import numpy as np
import pytest

from paper_2103_02903_b200 import build_config, finest_cells, initial_finest
from paper_2103_02903_b200.abi import level_extent
from oracle import pyoracle
from uniform_ref import UniformLBM

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def make_oracle(cid, J, eps=-1.0):
    sc, rc = build_config(cid, J, eps)
    o = pyoracle.Oracle(sc, rc)
    f0 = initial_finest(cid, sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), f0)
    o.commit()
    return sc, rc, o, f0


@pytest.mark.parametrize("cid,J,steps", [(1, 6, 60), (2, 6, 40), (3, 5, 100), (4, 5, 40), (5, 5, 60)])
def test_uniform_equivalence(cid, J, steps):
    """epsilon = 0 on the full finest mesh == uniform reference LBM (<= 1e-12 per step)."""
    sc, rc, o, f0 = make_oracle(cid, J, 0.0)
    ref = UniformLBM(sc, rc, f0)
    for k in range(steps):
        # per-step check: both solvers start the step from the same state, so
        # round-off amplification of unstable data (config 2) is excluded
        ref.f = o.read_leaves(rc.j_max)[1].reshape(ref.f.shape).copy()
        o.step(1)
        ref.step()
        for lv in range(rc.j_min, rc.j_max):
            assert o.level_count(lv) == 0, "epsilon = 0 must keep the full finest mesh"
        idx, f = o.read_leaves(rc.j_max)
        scale = max(1.0, float(np.abs(ref.soa()).max()))
        err = float(np.abs(f - ref.soa()).max()) / scale
        assert err <= 1e-12, f"step {k}: {err}"


def test_config2_blowup_detected():
    """Config 2 violates the lattice CFL bound (|u|+c = 4.03 > lambda = 3):
    the non-finite state must be reported as a numerical error."""
    sc, rc, o, _ = make_oracle(2, 8)
    with pytest.raises(FloatingPointError):
        o.step(80)


def leaves_all(o, sc, rc):
    out = {}
    for lv in range(rc.j_min, rc.j_max + 1):
        out[lv] = o.read_leaves(lv)
    return out


def conserved_mass(o, sc, rc):
    M = np.array(sc.M[: sc.q * sc.q]).reshape(sc.q, sc.q)
    tot = np.zeros(sc.q)
    for lv in range(rc.j_min, rc.j_max + 1):
        idx, f = o.read_leaves(lv)
        if f.shape[1]:
            tot += (M @ f).sum(axis=1) * 2.0 ** (-sc.d * lv)
    return tot


def test_periodic_conservation():
    """Adaptive periodic advection conserves mass to round-off.

    Uses (a, b) = (0.5, 0.5): the BASELINE speed (1, 1) violates the D2Q4 lattice
    CFL bound |a| + |b| <= lambda and grows exponentially (DESIGN.md Findings)."""
    sc, rc = build_config(3, 6)
    sc.eq_params[0] = sc.eq_params[1] = 0.5
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(3, sc, rc))
    o.commit()
    m0 = conserved_mass(o, sc, rc)[0]
    prev = m0
    for k in range(40):
        o.step(1)
        m = conserved_mass(o, sc, rc)[0]
        # per step: E/A rim fluxes of neighbouring leaves are the same
        # reconstruction evaluated by table vs recursion -> equal up to round-off
        assert abs(m - prev) <= 1e-12 * abs(m0), (k, m, prev)
        prev = m
    assert abs(prev - m0) <= 1e-10 * abs(m0)


def test_partition_and_grading():
    """Complete leaves tile the domain exactly once every step; the
    mesh adapts (fewer leaves than the full mesh)."""
    sc, rc, o, _ = make_oracle(4, 6)
    nx, ny = level_extent(rc, sc.d, rc.j_max)
    for k in range(10):
        o.step(1)
        cover = np.zeros((nx, ny), dtype=np.int32)
        for lv in range(rc.j_min, rc.j_max + 1):
            idx, _ = o.read_leaves(lv)
            sh = rc.j_max - lv
            for x, y in idx:
                cover[x << sh:(x + 1) << sh, y << sh:(y + 1) << sh] += 1
        assert (cover == 1).all()
    total = sum(o.level_count(lv) for lv in range(rc.j_min, rc.j_max + 1))
    assert total < nx * ny


def test_constant_field_collapses():
    """Constant datum: the mesh collapses to the coarsest level and the field stays
    constant."""
    sc, rc = build_config(3, 6)
    nx, ny = level_extent(rc, 2, rc.j_max)
    M = np.array(sc.M[:16]).reshape(4, 4)
    Minv = np.array(sc.Minv[:16]).reshape(4, 4)
    u = 0.7
    feq = Minv @ np.array([u, u, u, 0.0])
    f0 = np.repeat(feq[:, None], nx * ny, axis=1)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), f0)
    o.commit()
    o.step(3)
    assert o.level_count(rc.j_min) == 16
    assert sum(o.level_count(lv) for lv in range(rc.j_min + 1, rc.j_max + 1)) == 0
    idx, f = o.read_leaves(rc.j_min)
    rho = (M @ f)[0]
    assert np.allclose(rho, u, rtol=0, atol=1e-14)


def test_epsilon_zero_keeps_mesh():
    sc, rc, o, _ = make_oracle(1, 6, 0.0)
    o.step(5)
    nx, _ = level_extent(rc, 1, rc.j_max)
    assert o.level_count(rc.j_max) == nx


def test_load_rejects_non_partition():
    sc, rc = build_config(3, 5)
    o = pyoracle.Oracle(sc, rc)
    idx = finest_cells(sc, rc)[:-1]
    f = np.zeros((sc.q, idx.shape[0]))
    o.load_leaves(rc.j_max, idx, f)
    with pytest.raises(ValueError):
        o.commit()


@pytest.mark.parametrize("name", sorted(f for f in os.listdir(GOLDEN) if f.startswith("oracle_") and f.endswith(".npz")) if os.path.isdir(GOLDEN) else [])
def test_golden(name):
    """Regression pin: oracle output on committed small cases (tests/golden/make_golden.py)."""
    data = np.load(os.path.join(GOLDEN, name))
    cid, J, eps, steps = (int(data["cid"]), int(data["J"]), float(data["eps"]), int(data["steps"]))
    sc, rc, o, _ = make_oracle(cid, J, eps)
    o.step(steps)
    for lv in range(rc.j_min, rc.j_max + 1):
        idx, f = o.read_leaves(lv)
        assert np.array_equal(idx, data[f"idx{lv}"])
        assert np.array_equal(f.view(np.uint64), data[f"f{lv}"].view(np.uint64))
