"""The 3D path: D3Q6 advection of a sphere indicator (PAPER.md:1462-1518,
SPEC.md:408-416).  CPU: the 3D flattened tables (product push builder vs the oracle's pull
recursion over the reference predict<3>), the 3D prediction known answers, the oracle's
step properties.  GPU: step-by-step parity of the CUDA 3D engine against the oracle
instantiated at D = 3, epsilon = 0 uniform mode, and the paper's compression result
(MeshOR <= 0.05 at J = 8).
"""
import numpy as np
import pytest

from paper_2103_02903_b200 import build_config, config_steps, finest_cells, initial_finest, stream_table

ETAS = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]


def test_tables_3d_product_equals_oracle_bitwise():
    from oracle import pyoracle
    for gap in range(0, 5):
        for eta in ETAS:
            for side in (0, 1):
                po, pw = stream_table(3, gap, eta, side)
                oo, ow = pyoracle.stream_table(3, gap, eta, side)
                assert np.array_equal(po, oo), (gap, eta, side)
                assert np.array_equal(pw.view(np.uint64), ow.view(np.uint64)), (gap, eta, side)
                # a table sums f^^ over the 4^gap rim cells: exact on constants
                assert abs(pw.sum() - 4.0 ** gap) <= 1e-12 * 4.0 ** gap


def test_predict3_one_hot_fan():
    """Weights of the reference predict<3> (prediction.hpp:160-172): centre 1, axis -/+1/8,
    plane terms with the reference's minus sign, corner -/+1/512; the 8 children average
    back to the parent (consistency, Eq. 7)."""
    from oracle import pyoracle
    L = pyoracle.ref_lib()
    import ctypes as C
    W = np.zeros((8, 27))
    for code in range(8):
        delta = (C.c_int * 3)((code >> 2) & 1, (code >> 1) & 1, code & 1)
        for o in range(27):
            st = np.zeros(27)
            st[o] = 1.0
            W[code, o] = L.ref_predict(3, 1, st.ctypes.data_as(C.c_void_p), delta)
    assert np.allclose(W[:, 13], 1.0)
    assert W[0, 13 + 9] == -0.125 and W[0, 13 - 9] == 0.125          # +x / -x for delta_x = 0
    assert W[0, 13 + 9 + 3] == -1.0 / 64 and W[0, 13 + 9 - 3] == 1.0 / 64  # plane term: minus sign
    assert W[0, 26] == -1.0 / 512 and W[0, 0] == 1.0 / 512
    mean = W.mean(axis=0)
    assert np.array_equal(mean, np.eye(27)[13])


def test_oracle_3d_step_properties():
    """Oracle at D = 3 (J = 5): the leaves partition the cube, the mass is conserved to
    round-off while the support is away from the walls, the mesh compresses."""
    from oracle import pyoracle
    sc, rc = pyoracle.build_config(6, 5)
    assert sc.d == 3 and sc.q == 6 and rc.j_min == 1 and rc.mu == 2
    idx, f0 = pyoracle.finest_cells(sc, rc), pyoracle.initial_finest(6, sc, rc)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, idx, f0)
    o.commit()
    m0 = f0.sum() * 2.0 ** (-3 * rc.j_max)
    for step in range(4):
        o.step(1)
        vol, mass, n = 0.0, 0.0, 0
        for lv in range(rc.j_min, rc.j_max + 1):
            li, lf = o.read_leaves(lv)
            vol += li.shape[0] * 2.0 ** (-3 * lv)
            mass += lf.sum() * 2.0 ** (-3 * lv)
            n += li.shape[0]
        assert vol == 1.0
        assert abs(mass - m0) <= 1e-12 * m0
        assert n < idx.shape[0] // 4
    o.close()


def _uniform_d3q6(sc, rc, f, steps):
    """Independent numpy uniform-grid D3Q6 LBM: stream with the copy
    closure, then m = M f, m' = (1 - s) m + s m^eq, f = M^-1 m'."""
    n = 2 << (rc.j_max - rc.j_min)
    f = f.reshape(6, n, n, n).copy()
    M = np.array(sc.M[:36]).reshape(6, 6)
    Mi = np.array(sc.Minv[:36]).reshape(6, 6)
    sv = np.array(sc.s[:6])[:, None, None, None]
    V = [sc.eq_params[a] for a in range(3)]
    ar = np.arange(n)
    for _ in range(steps):
        new = np.empty_like(f)
        for h in range(6):
            ix = [np.clip(ar - sc.eta[h][a], 0, n - 1) for a in range(3)]
            new[h] = f[h][np.ix_(ix[0], ix[1], ix[2])]
        m = np.einsum("ij,jxyz->ixyz", M, new)
        meq = np.zeros_like(m)
        meq[0] = m[0]
        for a in range(3):
            meq[1 + a] = V[a] * m[0]
        f = np.einsum("ij,jxyz->ixyz", Mi, (1.0 - sv) * m + sv * meq)
    return f.reshape(6, -1)


def test_oracle_3d_uniform_mode_matches_numpy_lbm():
    """epsilon = 0 equivalence (acceptance 3) at D = 3: the adaptive oracle on
    the full finest mesh against an independent uniform D3Q6 solver, <= 1e-12 per step."""
    from oracle import pyoracle
    sc, rc = pyoracle.build_config(6, 4, 0.0)
    idx, f0 = pyoracle.finest_cells(sc, rc), pyoracle.initial_finest(6, sc, rc)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, idx, f0)
    o.commit()
    steps = 8
    o.step(steps)
    assert o.level_count(rc.j_max) == idx.shape[0]
    _, fo = o.read_leaves(rc.j_max)
    fu = _uniform_d3q6(sc, rc, f0, steps)
    scale = np.abs(fu).max()
    assert np.max(np.abs(fo - fu)) <= 1e-12 * steps * scale
    o.close()


def test_snapshot_roundtrip_3d(tmp_path):
    """cells_<step>.csv of a 3D state: three index and three coordinate
    columns, 17 significant digits, exact reload of the conserved moment."""
    from oracle import pyoracle
    from paper_2103_02903_b200.snapshot import read_snapshot, write_snapshot
    sc, rc = pyoracle.build_config(6, 4)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, pyoracle.finest_cells(sc, rc), pyoracle.initial_finest(6, sc, rc))
    o.commit()
    o.step(2)
    o.scheme, o.cfg = sc, rc
    path = write_snapshot(o, 2, str(tmp_path))
    per, hdr = read_snapshot(path)
    assert hdr[:8] == ["level", "k0", "k1", "k2", "x0", "x1", "x2", "edge"] and hdr[8:] == ["m0"]
    for lv in range(rc.j_min, rc.j_max + 1):
        idx, f = o.read_leaves(lv)
        if idx.shape[0] == 0:
            assert lv not in per
            continue
        ridx, rm = per[lv]
        assert np.array_equal(ridx, idx)
        u = np.zeros(idx.shape[0])
        for h in range(6):
            u = u + sc.M[h] * f[h]
        assert np.array_equal(rm[0].view(np.uint64), u.view(np.uint64))
    o.close()


def test_config6_descriptor_values():
    sc, rc = build_config(6)
    assert [tuple(sc.eta[h][:3]) for h in range(6)] == ETAS
    assert list(sc.s[:6]) == [0.0, 1.4, 1.4, 1.4, 1.0, 1.0]
    assert rc.j_min == 1 and rc.j_max == 8 and rc.epsilon == 1e-3 and rc.mu == 2
    assert config_steps(6, rc) == 200  # T = 0.78125 at dt = 2^-8
    M = np.array(sc.M[:36]).reshape(6, 6)
    Mi = np.array(sc.Minv[:36]).reshape(6, 6)
    assert np.allclose(M @ Mi, np.eye(6), atol=1e-15)


# ----------------------------------------------------------------------------- GPU
def _pair(J, eps=-1.0):
    from parity_util import make_pair
    return make_pair(6, J, eps)


@pytest.mark.gpu
@pytest.mark.parametrize("J,eps,steps", [(4, -1.0, 12), (5, -1.0, 16), (4, 0.0, 8), (6, -1.0, 6), (7, -1.0, 4)])
def test_gpu_3d_step_parity(J, eps, steps):
    """CUDA 3D engine vs the oracle at D = 3, after every step: identical leaf sets,
    fields within 1e-12 relative (north_star) -- bit-identical in practice."""
    from parity_util import compare
    sc, rc, gpu, ora = _pair(J, eps)
    allbit = True
    for k in range(steps):
        st = gpu.step(1)
        ora.step(1)
        rel, bitwise, total = compare(gpu, ora, rc, f"config 6 J={J} step {k}")
        assert rel <= 1e-12, f"config 6 J={J} step {k}: rel diff {rel}"
        allbit = allbit and bitwise
        assert st.fallback_leaves == ora.fallback_leaves()
    assert allbit
    assert gpu.tie_log() == ora.tie_log()
    gpu.close()
    ora.close()


@pytest.mark.gpu
def test_gpu_3d_reload_roundtrip():
    """read_leaves -> load_leaves of an adapted 3D mesh into a second context continues
    bit-identically (the snapshot contract either side of the step)."""
    from paper_2103_02903_b200 import Solver
    sc, rc = build_config(6, 5)
    a = Solver(sc, rc)
    a.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(6, sc, rc))
    a.commit()
    a.step(5)
    b = Solver(sc, rc)
    for lv in range(rc.j_min, rc.j_max + 1):
        i, f = a.read_leaves(lv)
        b.load_leaves(lv, i, f)
    b.commit()
    a.step(3)
    b.step(3)
    for lv in range(rc.j_min, rc.j_max + 1):
        ai, af = a.read_leaves(lv)
        bi, bf = b.read_leaves(lv)
        assert np.array_equal(ai, bi) and np.array_equal(af.view(np.uint64), bf.view(np.uint64))
    a.close()
    b.close()


@pytest.mark.gpu
def test_gpu_3d_restart_window_J8():
    """Parity at the paper's size (levels 1..8, 256^3 finest): the GPU state after 60 steps is
    read back through the ABI and loaded into the oracle and into a second GPU context; three
    more steps on each, compared bit for bit on every level after every step (gaps up to 5:
    the long-rim recursive path of the coarse leaves)."""
    from oracle import pyoracle
    from paper_2103_02903_b200 import Solver
    from parity_util import compare
    sc, rc = build_config(6)
    a = Solver(sc, rc)
    idx = finest_cells(sc, rc)
    a.load_leaves(rc.j_max, idx, initial_finest(6, sc, rc))
    del idx
    a.commit()
    a.step(60)
    b = Solver(sc, rc)
    o = pyoracle.Oracle(sc, rc)
    total = 0
    for lv in range(rc.j_min, rc.j_max + 1):
        i, f = a.read_leaves(lv)
        total += i.shape[0]
        if i.shape[0]:
            b.load_leaves(lv, i, f)
            o.load_leaves(lv, i, f)
    b.commit()
    o.commit()
    assert 200_000 < total < 600_000
    for k in range(3):
        sa = a.step(1)
        b.step(1)
        o.step(1)
        rel, bitwise, n = compare(b, o, rc, f"config 6 J=8 window step {60 + k}")
        assert bitwise, rel
        rel2, bitwise2, _ = compare(a, o, rc, f"config 6 J=8 continued run step {60 + k}")
        assert bitwise2, rel2
        assert sa.fallback_leaves == o.fallback_leaves()
    for s_ in (a, b, o):
        s_.close()


@pytest.mark.gpu
def test_gpu_3d_compression_J8():
    """advection3d with J_min = 1, J = 8, mu = 2, eps = 1e-3
    reaches a post-transient MeshOR <= 0.05 (the paper reports ~0.03); mass conserved."""
    from paper_2103_02903_b200 import Solver
    sc, rc = build_config(6)
    s = Solver(sc, rc)
    idx, f0 = finest_cells(sc, rc), initial_finest(6, sc, rc)
    n_fine = idx.shape[0]
    m0 = f0.sum() * 2.0 ** (-3 * rc.j_max)
    s.load_leaves(rc.j_max, idx, f0)
    s.commit()
    del idx, f0
    nsteps = config_steps(6, rc)
    ors = []
    for k in range(0, nsteps, 10):
        st = s.step(10)
        ors.append(sum(int(st.leaves[i]) for i in range(st.levels)) / n_fine)
    assert max(ors[2:]) <= 0.05, ors
    mass = 0.0
    for lv in range(rc.j_min, rc.j_max + 1):
        _, lf = s.read_leaves(lv)
        mass += lf.sum() * 2.0 ** (-3 * lv)
    # round-off per step plus the exponentially small tails that reach the copy (outflow) walls
    assert abs(mass - m0) <= 1e-6 * m0
    print("MeshOR over the run:", [round(v, 4) for v in ors])
    s.close()


# ----------------------------------------------------------------------------- ties in 3D
TIE_CELL = (5, 9, 6)


def _crafted3(delta, eps=7.0, J=4):
    """All populations 0 except population 0 of one finest cell = delta: the projected parent is
    delta / 8, its neighbours 0, so the group metric is exactly 7 delta / 8; with delta = 8 and
    eps = 7 it equals eps_l = 2^{3(l-J)} eps at every level (the 3D form of tests/test_ties.py)."""
    sc, rc = build_config(6, J, eps)
    idx = finest_cells(sc, rc)
    f = np.zeros((sc.q, idx.shape[0]))
    n = 2 << (J - rc.j_min)
    f[0, (TIE_CELL[0] * n + TIE_CELL[1]) * n + TIE_CELL[2]] = delta
    return sc, rc, idx, f


def _expected_ties3(rc, eps=7.0):
    out = []
    # (not l = J_min + 1: the level-1 box is 2^3 cells, so the parent's clamped stencil holds the
    # parent itself and the metric there is not 7/8 of the value)
    for l in range(rc.j_min + 2, rc.j_max + 1):
        sh = rc.j_max - l + 1
        thr = float(np.ldexp(eps, 3 * (l - rc.j_max)))
        out.append((1, l, TIE_CELL[0] >> sh, TIE_CELL[1] >> sh, TIE_CELL[2] >> sh, 0, thr, thr))
    return out


def test_oracle_3d_exact_ties_logged_and_kept():
    from oracle import pyoracle
    sc, rc, idx, f = _crafted3(8.0)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, idx, f)
    o.commit()
    o.step(1)
    assert o.tie_log() == _expected_ties3(rc)
    li, _ = o.read_leaves(rc.j_max)
    sib = {tuple(2 * (TIE_CELL[a] // 2) + b[a] for a in range(3)) for b in np.ndindex(2, 2, 2)}
    assert sib <= {tuple(r) for r in li}  # inclusive threshold: the group is kept
    o.close()


@pytest.mark.gpu
@pytest.mark.parametrize("delta", [8.0, 8.0 * (1 + 5e-13), 8.0 * (1 - 5e-13), 8.0 * (1 + 1e-11)])
def test_gpu_3d_tie_log_matches_oracle(delta):
    from oracle import pyoracle
    from paper_2103_02903_b200 import Solver
    from parity_util import compare
    sc, rc, idx, f = _crafted3(delta)
    g = Solver(sc, rc)
    o = pyoracle.Oracle(sc, rc)
    for s_ in (g, o):
        s_.load_leaves(rc.j_max, idx, f)
        s_.commit()
        s_.step(1)
    assert g.tie_log() == o.tie_log()
    if delta == 8.0:
        assert g.tie_log() == _expected_ties3(rc)
    if delta == 8.0 * (1 + 1e-11):
        assert [t for t in g.tie_log() if t[1] == rc.j_max] == []
    rel, bitwise, _ = compare(g, o, rc, f"3D ties delta={delta}")
    assert bitwise
    g.close()
    o.close()
