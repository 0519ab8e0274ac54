"""GPU parity: the CUDA step vs the CPU oracle, step by step, through the C-ABI.

Integer state (leaf sets per level) must be identical; fields within 1e-12
relative per step (north_star) -- in practice they are bit-identical because
both sides use the reference operation order without FMA.
"""
import numpy as np
import pytest

from parity_util import make_pair, compare

pytestmark = pytest.mark.gpu

CASES = [
    # (config, J_bar, epsilon override, steps)
    (1, 7, -1.0, 40),
    (2, 8, -1.0, 40),
    (3, 6, -1.0, 30),
    (3, 5, 0.0, 20),     # uniform-mesh mode (epsilon = 0)
    (4, 6, -1.0, 20),
    (5, 6, -1.0, 20),
]


@pytest.mark.parametrize("cid,J,eps,steps", CASES)
def test_step_parity(cid, J, eps, steps):
    sc, rc, gpu, ora = make_pair(cid, J, eps)
    worst = 0.0
    for k in range(steps):
        gpu.step(1)
        ora.step(1)
        rel, bitwise, total = compare(gpu, ora, rc, f"config {cid} step {k}")
        assert rel <= 1e-12, f"config {cid} step {k}: rel diff {rel}"
        worst = max(worst, rel)
    gpu.close()
    ora.close()
    print(f"config {cid} J={J} eps={eps}: {steps} steps, worst rel {worst:.3e}")


def test_config2_blowup_same_step():
    """Both sides report the non-finite state (status 3) at the same step."""
    sc, rc, gpu, ora = make_pair(2, 8)
    def first_fail(s):
        for k in range(120):
            try:
                s.step(1)
            except FloatingPointError:
                return k
        return None
    kg, ko = first_fail(gpu), first_fail(ora)
    assert kg is not None and kg == ko


def test_gpu_matches_golden_fixtures():
    """GPU output on the committed oracle fixtures (tests/golden), bitwise."""
    import os
    from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
    gdir = os.path.join(os.path.dirname(__file__), "golden")
    names = sorted(f for f in os.listdir(gdir) if f.startswith("oracle_") and f.endswith(".npz"))
    assert names
    for name in names:
        data = np.load(os.path.join(gdir, name))
        cid, J, eps, steps = int(data["cid"]), int(data["J"]), float(data["eps"]), int(data["steps"])
        sc, rc = build_config(cid, J, eps)
        s = Solver(sc, rc)
        s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(cid, sc, rc))
        s.commit()
        s.step(steps)
        for lv in range(rc.j_min, rc.j_max + 1):
            idx, f = s.read_leaves(lv)
            assert np.array_equal(idx, data[f"idx{lv}"]), (name, lv)
            assert np.array_equal(f.view(np.uint64), data[f"f{lv}"].view(np.uint64)), (name, lv)
        s.close()


@pytest.mark.parametrize("cid,J", [(3, 6), (4, 6), (5, 6)])
def test_generic_table_path_parity(cid, J, monkeypatch):
    """The generic (non-generated) table loop stays bit-identical to the oracle."""
    monkeypatch.setenv("MRLBM_NO_GEN", "1")
    sc, rc, gpu, ora = make_pair(cid, J)
    for k in range(12):
        gpu.step(1)
        ora.step(1)
        rel, bitwise, _ = compare(gpu, ora, rc, f"generic config {cid} step {k}")
        assert rel <= 1e-12
    gpu.close()
    ora.close()


@pytest.mark.parametrize("env", ["MRLBM_FUSE_PD", "MRLBM_NO_FB1T", "MRLBM_RIM_TPL", "MRLBM_K8_WARP", "MRLBM_K8_BLOCK",
                                 "MRLBM_K8_LONG_GAP=0", "MRLBM_K8_LONG_GAP=2", "MRLBM_K8_OCC=2", "MRLBM_SERIAL_STREAM"])
@pytest.mark.parametrize("cid,J", [(3, 6), (4, 6), (5, 7)])
def test_kernel_variant_parity(cid, J, env, monkeypatch):
    """The alternative kernel schedules stay bit-identical to the oracle: fused
    projection + details; all gap-1 fallback leaves in the block kernel k_fb1 (slot
    scan, no segment lists); boundary-rim gap-1 leaves thread per leaf (K7 MODE 3); the K8
    variants (one warp / one block per chunk, every deep-gap leaf
    in the thread kernel or in the warp-cooperative one, another register budget); the step graph
    without forked streams."""
    name, _, val = env.partition("=")
    monkeypatch.setenv(name, val or "1")
    sc, rc, gpu, ora = make_pair(cid, J)
    for k in range(12):
        gpu.step(1)
        ora.step(1)
        rel, bitwise, _ = compare(gpu, ora, rc, f"{env} config {cid} step {k}")
        assert rel <= 1e-12
    gpu.close()
    ora.close()


@pytest.mark.parametrize("cid,J", [(5, 7), (3, 6), (1, 8)])
def test_profiling_modes_do_not_change_the_state(cid, J):
    """mrlbm_set_profiling 0 (step graph), 1 (an event after every kernel, one stream) and 2
    (phase events, the graph's forks active) evolve the state bit-identically; mode 2's phase
    times add up to the step."""
    from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
    sc, rc = build_config(cid, J)
    outs = []
    for mode in (0, 1, 2):
        s = Solver(sc, rc)
        s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(cid, sc, rc))
        s.commit()
        s.set_profiling(mode)
        st = s.step(15)
        outs.append([s.read_leaves(lv) for lv in range(rc.j_min, rc.j_max + 1)])
        phases = sum(st.ms_phase[i] for i in range(6))
        if mode == 0:
            assert phases == 0.0
        else:
            assert 0.5 * st.ms_total <= phases <= 1.05 * st.ms_total
        s.close()
    for other in outs[1:]:
        for (ai, af), (bi, bf) in zip(outs[0], other):
            assert np.array_equal(ai, bi) and np.array_equal(af.view(np.uint64), bf.view(np.uint64))
