"""Shared helpers: run the GPU product and the CPU oracle side by side."""
import numpy as np

from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest


def make_pair(cid, J, eps=-1.0, seed=2103_02903):
    from oracle import pyoracle
    sc, rc = build_config(cid, J, eps)
    idx, f0 = finest_cells(sc, rc), initial_finest(cid, sc, rc, seed)
    gpu = Solver(sc, rc)
    gpu.load_leaves(rc.j_max, idx, f0)
    gpu.commit()
    ora = pyoracle.Oracle(sc, rc)
    ora.load_leaves(rc.j_max, idx, f0)
    ora.commit()
    return sc, rc, gpu, ora


def compare(gpu, ora, rc, tag=""):
    """Leaf sets must be identical; fields within 1e-12 relative. Returns
    (max relative difference, bitwise-equal flag, total leaves)."""
    worst, bitwise, total = 0.0, True, 0
    for lv in range(rc.j_min, rc.j_max + 1):
        gi, gf = gpu.read_leaves(lv)
        oi, of = ora.read_leaves(lv)
        assert gi.shape == oi.shape and np.array_equal(gi, oi), f"{tag}: leaf set differs at level {lv}"
        total += gi.shape[0]
        if gf.size:
            d = np.abs(gf - of)
            rel = float(np.max(d / np.maximum(np.abs(of), 1e-300)))
            worst = max(worst, rel)
            bitwise = bitwise and np.array_equal(gf.view(np.uint64), of.view(np.uint64))
    return worst, bitwise, total
