"""Generate the golden regression fixtures for the oracle (tests/golden/*.npz).

The reference ships no golden vectors for the step; these pin the
oracle's own output on small cases so later changes to the checker are caught.
Run from the repo root: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2103_02903_b200 import build_config, finest_cells, initial_finest  # noqa: E402
from oracle import pyoracle  # noqa: E402

CASES = [(1, 6, -1.0, 12), (3, 5, -1.0, 6), (4, 5, -1.0, 6), (5, 5, -1.0, 8), (6, 4, -1.0, 10)]


def main():
    out = os.path.dirname(os.path.abspath(__file__))
    force = "--force" in sys.argv
    for cid, J, eps, steps in CASES:
        path = os.path.join(out, f"oracle_c{cid}_J{J}_s{steps}.npz")
        if os.path.exists(path) and not force:
            continue  # existing fixtures are kept (run with --force to regenerate them all)
        sc, rc = build_config(cid, J, eps)
        o = pyoracle.Oracle(sc, rc)
        o.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(cid, sc, rc))
        o.commit()
        o.step(steps)
        data = {"cid": cid, "J": J, "eps": eps, "steps": steps}
        for lv in range(rc.j_min, rc.j_max + 1):
            idx, f = o.read_leaves(lv)
            data[f"idx{lv}"] = idx
            data[f"f{lv}"] = f
        np.savez_compressed(path, **data)
        print("wrote", cid, J, steps)
    # snapshot golden file: config 1, J=6, 5 steps, written by the product's writer
    if os.path.exists(os.path.join(out, "cells_c1_J6_s5.csv")) and not force:
        return
    from paper_2103_02903_b200.snapshot import write_snapshot
    sc, rc = build_config(1, 6)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(1, sc, rc))
    o.commit()
    o.step(5)
    o.scheme, o.cfg = sc, rc
    p = write_snapshot(o, 5, out)
    os.replace(p, os.path.join(out, "cells_c1_J6_s5.csv"))
    print("wrote snapshot golden")


if __name__ == "__main__":
    main()
