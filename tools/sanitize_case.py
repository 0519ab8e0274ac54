"""Small adaptive runs of every config for compute-sanitizer (memcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest  # noqa: E402

for cid, J in [(1, 6), (2, 6), (3, 5), (4, 5), (5, 6)]:
    sc, rc = build_config(cid, J)
    s = Solver(sc, rc)
    s.set_graph(False)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(cid, sc, rc))
    s.commit()
    s.step(6)
    for lv in range(rc.j_min, rc.j_max + 1):
        s.read_leaves(lv)
    s.close()
    print("config", cid, "ok", flush=True)
