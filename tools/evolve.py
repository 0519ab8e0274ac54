"""Run a config on the GPU and print per-step mesh statistics and device time."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--jmax", type=int, default=0)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--every", type=int, default=10)
a = ap.parse_args()
sc, rc = build_config(a.config, a.jmax)
s = Solver(sc, rc)
s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(a.config, sc, rc))
s.commit()
done = 0
while done < a.steps:
    st = s.step(a.every)
    done += a.every
    print(json.dumps({"step": done, "ms_per_step": st.ms_total / a.every,
                      "leaves": [int(st.leaves[i]) for i in range(st.levels)],
                      "fallback": int(st.fallback_leaves),
                      "virtual": int(sum(st.virtual_cells[i] for i in range(st.levels))),
                      "updates_per_s": (st.leaf_updates) / done / (st.ms_total / a.every / 1e3) if st.ms_total else 0}),
          flush=True)
