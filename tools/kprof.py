"""Warm per-kernel device times (CUDA events after every launch) for a config.

  python tools/kprof.py --config 5 --warmup 3 --steps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--jmax", type=int, default=0)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
sc, rc = build_config(a.config, a.jmax)
s = Solver(sc, rc)
s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(a.config, sc, rc))
s.commit()
st = s.step(a.warmup)
g = s.step(a.steps)
print(f"graph: {g.ms_total / a.steps:.3f} ms/step, leaves {[int(g.leaves[i]) for i in range(g.levels)]}, "
      f"fallback {g.fallback_leaves}, virtual {sum(g.virtual_cells[i] for i in range(g.levels))}")
s.set_profiling(True)
p = s.step(a.steps)
s.set_profiling(False)
prof = s.profile_text()
tot = sum(v[0] for v in prof.values()) / a.steps
print(f"profiled: {p.ms_total / a.steps:.3f} ms/step (sum of kernels {tot:.3f} ms)")
by_kernel = {}
for (k, lv), (ms, n) in prof.items():
    by_kernel[k] = by_kernel.get(k, 0.0) + ms / a.steps
for k, v in sorted(by_kernel.items(), key=lambda x: -x[1]):
    print(f"  {k:22s} {v * 1e3:9.1f} us/step  {100 * v / tot:5.1f}%")
print("top launches:")
for (k, lv), (ms, n) in sorted(prof.items(), key=lambda x: -x[1][0])[: a.top]:
    print(f"  {k:22s} L{lv:<3d} {ms / a.steps * 1e3:9.1f} us")
