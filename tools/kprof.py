"""Warm per-kernel device times (CUDA events after every launch) over a bench window.

  python tools/kprof.py --config 5 --warmup 5 --steps 20

The graph-timed steps and the profiled (eager, event after every kernel) steps are
the SAME window: both contexts start from the post-warm-up state.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--jmax", type=int, default=0)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
sc, rc = build_config(a.config, a.jmax)
s = Solver(sc, rc)
s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(a.config, sc, rc))
s.commit()
s.step(a.warmup)
snap = {lv: s.read_leaves(lv) for lv in range(rc.j_min, rc.j_max + 1)}
g = s.step(a.steps)
print(f"graph: {g.ms_total / a.steps:.3f} ms/step (steps {a.warmup}..{a.warmup + a.steps - 1}), last leaves "
      f"{[int(g.leaves[i]) for i in range(g.levels)]}, fallback {g.fallback_leaves}, "
      f"virtual {sum(g.virtual_cells[i] for i in range(g.levels))}")
s.close()
p = Solver(sc, rc)
for lv, (ix, ff) in snap.items():
    if ix.shape[0]:
        p.load_leaves(lv, ix, ff)
p.commit()
p.set_profiling(True)
st = p.step(a.steps)
prof = p.profile_text()
tot = sum(v[0] for v in prof.values()) / a.steps
print(f"profiled: {st.ms_total / a.steps:.3f} ms/step (sum of kernels {tot:.3f} ms)")
by_kernel = {}
for (k, lv), (ms, n) in prof.items():
    by_kernel[k] = by_kernel.get(k, 0.0) + ms / a.steps
for k, v in sorted(by_kernel.items(), key=lambda x: -x[1]):
    print(f"  {k:22s} {v * 1e3:9.1f} us/step  {100 * v / tot:5.1f}%")
print("top launches:")
for (k, lv), (ms, n) in sorted(prof.items(), key=lambda x: -x[1][0])[: a.top]:
    print(f"  {k:22s} L{lv:<3d} {ms / a.steps * 1e3:9.1f} us")
