"""Error-control slope experiments: E[u](eps) against the eps = 0 run."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest

def run(cid, J, eps, steps, ab=None):
    sc, rc = build_config(cid, J, eps)
    if ab is not None:
        sc.eq_params[0], sc.eq_params[1] = ab
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(cid, sc, rc))
    s.commit()
    s.step(steps)
    return s

EPS = [1e-2, 5e-3, 1e-3, 5e-4, 1e-4]
for name, cid, J, steps, ab, row in [("burgers T=0.5", 1, 10, 512, None, [1.0, 1.0]),
                                      ("burgers T=0.25", 1, 10, 256, None, [1.0, 1.0]),
                                      ("burgers T=1", 1, 10, 1024, None, [1.0, 1.0]),
                                      ("d2q4 adv (.5,.5) 128 steps", 3, 8, 128, (0.5, 0.5), [1.0] * 4),
                                      ("d2q4 adv (.25,.25) 256 steps", 3, 8, 256, (0.25, 0.25), [1.0] * 4)]:
    ref = run(cid, J, 0.0, steps, ab)
    Es = []
    for eps in EPS:
        g = run(cid, J, eps, steps, ab)
        Es.append(g.additional_error(ref, row)[0])
        g.close()
    sl = np.polyfit(np.log10(EPS), np.log10(Es), 1)[0]
    sl4 = np.polyfit(np.log10(EPS[:4]), np.log10(Es[:4]), 1)[0]
    print(name, "E", ["%.3e" % e for e in Es], "slope(all)", round(sl, 3), "slope(first 4)", round(sl4, 3), flush=True)
    ref.close()
