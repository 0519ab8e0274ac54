import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest, config_steps
J = int(sys.argv[1])
for V in [float(v) for v in sys.argv[2:]]:
    sc, rc = build_config(6, J)
    for a in range(3):
        sc.eq_params[a] = V
    idx, f0 = finest_cells(sc, rc), initial_finest(6, sc, rc)
    n = idx.shape[0]
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, idx, f0); s.commit()
    ors = []; ms = []
    for k in range(0, config_steps(6, rc), 10):
        st = s.step(10)
        ors.append(round(sum(int(st.leaves[i]) for i in range(st.levels)) / n, 4)); ms.append(round(st.ms_total / 10, 3))
    lv = [int(st.leaves[i]) for i in range(st.levels)]
    umax = max(np.abs(s.read_leaves(l)[1].sum(axis=0)).max() if s.level_count(l) else 0 for l in range(rc.j_min, rc.j_max + 1))
    print('V', V, 'MeshOR', ors, 'ms/step', ms, 'leaves', lv, 'fb', st.fallback_leaves, 'umax', umax, flush=True)
    s.close()
