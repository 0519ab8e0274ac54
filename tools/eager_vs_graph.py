import sys, os
sys.path.insert(0, os.getcwd())
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
sc, rc = build_config(5, 12)
res = {}
for mode in ["graph", "eager", "profiled", "graph2"]:
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc))
    s.commit()
    s.step(8)
    if mode == "eager":
        s.set_graph(False)
    if mode == "profiled":
        s.set_profiling(True)
    st = s.step(3)
    res[mode] = st.ms_total / 3
    if mode == "profiled":
        prof = s.profile_text()
        tot = {}
        for (k, lv), (ms, n) in prof.items():
            tot[k] = tot.get(k, 0) + ms / 3
        print(sorted(tot.items(), key=lambda x: -x[1])[:6])
    s.close()
print(res)
