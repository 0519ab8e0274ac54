import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
for cid,J in ((5,8),(3,6),(1,8)):
    sc, rc = build_config(cid, J)
    outs=[]
    for mode in (0,1,2):
        s = Solver(sc, rc); s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(cid, sc, rc)); s.commit()
        s.set_profiling(mode); st=s.step(30)
        outs.append([s.read_leaves(l) for l in range(rc.j_min, rc.j_max+1)])
        print(cid, 'mode', mode, 'phases', [round(st.ms_phase[i],3) for i in range(6)], 'total', round(st.ms_total,3))
        s.close()
    for a,b in zip(outs[0], outs[1]): assert np.array_equal(a[0],b[0]) and np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))
    for a,b in zip(outs[0], outs[2]): assert np.array_equal(a[0],b[0]) and np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))
print('modes agree bitwise')
