import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
sc, rc = build_config(5, 12)
s = Solver(sc, rc)
s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc)); s.commit(); s.step(3)
snap = {lv: s.read_leaves(lv) for lv in range(rc.j_min, rc.j_max + 1)}
def pinned_like(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype).pin_memory(); return t.numpy()
sp = {}
for lv,(ix,ff) in snap.items():
    a,b = pinned_like(ix), pinned_like(ff); a[...] = ix; b[...] = ff; sp[lv]=(a,b)
for rep in range(2):
    s2 = Solver(sc, rc)
    t0=time.perf_counter()
    for lv,(ix,ff) in sp.items(): s2.load_leaves(lv, ix, ff)
    s2.synchronize(); t1=time.perf_counter()
    s2.commit(); s2.synchronize(); t2=time.perf_counter()
    st=s2.step(10); s2.synchronize(); t3=time.perf_counter()
    out={}
    for lv in range(rc.j_min, rc.j_max+1):
        n=s2.level_count(lv)
        bi=pinned_like(np.zeros((n,2),np.int32)); bf=pinned_like(np.zeros((9,n)))
        out[lv]=(bi,bf)
    t4=time.perf_counter()
    for lv in range(rc.j_min, rc.j_max+1):
        s2.read_leaves_into(lv, *out[lv])
    t5=time.perf_counter()
    print(f"load {1e3*(t1-t0):.1f} ms, commit {1e3*(t2-t1):.1f} ms, 10 steps {1e3*(t3-t2):.1f} ms, (alloc {1e3*(t4-t3):.1f}), read {1e3*(t5-t4):.1f} ms")
    s2.close()
