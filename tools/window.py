"""Config 5 at J=12: W warm steps, then K steps inside a cuProfilerStart/Stop window
(for `ncu --profile-from-start off`, so only the window's kernels are captured).

usage: python tools/window.py [W=8] [K=1]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest  # noqa: E402


def main():
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    sc, rc = build_config(5, 12)
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc))
    s.commit()
    s.step(w)
    s.synchronize()
    cuda = C.CDLL("libcuda.so.1")
    cuda.cuProfilerStart()
    st = s.step(k)
    s.synchronize()
    cuda.cuProfilerStop()
    print("window steps", k, "ms/step", st.ms_total / k, "leaves", sum(int(st.leaves[i]) for i in range(st.levels)))


if __name__ == "__main__":
    main()
