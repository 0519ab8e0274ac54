"""Config 6 (D3Q6, 3D) at J=8: W warm steps, then K steps inside a cuProfilerStart/Stop window
(for `ncu --profile-from-start off`).  MRLBM_E3_PROF=1 prints the engine's per-kernel times.

usage: python tools/window3d.py [W=30] [K=1] [J=8]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest  # noqa: E402


def main():
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    J = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    sc, rc = build_config(6, J)
    s = Solver(sc, rc)
    idx = finest_cells(sc, rc)
    s.load_leaves(rc.j_max, idx, initial_finest(6, sc, rc))
    n_fine = idx.shape[0]
    del idx
    s.commit()
    s.step(w)
    s.synchronize()
    cuda = C.CDLL("libcuda.so.1")
    cuda.cuProfilerStart()
    st = s.step(k)
    s.synchronize()
    cuda.cuProfilerStop()
    leaves = sum(int(st.leaves[i]) for i in range(st.levels))
    print("window steps", k, "ms/step", st.ms_total / k, "leaves", leaves, "MeshOR", leaves / n_fine,
          "fallback", int(st.fallback_leaves))
    s.close()


if __name__ == "__main__":
    main()
