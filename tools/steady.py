"""Config 5 at J=12 in the settled regime: N warm steps, then K profiled steps.

usage: python tools/steady.py [N=200] [K=2]
Run under ncu with --launch-skip N*launches_per_step to capture only the last steps.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    sc, rc = build_config(5, 12)
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc))
    s.commit()
    st = s.step(n)
    st = s.step(k)
    print("launches/step", st.kernel_launches // k, "ms/step", st.ms_total / k,
          "leaves", sum(int(st.leaves[i]) for i in range(st.levels)))


if __name__ == "__main__":
    main()
