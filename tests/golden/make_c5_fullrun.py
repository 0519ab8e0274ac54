"""Generate the full-run fixture of config 5 at J_bar = 9 (tests/golden/c5_J9_fullrun.npz).

The oracle runs the whole BASELINE config-5 run (50 000 steps, T = 12.2) at
J_bar = 9 (512 x 256 finest) from the seeded initial datum.  Every 1000 steps
it records a SHA-256 of the complete mesh state (per level: leaf coordinates
and populations, CellIndex order); at the end it stores the leaves and fields
of every level.  tests/test_gpu_fullrun.py runs the GPU product over the same
50 000 steps and checks the hashes (bit-exact trajectory) and the final fields
(L1 <= 1e-9, north_star).  The oracle takes ~2 h on 8 host cores, which is why
this is a committed fixture and not a live comparison.

Run from the repo root: python tests/golden/make_c5_fullrun.py [threads]
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2103_02903_b200 import build_config, config_steps, finest_cells, initial_finest  # noqa: E402
from oracle import pyoracle  # noqa: E402

CID, J, EVERY = 5, 9, 1000


def state_hash(o, rc):
    h = hashlib.sha256()
    for lv in range(rc.j_min, rc.j_max + 1):
        idx, f = o.read_leaves(lv)
        h.update(np.int64(lv).tobytes())
        h.update(np.ascontiguousarray(idx, dtype=np.int32).tobytes())
        h.update(np.ascontiguousarray(f, dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    pyoracle.set_threads(threads)
    sc, rc = build_config(CID, J)
    nsteps = config_steps(CID, rc)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(CID, sc, rc))
    o.commit()
    hashes, leaves, t0 = [], [], time.time()
    done = 0
    while done < nsteps:
        n = min(EVERY, nsteps - done)
        o.step(n)
        done += n
        hashes.append(state_hash(o, rc))
        leaves.append(sum(o.level_count(lv) for lv in range(rc.j_min, rc.j_max + 1)))
        print(f"step {done}: {leaves[-1]} leaves, {time.time() - t0:.0f} s", flush=True)
    data = {"cid": CID, "J": J, "steps": nsteps, "every": EVERY, "hashes": np.array(hashes),
            "leaves": np.array(leaves, dtype=np.int64)}
    for lv in range(rc.j_min, rc.j_max + 1):
        idx, f = o.read_leaves(lv)
        data[f"idx{lv}"] = idx
        data[f"f{lv}"] = f
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"c{CID}_J{J}_fullrun.npz")
    np.savez_compressed(out, **data)
    print("wrote", out, f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
