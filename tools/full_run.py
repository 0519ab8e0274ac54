"""BASELINE config 5 end to end on one GPU: D2Q9 cylinder, levels 2..J (default 12,
finest 8192 x 4096), the full step count (default 50 000 = ceil(T / dt)), with the
obstacle force recorded on the device every step (mrlbm_set_force_tracking).

Reports wall / device time, leaf counts and leaf-updates/s per chunk of steps,
the drag / lift coefficients and the Strouhal number of the
lift series when it has a dominant peak.

usage: python tools/full_run.py [--jmax 12] [--steps 50000] [--chunk 1000] [--out profiles/x.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_02903_b200 import (Solver, build_config, config_steps, drag_lift, finest_cells,  # noqa: E402
                                   initial_finest, strouhal)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jmax", type=int, default=12)
    ap.add_argument("--steps", type=int, default=0, help="0: the config's own count ceil(T / dt)")
    ap.add_argument("--chunk", type=int, default=1000)
    ap.add_argument("--out", default="")
    ap.add_argument("--series", default="", help="optional .npz with the per-step Fx, Fy, leaves")
    ap.add_argument("--no-forces", dest="forces", action="store_false", help="run without force tracking")
    a = ap.parse_args()
    sc, rc = build_config(5, a.jmax)
    n = a.steps or int(config_steps(5, rc))
    s = Solver(sc, rc)
    t0 = time.time()
    s.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(5, sc, rc))
    s.commit()
    if a.forces:
        s.set_force_tracking(n)
    dt = 2.0 ** (-rc.j_max) / sc.lam
    chunks, done, dev_ms, updates = [], 0, 0.0, 0
    leaves_hist = []
    upd0 = 0  # stats.leaf_updates is cumulative over the context's steps
    while done < n:
        k = min(a.chunk, n - done)
        st = s.step(k)
        done += k
        dev_ms += st.ms_total
        du = st.leaf_updates - upd0
        upd0 = st.leaf_updates
        updates += du
        nl = sum(int(st.leaves[i]) for i in range(st.levels))
        leaves_hist.append((done, nl))
        chunks.append({"steps_done": done, "ms_per_step": st.ms_total / k, "leaves_last": nl,
                       "leaf_updates_per_s": du / (st.ms_total * 1e-3)})
    wall = time.time() - t0
    res = {
        "workload": f"config 5 (D2Q9 cylinder, Re=1200), levels {rc.j_min}..{rc.j_max}, eps={rc.epsilon}",
        "steps": n, "dt": dt, "T": n * dt, "force_tracking": a.forces,
        "device_s": dev_ms * 1e-3, "wall_s": wall,
        "leaf_updates": int(updates), "leaf_updates_per_s": updates / (dev_ms * 1e-3),
        "ms_per_step_mean": dev_ms / n,
        "leaves_final": leaves_hist[-1][1],
        "finest_cells": int(finest_cells(sc, rc).shape[0]),
        "chunks": chunks,
    }
    if not a.forces:
        print(json.dumps(res, indent=1))
        if a.out:
            with open(a.out, "w") as fh:
                fh.write(json.dumps(res, indent=1) + "\n")
        return
    fx, fy = s.force_history()
    L = 2 * rc.obstacle_radius
    u0 = 0.05
    cd = np.array([drag_lift(x, y, 1.0, u0, L)[0] for x, y in zip(fx, fy)])
    cl = np.array([drag_lift(x, y, 1.0, u0, L)[1] for x, y in zip(fx, fy)])
    half = n // 2
    res.update({
        "cd_mean_second_half": float(np.mean(cd[half:])), "cl_rms_second_half": float(np.sqrt(np.mean(cl[half:] ** 2))),
        "cd_last": float(cd[-1]), "cl_last": float(cl[-1]),
    })
    try:
        st_, df = strouhal(cl, dt, u0, L, skip=half)
        res["strouhal"] = st_
        res["strouhal_resolution"] = L * df / u0
    except FloatingPointError as e:
        res["strouhal"] = None
        res["strouhal_note"] = f"no dominant peak in the second half of the lift series ({e})"
    s.close()
    txt = json.dumps(res, indent=1)
    print(txt)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w") as fh:
            fh.write(txt + "\n")
    if a.series:
        np.savez_compressed(a.series, fx=fx, fy=fy, cd=cd, cl=cl, leaves=np.array(leaves_hist))


if __name__ == "__main__":
    main()
