#!/usr/bin/env python3
"""Benchmark of the adaptive MR-LBM time step (BASELINE.json metric: leaf-cell
updates/s for the full step incl. adaptation; HBM GB/s vs peak).

Workload (config.workload): BASELINE configs[4], D2Q9 Navier-Stokes past a
cylinder, levels 2..12 (finest 8192 x 4096), epsilon = 1e-4, from its seeded
initial datum.  A "step" is one Algorithm-1 iteration (adapt -> transfer ->
stream -> collide -> obstacle) over the whole adaptive mesh.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl product|reference]

--impl reference times the CPU restatement of the reference path (the oracle;
the reference ships no step of its own) on the host cores.
Multi-GPU: the path does not shard in this tier (replicas only);
every rank runs an independent replica, value = total updates / max time.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_ID = 5
METRIC = "MR-LBM leaf-cell updates/s (full step incl. adaptation)"
UNIT = "leaf-updates/s"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 9]
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows)
        smax = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": smax, "reasons": reasons, "samples": len(rows)}


def reduce_replicas(ms, updates, device, world):
    """Replicas-only aggregation: max device time over ranks, summed
    leaf updates.  Works with any torch.distributed backend (gloo tests on CPU)."""
    import torch
    t = torch.tensor([float(ms)], device=device, dtype=torch.float64)
    u = torch.tensor([float(updates)], device=device, dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def snapshot(s, rc):
    out = {}
    for lv in range(rc.j_min, rc.j_max + 1):
        out[lv] = s.read_leaves(lv)
    return out


def run_cpu_sample(min_seconds=10.0, max_steps=40, jmax=10, threads=None):
    """CPU oracle (the reference path restated on the reference headers) on a
    bounded sample: config 5 at J_bar = jmax from its initial datum, stepping
    until min_seconds of step time (at least 2 steps, at most max_steps)."""
    from oracle import pyoracle
    from paper_2103_02903_b200 import build_config, finest_cells, initial_finest
    cores = threads or os.cpu_count() or 1
    pyoracle.set_threads(cores)
    sc, rc = build_config(CONFIG_ID, jmax)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(CONFIG_ID, sc, rc))
    o.commit()
    upd, secs, steps = 0, 0.0, 0
    while steps < max_steps and (steps < 2 or secs < min_seconds):
        t = time.perf_counter()
        o.step(1)
        secs += time.perf_counter() - t
        upd += sum(o.level_count(lv) for lv in range(rc.j_min, rc.j_max + 1))
        steps += 1
    o.close()
    return {"value": upd / secs, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"config 5 (D2Q9 cylinder) at J_bar={jmax} ({(8 << (jmax - 2)) * (4 << (jmax - 2))} finest cells), "
                      f"{steps} oracle steps from the initial datum, {cores} threads, {secs:.2f} s"}


def bench_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # each step: one oracle step of the bounded sample (config 5 at J_bar = 9)
    from oracle import pyoracle
    from paper_2103_02903_b200 import build_config, finest_cells, initial_finest
    cores = os.cpu_count() or 1
    pyoracle.set_threads(cores)
    jmax = 9
    sc, rc = build_config(CONFIG_ID, jmax)
    o = pyoracle.Oracle(sc, rc)
    o.load_leaves(rc.j_max, finest_cells(sc, rc), initial_finest(CONFIG_ID, sc, rc))
    o.commit()
    for _ in range(args.warmup):
        o.step(1)
    upd, secs = 0, 0.0
    for _ in range(args.steps):
        t = time.perf_counter()
        o.step(1)
        secs += time.perf_counter() - t
        upd += sum(o.level_count(lv) for lv in range(rc.j_min, rc.j_max + 1))
    v = upd / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (config 5 initial datum, seeded perturbation)",
        "config": {"workload": f"config 5 D2Q9 cylinder, levels 2..{jmax} (bounded CPU sample of levels 2..12)",
                   "epsilon": rc.epsilon},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"config 5 at J_bar={jmax}, {args.steps} timed oracle steps after {args.warmup} warm-up"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def bench_product(args):
    import numpy as np
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2103_02903_b200 import Solver, build_config, finest_cells, initial_finest
    from paper_2103_02903_b200.abi import PHASES

    sc, rc = build_config(CONFIG_ID, args.jmax)
    idx0, f0 = finest_cells(sc, rc), initial_finest(CONFIG_ID, sc, rc)
    s = Solver(sc, rc)
    s.load_leaves(rc.j_max, idx0, f0)
    s.commit()
    stream = torch.cuda.ExternalStream(s.stream_handle(), device=dev)
    # warm-up (also evolves the state into the measured regime)
    st = s.step(args.warmup)
    # state snapshot for the e2e leg (same K steps, through host buffers)
    snap = snapshot(s, rc)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- device-timed region: K steps, L2 flushed between steps (outside the events)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    u0 = st.leaf_updates
    barrier()
    launches = 0
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)
            evs[k][0].record(stream)
            st = s.step(1)
            evs[k][1].record(stream)
            launches += st.kernel_launches
    barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    updates = st.leaf_updates - u0
    clocks = clk.summary()
    ms_max, utot = reduce_replicas(ms, updates, dev, world)
    value = utot / (ms_max / 1e3)
    state_bytes = 8 * sc.q * sum(int(st.leaves[i]) for i in range(st.levels))

    end_counts = {lv: s.level_count(lv) for lv in range(rc.j_min, rc.j_max + 1)}

    # ---- phase breakdown over the SAME K steps as the timed window: a second context
    # restarts from the post-warm-up state (bit-identical evolution) with eager launches
    # and CUDA events after every phase / kernel on the context's stream (~5-9 % slower
    # than the graph, so the per-phase bandwidths below are conservative)
    sprof = Solver(sc, rc)
    for lv, (ix, ff) in snap.items():
        sprof.load_leaves(lv, ix, ff)
    sprof.commit()
    sprof.set_profiling(True)
    nprof = args.steps
    phase_tot = [0.0] * len(PHASES)
    stream_bytes_tot, model_bytes_tot, fin_bytes_tot = 0, 0, 0
    for _ in range(nprof):
        sp = sprof.step(1)
        for i in range(len(PHASES)):
            phase_tot[i] += sp.ms_phase[i]
        stream_bytes_tot += sp.bytes_stream      # per-step algorithmic bytes
        model_bytes_tot += sp.bytes_model
        # finest-level table stream + collision (K7 gap 0): read f* of the level's leaves and
        # ghosts, write the leaves (boundary-rim fallback leaves are a negligible part)
        nl, nv = int(sp.leaves[sp.levels - 1]), int(sp.virtual_cells[sp.levels - 1])
        fin_bytes_tot += 8 * sc.q * (2 * nl + nv)
    kern_prof = sprof.profile_text()
    sprof.close()
    phase_ms = {p: phase_tot[i] / nprof for i, p in enumerate(PHASES)}
    stream_kernels = {}
    for (kname, lv), (kms, kn) in kern_prof.items():
        if kname.startswith(("k_stream", "k_fb1")):
            stream_kernels[kname] = stream_kernels.get(kname, 0.0) + kms / nprof
    fin_ms = kern_prof.get(("k_stream_collide", rc.j_max), (0.0, 0))[0] / nprof
    fin_bytes = fin_bytes_tot / nprof
    dom = max(phase_ms, key=phase_ms.get)
    peak, peak_kind = load_peaks()
    stream_bytes = stream_bytes_tot / nprof
    model_bytes = model_bytes_tot / nprof
    achieved = stream_bytes / (phase_ms["stream"] / 1e3) / 1e9 if phase_ms["stream"] > 0 else 0.0
    step_ms_prof = sum(phase_ms.values())
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_stream_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("bytes_per_step")
        except Exception:
            traffic = None

    # ---- steady regime (context only, not the headline): after the white-noise
    # transient the mesh settles (~0.9 M leaves); continue the run to step 200
    steady = None
    if args.steady and world == 1:
        done = args.warmup + args.steps
        if done < 200:
            s.step(200 - done)
        ss = s.step(20)
        steady = {"after_steps": 200, "steps": 20, "ms_per_step": ss.ms_total / 20,
                  "value": ss.leaf_updates and (sum(int(ss.leaves[i]) for i in range(ss.levels)) / (ss.ms_total / 20 / 1e3)),
                  "leaves": sum(int(ss.leaves[i]) for i in range(ss.levels))}

    # ---- e2e through the C-ABI with host buffers: load snapshot -> commit -> K steps -> read back.
    # Host buffers are pinned (page-locked) as the contract asks; allocation is outside the timing.
    def pinned_like(a):
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype).pin_memory()
        return t.numpy()

    snap_p = {}
    for lv, (ix, ff) in snap.items():
        pi_, pf_ = pinned_like(ix), pinned_like(ff)
        pi_[...] = ix
        pf_[...] = ff
        snap_p[lv] = (pi_, pf_)
    # read-back buffers: pinned, sized by the level counts the timed run ended with (the
    # e2e context replays the same deterministic K steps from the same state)
    out_flat = {lv: (pinned_like(np.zeros(sc.d * end_counts[lv] + 16, np.int32)),
                     pinned_like(np.zeros(sc.q * end_counts[lv] + 16)))
                for lv in snap}
    s2 = Solver(sc, rc)
    h2d = sum(v[0].nbytes + v[1].nbytes for v in snap_p.values())
    barrier()
    t0 = time.perf_counter()
    for lv, (ix, ff) in snap_p.items():
        s2.load_leaves(lv, ix, ff)
    s2.commit()
    st2 = s2.step(args.steps)
    d2h = 0
    for lv in range(rc.j_min, rc.j_max + 1):
        n = s2.level_count(lv)
        fi, ffl = out_flat[lv]
        if n * sc.d > fi.size or n * sc.q > ffl.size:
            fi, ffl = np.zeros(n * sc.d + 1, np.int32), np.zeros(n * sc.q + 1)  # pageable overflow
        bi, bf = fi[: n * sc.d].reshape(n, sc.d), ffl[: n * sc.q].reshape(sc.q, n)
        s2.read_leaves_into(lv, bi, bf)
        d2h += bi.nbytes + bf.nbytes
    barrier()
    e2e_s = time.perf_counter() - t0
    e2e_smax, e2e_u = reduce_replicas(e2e_s, st2.leaf_updates, dev, world)
    e2e_val = e2e_u / e2e_smax
    s2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = run_cpu_sample()

    if rank == 0:
        leaves_last = [int(st.leaves[i]) for i in range(st.levels)]
        internal_last = [int(st.internal[i]) for i in range(st.levels)]
        virtual_last = [int(st.virtual_cells[i]) for i in range(st.levels)]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (config 5 initial datum: rest + seeded 1e-3 transverse perturbation)",
            "config": {"workload": "config 5: D2Q9 Navier-Stokes past a cylinder, levels 2..%d (finest %dx%d), "
                                   "eps=1e-4, Re=1200" % (rc.j_max, 8 << (rc.j_max - 2), 4 << (rc.j_max - 2)),
                       "parallelism": "replicas" if world > 1 else "single-gpu",
                       "l2": f"flushed between timed steps (256 MiB write); state {state_bytes / 1e6:.0f} MB",
                       "leaves_per_level_last_step": leaves_last,
                       "internal_per_level_last_step": internal_last,
                       "virtual_per_level_last_step": virtual_last,
                       "fallback_leaves_last_step": int(st.fallback_leaves)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "stream+collide phase per step (K8 k_stream_fallback, k_fb1, K7 k_stream_collide: "
                                   "gap-1 fallback thread-per-leaf k_fb1t, finest level, coarser levels, other fallback)",
                         "algorithmic_bytes": stream_bytes, "peak_kind": peak_kind,
                         "timing": "CUDA events per kernel on the context stream over the same K steps as the "
                                   "timed window (eager replay from the post-warm-up state)",
                         "kernels_ms_per_step": stream_kernels},
            "kernel_roofline": {"kernel": "K7 finest level (gap-0 table stream + MRT collision), per launch",
                                "algorithmic_bytes": fin_bytes, "ms": fin_ms,
                                "achieved_gbs": fin_bytes / (fin_ms / 1e3) / 1e9 if fin_ms > 0 else 0.0,
                                "frac": (fin_bytes / (fin_ms / 1e3) / 1e9 / peak) if fin_ms > 0 else 0.0},
            "step_roofline": {"bytes_model_per_step": model_bytes,
                              "achieved_gbs": model_bytes / (ms_max / args.steps / 1e3) / 1e9,
                              "frac": model_bytes / (ms_max / args.steps / 1e3) / 1e9 / peak},
            "phases_ms": phase_ms, "dominant_phase": dom,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                    "d2h_bytes_per_step": d2h // args.steps},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if steady is not None:
            line["steady_state"] = steady
        print(json.dumps(line))
    s.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--jmax", type=int, default=0, help="override J_bar (default: config value 12)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-steady", dest="steady", action="store_false", help="skip the steady-regime context run")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_product(args)


if __name__ == "__main__":
    main()
