"""Aggregate an ncu launch list (gpu__time_duration.sum CSV) over every step it holds.

usage: python tools/launch_window.py launches.csv
Steps start at k_zero_flags launches; prints per-kernel us/step and share.
"""
import csv
import sys
from collections import defaultdict


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    data = [dict(zip(h, r)) for r in rows[1:]]
    nsteps = sum(1 for d in data if "k_zero_flags" in d["Kernel Name"])
    acc, cnt = defaultdict(float), defaultdict(int)
    for d in data:
        nm = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mrlbm_b200::", "")
        if "k_stream_collide" in nm:
            nm = "k_stream_collide" + nm[nm.find("<"):]
        else:
            nm = nm.split("<")[0]
        v = float(d["Metric Value"].replace(",", ""))
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        acc[nm] += us
        cnt[nm] += 1
    tot = sum(acc.values())
    print(f"{nsteps} steps, {len(data)} launches, {tot / nsteps:.1f} us/step (cold, serialised)")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
        print(f"{v / nsteps:9.1f} us/step {100 * v / tot:5.1f}%  x{cnt[k] / nsteps:5.1f}/step  {k}")


if __name__ == "__main__":
    main()
