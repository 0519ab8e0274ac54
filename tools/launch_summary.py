"""Summarise an ncu launch list (gpu__time_duration.sum CSV) for one step.

usage: python tools/launch_summary.py launches.csv STEP_INDEX
A step starts at a k_zero_flags launch; STEP_INDEX counts them from 0.
"""
import csv
import sys
from collections import defaultdict


def main():
    path, step = sys.argv[1], int(sys.argv[2])
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    data = [dict(zip(h, r)) for r in rows[1:]]
    starts = [i for i, d in enumerate(data) if "k_zero_flags" in d["Kernel Name"]]
    a = starts[step]
    b = starts[step + 1] if step + 1 < len(starts) else len(data)
    acc = defaultdict(float)
    cnt = defaultdict(int)
    for d in data[a:b]:
        nm = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mrlbm_b200::", "")
        if "k_stream_collide" in nm:
            nm = "k_stream_collide" + nm[nm.find("<"):]
        else:
            nm = nm.split("<")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit]
        acc[nm] += us
        cnt[nm] += 1
    tot = sum(acc.values())
    print(f"step {step}: {b - a} launches, {tot:.1f} us")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
        print(f"{v:9.1f} us {100 * v / tot:5.1f}%  x{cnt[k]:3d}  {k}")


if __name__ == "__main__":
    main()
