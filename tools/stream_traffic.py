"""profiles/ncu_stream_traffic.json from an ncu CSV metric dump (``ncu --csv --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum``) of the stream-phase
launches (K8 k_stream_fallback, k_fb1, K7 k_stream_collide variants) of K steps: DRAM
bytes per step = total / K.

usage: python tools/stream_traffic.py dump.csv K "how it was captured"
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def main():
    path, k, how = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ix = {c: i for i, c in enumerate(h)}
    per = {}
    for r in rows[1:]:
        lid, name = r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0]
        d = per.setdefault(lid, {"kernel": name})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * SCALE[r[ix["Metric Unit"]]]
    by = {}
    rd = wr = tt = 0.0
    for d in per.values():
        b = by.setdefault(d["kernel"], {"dram_read": 0.0, "dram_write": 0.0, "time_s": 0.0, "launches": 0})
        b["dram_read"] += d.get("dram__bytes_read.sum", 0.0) / k
        b["dram_write"] += d.get("dram__bytes_write.sum", 0.0) / k
        b["time_s"] += d.get("gpu__time_duration.sum", 0.0) / k
        b["launches"] += 1
        rd += d.get("dram__bytes_read.sum", 0.0) / k
        wr += d.get("dram__bytes_write.sum", 0.0) / k
        tt += d.get("gpu__time_duration.sum", 0.0) / k
    res = {"bytes_per_step": rd + wr, "read": rd, "write": wr, "steps": k, "kernels_per_step": by,
           "ncu_time_ms_per_step": tt * 1e3, "how": how}
    out = os.path.join(ROOT, "profiles", "ncu_stream_traffic.json")
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({kk: v for kk, v in res.items() if kk != "kernels_per_step"}))


if __name__ == "__main__":
    main()
