"""profiles/ncu_stream_traffic.json from an ncu --set full report of one step's
stream-phase launches (K8 k_stream_fallback, k_fb1, K7 k_stream_collide x3).

usage: python tools/stream_traffic.py report.ncu-rep "how it was captured"
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, how = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
             "msecond": 1e-3, "second": 1.0}
    ks, rd, wr, tt = [], 0.0, 0.0, 0.0
    for r in rows[2:]:
        d = dict(zip(h, r))

        def val(k):
            return float(d[k].replace(",", "")) * scale[units[h.index(k)]]

        k = {"kernel": d["Kernel Name"].split("(")[0], "grid": d.get("launch__grid_size", ""),
             "dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum"),
             "time_s": val("gpu__time_duration.sum")}
        ks.append(k)
        rd += k["dram_read"]
        wr += k["dram_write"]
        tt += k["time_s"]
    res = {"bytes_per_step": rd + wr, "read": rd, "write": wr, "kernels": ks, "ncu_time_ms": tt * 1e3, "how": how}
    path = os.path.join(ROOT, "profiles", "ncu_stream_traffic.json")
    json.dump(res, open(path, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}))


if __name__ == "__main__":
    main()
