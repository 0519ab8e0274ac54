"""Compact per-launch table from an `ncu --page raw --csv` export: duration, DRAM
read/write, issue-active, warps-active, L1/L2 hit rates, sectors per request.
usage: python tools/ncu_table.py raw.csv [min_us]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    lim = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
    h, u = rows[0], rows[1]
    ix = {k: i for i, k in enumerate(h)}
    scale = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}

    def g(r, k):
        try:
            return float(r[ix[k]].replace(",", "")) * scale.get(u[ix[k]], 1.0)
        except (KeyError, ValueError):
            return float("nan")
    tot = 0.0
    for r in rows[2:]:
        d = g(r, "gpu__time_duration.sum")
        tot += d
        if d < lim:
            continue
        rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
        req = g(r, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
        sec = g(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
        print(f"{d:8.1f}us {r[ix['Kernel Name']][:34]:34s} rd {rd:7.1f} wr {wr:6.1f} MB {(rd + wr) / d:5.2f} TB/s "
              f"iss {g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):4.1f} "
              f"wrp {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):4.1f} "
              f"L1h {g(r, 'l1tex__t_sector_hit_rate.pct'):4.1f} L2h {g(r, 'lts__t_sector_hit_rate.pct'):4.1f} "
              f"sec/req {sec / max(req, 1.0):4.1f}")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main()
