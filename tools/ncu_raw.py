"""Print selected metrics per kernel launch from an exported ncu raw CSV (.csv or .csv.gz)."""
import csv
import gzip
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
     "l1tex__t_sector_hit_rate.pct", "launch__grid_size"]


def main():
    p = sys.argv[1]
    f = gzip.open(p, "rt") if p.endswith(".gz") else open(p)
    r = list(csv.reader(f))
    h = r[0]
    idx = [h.index(m) if m in h else -1 for m in M]
    print("kernel | " + " | ".join(m.split("__")[1][:22] for m in M))
    for x in r[2:]:
        name = x[h.index("Kernel Name")]
        name = name.replace("void ", "").split("(")[0][:60]
        print(name, "|", " | ".join(x[i] if i >= 0 else "-" for i in idx))


if __name__ == "__main__":
    main()
