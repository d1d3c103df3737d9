"""Markdown table of selected metrics from `ncu -i REPORT --page raw --csv` output (one row per captured
launch).  python tools/r2/ncu_raw_table.py RAW.csv"""
import csv
import sys

COLS = [("gpu__time_duration.sum", "ms", 1e-6, "%.3f"),
        ("dram__bytes_read.sum", "DRAM rd GB", None, "%.3f"),
        ("dram__bytes_write.sum", "DRAM wr GB", None, "%.3f"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1, "%.1f"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %", 1, "%.1f"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thr %", 1, "%.1f"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor % (elapsed)", 1, "%.1f"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor % (active)", 1, "%.1f"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1, "%.1f"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1, "%.1f"),
        ("launch__registers_per_thread", "regs", 1, "%.0f")]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    have = [(c, n, f, fmt) for c, n, f, fmt in COLS if c in h]
    print("| kernel | " + " | ".join(n for _, n, _, _ in have) + " |")
    print("|---|" + "---|" * len(have))
    for r in rows[2:]:
        vals = []
        for c, n, f, fmt in have:
            i = h.index(c)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                vals.append(r[i])
                continue
            u = units[i]
            if f is None:  # bytes: normalise to GB
                v *= {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1.0)
            elif c.startswith("gpu__time_duration"):
                v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1.0)
            vals.append(fmt % v)
        k = r[ki].split("(")[0].replace("void ", "")[:40]
        print("| %s | %s |" % (k, " | ".join(vals)))


if __name__ == "__main__":
    main()
