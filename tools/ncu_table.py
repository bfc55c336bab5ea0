"""Compact table of key ncu metrics from `--page raw --csv` exports
(profiling aid): one line per kernel."""
import csv
import sys

COLS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("lts__t_sector_hit_rate.pct", "L2hit%"), ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "lsb"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tc%")]


def main(paths):
    print("kernel".ljust(48) + "".join(n.rjust(11) for _, n in COLS))
    for p in paths:
        rows = list(csv.reader(open(p)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
            cells = []
            for m, _ in COLS:
                if m not in hdr:
                    cells.append("-")
                    continue
                i = hdr.index(m)
                v, u = r[i].replace(",", ""), units[i]
                try:
                    x = float(v)
                    if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                        cells.append(f"{x / 1e9:.3f}G")
                    elif u in ("usecond", "msecond", "nsecond", "us", "ms", "ns"):
                        x *= {"usecond": 1e-3, "msecond": 1, "nsecond": 1e-6, "us": 1e-3, "ms": 1, "ns": 1e-6}[u]
                        cells.append(f"{x:.4f}ms")
                    else:
                        cells.append(f"{x:.1f}")
                except ValueError:
                    cells.append(v[:10])
            print(name.split("(")[0][:47].ljust(48) + "".join(c.rjust(11) for c in cells))


if __name__ == "__main__":
    main(sys.argv[1:])
