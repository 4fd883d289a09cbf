"""Summarise `ncu -i REP --page raw --csv` exports: one line per kernel with
duration, DRAM bytes, cache hit rates, L2 throughput, occupancy, registers,
grid, and the top warp-stall reasons (pc sampling).  Usage:
    python tools/ncu_csv_summary.py TITLE raw1.csv [raw2.csv ...]
"""
import csv
import sys

WANT = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"), ("l1tex__t_sector_hit_rate.pct", "L1hit"),
        ("lts__t_sector_hit_rate.pct", "L2hit"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2thru"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAMthru"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]


def main():
    print(f"# {sys.argv[1]}")
    for path in sys.argv[2:]:
        rows = list(csv.reader(open(path)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            name = name.replace("vl::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
            cells = []
            for key, label in WANT:
                if key in hdr:
                    cells.append(f"{label}={r[hdr.index(key)]}{units[hdr.index(key)].replace('register/thread', '')}")
            tot = sum(float(r[hdr.index(h)] or 0) for h in stalls) or 1.0
            top = sorted(((float(r[hdr.index(h)] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                          for h in stalls), reverse=True)[:5]
            print(name[:110])
            print("    " + " | ".join(cells))
            print("    stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top))


if __name__ == "__main__":
    main()
