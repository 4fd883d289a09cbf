"""One line per captured kernel of an ncu --set full report: duration, DRAM
bytes, cache hit rates, occupancy, registers, grid (for profiles/)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = {
    "gpu__time_duration.sum": "time_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "l1tex__t_sector_hit_rate.pct": "L1hit%",
    "lts__t_sector_hit_rate.pct": "L2hit%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active%",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}
idx = {k: hdr.index(k) for k in want if k in hdr}
units = rows[1] if len(rows) > 1 else []
print("# kernel | " + " | ".join(want[k] for k in idx))
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:70]
    vals = []
    for k, i in idx.items():
        v = r[i].replace(",", "")
        u = units[i] if units else ""
        try:
            x = float(v)
            if k.startswith("dram__bytes"):
                x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) / 1e6
                v = f"{x:.1f}MB"
            elif k == "gpu__time_duration.sum":
                x = x * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
                v = f"{x:.1f}"
        except ValueError:
            pass
        vals.append(v)
    print(f"{name} | " + " | ".join(vals))
