"""Aggregate an ncu 'cuda,sass' source page (csv) per CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > x.csv; python tools/ncu_hot.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur_file, hdr, agg = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg.append((cur_file, r[0], r[1][:90], float(d["Warp Stall Sampling (All Samples)"] or 0),
                    float(d["Instructions Executed"] or 0)))
    except (KeyError, ValueError):
        pass
ts = sum(a[3] for a in agg) or 1
ti = sum(a[4] for a in agg) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3g}")
for f, ln, src, s, i in sorted(agg, key=lambda a: -a[3])[:top]:
    print(f"{s / ts * 100:5.1f}% stall {i / ti * 100:5.1f}% inst  {f}:{ln}  {src}")
