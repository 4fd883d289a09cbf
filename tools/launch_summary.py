"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per
kernel family, launches, total and mean duration, share of the sum."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    fam = re.sub(r"\(.*", "", name)
    m = re.match(r"void vl::(?:\(anonymous namespace\)::)?(\w+)<(.*)>", name)
    if m:
        body = re.findall(r"vl::(?:\(anonymous namespace\)::)?(?:cg::)?(\w+)", m.group(2))
        fam = m.group(1) + ("<" + ",".join(b for b in body[:2]) + ">" if body else "")
    unit = d.get("Metric Unit", "ns")
    v = float(d["Metric Value"].replace(",", ""))
    v = v / 1e3 if unit == "ns" else (v * 1e3 if unit in ("ms", "msecond") else v)  # -> us
    if unit == "usecond":
        v = float(d["Metric Value"].replace(",", ""))
    agg[fam][0] += 1
    agg[fam][1] += v
tot = sum(v for _, v in agg.values()) or 1.0
print(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>6s}")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{k[:70]:70s} {c:8d} {v:12.1f} {v / c:10.2f} {v / tot * 100:5.1f}%")
print(f"total {sum(c for c, _ in agg.values())} launches, {tot / 1e3:.1f} ms")
