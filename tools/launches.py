"""Summarise an ncu --csv launch list: per-kernel mean time and DRAM bytes."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    per[r[idi]][r[mi]] = v * scale
    names[r[idi]] = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:58]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':58s} {'n':>3s} {'mean us':>9s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>7s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:58s} {n:3d} {t / n:9.1f} {t / tot:6.1%} {b / n / 1e6:10.1f} {b / t / 1e3 if t else 0:7.0f}")
