"""Mean duration per kernel of an ncu --csv launch list: python tools/launch_summary.py launches.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
h, out = None, {}
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d["Metric Name"] == "gpu__time_duration.sum":
        v = float(d["Metric Value"].replace(",", ""))
        if d.get("Metric Unit") == "ns":
            v /= 1000.0
        elif d.get("Metric Unit") == "ms":
            v *= 1000.0
        out.setdefault(d["Kernel Name"][:60], []).append(v)
for k, v in sorted(out.items(), key=lambda x: -sum(x[1]) / len(x[1]))[:top]:
    print(f"{sum(v) / len(v):9.1f} us  x{len(v):<3d} {k}")
