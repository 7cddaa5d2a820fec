"""Stall samples per SASS instruction of one kernel in an ncu report, with the
instruction's index so that waits of different warp roles can be told apart:
python tools/sass_hot.py report.ncu-rep kernel_regex [top] [nth match, default 0]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
nth = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, h, seen, name, kname = [], None, -1, "", ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "Kernel Name":
        name = r[1] if len(r) > 1 else ""
        continue
    if r[0] == "Address":
        if seen + 1 == nth:
            kname = name
        seen += 1
        if seen > nth:
            break
        h = r if seen == nth else None
        continue
    if h and len(r) == len(h):
        rows.append(dict(zip(h, r)))
tot = sum(int(r["Warp Stall Sampling (All Samples)"]) for r in rows) or 1
ins = sum(int(r["Instructions Executed"]) for r in rows) or 1
print(kname[:100])
print(f"{len(rows)} SASS lines, {tot} samples, {ins} warp instructions")
for i, r in sorted(enumerate(rows), key=lambda x: -int(x[1]["Warp Stall Sampling (All Samples)"]))[:top]:
    s = int(r["Warp Stall Sampling (All Samples)"])
    print(f"{i:5d} {100 * s / tot:5.1f}% {int(r['Instructions Executed']):10d}  {r['Source'].strip()[:90]}")
