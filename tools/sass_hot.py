"""Per-SASS-instruction hotspots of one kernel in an ncu report:
python tools/sass_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# several matching kernels: keep the block of the first (or the one whose
# name contains argv[4])
pick = sys.argv[4] if len(sys.argv) > 4 else None
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
blk = 0
if pick:
    blk = next(b for b in range(len(starts) - 1) if pick in rows[starts[b]][1])
print(rows[starts[blk]][1][:100])
rows = rows[starts[blk]:starts[blk + 1]]
h = rows[1]
ai, si, wi, ii = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) <= ii:
        continue
    try:
        data.append((int(r[wi] or 0), int(r[ii] or 0), r[si].strip()))
    except ValueError:
        pass
ts = sum(d[0] for d in data) or 1
ti = sum(d[1] for d in data) or 1
print(f"total stall samples {ts}, instructions {ti}")
ops = {}
for s, n, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    a = ops.setdefault(op, [0, 0])
    a[0] += s
    a[1] += n
print("by opcode (stall%, instr%):")
for op, (s, n) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:18]:
    print(f"  {op:10s} {100*s/ts:5.1f}% {100*n/ti:5.1f}%")
print("hottest instructions:")
for s, n, src in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"  {100*s/ts:5.1f}%  {n:9d}  {src[:90]}")
