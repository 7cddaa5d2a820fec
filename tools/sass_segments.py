"""Execution-count segments of a kernel's SASS from an ncu report (where the
instructions and stalls go): python tools/sass_segments.py rep.ncu-rep kernel_regex [name_substring] [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
pick = sys.argv[3] if len(sys.argv) > 3 else None
top = int(sys.argv[4]) if len(sys.argv) > 4 else 14
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
blk = 0
if pick:
    blk = next(b for b in range(len(starts) - 1) if pick in rows[starts[b]][1])
print(rows[starts[blk]][1][:110])
rows = rows[starts[blk]:starts[blk + 1]]
h = rows[1]
si, ii, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((r[si].strip(), int(r[ii] or 0), int(r[wi] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(d[1] for d in data) or 1
ts = sum(d[2] for d in data) or 1
print(f"instructions {tot}, static {len(data)}, stall samples {ts}")
segs, cur, start = [], None, 0
for i, (_, c, _) in enumerate(data):
    if c != cur:
        if cur is not None:
            segs.append((start, i - 1, cur))
        cur, start = c, i
segs.append((start, len(data) - 1, cur))
for s, e, c in sorted(segs, key=lambda x: -x[2] * (x[1] - x[0] + 1))[:top]:
    n = e - s + 1
    st = sum(d[2] for d in data[s:e + 1])
    ops = {}
    for src, _, _ in data[s:e + 1]:
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top_ops = ", ".join(f"{k} {v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:6])
    print(f"[{s:5d}-{e:5d}] x{c:9d} * {n:4d} = {100 * c * n / tot:5.1f}% instr {100 * st / ts:5.1f}% stall | {top_ops}")
