"""Stall samples and executed instructions per CUDA source line of one kernel
in an ncu report (--import-source on; compile with -lineinfo):
python tools/src_hot.py report.ncu-rep kernel_regex [top] [function-name substring]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
pick = sys.argv[4] if len(sys.argv) > 4 else None  # substring of the function name
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0, ""])
cur_file = cur_line = None
cur_src = ""
fn0 = None
skip = True
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "Function Name":
        if fn0 is None and (pick is None or pick in r[1]):
            fn0 = r[1]
        skip = fn0 is None or r[1] != fn0
        if fn0 is not None and r[1] != fn0 and agg:
            break  # first matching kernel only
        continue
    if fn0 is None or skip:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        continue
    if r[0] != "":
        cur_line, cur_src = r[0], r[1][:100]
    if len(r) > 7 and r[2] != "":
        try:
            st, ins = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        a = agg[(cur_file, cur_line)]
        a[0] += st
        a[1] += ins
        a[2] = cur_src
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"stall% instr%  file:line source   (total instructions {toti})")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% {100 * v[1] / toti:5.1f}%  {k[0]}:{k[1]}: {v[2]}")
