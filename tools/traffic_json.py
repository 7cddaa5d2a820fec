"""Per-stage DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
one C2 time point from an ncu launch list of tools/profile_stages.py --reps 1,
written to profiles/ncu_traffic.json for bench.py's roofline "traffic" field.
python tools/traffic_json.py gpurun_out/launchesNN.csv"""
import collections
import csv
import json
import os
import sys

STAGES = {
    "K1 gaussian": ("tc_prep", "tc_pass_xy", "tc_pass_z", "fix_p1", "fix_p2q", "gauss_fixup", "gauss_strided",
                    "gauss_contig"),
    "K2 median+hist": ("median3",),
    "K5 ccl": ("ccl_",),
    "K6 table": ("tab_",),
    "K7 mrf": ("mrf_", "pw_", "delta_from_hist", "lap_mean"),
    "K8 edt": ("edt_",),
}
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.defaultdict(float)
names = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        continue
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
    per[r[idi]] += float(r[vi].replace(",", "")) * scale
    names[r[idi]] = r[ki].replace("void ", "").replace("<unnamed>::", "")
out = {}
for stage, pats in STAGES.items():
    tot = sum(b for i, b in per.items() if names[i].startswith(pats))
    if tot:
        out[stage] = tot
out["_note"] = ("DRAM bytes per C2 time point and stage (sum over the stage's kernels, cold-cache ncu "
                f"replay) from {os.path.basename(sys.argv[1])}")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
