"""Per-kernel counts of the Blackwell-specific SASS in libct.so (tcgen05 MMA /
TMEM loads and stores / TMA bulk-tensor loads / mbarrier ops / cp.async) from
`cuobjdump -sass`, plus one excerpt of each kind.  Run here (no GPU needed):

    python tools/sass_evidence.py [paper_1407_2089_b200/libct.so] > profiles/rNN_sass_evidence.txt
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict

so = sys.argv[1] if len(sys.argv) > 1 else "paper_1407_2089_b200/libct.so"
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
KINDS = {
    "UTCIMMA": "tcgen05.mma kind::i8 (tensor core, TMEM accumulator)",
    "UTCHMMA": "tcgen05.mma kind::f16",
    "UTCBAR": "tcgen05.commit -> mbarrier",
    "LDTM": "tcgen05.ld (TMEM -> registers)",
    "STTM": "tcgen05.st (registers -> TMEM)",
    "UTCATOMSWS": "tcgen05.alloc / dealloc (TMEM allocator)",
    "UTMALDG": "cp.async.bulk.tensor (TMA tile load)",
    "UTMASTG": "cp.async.bulk.tensor shared -> global (TMA tile store)",
    "UBLKCP": "cp.async.bulk (bulk copy)",
    "SYNCS": "mbarrier arrive / try_wait",
    "LDGSTS": "cp.async (Ampere-style async copy)",
}
pat = re.compile(r"\b(" + "|".join(KINDS) + r")[A-Z0-9_.]*")
per_fn = defaultdict(Counter)
example = {}
fn = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    if fn is None:
        continue
    for mm in pat.finditer(line):
        per_fn[fn][mm.group(1)] += 1
        example.setdefault(mm.group(1), (fn, line.strip()))


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out)) if len(out) == len(names) else {n: n for n in names}


n_fn = len(re.findall(r"Function : ", sass))
print(f"# SASS evidence: {so} ({n_fn} kernels), cuobjdump -sass, sm_100a")
print("# mnemonic -> PTX meaning")
for k, v in KINDS.items():
    print(f"#   {k:11s} {v}")
print()
dm = demangle(sorted(per_fn))
for f in sorted(per_fn, key=lambda f: -sum(per_fn[f].values())):
    c = per_fn[f]
    print(f"{dm[f][:110]}")
    print("    " + ", ".join(f"{k} x{c[k]}" for k in KINDS if c[k]))
print()
print("# one instance of each")
for k in KINDS:
    if k in example:
        f, ln = example[k]
        print(f"{k:11s} {dm.get(f, f)[:60]}: {ln[:150]}")
