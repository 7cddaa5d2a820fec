"""Run the fused pipeline on one BASELINE config (default C4) and report
per-frame device time and sanity properties.  python tools/run_config.py C4"""
import sys
import os
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
spec = getattr(synth, name)
t0 = time.perf_counter()
pipe = FramePipeline(spec.dims, spec.dtype, VoxelSpacing(0.8, 0.8, 1.0), capacity=1 << 21)
rc = synth.generate(spec, 0, synth.CELL)
rv = synth.generate(spec, 0, synth.VESSEL)
torch.cuda.synchronize()
print(f"{name} {spec.dims} {spec.dtype}: setup {time.perf_counter() - t0:.1f} s, "
      f"mem {torch.cuda.memory_allocated() / 2**30:.1f} GiB, k1 path {'tensor' if pipe.k1_path_tc else 'fp64'}")
for rep in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    res = pipe.cell(rc, frame=0)
    e[1].record()
    vres = pipe.vessel(rv)
    e[2].record()
    torch.cuda.synchronize()
    cnt, rows = pipe.finish_cell(res)
    print(f"  rep {rep}: cell {e[0].elapsed_time(e[1]):.1f} ms, vessel {e[1].elapsed_time(e[2]):.1f} ms, "
          f"cells {len(rows)}, fg voxels {int(cnt[0])}, vessel decision {int(vres.state[5].item())}")
lab = pipe.labels
n = spec.nx * spec.ny * spec.nz
print("  labels in [-1, cells):", int(lab.min()) >= -1 and int(lab.max()) < len(rows),
      " counts match:", int((lab >= 0).sum()) == int(rows["count"].sum()))
d = vres.distance
print("  edt zero on mask:", bool(((d == 0) == vres.mask.bool()).all()), f" max dist {float(d.max()):.2f} um")
vox = n * 2 / 1e9
tot = e[0].elapsed_time(e[2])
print(f"  {2 * n / (tot / 1e3):.3e} voxels/s ({tot:.1f} ms per 2-channel time point, {vox:.2f} Gvoxels)")
