"""Run the fused per-frame pipeline serially on C2 frames (for ncu launch
lists and per-stage timings).  python tools/profile_stages.py [--reps N]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--config", default="C2")
ap.add_argument("--only", default="both", choices=["both", "cell", "vessel"])
a = ap.parse_args()
spec = getattr(synth, a.config)
pipe = FramePipeline(spec.dims, spec.dtype, VoxelSpacing(0.8, 0.8, 1.0))
rc = synth.generate(spec, 0, synth.CELL)
rv = synth.generate(spec, 0, synth.VESSEL)
ap_warm = os.environ.get("PS_WARM", "0") == "1"
if ap_warm:  # one untimed rep (module load, first-launch costs)
    if a.only in ("both", "cell"):
        pipe.cell(rc)
    if a.only in ("both", "vessel"):
        pipe.vessel(rv)
torch.cuda.synchronize()
pipe.marks = []
for _ in range(a.reps):
    if a.only in ("both", "cell"):
        pipe.cell(rc)
    if a.only in ("both", "vessel"):
        pipe.vessel(rv)
torch.cuda.synchronize()
for k, v in pipe.stage_times_ms().items():
    print(f"{k:28s} {v:8.3f} ms")
