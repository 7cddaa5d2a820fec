"""Certified-K1 fix-up list size on the C2 cell frames (how many voxels the
exact recompute handles): python tools/fix_count.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402

spec = synth.C2
pipe = FramePipeline(spec.dims, spec.dtype, VoxelSpacing(0.8, 0.8, 1.0), vessel=False)
for t in range(3):
    rc = synth.generate(spec, t, synth.CELL)
    pipe.cell(rc)
    torch.cuda.synchronize()
    print(f"t={t}: fix entries {int(pipe.fix[0].item())}, overflow {int(pipe.fix[1].item())}")
