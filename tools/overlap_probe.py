"""Step time of the C2 time point with the cell channel only, the vessel
channel only, and both (two streams, graph replays as in bench.py), to see
what each channel costs in the overlapped step.  python tools/overlap_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402

spec = synth.C2
dev = torch.device("cuda", 0)
pipe = FramePipeline(spec.dims, "u8", VoxelSpacing(0.8, 0.8, 1.0))
ring = 6
inputs = [{ch: synth.generate(spec, t, ch) for ch in (synth.CELL, synth.VESSEL)} for t in range(ring)]
s_cell = torch.cuda.Stream(dev, priority=-1)
s_vess = torch.cuda.Stream(dev, priority=0)
for i in range(ring):
    pipe.cell(inputs[i][synth.CELL])
    pipe.vessel(inputs[i][synth.VESSEL])
torch.cuda.synchronize()
gc = [pipe.capture(lambda i=i: pipe.cell(inputs[i][synth.CELL])) for i in range(ring)]
gv = [pipe.capture(lambda i=i: pipe.vessel(inputs[i][synth.VESSEL])) for i in range(ring)]
torch.cuda.synchronize()


def timeit(cell, vess, steps=200):
    main = torch.cuda.current_stream()
    for i in range(10):
        if cell:
            with torch.cuda.stream(s_cell):
                gc[i % ring].replay()
        if vess:
            with torch.cuda.stream(s_vess):
                gv[i % ring].replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s_cell.wait_stream(main)
    s_vess.wait_stream(main)
    for i in range(steps):
        if cell:
            with torch.cuda.stream(s_cell):
                gc[i % ring].replay()
        if vess:
            with torch.cuda.stream(s_vess):
                gv[i % ring].replay()
    main.wait_stream(s_cell)
    main.wait_stream(s_vess)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


for name, c, v in (("cell only", True, False), ("vessel only", False, True), ("both", True, True)):
    print(f"{name:12s} {timeit(c, v):.3f} ms per time point", flush=True)
