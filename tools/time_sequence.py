"""Wall time per frame of sequence.segment_frames on C2 pinned frames
(materialised, no hulls), N frames after a warm-up call.
python tools/time_sequence.py [N] [depth]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.sequence import segment_frames  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = synth.C2
host = []
for i in range(2):
    fr = {}
    for ch in (synth.CELL, synth.VESSEL):
        h = torch.empty(spec.dims, dtype=spec.torch_dtype, pin_memory=True)
        h.copy_(synth.generate(spec, 60 + i, ch).cpu())
        fr[ch] = h
    host.append(fr)
sp = VoxelSpacing(0.8, 0.8, 1.0)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    last = {}
    segment_frames(range(n), lambda t: host[t % 2][synth.CELL], lambda t: host[t % 2][synth.VESSEL],
                   spacing=sp, materialize=True, with_hull=False, depth=depth, on_frame=lambda fo: last.update(fo=fo))
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    print(f"rep {rep}: {n} frames depth {depth}: {ms / n:.2f} ms/frame, {len(last['fo'].detections)} dets", flush=True)
