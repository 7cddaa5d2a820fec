"""cProfile of sequence.segment_frames on C2 pinned frames (host side of the
materialised drop-in path).  python tools/prof_sequence.py"""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.sequence import segment_frames  # noqa: E402

spec = synth.C2
host = [{ch: synth.generate(spec, 60 + i, ch).cpu().pin_memory() for ch in (synth.CELL, synth.VESSEL)}
        for i in range(2)]
sp = VoxelSpacing(0.8, 0.8, 1.0)


def run(n):
    return segment_frames(range(n), lambda t: host[t % 2][synth.CELL], lambda t: host[t % 2][synth.VESSEL],
                          spacing=sp, materialize=True, with_hull=False)


run(3)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
run(10)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
