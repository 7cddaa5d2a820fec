import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1407_2089_b200 import synth
from paper_1407_2089_b200.imaging import VoxelSpacing
from paper_1407_2089_b200.pipeline import FramePipeline
from paper_1407_2089_b200._lib import CELL_DTYPE
spec = synth.C2
pipe = FramePipeline(spec.dims, spec.dtype, VoxelSpacing(0.8, 0.8, 1.0))
rc = synth.generate(spec, 0, synth.CELL)
pipe.cell(rc)
torch.cuda.synchronize()
c = pipe.counters.cpu().numpy()
nk = int(c[2])
tab = pipe.table[:nk * CELL_DTYPE.itemsize].cpu().numpy().view(CELL_DTYPE)
box = (tab['bbox_hi'] - tab['bbox_lo'] + 1).prod(axis=1)
print('kept', nk, 'count max/mean', tab['count'].max(), tab['count'].mean(), 'bbox max/mean', box.max(), box.mean())
print('top counts', sorted(tab['count'])[-5:], 'top boxes', sorted(box)[-5:])
